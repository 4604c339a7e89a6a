// Microbenchmark of the GS-2D 9-point unit chain (K6's steady body without
// synchronisation): per iteration a lane reads NE / E / SE inputs from a
// shared ring, takes SE from lane-1 by shuffle, runs the unfused sorted-tap
// chain and stores its output.  Variants: warps per block, independent
// chains per lane (NCH), shuffle on/off.  Reports SM cycles per iteration and
// units per clock per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gs_chain_bench tools/gs_chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kSl = 34;
constexpr int kRing = 8;

template <int NCH, bool SH>
__global__ void chain(int iters, double* sink, long long* cyc, const double* wv) {
  extern __shared__ double ring[];  // [warp][kRing][kSl]
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  double* my = ring + (size_t)wi * kRing * kSl * NCH;
  for (int i = threadIdx.x; i < (int)(blockDim.x / 32) * kRing * kSl * NCH; i += blockDim.x) ring[i] = 0.001 * (i % 97);
  __syncthreads();
  double w[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) w[k] = __shfl_sync(0xffffffffu, wv[k], 0);
  double nw[NCH], nn[NCH], ne[NCH], cc[NCH], ee[NCH], sw[NCH], ss[NCH], se[NCH], ww[NCH], out[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) nw[c] = nn[c] = ne[c] = cc[c] = ee[c] = sw[c] = ss[c] = se[c] = ww[c] = out[c] = 0.5 + c;
  const long long t0 = clock64();
  for (int it = 0; it < iters; it += 4) {
    double in_ne[NCH][4], in_e[NCH][4], in_se[NCH][4];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* rb = my + (size_t)c * kRing * kSl + ((it + u) & (kRing - 1)) * kSl;
        in_ne[c][u] = rb[lane + 2];
        in_e[c][u] = rb[lane + 1];
        in_se[c][u] = rb[1];
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        double sev = in_se[c][u];
        if (SH) {
          const double sh = __shfl_up_sync(0xffffffffu, out[c], 1);
          sev = lane == 0 ? in_se[c][u] : sh;
        }
        nw[c] = nn[c]; nn[c] = ne[c]; ne[c] = in_ne[c][u];
        cc[c] = ee[c]; ee[c] = in_e[c][u];
        sw[c] = ss[c]; ss[c] = se[c]; se[c] = sev;
        double acc = __dmul_rn(w[0], nw[c]);
        acc = __dadd_rn(__dmul_rn(w[1], nn[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[2], ne[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[3], ww[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[4], cc[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[5], ee[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[6], sw[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[7], ss[c]), acc);
        acc = __dadd_rn(__dmul_rn(w[8], se[c]), acc);
        out[c] = acc;
        ww[c] = acc;
        my[(size_t)c * kRing * kSl + ((it + u + 4) & (kRing - 1)) * kSl + lane + 2] = acc;
      }
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += out[c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NCH, bool SH>
void run(int warps, int iters) {
  double *sink, *wv;
  long long* cyc;
  cudaMalloc(&sink, 148 * 1024 * sizeof(double));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&wv, 9 * sizeof(double));
  double h[9] = {0.1, 0.11, 0.12, 0.13, 0.1, 0.09, 0.11, 0.12, 0.12};
  cudaMemcpy(wv, h, sizeof h, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)warps * kRing * kSl * NCH * sizeof(double);
  cudaFuncSetAttribute(chain<NCH, SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chain<NCH, SH><<<148, warps * 32, smem>>>(iters, sink, cyc, wv);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<NCH, SH><<<148, warps * 32, smem>>>(iters, sink, cyc, wv);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  const cudaError_t err = cudaGetLastError();
  const double units = 148.0 * warps * 32 * NCH * iters;
  printf("warps %2d NCH %d shfl %d smem %6zu: %7.1f cyc/iter  %.2f units/clk/SM  %.1f GSt/s  %s\n", warps, NCH, SH ? 1 : 0,
         smem, (double)c / iters, (double)warps * 32 * NCH * iters / c, units / ms / 1e6,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(sink);
  cudaFree(cyc);
  cudaFree(wv);
}

int main() {
  const int it = 1 << 14;
  for (int w : {4, 8, 16, 24, 32}) run<1, true>(w, it);
  for (int w : {8, 16}) run<1, false>(w, it);
  for (int w : {4, 8, 16}) run<2, true>(w, it);
  for (int w : {4, 8}) run<3, true>(w, it);
  for (int w : {4, 8}) run<4, true>(w, it);
  return 0;
}
