// Micro-benchmarks that ground the kernel designs (DESIGN.md §"measured
// constants"): FP64 dependent-op latency, 64-bit shuffle latency, FP64
// throughput under full load, and the GS-1D inner chain (DMUL->DADD->DADD).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void lat_dadd(double* out, long long* cyc, int n, double a) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); }
  long long t1 = clock64();
  out[threadIdx.x + 1] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dmul(double* out, long long* cyc, int n, double a) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dmul_rn(x, a); x = __dmul_rn(x, a); x = __dmul_rn(x, a); x = __dmul_rn(x, a); }
  long long t1 = clock64();
  out[threadIdx.x + 1] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dfma(double* out, long long* cyc, int n, double a) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, a); x = fma(x, a, a); x = fma(x, a, a); x = fma(x, a, a); }
  long long t1 = clock64();
  out[threadIdx.x + 1] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// the GS-1D chain: acc = w0*L; acc = w1*C + acc; acc = w2*R + acc; L = acc
__global__ void lat_gschain(double* out, long long* cyc, int n, double w0, double w1, double w2) {
  double L = out[0], C = out[1], R = out[2];
  double pc = __dmul_rn(w1, C), pr = __dmul_rn(w2, R);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double acc = __dmul_rn(w0, L); acc = __dadd_rn(pc, acc); acc = __dadd_rn(pr, acc); L = acc;
  }
  long long t1 = clock64();
  out[threadIdx.x + 3] = L; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(double* out, long long* cyc, int n) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1); }
  long long t1 = clock64();
  out[threadIdx.x + 64] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ int idx[64];
  idx[threadIdx.x] = (threadIdx.x + 1) & 31;
  __syncwarp();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { j = idx[j]; j = idx[j]; }
  long long t1 = clock64();
  out[threadIdx.x] = j; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread, full grid
__global__ void thr_dmuladd(double* out, int n, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
#define OP(x) x = __dadd_rn(__dmul_rn(x, a), b);
    OP(x0) OP(x1) OP(x2) OP(x3) OP(x4) OP(x5) OP(x6) OP(x7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void thr_dfma(double* out, int n, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
#define OPF(x) x = fma(x, a, b);
    OPF(x0) OPF(x1) OPF(x2) OPF(x3) OPF(x4) OPF(x5) OPF(x6) OPF(x7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copyk(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s sms %d l2 %d MB smem/blk optin %zu clock_khz %d\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, clk);
  double* d; long long* c; CK(cudaMalloc(&d, 1 << 24)); CK(cudaMalloc(&c, 64));
  CK(cudaMemset(d, 0, 1 << 24));
  long long h; const int n = 4096;
  lat_dadd<<<1, 1>>>(d, c, n, 1e-3); CK(cudaDeviceSynchronize());
  lat_dadd<<<1, 1>>>(d, c, n, 1e-3); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost)); printf("DADD latency %.2f cyc\n", h / (4.0 * n));
  lat_dmul<<<1, 1>>>(d, c, n, 1.0000001); lat_dmul<<<1, 1>>>(d, c, n, 1.0000001); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost)); printf("DMUL latency %.2f cyc\n", h / (4.0 * n));
  lat_dfma<<<1, 1>>>(d, c, n, 0.5); lat_dfma<<<1, 1>>>(d, c, n, 0.5); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost)); printf("DFMA latency %.2f cyc\n", h / (4.0 * n));
  lat_gschain<<<1, 1>>>(d, c, n, 0.3, 0.4, 0.3); lat_gschain<<<1, 1>>>(d, c, n, 0.3, 0.4, 0.3); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost)); printf("GS chain (DMUL,DADD,DADD) %.2f cyc/iter\n", h / (1.0 * n));
  lat_shfl<<<1, 32>>>(d, c, n); lat_shfl<<<1, 32>>>(d, c, n); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost)); printf("SHFL.64 (2x32) latency %.2f cyc\n", h / (2.0 * n));
  lat_lds<<<1, 32>>>(d, c, n); lat_lds<<<1, 32>>>(d, c, n); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost)); printf("LDS latency %.2f cyc\n", h / (2.0 * n));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, it = 20000;
  thr_dmuladd<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); thr_dmuladd<<<blocks, threads>>>(d, it, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 2.0 * 8 * it * (double)blocks * threads;
  printf("DMUL+DADD throughput %.2f Tops/s (%.1f ops/clk/SM at %d kHz)\n", ops / ms / 1e9, ops / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3), clk);
  cudaEventRecord(e0); thr_dfma<<<blocks, threads>>>(d, it, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1); ops = 1.0 * 8 * it * (double)blocks * threads;
  printf("DFMA throughput %.2f Tinstr/s (%.1f /clk/SM)\n", ops / ms / 1e9, ops / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3));
  size_t bytes = size_t(4) << 30; double4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 0, bytes);
  size_t n4 = bytes / 32;
  copyk<<<p.multiProcessorCount * 16, 512>>>(a, b, n4); CK(cudaDeviceSynchronize());
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); copyk<<<p.multiProcessorCount * 16, 512>>>(a, b, n4); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("copy 4GiB: %.1f GB/s (r+w)\n", 2.0 * bytes / best / 1e6);
  return 0;
}
