// PCIe duplex with SM-driven downloads: copy-engine H2D of 2 GiB while a
// kernel streams 2 GiB from HBM into page-locked host memory (mapped, UVA)
// vs two copy-engine copies.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -o tools/zc_probe tools/zc_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                            \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void d2h_kernel(const double2* __restrict__ src, double2* dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

int main() {
  const size_t bytes = 2ull << 30, n2 = bytes / sizeof(double2);
  double *h_in, *h_out, *d_a, *d_b;
  CK(cudaHostAlloc(&h_in, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_out, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaMalloc(&d_a, bytes));
  CK(cudaMalloc(&d_b, bytes));
  for (size_t i = 0; i < bytes / 8; i += 512) h_in[i] = 1.0, h_out[i] = 2.0;
  CK(cudaMemset(d_b, 0, bytes));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto fn) {
    float best = 1e9f;
    for (int r = 0; r < 3; ++r) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      fn();
      cudaDeviceSynchronize();
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  const double gb = bytes / 1e9;
  float t = timed([&] { cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2); });
  printf("CE D2H alone        %6.1f ms %5.1f GB/s\n", t, gb / t * 1e3);
  t = timed([&] {
    cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
  });
  printf("CE H2D + CE D2H     %6.1f ms\n", t);
  for (int blocks : {4, 8, 16, 32, 64, 148}) {
    t = timed([&] { d2h_kernel<<<blocks, 512, 0, s2>>>((const double2*)d_b, (double2*)h_out, n2); });
    printf("SM D2H alone %3d blocks %6.1f ms %5.1f GB/s\n", blocks, t, gb / t * 1e3);
    t = timed([&] {
      cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
      d2h_kernel<<<blocks, 512, 0, s2>>>((const double2*)d_b, (double2*)h_out, n2);
    });
    printf("CE H2D + SM D2H %3d %6.1f ms\n", blocks, t);
  }
  CK(cudaGetLastError());
  return 0;
}
