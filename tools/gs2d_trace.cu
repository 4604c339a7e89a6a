// Standalone latency trace of the GS-2D pipeline (tools only):
//   nvcc -DGS2P_TRACE ... tools/gs2d_trace.cu build/{api,...}.o   (see tools/build_trace.sh)
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../include/tvstencil.h"
namespace tvs { extern __device__ unsigned long long g_trace[4096][8]; extern __device__ unsigned long long g_wait[2][6][2]; }
int main() {
  const int64_t ext[3] = {8192, 8192, 1};
  tvs_stencil st{};
  st.dim = 2; st.kind = TVS_GAUSS_SEIDEL; st.ntaps = 9; st.radius = 1;
  int k = 0;
  for (int i = -1; i <= 1; ++i) for (int j = -1; j <= 1; ++j) { st.offsets[k][0] = i; st.offsets[k][1] = j; st.coeffs[k] = 1.0 / 9; ++k; }
  tvs_exec ex{}; ex.fma_policy = TVS_FMA_NEVER;
  tvs_plan* p = nullptr;
  if (tvs_plan_create(&st, 2, ext, &ex, &p)) { printf("create: %s\n", tvs_last_error()); return 1; }
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(&tvs::g_trace, 0, 0);  // no-op placeholder
    std::vector<unsigned long long> zero(4096 * 8, 0);
    cudaMemcpyToSymbol(tvs::g_trace, zero.data(), zero.size() * 8);
    cudaMemcpyToSymbol(tvs::g_wait, zero.data(), 2 * 6 * 2 * 8);
    if (tvs_plan_run(p, 100)) { printf("run: %s\n", tvs_last_error()); return 1; }
    tvs_plan_synchronize(p);
    float ms; tvs_plan_last_ms(p, &ms);
    std::vector<unsigned long long> tr(4096 * 8);
    cudaMemcpyFromSymbol(tr.data(), tvs::g_trace, tr.size() * 8);
    unsigned long long t0 = tr[0 * 8 + 0];
    printf("rep %d: %.3f ms\n", rep, ms);
    unsigned long long wt[2][6][2];
    cudaMemcpyFromSymbol(wt, tvs::g_wait, sizeof(wt));
    const char* names[6] = {"w(0,0)", "w(0,3)", "w(3,0)", "w(3,3)", "loader", "drainer"};
    for (int c = 0; c < 2; ++c)
      for (int r = 0; r < 6; ++r)
        printf("cta %d %-8s wait %10llu of %10llu cycles (%.0f%%)\n", c, names[r], wt[c][r][0], wt[c][r][1],
               wt[c][r][1] ? 100.0 * wt[c][r][0] / wt[c][r][1] : 0.0);
    for (int n : {0, 1, 2, 3, 10, 50, 100, 147, 148, 149, 200, 500, 1000, 2000, 2079}) {
      auto* e = &tr[n * 8];
      printf("cta %4d start %9.1f us  g0c0 %9.1f  g0c100 %9.1f  g3c100 %9.1f  pub1 %9.1f\n", n,
             (e[0] - t0) / 1e3, e[1] ? (e[1] - t0) / 1e3 : -1, e[2] ? (e[2] - t0) / 1e3 : -1,
             e[3] ? (e[3] - t0) / 1e3 : -1, e[4] ? (e[4] - t0) / 1e3 : -1);
    }
  }
  tvs_plan_destroy(p);
  return 0;
}
