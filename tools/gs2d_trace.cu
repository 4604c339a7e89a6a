// Standalone timeline trace of the GS-2D pipeline (tools only; see tools/build_trace.sh):
//   build/var/gs2d_trace ROWS COLS T      (TVS_GS2D_CLUSTER selects the cluster size)
// Per block n (g_trace[n]): 0 start, 1 group-0 chunk 0, 2 group-0 chunk 100,
// 3 last group chunk 100, 4 first downstream publish, 5 last group done,
// 6 exit, 7 SM id.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../include/tvstencil.h"
namespace tvs { extern __device__ unsigned long long g_trace[4096][8]; extern __device__ unsigned long long g_wait[2][6][2]; }
int main(int argc, char** argv) {
  const int64_t ext[3] = {argc > 1 ? atoll(argv[1]) : 8192, argc > 2 ? atoll(argv[2]) : 8192, 1};
  const int T = argc > 3 ? atoi(argv[3]) : 100;
  const char* cse = getenv("TVS_GS2D_CLUSTER");
  const int CS = cse ? atoi(cse) : 4;
  tvs_stencil st{};
  st.dim = 2; st.kind = TVS_GAUSS_SEIDEL; st.ntaps = 9; st.radius = 1;
  int k = 0;
  for (int i = -1; i <= 1; ++i) for (int j = -1; j <= 1; ++j) { st.offsets[k][0] = i; st.offsets[k][1] = j; st.coeffs[k] = 1.0 / 9; ++k; }
  tvs_exec ex{}; ex.fma_policy = TVS_FMA_NEVER;
  tvs_plan* p = nullptr;
  if (tvs_plan_create(&st, 2, ext, &ex, &p)) { printf("create: %s\n", tvs_last_error()); return 1; }
  const int nblk = std::min<int>(4096, (int)((ext[0] + 127 + 3) / 4 + CS - 1) / CS * CS);
  for (int rep = 0; rep < 2; ++rep) {
    std::vector<unsigned long long> zero(4096 * 8, 0);
    cudaMemcpyToSymbol(tvs::g_trace, zero.data(), zero.size() * 8);
    cudaMemcpyToSymbol(tvs::g_wait, zero.data(), 2 * 6 * 2 * 8);
    if (tvs_plan_run(p, T)) { printf("run: %s\n", tvs_last_error()); return 1; }
    tvs_plan_synchronize(p);
    float ms; tvs_plan_last_ms(p, &ms);
    std::vector<unsigned long long> tr(4096 * 8);
    cudaMemcpyFromSymbol(tr.data(), tvs::g_trace, tr.size() * 8);
    unsigned long long t0 = ~0ull;
    for (int n = 0; n < nblk; ++n) if (tr[n * 8]) t0 = std::min(t0, tr[n * 8]);
    auto at = [&](int n, int e) { return tr[n * 8 + e] ? (tr[n * 8 + e] - t0) / 1e3 : -1.0; };
    printf("rep %d: %.3f ms, %d blocks, cluster %d\n", rep, ms, nblk, CS);
    if (rep == 0) continue;
    unsigned long long wt[2][6][2];
    cudaMemcpyFromSymbol(wt, tvs::g_wait, sizeof(wt));
    const char* names[6] = {"warp(g0,w0)", "warp(g0,w3)", "warp(g3,w0)", "warp(g3,w3)", "loader", "drainer"};
    for (int c = 0; c < 2; ++c)
      for (int r = 0; r < 6; ++r)
        printf("block %d %-12s first 100 chunks: %9llu cycles, waiting %9llu (%.0f%%)\n", c, names[r], wt[c][r][1],
               wt[c][r][0], wt[c][r][1] ? 100.0 * wt[c][r][0] / wt[c][r][1] : 0.0);
    double life = 0, gin = 0, gout = 0, live = 0;
    int nin = 0, nout = 0;
    for (int n = 0; n < nblk; ++n) life += at(n, 6) - at(n, 0);
    for (int n = 1; n < nblk; ++n) {
      const double d = at(n, 2) - at(n - 1, 2);
      if (n % CS) { gin += d; ++nin; } else { gout += d; ++nout; }
    }
    // average number of blocks between start and exit at the midpoint of the run
    const double mid = ms * 500;
    for (int n = 0; n < nblk; ++n) live += (at(n, 0) <= mid && at(n, 6) >= mid);
    printf("mean lifetime %.1f us; group-0 chunk-100 lag: within cluster %.2f us (%d), across %.2f us (%d); live at mid %.0f\n",
           life / nblk, nin ? gin / nin : 0.0, nin, nout ? gout / nout : 0.0, nout, live);
    for (int n : {0, 1, 2, 3, 4, 5, 8, 9, 100, 101, 147, 148, 149, 500, 1000, 2000, nblk - 1}) {
      if (n >= nblk) continue;
      printf("blk %4d sm %3llu start %9.1f  g0c0 %9.1f  g0c100 %9.1f  g3c100 %9.1f  g3done %9.1f  exit %9.1f\n", n,
             tr[n * 8 + 7], at(n, 0), at(n, 1), at(n, 2), at(n, 3), at(n, 5), at(n, 6));
    }
  }
  tvs_plan_destroy(p);
  return 0;
}
