// K6: 2D radius-1 Gauss-Seidel (lexicographic order) as a time-lane pipeline.
//
// Replaces gs2d_temporal (reference kernels_nd.py:48-50, star-only there) for
// the row-major in-place sweep of BASELINE config 4 (9-point box), bit-exact
// with the oracle's lexicographic loop (oracle/oracle.py gs_sweep_loop; the
// reference loop test test_baselines.py:39-52).
//
// The paper's time lanes, on a GPU: lane t of a "group" runs sweep t, and
// group d owns the units {(sweep t, row d - t)}: a diagonal through
// (time, row) space.  With a lexicographic sweep every input of unit
// (t, i) comes from exactly three places:
//   * row i-1, sweep t   (NW, N, NE: new)      = group d-1, lane t
//   * row i,   sweep t-1 (C, E: old)           = group d-1, lane t-1
//   * row i+1, sweep t-1 (SW, S, SE: old)      = group d,   lane t-1
// plus W = the lane's own previous output.  So data only ever flows from
// group d-1 to group d and from lane t-1 to lane t: a one-directional chain.
//
//   * lanes:  lane t trails lane t-1 by lambda = 2 columns (its SE input is
//             what lane t-1 produced one step earlier: __shfl_up);
//   * warps:  a group is 4 warps (128 lanes = 128 sweeps); warp w trails
//             warp w-1 by mu extra columns (its lane 0 reads lane 31 of the
//             previous warp from shared memory);
//   * groups: group g of a block trails group g-1 by Lambda columns and
//             reads its outputs from a shared-memory ring indexed by
//             *iteration* (not column), so the 254-column lane skew inside a
//             group costs no ring space;
//   * blocks: G = 4 groups per block; one IO warp per block streams in the
//             previous block's last group (a tagged global ring, L2-resident)
//             and the grid rows the chain starts from, and drains this
//             block's last group to the next block.  Blocks take tickets and
//             only wait on lower tickets (plus bounded back-pressure), so the
//             launch is deadlock-free.
// "Virtual lane -1" of group g (ring slot 0) is grid row d_g + 1 at sweep
// t0 - 1: lane 0 reads its old own row / row below from there.  Lane lf = T - 1 (the last
// requested sweep of the pass) writes the final value of row d - lf back to
// the grid in place; lanes past it compute values nothing reads.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace tvs {

#ifdef GS2P_TRACE
// [cta][event] globaltimer stamps: 0 start, 1 group0 chunk 0 begins, 2 group0 chunk 100,
// 3 last group chunk 100, 4 first downstream publish, 5 compute done
__device__ unsigned long long g_trace[4096][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(n, e) do { if ((n) < 4096) g_trace[(n)][(e)] = gtimer(); } while (0)
// [cta<2][role] = {wait cycles, total cycles} over the first 100 chunks
// roles: 0 warp(0,0) 1 warp(0,3) 2 warp(3,0) 3 warp(3,3) 4 loader 5 drainer
__device__ unsigned long long g_wait[2][6][2];
#define WAITACC(n, r, w, t) do { if ((n) < 2) { atomicAdd(&g_wait[(n)][(r)][0], (w)); atomicAdd(&g_wait[(n)][(r)][1], (t)); } } while (0)
#else
#define TRACE(n, e) do { } while (0)
#endif

namespace gs2p {
constexpr int kLanes = 128;          // sweeps per pass (4 warps)
constexpr int kWarpsG = 4;
#ifndef GS2P_KG
#define GS2P_KG 4
#endif
constexpr int kG = GS2P_KG;          // groups per block
constexpr int kC = 4;                // iterations per chunk (sync granularity)
constexpr int kR = 32;               // ring depth (iterations), power of two
constexpr int kSlots = kLanes + 2;   // [0] virtual lane -1, [1] pad, [2 + t] lane t (16-B aligned pairs)
constexpr int kLam = 2;              // column lag lane t-1 -> t
constexpr int kMu = 3;               // extra lag warp w-1 -> w (>= kC + 1 - kLam)
constexpr int kBig = 5;              // lag group g-1 -> g (>= kC + 1)
constexpr int kBase = 10;            // every producer starts left of column 0 (>= kLam + kBig + 2)
// Global ring between clusters (blocks when CS = 1): rg iterations per
// boundary, kslots boundaries in flight — both sized at launch.  With G chain
// units resident, the oldest can run at most G * rg iterations ahead of the
// first unit not yet resident, and must reach c_end to retire, so the host
// makes G * rg >= 2 * c_end (no back-pressure deadlock for any width).
#ifndef GS2P_PUB
#define GS2P_PUB 4  // 8192^2 T=100: 1 55.5, 2 35.7, 4 31.7, 6 34.7, 8 39.6 ms
#endif
constexpr int kPub = GS2P_PUB;       // IO warps publish up/downstream every kPub chunks
constexpr int kComputeWarps = kG * kWarpsG;
constexpr int kPhLag = kBig * kG / kC;  // phantom chunk kl = producer chunk kl + kPhLag
constexpr bool kClusterOK = kBig * kG % kC == 0;  // DSMEM push needs a whole-chunk phantom lag
#ifndef GS2P_PUBLISHER
#define GS2P_PUBLISHER 1  // 1: a publisher warp takes the GPU-scope fence + progress store off the drainer
#endif
#ifndef GS2P_PUBP
#define GS2P_PUBP 2       // publisher: chunks per publication
#endif
constexpr int kPubP = GS2P_PUBP;
constexpr int kThreads = (kComputeWarps + 2 + GS2P_PUBLISHER) * 32;  // + loader, drainer (+ publisher)
constexpr int kRows = kR + kC;       // ring rows incl. kC mirror rows (chunk reads never wrap)
constexpr size_t kSmem = sizeof(double) * (size_t)(kG + 1) * kRows * kSlots;
static_assert(kMu >= kC + 1 - kLam && kBig >= kC + 1, "lags too small for chunked sync");
}  // namespace gs2p

struct Gs2pArgs {
  double* a;                 // interior origin (in place)
  long long s0;              // row pitch (elements)
  int e0, e1;                // rows, columns
  int sweeps;                // real sweeps this pass (<= 128)
  int nctas;
  int c_end;                 // iterations per warp (multiple of kC)
  double* gring;             // kslots * rg * 128
  int rg;                    // global ring depth (iterations, power of two)
  int kslots;                // global ring slots (boundaries in flight)
  unsigned long long* gprod; // kK tagged counters: (boundary+1) << 32 | iterations written
  unsigned long long* gcons; // kK tagged counters: (boundary+1) << 32 | iterations consumed
  int* ticket;
  const double* bndpad;       // 32 copies of the boundary value
  const unsigned* rows_ready; // drop-in pipeline: grid rows uploaded so far (nullptr: all resident)
  unsigned* blocks_done;      // drop-in pipeline: blocks finished, published in ticket order (or nullptr)
  double w[9];
  double bnd;
};

__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
// loader publication of io_load (experiment switch GS2P_RELAXED_LOAD)
__device__ __forceinline__ void st_io_load(int* p, int v) {
#ifdef GS2P_RELAXED_LOAD
  asm volatile("st.volatile.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
#else
  st_rel_cta(p, v);
#endif
}
__device__ __forceinline__ unsigned long long ld_acq_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- mbarrier chunk-completion rings (hardware-suspended waits) ----
// Warp X (compute warps 0..15, loader 16, drainer 17) completes its chunks in
// order; completion of chunk m is phase (m >> 3) of barrier bar[X][m & 7].
// Every waiter is at most 5 chunks behind / 3 ahead of the warp it waits on
// (RAW/WAR bounds), so a slot never wraps under a waiter (no ABA).
// ---- thread-block cluster helpers (distributed shared memory) ----
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}
// shared::cta address -> the same variable in CTA `rank` of the cluster
__device__ __forceinline__ unsigned mapa(const void* local, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smaddr(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ void remote_arrive(unsigned rbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void remote_arrive_tx(unsigned rbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar), "r"(bytes)
               : "memory");
}
// local shared memory -> shared memory of another CTA in the cluster, completion
// counted as transaction bytes on that CTA's mbarrier
__device__ __forceinline__ void push_s2s(unsigned rdst, const void* src, unsigned bytes, unsigned rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(rdst), "r"(smaddr(src)), "r"(bytes), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* b, unsigned parity) {
  // acquire at cluster scope: the phase was completed by another CTA
  auto try1 = [&] {
    unsigned ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smaddr(b)), "r"(parity) : "memory");
    return ok != 0;
  };
  if (try1()) return;
  const long long t0 = clock64();
  while (!try1())
    if (clock64() - t0 > (1ll << 34)) __trap();
}

// Wait until a shared-memory progress counter reaches `v`; back off so the
// spinning warps do not starve the IO warp of issue slots.
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  if (ld_acq_cta(p) >= v) return;
  SpinGuard sg;
  while (ld_acq_cta(p) < v) {
    __nanosleep(40);
    sg.tick();
  }
}

// taps in sorted order: NW N NE W C E SW S SE (mask bit k = position k)
template <unsigned MASK>
__device__ __forceinline__ double gs9(const double* w, double nw, double n, double ne, double ww, double c, double e,
                                      double sw, double s, double se) {
  const double v[9] = {nw, n, ne, ww, c, e, sw, s, se};
  double acc = 0.0;
  bool first = true;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if ((MASK >> k) & 1u) {
      acc = first ? tap_first(w[k], v[k]) : tap_next<false>(w[k], v[k], acc);
      first = false;
    }
  }
  return acc;
}

// CS > 1: consecutive blocks of the chain form a thread-block cluster; block
// r+1 of a cluster receives block r's last group through distributed shared
// memory (one bulk copy per chunk pushed by block r's drainer straight into
// block r+1's phantom ring, completing on block r+1's mbarrier) instead of the
// global ring — no GPU-scope fence on those hops.  Only the first block of a
// cluster reads the global ring.  WAR: block r+1's loader returns a credit
// (remote arrive) for phantom chunk kl once its group 0 finished chunk kl - 5;
// credit kl also tells block r that its chunk kl push completed, which lets
// block r's last group reuse those ring rows (pushed[]).
template <unsigned MASK, int CS>
__global__ void __launch_bounds__(gs2p::kThreads, 1) gs2d_pipe_kernel(Gs2pArgs p) {
  using namespace gs2p;
  extern __shared__ __align__(16) double smem[];
  // rings[0] = phantom (previous block's last group), rings[g+1] = group g
  auto ring = [&](int gi, int it, int slot) -> double& {
    return smem[((size_t)gi * kRows + (it & (kR - 1))) * kSlots + (slot == 0 ? 0 : slot + 1)];
  };
  auto ring_lane0 = [&](int gi, int it) -> double* { return &smem[((size_t)gi * kRows + (it & (kR - 1))) * kSlots + 2]; };
  // a write of ring row r < kC also goes to mirror row kR + r
  auto mirror_of = [&](double* p_row_elem, int it) -> double* { return (it & (kR - 1)) < kC ? p_row_elem + (size_t)kR * kSlots : nullptr; };
  constexpr int kLoader = kComputeWarps, kDrainer = kComputeWarps + 1;
  __shared__ unsigned long long bar[kComputeWarps + 2][8];
  // cluster hand-off: pbar = phantom chunk arrived (pushed by block r-1 or
  // filled by my loader), cbar = credits from block r+1, pushed = my chunk's
  // push to block r+1 complete
  __shared__ unsigned long long pbar[8], cbar[8], pushed[8];
  __shared__ int s_ticket;
  __shared__ int s_drained;  // chunks the drainer has finished (publisher warp)
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const unsigned crank = CS > 1 ? cluster_rank() : 0u;
  if (threadIdx.x == 0) {
    if (crank == 0) s_ticket = atomicAdd(p.ticket, 1) * CS;
    for (int x = 0; x < kComputeWarps + 2; ++x)
      for (int q = 0; q < 8; ++q) mbar_init(&bar[x][q], x == kLoader ? 32u : 1u);
    for (int q = 0; q < 8; ++q) {
      mbar_init(&pbar[q], 1u);
      mbar_init(&cbar[q], 1u);
      mbar_init(&pushed[q], 1u);
    }
    s_drained = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int n;  // block index along the chain
  if constexpr (CS > 1) {
    cluster_sync_all();  // every block's barriers initialised before any remote access
    int t0;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(t0) : "r"(mapa(&s_ticket, 0)) : "memory");
    n = t0 + (int)crank;
  } else {
    __syncthreads();
    n = s_ticket;
  }
  // "warp x completed chunk m" / "I completed chunk m"
  auto wait_chunk = [&](int x, int m) {
#ifndef GS2P_NOWAIT
    if (m >= 0) mbar_wait(&bar[x][m & 7], (unsigned)(m >> 3) & 1u);
#endif
  };
  if (threadIdx.x == 0) TRACE(n, 0);
  const int d0 = n * kG;            // first group (diagonal) of this block
  const int nch = p.c_end / kC;
  const double bnd = p.bnd;
  const int e0 = p.e0, e1 = p.e1;

  const bool has_up = n > 0, has_down = n + 1 < p.nctas;
  // lane lf = sweeps - 1 runs the last requested sweep: group d's lane lf
  // emits the final value of row d - lf.  Lanes past it compute values no
  // real lane or output ever reads, so no lane selects between sweep and
  // identity and every warp inside the grid runs the pure body.
  const int lf = p.sweeps - 1, lf_warp = lf / 32;
  const bool up_cl = CS > 1 && crank > 0;                 // phantom pushed by block n-1 (same cluster)
  const bool dn_cl = CS > 1 && crank + 1 < CS && has_down;  // push to block n+1 (same cluster)
  const bool up_gl = has_up && !up_cl, dn_gl = has_down && !dn_cl;
  auto ring_row = [&](int gi, int r) -> double* { return &smem[((size_t)gi * kRows + r) * kSlots]; };
  // global boundaries are between clusters: bd after my cluster, bd - 1 before
  const int kK = p.kslots, kRG = p.rg;
  const int bd = n / CS;
  const int up_slot = (bd - 1 + kK) % kK, dn_slot = bd % kK;
  const unsigned long long up_tag = (unsigned long long)bd << 32;        // boundary bd-1 -> tag bd
  const unsigned long long dn_tag = (unsigned long long)(bd + 1) << 32;  // boundary bd -> tag bd+1
  if (wi == kComputeWarps) {
    // ============ loader warp: grid rows (slot 0) + previous block's last group ============
    const double* up_ring = p.gring + (size_t)up_slot * kRG * kLanes;
    unsigned long long up_seen = 0;
#ifdef GS2P_TRACE
    long long lw = 0, lt0 = clock64();
#endif
    const double* bndsrc = p.bndpad;  // 32 copies of the boundary value (cp.async source)
    if (p.rows_ready) {
      // the drop-in path uploads row bands while this kernel runs: the only
      // grid rows a block reads are rows d0 .. d0 + kG (slot 0 of its rings)
      const unsigned need = (unsigned)min(e0, d0 + kG + 1);
      SpinGuard sg;
      unsigned have;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(have) : "l"(p.rows_ready) : "memory");
        if (have >= need) break;
        __nanosleep(256);
        sg.tick();
      }
    }
    for (int kl = 0; kl < nch; ++kl) {
#ifdef GS2P_TRACE
      const long long lws = clock64();
      if (kl == 100 && lane == 0) WAITACC(n, 4, (unsigned long long)lw, (unsigned long long)(lws - lt0));
#endif
      const int it_lo = kl * kC, it_hi = it_lo + kC;
      // WAR: the readers of the slots written below (group 0 -> phantom slots,
      // every group's warp 0 -> slot 0) finished chunk kl-5 (ring chunk kl-8 reusable)
      for (int q = 0; q < kWarpsG; ++q) wait_chunk(q, kl - 5);
      for (int g = 1; g < kG; ++g) wait_chunk(g * kWarpsG, kl - 5);
      if (up_cl && lane == 0) remote_arrive(mapa(&cbar[kl & 7], crank - 1));  // credit: phantom chunk kl writable
      // upstream data for producer iterations up to it_hi + Lambda*G
      if (up_gl) {
        const int up_need = min(it_hi + kBig * kG, p.c_end);
        SpinGuard guard;
        while ((up_seen >> 32) != (up_tag >> 32) || (up_seen & 0xffffffffull) < (unsigned long long)up_need) {
          up_seen = lane == 0 ? ld_acq_gpu(p.gprod + up_slot) : 0ull;
          up_seen = __shfl_sync(0xffffffffu, up_seen, 0);
          if ((up_seen >> 32) == (up_tag >> 32) && (up_seen & 0xffffffffull) >= (unsigned long long)up_need) break;
          __nanosleep(64);
          guard.tick();
        }
      }
#ifdef GS2P_TRACE
      lw += clock64() - lws;
#endif
      // slot 0 of rings -1..G-1: grid row d0+g+1 at column it + lam - Lambda*g - base
      // (also for a pushed phantom ring: the push carries only the lane slots,
      // block n-1's own slot 0 of those rows is reloaded by its loader)
      if (lane < (kG + 1) * kC) {
        const int g = lane / kC - 1, it = it_lo + lane % kC;
        const int row = d0 + g + 1, col = it + kLam - kBig * g - kBase;
        double* dst = &ring(g + 1, it, 0);
        double* mir = mirror_of(dst, it);
        const double* src = (row >= 0 && row < e0 && col >= 0 && col < e1) ? p.a + (long long)row * p.s0 + col : bndsrc;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smaddr(dst)), "l"(src));
        if (mir) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smaddr(mir)), "l"(src));
      }
      // phantom lanes: 4 iterations x 64 pairs, 16-byte copies (L2 only: the
      // global ring is rewritten every kRG iterations)
      if (!up_cl) {
#pragma unroll
        for (int q = 0; q < kC * kLanes / 64; ++q) {
          const int e = lane + 32 * q;  // pair index
          const int it = it_lo + e / (kLanes / 2), t = 2 * (e % (kLanes / 2));
          const int pit = it + kBig * kG;
          double* dst = ring_lane0(0, it) + t;
          double* mir = mirror_of(dst, it);
          const double* src = (has_up && pit < p.c_end) ? up_ring + (size_t)(pit & (kRG - 1)) * kLanes + t : bndsrc;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smaddr(dst)), "l"(src));
          if (mir) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smaddr(mir)), "l"(src));
        }
      } else if (it_hi + kBig * kG > p.c_end) {
        // block n-1 has no iterations left for these phantom rows: boundary
        for (int e = lane; e < kC * kLanes; e += 32) {
          const int r = (it_lo & (kR - 1)) + e / kLanes;
          ring_row(0, r)[2 + e % kLanes] = bnd;
          if (r < kC) ring_row(0, r + kR)[2 + e % kLanes] = bnd;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pbar[kl & 7]);
      }
      // the chunk's barrier phase completes when every lane's copies landed
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smaddr(&bar[kLoader][kl & 7])) : "memory");
      if (up_gl && ((kl + 1) % kPub == 0 || kl + 1 == nch)) {
        // producer iterations below it_hi + Lambda*G are no longer read from
        // the global ring once this chunk's copies completed
        wait_chunk(kLoader, kl);
        if (lane == 0) st_rel_gpu(p.gcons + up_slot, up_tag | (unsigned long long)min(it_hi + kBig * kG, p.c_end));
      }
    }
  } else if (wi == kComputeWarps + 1) {
    // ============ drainer warp: last group -> next block (global ring) ============
    double* dn_ring = p.gring + (size_t)dn_slot * kRG * kLanes;
    bool slot_ok = !dn_gl || bd < kK;
    unsigned long long dn_cons_seen = 0;
    SpinGuard guard;
#ifdef GS2P_TRACE
    long long dw = 0, dt0 = clock64();
#endif
    for (int ks = 0; ks < nch; ++ks) {
      const int lo = ks * kC;
#ifdef GS2P_TRACE
      const long long dws = clock64();
      if (ks == 100 && lane == 0) WAITACC(n, 5, (unsigned long long)dw, (unsigned long long)(dws - dt0));
#endif
      // the last group (forwarded downstream) and every group's warp lf_warp
      // (lane lf = the final sweep, written back to the grid here)
      for (int q = 0; q < kWarpsG; ++q) wait_chunk((kG - 1) * kWarpsG + q, ks);
      for (int g = 0; g + 1 < kG; ++g) wait_chunk(g * kWarpsG + lf_warp, ks);
      for (;;) {
        bool ok = true;
        if (ok && dn_gl && !slot_ok) {  // previous user of this global slot fully consumed
          unsigned long long v = lane == 0 ? ld_acq_gpu(p.gcons + dn_slot) : 0ull;
          v = __shfl_sync(0xffffffffu, v, 0);
          slot_ok = v >= (((unsigned long long)(bd + 1 - kK) << 32) | (unsigned long long)p.c_end);
          ok = slot_ok;
        }
        if (ok && dn_gl && lo + kC > kRG) {  // global back-pressure
          const unsigned long long need = dn_tag | (unsigned long long)(lo + kC - kRG);
          if (dn_cons_seen < need) {
            unsigned long long v = lane == 0 ? ld_acq_gpu(p.gcons + dn_slot) : 0ull;
            dn_cons_seen = __shfl_sync(0xffffffffu, v, 0);
          }
          ok = dn_cons_seen >= need;
        }
        if (ok) break;
        __nanosleep(20);
        guard.tick();
      }
#ifdef GS2P_TRACE
      dw += clock64() - dws;
#endif
      if (dn_cl && ks >= kPhLag) {
        // my chunk ks -> phantom chunk kl = ks - kPhLag of block n+1 (pit = it + kBig * kG)
        const int kl = ks - kPhLag;
        mbar_wait_cluster(&cbar[kl & 7], (unsigned)(kl >> 3) & 1u);  // block n+1 freed those rows
        if (lane == 0) {
          mbar_arrive(&pushed[kl & 7]);  // credit kl => my chunk kl push completed
          fence_proxy_async_smem();      // compute warps' ring writes -> async-proxy read
          // lane slots only: slot 0 of these rows is refilled by my loader
          // as soon as my compute warps are done with them
          const unsigned rb = mapa(&pbar[kl & 7], crank + 1);
          const int rdst = (kl * kC) & (kR - 1), rsrc = lo & (kR - 1);
          const unsigned bytes = (unsigned)(kLanes * sizeof(double));
          remote_arrive_tx(rb, (rdst < kC ? 2u : 1u) * kC * bytes);
#pragma unroll
          for (int u = 0; u < kC; ++u) {
            const double* src = ring_row(kG, rsrc + u) + 2;
            push_s2s(mapa(ring_row(0, rdst + u) + 2, crank + 1), src, bytes, rb);
            if (rdst < kC) push_s2s(mapa(ring_row(0, rdst + kR + u) + 2, crank + 1), src, bytes, rb);
          }
        }
      }
#ifndef GS2P_NODRAIN
      if (dn_gl) {
#pragma unroll
        for (int q = 0; q < kC * kLanes / 64; ++q) {
          const int e = lane + 32 * q;
          const int it = lo + e / (kLanes / 2), t = 2 * (e % (kLanes / 2));
          const double2 v = *reinterpret_cast<const double2*>(ring_lane0(kG, it) + t);
          *reinterpret_cast<double2*>(dn_ring + (size_t)(it & (kRG - 1)) * kLanes + t) = v;
        }
      }
      if (lane < kG * kC) {  // final outputs: lane lf of group g = row d_g - lf
        const int g = lane / kC, it = lo + lane % kC;
        const int row = d0 + g - lf;
        const int col = it - (kBase + kLam * lf + kMu * lf_warp + kBig * g);
        if (row >= 0 && row < e0 && col >= 0 && col < e1) p.a[(long long)row * p.s0 + col] = ring(g + 1, it, lf + 1);
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[kDrainer][ks & 7]);
#if GS2P_PUBLISHER
      if (lane == 0) st_rel_cta(&s_drained, ks + 1);  // monotone count for the publisher warp
#else
      if (dn_gl && ((ks + 1) % kPub == 0 || ks + 1 == nch)) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_rel_gpu(p.gprod + dn_slot, dn_tag | (unsigned long long)(lo + kC));
        if (lane == 0 && ks + 1 == kPub) TRACE(n, 4);
      }
#endif
    }
#if GS2P_PUBLISHER
  } else if (wi == kComputeWarps + 2) {
    // ============ publisher warp: GPU-scope progress for the next block ============
    // Waits for the drainer's chunks (its global-ring writes are then visible
    // here at CTA scope through the mbarrier's release/acquire), fences once
    // per kPubP chunks and stores the progress with release semantics: the
    // fence is cumulative over the drainer's writes, and the drainer never
    // stalls on it.  Lagging behind only delays (never advances) a publication.
    if (dn_gl) {
      int published = 0;
      SpinGuard guard;
      while (published < nch) {
        const int c = ld_acq_cta(&s_drained);  // chunks the drainer finished (monotone)
        if (c >= published + kPubP || (c == nch && c > published)) {
          __threadfence();
          __syncwarp();
          if (lane == 0) st_rel_gpu(p.gprod + dn_slot, dn_tag | (unsigned long long)(c * kC));
          published = c;
        } else {
          __nanosleep(32);
          guard.tick();
        }
      }
    }
#endif
  } else {

  // ======================= compute warps =======================
  const int g = wi / kWarpsG, w = wi % kWarpsG;
  const int t = w * 32 + lane;           // lane index in the group = sweep offset
  const int d = d0 + g;                  // diagonal of this group
  const int row = d - t;
  const bool row_ok = row >= 0 && row < e0;
  // per-lane output mode: 0 compute, 2 outside the grid (emits the boundary)
  const int mode = row_ok ? 0 : 2;
  const bool warp_pure = __all_sync(0xffffffffu, mode == 0);
  const int col_off = kBase + kLam * t + kMu * w + kBig * g;  // column = iteration - col_off
  const int offE = 1 - kLam - kBig - ((lane == 0 && w > 0) ? kMu : 0);
  const int offSE = 1 - kLam - (w > 0 ? kMu : 0);   // lane 0 only
  const int idxE = t == 0 ? 0 : t + 1;               // element index of lane t-1's slot (or virtual lane -1)
  const int idxSE = w == 0 ? 0 : 32 * w + 1;         // lane 32w-1 (or virtual lane -1)
  double* const base_prev = smem + (size_t)g * kRows * kSlots;        // ring of group g-1 (or phantom)
  double* const base_cur = smem + (size_t)(g + 1) * kRows * kSlots;   // ring of group g
  double wk[9];  // coefficients in registers (a shuffle makes them runtime values)
#pragma unroll
  for (int k = 0; k < 9; ++k) wk[k] = __shfl_sync(0xffffffffu, p.w[k], 0);
  // progress of the warps I read from / that read me
  // warps I read from (RAW, chunk k-1) and that read me (WAR, chunk k-5)
  const int dep_prev = g > 0 ? (g - 1) * kWarpsG + w : kLoader;
  const int dep_prev2 = (g > 0 && w > 0) ? (g - 1) * kWarpsG + w - 1 : -1;
  const int dep_left = w > 0 ? g * kWarpsG + w - 1 : -1;
  const bool needs_io = g == 0 || w == 0;
  const int war0 = g + 1 < kG ? (g + 1) * kWarpsG + w : kDrainer;
  const int war1 = (g + 1 < kG && w + 1 < kWarpsG) ? (g + 1) * kWarpsG + w + 1 : -1;
  // lane 31 of warp w is read by warp w+1 (warp 3's by the drainer, which
  // forwards / writes it); lane lf by the drainer (war3 below)
  const int war2 = w + 1 < kWarpsG ? g * kWarpsG + w + 1 : kDrainer;
  // the drainer also reads lane lf's slots (final outputs)
  const int war3 = (w == lf_warp && w + 1 < kWarpsG) ? kDrainer : -1;

  // shared::cta addresses of the chunk-completion rings this warp waits on
  const unsigned a_prev = smaddr(&bar[g > 0 ? dep_prev : 0][0]);
  const unsigned a_prev2 = smaddr(&bar[dep_prev2 >= 0 ? dep_prev2 : 0][0]);
  const unsigned a_left = smaddr(&bar[dep_left >= 0 ? dep_left : 0][0]);
  const unsigned a_loader = smaddr(&bar[kLoader][0]);
  const unsigned a_war0 = smaddr(&bar[war0][0]);
  const unsigned a_war1 = smaddr(&bar[war1 >= 0 ? war1 : 0][0]);
  const unsigned a_war2 = smaddr(&bar[war2][0]);
  const unsigned a_war3 = smaddr(&bar[war3 >= 0 ? war3 : 0][0]);
  double nw = bnd, nn = bnd, ne = bnd, cc = bnd, ee = bnd, sw = bnd, ss = bnd, se = bnd, ww = bnd, out = bnd;
#ifdef GS2P_TRACE
  long long t_wait = 0, t_start = 0;
#endif

  for (int k = 0; k < nch; ++k) {
    const int cb = k * kC;
    if (lane == 0 && w == 0 && g == 0 && (k == 0 || k == 100)) TRACE(n, k == 0 ? 1 : 2);
    if (lane == 0 && w == kWarpsG - 1 && g == kG - 1 && k == 100) TRACE(n, 3);
    if (lane == 0 && w == kWarpsG - 1 && g == kG - 1 && k == nch - 1) TRACE(n, 5);
#ifdef GS2P_TRACE
    const long long tw0 = clock64();
    if (k == 0) t_start = tw0;
#endif
    // RAW: producers finished chunk k-1 (the loader: chunk k); WAR: readers
    // of my ring slots finished chunk k-5 (the ring holds 8 chunks)
#ifndef GS2P_NOWAIT
    {
      // slot offset / parity per chunk distance, barrier bases per warp (above)
      const unsigned o1 = (unsigned)((k - 1) & 7) * 8u, q1 = (unsigned)((k - 1) >> 3) & 1u;
      const unsigned o0 = (unsigned)(k & 7) * 8u, q0 = (unsigned)(k >> 3) & 1u;
      const unsigned o5 = (unsigned)((k - 5) & 7) * 8u, q5 = (unsigned)((k - 5) >> 3) & 1u;
      if (k >= 1) {
        if (g > 0) mbar_wait_a(a_prev + o1, q1);
        if (dep_prev2 >= 0) mbar_wait_a(a_prev2 + o1, q1);
        if (dep_left >= 0) mbar_wait_a(a_left + o1, q1);
      }
      if (needs_io) mbar_wait_a(a_loader + o0, q0);
      if (up_cl && g == 0) mbar_wait_cluster(&pbar[k & 7], q0);
      if (dn_cl && g == kG - 1 && k >= 8) mbar_wait(&pushed[(k - 8) & 7], (unsigned)((k - 8) >> 3) & 1u);
      if (k >= 5) {
        mbar_wait_a(a_war0 + o5, q5);
        if (war1 >= 0) mbar_wait_a(a_war1 + o5, q5);
        mbar_wait_a(a_war2 + o5, q5);
        if (war3 >= 0) mbar_wait_a(a_war3 + o5, q5);
      }
    }
#endif
#ifdef GS2P_TRACE
    t_wait += clock64() - tw0;
    if (k == 100 && lane == 0) {
      const int role = (g == 0 && w == 0) ? 0 : (g == 0 && w == kWarpsG - 1) ? 1 : (g == kG - 1 && w == 0) ? 2 : (g == kG - 1 && w == kWarpsG - 1) ? 3 : -1;
      if (role >= 0) WAITACC(n, role, (unsigned long long)t_wait, (unsigned long long)(clock64() - t_start));
    }
#endif
    // steady chunk: every column of the chunk inside [0, e1) for every lane
    // of the warp and no negative ring iteration -> no guards, base pointers
    // with immediate per-iteration offsets (the ring has kC mirror rows)
    const int jmin = cb - (kBase + kLam * (w * 32 + 31) + kMu * w + kBig * g);
    const int jmax = cb + kC - 1 - (kBase + kLam * (w * 32) + kMu * w + kBig * g);
    const bool steady = jmin >= 0 && jmax < e1 && cb + offSE - kBig - kMu >= 0;
    if (steady) {
      const double* pNE = base_prev + ((cb + 1 - kBig) & (kR - 1)) * kSlots + t + 2;
      const double* pE = base_prev + ((cb + offE) & (kR - 1)) * kSlots + idxE;
      const double* pSE = base_cur + ((cb + offSE) & (kR - 1)) * kSlots + idxSE;
      double* pOut = base_cur + (cb & (kR - 1)) * kSlots + t + 2;
      const bool mirror = (cb & (kR - 1)) == 0;  // rows 0..kC-1 are mirrored at kR..kR+kC-1
      double outs[kC];
      // every ring input of the chunk is loaded before the first ring store:
      // the compiler cannot prove the stores do not alias the loads, so
      // interleaved they would serialise each iteration's loads behind the
      // previous iteration's whole accumulation chain.  (They do not alias:
      // pNE/pE read group g-1's ring, pSE another warp's lane slot or the
      // loader's slot 0, and everything read was published before this chunk.)
      double in_ne[kC], in_e[kC], in_se[kC];
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        in_ne[u] = pNE[u * kSlots];
        in_e[u] = pE[u * kSlots];
        in_se[u] = pSE[u * kSlots];
      }
      auto body = [&](auto pure_tag) {
        constexpr bool PURE = decltype(pure_tag)::value;
#pragma unroll
        for (int u = 0; u < kC; ++u) {
          const double ne_new = in_ne[u];
          const double e_new = in_e[u];
          const double sh = __shfl_up_sync(0xffffffffu, out, 1);
          const double se_new = lane == 0 ? in_se[u] : sh;
          nw = nn; nn = ne; ne = ne_new;
          cc = ee; ee = e_new;
          sw = ss; ss = se; se = se_new;
          const double v = gs9<MASK>(wk, nw, nn, ne, ww, cc, ee, sw, ss, se);
          if constexpr (PURE) {
            out = v;
          } else {
            out = mode == 0 ? v : bnd;
          }
          ww = out;
          pOut[u * kSlots] = out;
          outs[u] = out;
        }
      };
      if (warp_pure)
        body(std::true_type{});
      else
        body(std::false_type{});
      if (mirror) {
#pragma unroll
        for (int u = 0; u < kC; ++u) pOut[(kR + u) * kSlots] = outs[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        const int c = cb + u;
        const int j = c - col_off;
        const int i1 = c + 1 - kBig, i2 = c + offE, i3 = c + offSE;
        const double ne_new = i1 >= 0 ? base_prev[(i1 & (kR - 1)) * kSlots + t + 2] : bnd;
        const double e_new = i2 >= 0 ? base_prev[(i2 & (kR - 1)) * kSlots + idxE] : bnd;
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const double sl = i3 >= 0 ? base_cur[(i3 & (kR - 1)) * kSlots + idxSE] : bnd;
        const double se_new = lane == 0 ? sl : sh;
        nw = nn; nn = ne; ne = ne_new;
        cc = ee; ee = e_new;
        sw = ss; ss = se; se = se_new;
        const double v = gs9<MASK>(wk, nw, nn, ne, ww, cc, ee, sw, ss, se);
        const bool inside = row_ok && j >= 0 && j < e1;
        out = inside ? v : bnd;
        ww = out;
        const int r = c & (kR - 1);
        base_cur[r * kSlots + t + 2] = out;
        if (r < kC) base_cur[(r + kR) * kSlots + t + 2] = out;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar[wi][k & 7]);
  }
  }  // compute warps
  // no block of a cluster leaves while a peer may still push into / credit it
  if constexpr (CS > 1) cluster_sync_all();
  if (p.blocks_done) {
    // publish "blocks 0..n done" in ticket order (block n-1 is resident and
    // never waits on n, so this cannot deadlock); the drop-in path's download
    // stream waits on this count for the rows whose final values are written
    __syncthreads();
    if (threadIdx.x == 0) {
      SpinGuard sg;
      unsigned seen;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.blocks_done) : "memory");
        if (seen >= (unsigned)n) break;
        sg.tick();
      }
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.blocks_done), "r"((unsigned)n + 1u) : "memory");
    }
  }
#ifdef GS2P_TRACE
  if (threadIdx.x == 0) {
    TRACE(n, 6);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (n < 4096) g_trace[n][7] = smid;
  }
#endif
}

static unsigned gs_mask2d(const tvs_stencil& st, double w[9]) {
  unsigned mask = 0;
  int last = -1;
  for (int k = 0; k < 9; ++k) w[k] = 0.0;
  for (int k = 0; k < st.ntaps; ++k) {
    const int pos = (st.offsets[k][0] + 1) * 3 + (st.offsets[k][1] + 1);
    if (pos <= last) return 0;
    last = pos;
    mask |= 1u << pos;
    w[pos] = st.coeffs[k];
  }
  return mask;
}

bool gs2d_pipe_supported(const tvs_stencil& st) {
  double w[9];
  const unsigned m = gs_mask2d(st, w);
  constexpr unsigned kStar = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);
  return m == 0x1FFu || m == kStar;
}

// Drop-in pipeline hooks (api.cu gs2d_pipelined): the number of blocks one
// pass publishes on `blocks_done`, and how many must have exited before row
// `row` holds its final value (group row + steps - 1 is the last writer).
// Derived from the kernel's own constants so a -DGS2P_KG build stays correct.
int64_t gs2d_pipe_blocks(int64_t rows) { return (rows + gs2p::kLanes - 1 + gs2p::kG - 1) / gs2p::kG; }
int64_t gs2d_pipe_blocks_for_row(int64_t row, int64_t steps) {
  return std::min(gs2d_pipe_blocks(row + 1), (row + steps - 1) / gs2p::kG + 1);
}
int gs2d_pipe_max_sweeps() { return gs2p::kLanes; }

int gs2d_pipeline(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, cudaStream_t s,
                  const unsigned* rows_ready, unsigned* blocks_done) {
  using namespace gs2p;
  double w[9];
  const unsigned mask = gs_mask2d(st, w);
  constexpr unsigned kStar = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);
  if (mask != 0x1FFu && mask != kStar) return fail(TVS_ERR_UNSUPPORTED, "gs2d_pipeline: tap set");
  if (g.extents[0] >= (1ll << 30) || g.extents[1] >= (1ll << 30)) return fail(TVS_ERR_UNSUPPORTED, "gs2d_pipeline: extent");
  Gs2pArgs a{};
  a.a = grid + g.origin;
  a.s0 = g.strides[0];
  a.e0 = (int)g.extents[0];
  a.e1 = (int)g.extents[1];
  const int ngroups = a.e0 + kLanes - 1;
  a.nctas = (ngroups + kG - 1) / kG;
  const int skew = kLam * (kLanes - 1) + kMu * (kWarpsG - 1) + kBig * (kG - 1);
  a.c_end = ((a.e1 + 2 + kBase + skew + kBig * kG + kC - 1) / kC) * kC;
  for (int k = 0; k < 9; ++k) a.w[k] = w[k];
  a.bnd = st.boundary;
  double* bndpad = static_cast<double*>(scratch(sizeof(double) * 32, 2));
  if (!bndpad) return fail(TVS_ERR_CUDA, "gs2d_pipeline: scratch");
  {
    double h[32];
    for (double& x : h) x = st.boundary;
    TVS_CUDA(cudaMemcpyAsync(bndpad, h, sizeof(h), cudaMemcpyHostToDevice, s));
  }
  a.bndpad = bndpad;
  a.rows_ready = rows_ready;
  a.blocks_done = blocks_done;
  // Cluster size.  Consecutive blocks of a cluster hand off through
  // distributed shared memory, which shortens the block->block chain (the
  // bound for narrow grids: 8192x2048 T=100 29.3 ms at 1, 20.2 ms at 8) but
  // couples the blocks tightly and leaves SMs idle at cluster granularity,
  // which costs wide grids whose time is set by per-block speed (8192x8192:
  // 31.4 ms at 1, 48.7 at 8).  Measured crossover: a block's iteration count
  // c_end ~ 148 x 50.  TVS_GS2D_CLUSTER = 1, 2, 4 or 8 overrides.
  static const int cs_env = [] {
    const char* e = getenv("TVS_GS2D_CLUSTER");
    const int v = e ? atoi(e) : 0;
    return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
  }();
  const int cs_req = cs_env ? cs_env : (a.c_end < 148 * 50 ? 8 : 1);
  auto launch = [&](auto cs_tag) -> int {
    constexpr int CS = decltype(cs_tag)::value;
    if constexpr (CS > 1 && !kClusterOK) {
      return TVS_ERR_UNSUPPORTED;  // cluster hand-off needs a whole-chunk phantom lag
    } else {
    auto kern = mask == 0x1FFu ? gs2d_pipe_kernel<0x1FFu, CS> : gs2d_pipe_kernel<kStar, CS>;
    TVS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    Gs2pArgs b = a;
    b.nctas = (a.nctas + CS - 1) / CS * CS;  // tail blocks hold only out-of-grid rows
    cudaLaunchConfig_t lc{};
    cudaLaunchAttribute attr[1];
    lc.gridDim = dim3((unsigned)b.nctas);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = kSmem;
    lc.stream = s;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    // resident chain units: clusters (CS > 1) or blocks
    int units = 0;
    if (CS > 1) {
      if (cudaOccupancyMaxActiveClusters(&units, kern, &lc) != cudaSuccess || units < 1) {
        cudaGetLastError();
        return TVS_ERR_UNSUPPORTED;  // caller retries with CS = 1
      }
    } else {
      int per_sm = 0, dev = 0, sms = 0;
      TVS_CUDA(cudaGetDevice(&dev));
      TVS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      TVS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, kSmem));
      units = std::max(1, per_sm * sms);
    }
    int rg = 256;
    while ((long long)rg * units < 2ll * b.c_end + 64) rg *= 2;
    b.rg = rg;
    b.kslots = units + 2;
    const size_t ring_bytes = sizeof(double) * (size_t)b.kslots * rg * kLanes;
    const size_t ctrl_bytes = sizeof(unsigned long long) * 2 * b.kslots + 64;
    b.gring = static_cast<double*>(scratch(ring_bytes, 0));
    char* ctrl = static_cast<char*>(scratch(ctrl_bytes, 1));
    if (!b.gring || !ctrl) return fail(TVS_ERR_CUDA, "gs2d_pipeline: scratch");
    b.gprod = reinterpret_cast<unsigned long long*>(ctrl);
    b.gcons = b.gprod + b.kslots;
    b.ticket = reinterpret_cast<int*>(b.gcons + b.kslots);
    for (int64_t done = 0; done < steps; done += kLanes) {
      b.sweeps = (int)std::min<int64_t>(kLanes, steps - done);
      TVS_CUDA(cudaMemsetAsync(ctrl, 0, ctrl_bytes, s));
      TVS_CUDA(cudaLaunchKernelEx(&lc, kern, b));
      TVS_LAUNCHED("gs2d_pipe_kernel");
    }
    return TVS_OK;
    }
  };
  int rc = TVS_ERR_UNSUPPORTED;
  if (cs_req == 8) rc = launch(std::integral_constant<int, 8>{});
  else if (cs_req == 4) rc = launch(std::integral_constant<int, 4>{});
  else if (cs_req == 2) rc = launch(std::integral_constant<int, 2>{});
  if (rc == TVS_ERR_UNSUPPORTED) rc = launch(std::integral_constant<int, 1>{});
  return rc;
}

}  // namespace tvs
