// K6v3: 2D radius-1 Gauss-Seidel (9-point box / 5-point star) as time-lane
// groups advancing in per-iteration lockstep, fed by decoupled loader warps.
//
// Replaces gs2d_temporal (reference kernels_nd.py:48-50, star-only there) for
// the row-major in-place sweep of BASELINE config 4, bit-exact with the
// oracle's lexicographic loop (oracle/stencil_oracle.c gs_lex; the reference
// loop test test_baselines.py:39-52) and, with order = reference, with the
// reference's anti-diagonal gather/scatter (baselines.py:83-107: the NE
// neighbour is read from the previous sweep).
//
// The paper's time lanes.  A "group" is lr lanes (the pass's sweeps, rounded
// up to even); lane l runs sweep t0 + l and group d owns the units
// {(sweep l, row d - l)} (a diagonal through (time, row) space), streaming
// left to right over the columns, one column per iteration.  Every input of
// unit (l, row r = d - l, column c) is
//   NW, N, NE  row r-1, sweep l    = group d-1, lane l     (smem ring)
//   W          row r,   sweep l    = my previous output    (register)
//   C, E       row r,   sweep l-1  = group d-1, lane l-1   (smem ring)
//   SW, S, SE  row r+1, sweep l-1  = group d,   lane l-1   (smem ring)
// (reference order: NE = row r-1, sweep l-1 = group d-2, lane l-1), where
// "lane -1" of group d is grid row d+1 as it was before the pass.  Lane l
// trails lane l-1 by 2 columns and group g trails group g-1 by 2 iterations
// (LAM): the hyperplane slope of the dependence graph (h = 2 row + column + 4
// sweep), so the pipeline is no longer than the computation's critical path.
// Taps are summed in sorted order (NW N NE W C E SW S SE), unfused: bit-exact.
//
// CTA = G groups packed back to back into compute warps (T = 100: 5 x 100
// units on 16 warps; lanes beyond the pass's sweeps would cost the same as
// real ones) + 2 loader warps (4 in reference order), two CTAs per SM.  The
// compute warps meet at one named barrier per iteration (every warp does
// identical work; all ring reads are at compile-time offsets).  The loader
// warps are NOT in that barrier: they hand 4-iteration blocks over through
// named producer / consumer barriers (bar.arrive / bar.sync, four per
// direction) and run up to two blocks ahead, so neither the L2 latency of the
// CTA-to-CTA hand-off nor the loaders' instruction stream sits on the
// per-iteration critical path (K6v2 had one loader warp inside the
// barrier: 19.1 ms at config 4, 14.5 ms with the hand-off compiled out; this
// kernel: 13.8 ms, 11.2 ms).  Per block the loaders
//   * copy lane -1 of every group (grid rows, prefetched by cp.async one
//     block ahead) into ring slot 1;
//   * copy the previous CTA's last group(s) ("phantom" groups) from an L2
//     ring into the phantom rings.  The hand-off is fence-free: the producer
//     stores every output to an L2 ring whose cells hold a signalling-NaN
//     sentinel until written (arithmetic never yields a signalling NaN; the
//     boundary value is checked on the host); the consumer prefetches blocks
//     by cp.async one block ahead, re-polls cells that still hold the
//     sentinel and puts the sentinel back, so the ring is clean for its next
//     use.
// The run is a chain: a CTA starts one hop (~7 us: 10 iterations of lag, the
// L2 round trips of its first rows) after its producer, 1659 CTAs at config
// 4, 296 of them resident.
// CTAs take tickets and only wait on lower tickets; a ring slot is reused
// only after its consumer has exited.  Units outside the grid output the
// boundary; lane Tp-1 (the pass's last sweep) writes its row's final values
// to the grid in place.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace tvs {
namespace gsl {
#ifndef GSL_SLACK
#define GSL_SLACK 0
#endif
// Group lag and lane skew: 2 is the dependence graph's own slope (a value is
// read the iteration after it is produced); 3 gives every cross-lane value a
// spare iteration, so the compute warps load the next iteration's inputs
// before the barrier and the shared-memory round trip leaves the
// per-iteration critical path (one more column of pipeline per lane / group).
constexpr int kLam = 2 + GSL_SLACK;  // group lag (iterations)
constexpr int kSk = 2 + GSL_SLACK;   // lane skew (columns)
constexpr bool kPrefetch = GSL_SLACK > 0;
constexpr int kB = 2;            // every lane starts >= 2 columns left of column 0
constexpr int kR = 16;           // smem ring rows (iterations, power of two; the unroll of the compute loop)
#ifndef GSL_BLK
#define GSL_BLK 4
#endif
#ifndef GSL_DIST
#define GSL_DIST 1  // config 4 lexicographic / reference order, 1 / 2 / 3 blocks: 14.6 / 15.6 / 17.0 and 19.7 / 21.3 / 23.6 ms (a longer hand-off lag lengthens the 332-CTA start-up ramp)
#endif
constexpr int kBlk = GSL_BLK;    // iterations per loader block
constexpr int kDist = GSL_DIST;  // blocks requested ahead of their hand-over (L2 / HBM latency)
constexpr int kProMax = 12;      // most rows handed over before iteration 0 (Cfg::ProRows)
#ifndef GSL_NL
#define GSL_NL 0
#endif
constexpr int kLR = 32;          // lane -1 staging ring (iterations), power of two
#ifndef GSL_SLOTS
#define GSL_SLOTS 320
#endif
constexpr int kNumSlots = GSL_SLOTS;  // global ring slots (CTA boundaries in flight) >= resident CTAs
// sentinel of an unwritten global-ring cell: a signalling NaN (quiet bit
// clear), which no arithmetic result can be
constexpr unsigned long long kSent = 0x7FF4DEADBEEF0001ull;

// REF: reference (anti-diagonal) order; LC: lane capacity of a group (ring
// pitch; 32 / 64 / 102 / 128 -- 102 holds T = 100 in one pass)
template <bool REF, int LC>
struct Cfg {
#ifndef GSL_G
#define GSL_G 0
#endif
  // groups per CTA (two CTAs per SM).  Config 4 lexicographic, packed lanes,
  // K6v2 loader: G 4 / 5 21.2 / 19.1 ms; without hand-off 12.0 / 11.5 ms
#ifndef GSL_GREF
#define GSL_GREF 0
#endif
  // reference order, config 4: G 4 / 5 18.85 / 17.95 ms
  static constexpr int G = REF ? (GSL_GREF > 0 ? GSL_GREF : (LC <= 102 ? 5 : 4)) : (GSL_G > 0 ? GSL_G : (LC <= 102 ? 5 : 4));
  static constexpr int Ph = REF ? 2 : 1;        // phantom groups (reads reach group d-2 in REF)
  static constexpr int S = LC + 2;              // ring row: [pad][lane -1][lanes 0..LC-1] (16-B aligned lanes)
  static constexpr int Rings = G + Ph;          // ring index = local group + Ph
  static constexpr int Compute = (G * LC + 31) / 32;  // compute warps at full capacity
  // loader warps: warp w hands over rows [w, w + 1) * kBlk / NL of every
  // block.  One warp could not keep up (config 4: 20.6 ms, the compute warps
  // waiting on it 44% of the time); lexicographic 2 / 4 warps: 15.6 / 17.0
  // ms, reference order (two phantom groups): 26.3 / 21.3 ms
  static constexpr int NL = GSL_NL > 0 ? GSL_NL : (REF ? 4 : 2);
  static_assert(kBlk % NL == 0, "loader warps split a block's rows");
  static constexpr int Threads = (Compute + NL) * 32;
  static constexpr int RowCells = Ph * LC;      // cells of one phantom row (L2 ring and staging pitch)
  static constexpr int Back = REF ? kSk + 2 * kLam - 1 : kSk + kLam - 1;  // deepest ring read behind m
  // ring row i is last read in iteration i + Back and overwritten by row
  // i + kR: the loader may write block b once block b - Ahead is complete
  static constexpr int Ahead = (kR - Back) / kBlk < 3 ? (kR - Back) / kBlk : 3;  // <= 3: four barriers per direction
  static_assert(Ahead >= 2, "the loader must be able to run a block ahead");
  // phantom / lane -1 rows handed over before iteration 0: the rows the first
  // iterations read behind them, in whole blocks (4 lexicographic, 8 reference order)
  static constexpr int ProRows = (Back + 1 + kBlk - 1) / kBlk * kBlk;
  static_assert(ProRows <= kProMax && kLam * G >= ProRows, "prologue rows must be rows the producer hands over");
  static constexpr int Stg = kDist + 1 > ProRows / kBlk ? kDist + 1 : ProRows / kBlk;  // phantom staging slots
  static constexpr size_t Smem =
      sizeof(double) * ((size_t)Rings * (kR * S + 16) + (size_t)Rings * kLR + (size_t)Stg * kBlk * RowCells);
  // CTAs per SM the shared memory (and 2048 threads) allow, at most 3
  static constexpr int MinB = (3 * (Smem + 1024) <= 227 * 1024 && 3 * Threads <= 2048) ? 3
                              : (2 * (Smem + 1024) <= 227 * 1024 ? 2 : 1);
  static_assert(Rings * kBlk <= 32, "one lane -1 cell per loader lane and block");
  static_assert(kLR >= (kDist + 1) * kBlk + kProMax, "lane -1 staging ring too shallow");
  static_assert(LC % 2 == 0 && (S * 8) % 16 == 0, "16-byte ring rows");
};
}  // namespace gsl

#ifdef GSL_TRACE
// [cta][0] start ns, [1] first iteration ns, [2] end ns, [3] loader cycles waiting for compute,
// [4] loader cycles re-polling the L2 ring, [5] compute warp 0 cycles waiting for the loader
__device__ unsigned long long g_gsl_trace[8192][8];
__device__ __forceinline__ unsigned long long gsl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

struct GslArgs {
  double* a;          // interior origin (in place)
  long long s0;       // row pitch (elements)
  int e0, e1;         // rows, columns
  int tp;             // sweeps of this pass (<= lr)
  int lr;             // lanes per group in use (even, <= LC): groups are packed into warps
  int nctas;
  int m_end;          // iterations per CTA (multiple of kR)
  double* gring;      // kNumSlots x m_end x RowCells (sentinel until written)
  int* done;          // [slot]: consumer CTAs of this slot that exited (their ticket)
  int* epoch;         // [slot]: boundary + 1 of the producer that owns the slot now
  int* ticket;
  const unsigned* rows_ready;  // drop-in pipeline: grid rows uploaded so far (nullptr: all resident)
  unsigned* blocks_done;       // drop-in pipeline: CTAs finished, published in ticket order (or nullptr)
  double w[9];
  double bnd;
};

// 9 sorted taps NW N NE W C E SW S SE (mask bit k = tap k), unfused
template <unsigned MASK>
__device__ __forceinline__ double gsl_taps(const double* w, double nw, double n, double ne, double ww, double c,
                                           double e, double sw, double s, double se) {
  const double v[9] = {nw, n, ne, ww, c, e, sw, s, se};
  double acc = 0.0;
  bool first = true;
#pragma unroll
  for (int k = 0; k < 9; ++k)
    if ((MASK >> k) & 1u) {
      acc = first ? tap_first(w[k], v[k]) : tap_next<false>(w[k], v[k], acc);
      first = false;
    }
  return acc;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smaddr(smem)), "l"(gmem));
}
// L2-only (cg): the ring cells are written by other SMs
__device__ __forceinline__ void cp_async16g(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smaddr(smem)), "l"(gmem));
}
__device__ __forceinline__ void st_relaxed_gpu(double* p, unsigned long long v) {
#if defined(GSL_ST_WEAK)
  asm volatile("st.weak.global.cg.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#elif defined(GSL_ST_NONE)
  (void)p; (void)v;
#else
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#endif
}
__device__ __forceinline__ int ld_acquire_gpu32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_relaxed_gpu2(const double* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool gsl_is_sent(const double2& v) {
  return (__double_as_longlong(v.x) == (long long)gsl::kSent) | (__double_as_longlong(v.y) == (long long)gsl::kSent);
}
// Named barriers.  1: the compute warps' per-iteration barrier (the loader is
// not part of it).  kBarFill + (b & 3): block b handed over -- the loader
// arrives, every compute warp waits (in place of barrier 1 at the end of the
// block's first iteration).  kBarDone + (b & 3): block b's iterations finished
// -- compute warp 0 arrives, the loader waits.  Waiting warps are suspended by
// the hardware (a spinning shared-memory poll starved the loader of issue
// slots: 32 ms instead of 19).  At most three blocks are outstanding on
// either side, so four barriers each never alias.
constexpr int kBarFill = 2, kBarDone = 6, kBarPro = 10;
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
template <unsigned MASK, bool REF, int LC>
__global__ void __launch_bounds__(gsl::Cfg<REF, LC>::Threads, gsl::Cfg<REF, LC>::MinB) gs2d_lane_kernel(GslArgs p) {
  using namespace gsl;
  using C = Cfg<REF, LC>;
  constexpr int kG = C::G, kPh = C::Ph, kS = C::S, kRings = C::Rings, kRowCells = C::RowCells, kNL = C::NL;
  extern __shared__ __align__(16) double smem[];
  // Ring g starts rstride cells after ring g-1: kR rows plus a pad chosen so
  // that a warp straddling two packed groups (lanes 96..99 of one, 0..27 of
  // the next at lr = 100) touches 32 consecutive banks instead of the same
  // ones twice (ncu: 9% of the kernel's shared-memory wavefronts were
  // conflicts).  The pad is exact for lr = 100 (T = 100, capacity 102) and
  // compile-time (a run-time stride costs the register the kernel lacks)
  constexpr int rstride = kR * kS + (LC == 102 ? 100 % 16 : 0);
  double* const lm1 = smem + (size_t)kRings * (kR * kS + 16);  // lane -1 staging [ring][kLR]
  double* const stg = lm1 + kRings * kLR;                 // phantom staging [Stg][kBlk][RowCells]
  __shared__ int s_ticket;
  // the warp index through a shuffle: the compiler then knows it is warp-uniform
  // (uniform branches and uniform registers for the role split)
  const int lane = threadIdx.x & 31, wi = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lr = p.lr, nunits = kG * lr;
  const int ncomp = (nunits + 31) >> 5;  // compute warps; the loader is warp ncomp
  const int cthreads = ncomp * 32;
  const double bnd = p.bnd;
  // every ring cell starts as the boundary (iterations before 0 are columns
  // left of the grid)
  for (int i = threadIdx.x; i < kRings * (kR * kS + 16 + kLR); i += blockDim.x) smem[i] = bnd;
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1);
  __syncthreads();
  const int n = s_ticket;  // position in the CTA chain
#ifdef GSL_TRACE
  if (threadIdx.x == 0 && n < 8192) g_gsl_trace[n][0] = gsl_now();
  long long tr_wait = 0, tr_poll = 0;
#endif
  const int d0 = n * kG;   // global group of local group 0
  const int m_end = p.m_end;
  const int e0 = p.e0, e1 = p.e1;
  const int slot_in = (n - 1 + kNumSlots) % kNumSlots, slot_out = n % kNumSlots;
#ifdef GSL_NO_UP  // experiment: no CTA-to-CTA hand-off (wrong results; timing only)
  const bool has_up = false, has_down = false;
#else
  const bool has_up = n > 0, has_down = n + 1 < p.nctas;
#endif
  double* const gin = p.gring + (size_t)slot_in * m_end * kRowCells;
  double* const gout = p.gring + (size_t)slot_out * m_end * kRowCells;
  if (has_down && threadIdx.x == 0) {
    // ring slot reuse: the consumer of boundary n - kNumSlots (a lower
    // ticket, so started) must have exited -- read and reset every cell --
    // before this CTA writes the slot; then the slot is published as mine
    if (n >= kNumSlots) {
      const long long t0 = clock64();
      while (ld_acquire_gpu32(p.done + slot_out) < n - kNumSlots + 1) {
        __nanosleep(256);
        if (clock64() - t0 > (1ll << 34)) __trap();
      }
    }
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.epoch + slot_out), "r"(n + 1) : "memory");
  }
  __syncthreads();
  // producer rows a consumer reads: its rows >= -ProRows, i.e. >= LAM*G - ProRows here
  const int ring_lo = kLam * kG - C::ProRows;

  if (wi < ncomp) {
    // ---------------- compute warp: packed unit = group g, lane l ----------
    // (the last warp's spare threads shadow the last unit and store nothing)
    const bool live = (int)threadIdx.x < nunits;
    const int unit = live ? (int)threadIdx.x : nunits - 1;
    const int g = unit / lr, l = unit - g * lr;
    const int d = d0 + g, row = d - l;
    const int col0 = -kLam * g - kSk * l - kB;  // my column at iteration 0
    double* const ring_me = smem + (size_t)(g + kPh) * rstride;
    const double* const ring_up = ring_me - rstride;
    const double* const ring_up2 = ring_me - 2 * rstride;
    const bool emit = live && l == p.tp - 1;  // last sweep of the pass: final values
    double* const arow = p.a + (long long)row * p.s0;
    const bool to_ring = live && has_down && g >= kG - kPh;  // phantom source of the next CTA
    double* const gdst = gout + (size_t)(g - (kG - kPh)) * LC + l;
    // this warp's units all inside the grid (rows, and columns for iterations
    // [m_in0, m_in1)): the steady body needs no selects
    const bool row_ok = row >= 0 && row < e0;
    const bool rows_in = __all_sync(0xffffffffu, row_ok);
    const int m_in0 = __reduce_max_sync(0xffffffffu, -col0), m_in1 = __reduce_min_sync(0xffffffffu, e1 - col0);
    double nw = bnd, nn = bnd, ne = bnd, ww = bnd, cc = bnd, ee = bnd, sw = bnd, ss = bnd, se = bnd;
    double out = bnd;
    bar_sync(kBarPro, cthreads + 32 * kNL);  // prologue rows handed over
    double ne_p = bnd, e_p = bnd, se_p = bnd, rn_p = bnd;  // inputs of the next iteration (kPrefetch)
    if constexpr (kPrefetch) {
      ne_p = ring_up[((-(kLam - 1)) & (kR - 1)) * kS + 2 + l];
      e_p = ring_up[((-(kSk + kLam - 1)) & (kR - 1)) * kS + 1 + l];
      se_p = ring_me[((-(kSk - 1)) & (kR - 1)) * kS + 1 + l];
      if constexpr (REF) rn_p = ring_up2[((-(kSk + 2 * kLam - 1)) & (kR - 1)) * kS + 1 + l];
    }
    (void)ne_p, (void)e_p, (void)se_p, (void)rn_p;
#ifdef GSL_TRACE
    if (wi == 0 && lane == 0 && n < 8192) g_gsl_trace[n][1] = gsl_now();
#endif
    for (int mb = 0; mb < m_end; mb += kR) {
      const bool steady = rows_in && mb >= m_in0 && mb + kR <= m_in1;
      auto block = [&](auto steady_tag) {
        constexpr bool ST = decltype(steady_tag)::value;
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const int m = mb + u;
          // every input is a shared-memory ring read at a compile-time offset
          // (slot 1 of a ring = its lane -1, a grid row, copied in by the
          // loader); no shuffles, no per-lane special cases
          // ring rows behind m: NE kLam - 1, SE kSk - 1, E kSk + kLam - 1 (REF NE: kSk + 2 kLam - 1)
          constexpr int dNE = kLam - 1, dSE = kSk - 1, dE = kSk + kLam - 1;
          [[maybe_unused]] constexpr int dRN = kSk + 2 * kLam - 1;
          double ne_use;
          if constexpr (kPrefetch) {
            // this iteration's inputs were loaded before the previous barrier;
            // the next iteration's (rows <= m - 1, visible since that barrier) go out now
            nw = nn; nn = ne; ne = ne_p;
            cc = ee; ee = e_p;
            sw = ss; ss = se; se = se_p;
            ne_use = REF ? rn_p : ne;
            ne_p = ring_up[((u + 1 - dNE) & (kR - 1)) * kS + 2 + l];
            e_p = ring_up[((u + 1 - dE) & (kR - 1)) * kS + 1 + l];
            se_p = ring_me[((u + 1 - dSE) & (kR - 1)) * kS + 1 + l];
            if constexpr (REF) rn_p = ring_up2[((u + 1 - dRN) & (kR - 1)) * kS + 1 + l];
          } else {
            const double ne_new = ring_up[((u - dNE) & (kR - 1)) * kS + 2 + l];  // group d-1, lane l
            const double e_new = ring_up[((u - dE) & (kR - 1)) * kS + 1 + l];    // group d-1, lane l-1 (lane 0: grid row d)
            const double se_new = ring_me[((u - dSE) & (kR - 1)) * kS + 1 + l];  // my group, lane l-1 (lane 0: grid row d+1)
            nw = nn; nn = ne; ne = ne_new;
            cc = ee; ee = e_new;
            sw = ss; ss = se; se = se_new;
            ne_use = ne;
            if constexpr (REF) ne_use = ring_up2[((u - dRN) & (kR - 1)) * kS + 1 + l];  // group d-2, lane l-1 (lane 0: grid row d-1)
          }
          const double v = gsl_taps<MASK>(p.w, nw, nn, ne_use, ww, cc, ee, sw, ss, se);
          bool inside = true;
          if constexpr (ST) {
            out = v;
          } else {
            const int c = col0 + m;
            inside = row_ok && c >= 0 && c < e1;
            out = inside ? v : bnd;
          }
          ww = out;
          if (live) ring_me[(u & (kR - 1)) * kS + 2 + l] = out;
          if (to_ring && m >= ring_lo) st_relaxed_gpu(gdst + (size_t)m * kRowCells, __double_as_longlong(out));
          if (emit && inside) arow[col0 + m] = out;
          // iteration m done in every compute warp; iteration m + 1 of a
          // block's first iteration reads the block's first loader row
          if (u % kBlk == 0) {
#ifdef GSL_TRACE
            const long long tw0 = clock64();
#endif
            bar_sync(kBarFill + ((u / kBlk) & 3), cthreads + 32 * kNL);
#ifdef GSL_TRACE
            tr_wait += clock64() - tw0;
#endif
          } else {
            bar_sync(1, cthreads);
          }
          if (u % kBlk == kBlk - 1 && wi == 0) bar_arrive(kBarDone + ((u / kBlk) & 3), 32 + 32 * kNL);
        }
      };
      if (steady)
        block(std::true_type{});
      else
        block(std::false_type{});
    }
#ifdef GSL_TRACE
    if (wi == 0 && lane == 0 && n < 8192) {
      g_gsl_trace[n][2] = gsl_now();
      g_gsl_trace[n][5] = tr_wait;
    }
#endif
  } else {
    // ---------------- loader (one warp, decoupled) ---------------------------
    // Block q = rows [4q, 4q + 4) of every ring:
    //  * lane -1 of ring ri (local group g = ri - kPh, global d0 + g) at row i
    //    = grid row d0 + g + 1 at column i - LAM*g + 2 - B;
    //  * phantom row i = the previous CTA's last kPh groups at producer
    //    iteration i + LAM*G (rows past its last iteration are columns right
    //    of the grid: the boundary).
    // request(q) starts the copies (grid rows -> lane -1 staging, L2 ring ->
    // phantom staging), finish(q) -- kDist blocks later -- validates the
    // phantom cells (sentinel: re-polled until written), resets them in the
    // L2 ring, copies everything into the rings and publishes the block.
    constexpr int kStgBlock = kBlk * kRowCells;
    // A lane's 16-byte pieces of a block sit at compile-time offsets from its
    // lane base: row r (< kBlk), cells 2 lane + 64 s and the next one, for
    // s < kSeg (the 32-lane segments of a row) -- no per-piece index
    // arithmetic (the first K6v3 loader spent ~400 dependent integer
    // instructions per block on it and was the kernel's bottleneck).
    constexpr int kSeg = (LC / 2 + 31) / 32;  // pieces per lane and row
    bool seg_on[kSeg];                        // the segment's pair lies inside the lanes in use
#pragma unroll
    for (int sg = 0; sg < kSeg; ++sg) seg_on[sg] = 2 * lane + 64 * sg < lr;
    // lane -1: loader lane t < kRings * kBlk owns ring t / kBlk, row offset t % kBlk
    const int lm_ri = lane / kBlk, lm_o = lane % kBlk, lm_g = lm_ri - kPh, lm_r = d0 + lm_g + 1;
    const int lw = wi - ncomp;  // loader warp: its rows of a block are [lw_r0, lw_r0 + kSubR)
    constexpr int kSubR = kBlk / kNL;
    const int lw_r0 = lw * kSubR;
    const bool lm_on = lw == 0 && lane < kRings * kBlk, lm_row = lm_r >= 0 && lm_r < e0;
    const int lm_c0 = lm_o - kLam * lm_g + kSk - kB;  // grid column of row 4q + lm_o at q = 0
    const double* const lm_src = p.a + (long long)lm_r * p.s0;
    auto rows_in_ring = [&](int i) { return has_up && i + kLam * kG < m_end; };
    // a ring cell only this lane stores in every finish() (read back before the hand-over):
    // its lane -1 slot, or -- lanes without one -- its first phantom pair (always inside the lanes in use)
    int lane_cell = 0;
    int rq_slot = 0, fin_slot = 0;  // phantom staging slots of the next request / finish
    auto request = [&](int q) {
      const int i0 = q * kBlk;
      if (lm_on) {
        const int c = i0 + lm_c0;
        double* dst = lm1 + lm_ri * kLR + ((i0 + lm_o) & (kLR - 1));
        if (lm_row && c >= 0 && c < e1)
          cp_async8(dst, lm_src + c);
        else
          *dst = bnd;
      }
      const bool full = rows_in_ring(i0 + kBlk - 1);
      if (full || rows_in_ring(i0)) {
#pragma unroll 1
        for (int ph = 0; ph < kPh; ++ph) {
          double* sb = stg + rq_slot * kStgBlock + lw_r0 * kRowCells + ph * LC + 2 * lane;
          const double* gb = gin + (long long)(i0 + lw_r0 + kLam * kG) * kRowCells + ph * LC + 2 * lane;
#pragma unroll
          for (int r = 0; r < kSubR; ++r)
#pragma unroll
            for (int sg = 0; sg < kSeg; ++sg)
              if (seg_on[sg] && (full || rows_in_ring(i0 + lw_r0 + r)))
                cp_async16g(sb + r * kRowCells + 64 * sg, gb + r * kRowCells + 64 * sg);
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      rq_slot = rq_slot == C::Stg - 1 ? 0 : rq_slot + 1;
    };
    auto finish = [&](int q) {
      const int i0 = q * kBlk;
      const bool full = rows_in_ring(i0 + kBlk - 1);
#pragma unroll 1
      for (int ph = 0; ph < kPh; ++ph) {
        {
          const int r0 = lw_r0;  // this loader warp's rows
          const double* sb = stg + fin_slot * kStgBlock + r0 * kRowCells + ph * LC + 2 * lane;
          double* const gb = gin + (long long)(i0 + r0 + kLam * kG) * kRowCells + ph * LC + 2 * lane;
          double* const rb = smem + (size_t)ph * rstride + ((i0 + r0) & (kR - 1)) * kS + 2 + 2 * lane;
          double2 got[kSubR * kSeg];
          unsigned live_mask = 0;  // pieces that come from the L2 ring
          bool bad = false;
#pragma unroll
          for (int r = 0; r < kSubR; ++r)
#pragma unroll
            for (int sg = 0; sg < kSeg; ++sg) {
              const int j = r * kSeg + sg;
              got[j] = make_double2(bnd, bnd);
              if (seg_on[sg] && (full || rows_in_ring(i0 + r0 + r))) {
                live_mask |= 1u << j;
                got[j] = *reinterpret_cast<const double2*>(sb + r * kRowCells + 64 * sg);
                bad |= gsl_is_sent(got[j]);
              }
            }
          if (__any_sync(0xffffffffu, bad)) {
            // late cells (the consumer caught up with its producer): re-read
            // every late pair at once until all have landed
            const long long t0 = clock64();
            do {
              bad = false;
#pragma unroll
              for (int r = 0; r < kSubR; ++r)
#pragma unroll
                for (int sg = 0; sg < kSeg; ++sg) {
                  const int j = r * kSeg + sg;
                  if ((live_mask >> j & 1u) && gsl_is_sent(got[j])) {
                    got[j] = ld_relaxed_gpu2(gb + r * kRowCells + 64 * sg);
                    bad |= gsl_is_sent(got[j]);
                  }
                }
              if (clock64() - t0 > (1ll << 34)) __trap();
            } while (__any_sync(0xffffffffu, bad));
#ifdef GSL_TRACE
            tr_poll += clock64() - t0;
#endif
          }
#pragma unroll
          for (int r = 0; r < kSubR; ++r)
#pragma unroll
            for (int sg = 0; sg < kSeg; ++sg) {
              const int j = r * kSeg + sg;
              if (seg_on[sg]) {
#ifndef GSL_NO_RESET
                if (live_mask >> j & 1u)
                  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(gb + r * kRowCells + 64 * sg),
                               "l"(kSent), "l"(kSent)
                               : "memory");
#endif
                *reinterpret_cast<double2*>(rb + r * kS + 64 * sg) = got[j];
              }
            }
        }
      }
      fin_slot = fin_slot == C::Stg - 1 ? 0 : fin_slot + 1;
      // lane -1 of every ring -> ring slot 1
      if (lm_on) {
        const int i = i0 + lm_o;
        lane_cell = lm_ri * rstride + (i & (kR - 1)) * kS + 1;
        smem[lane_cell] = lm1[lm_ri * kLR + (i & (kLR - 1))];
      } else {
        lane_cell = (kPh - 1) * rstride + ((i0 + lw_r0 + kSubR - 1) & (kR - 1)) * kS + 2 + 2 * lane;  // last row, segment 0
      }
    };
    // Hand-over: the block's shared-memory stores must be performed before
    // the arrival.  A block-scope fence would also wait for this warp's
    // global traffic in flight (the sentinel resets and the cp.async of the
    // next blocks: an L2 round trip per block, which made the loader the
    // kernel's bottleneck).  bar.arrive already orders the arriving
    // thread's earlier accesses for the threads the barrier releases; the
    // read-back of the last cell this lane stored additionally keeps the
    // arrival behind the stores in the warp's own instruction stream
    // (shared-memory accesses of a warp complete in order).
    auto publish = [&](int bar, const double* last_store) {
      unsigned long long echo;
      asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(echo) : "r"(smaddr(last_store)) : "memory");
      asm volatile("{ .reg .pred p; setp.eq.u64 p, %2, 0x7FF4DEADBEEF0002; @!p bar.arrive %0, %1; @p bar.arrive %0, %1; }"
                   ::"r"(bar), "r"(cthreads + 32 * kNL), "l"(echo) : "memory");
    };
    if (has_up) {
      // the incoming slot holds my producer's cells only once the producer
      // took it over (after its previous consumer reset every cell); before
      // that its cells may still hold the previous boundary's values
      const long long t0 = clock64();
      while (ld_acquire_gpu32(p.epoch + slot_in) != n) {
        __nanosleep(128);
        if (clock64() - t0 > (1ll << 35)) __trap();
      }
    }
    if (p.rows_ready) {
      // the drop-in path uploads row bands while this kernel runs: this
      // CTA reads grid rows d0 - kPh + 1 .. d0 + G (its rings' lane -1)
      const unsigned need = (unsigned)min(e0, d0 + kG + 1);
      const long long t0 = clock64();
      for (;;) {
        unsigned have;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(have) : "l"(p.rows_ready) : "memory");
        if (have >= need) break;
        __nanosleep(256);
        if (clock64() - t0 > (1ll << 35)) __trap();
      }
    }
    const int nb = m_end / kBlk;
    constexpr int kProBlocks = C::ProRows / kBlk;
    // prologue rows -ProRows..-1, then blocks 0 .. kDist-1 in flight
    static_assert(kProBlocks <= C::Stg, "prologue blocks share the staging slots");
    if constexpr (kProBlocks + kDist <= C::Stg) {
      // the prologue blocks and the first kDist blocks in one L2 round trip
      for (int q = -kProBlocks; q < kDist; ++q) request(q);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kDist) : "memory");  // the prologue blocks landed
      for (int q = -kProBlocks; q < 0; ++q) finish(q);
    } else {
      for (int q = -kProBlocks; q < 0; ++q) request(q);  // one L2 round trip for all of them
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      for (int q = -kProBlocks; q < 0; ++q) finish(q);
      for (int q = 0; q < kDist; ++q) request(q);
    }
    publish(kBarPro, smem + (size_t)lane_cell);
    for (int b = 0; b < nb; ++b) {
      if (b + kDist < nb)
        request(b + kDist);
      else
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kDist) : "memory");  // block b's copies landed
      if (b >= C::Ahead) {
        // ring rows of block b still hold block b - kR / kBlk, read until
        // block b - Ahead completes
#ifdef GSL_TRACE
        const long long tw0 = clock64();
#endif
        bar_sync(kBarDone + ((b - C::Ahead) & 3), 32 + 32 * kNL);
#ifdef GSL_TRACE
        tr_wait += clock64() - tw0;
#endif
      }
      finish(b);
      publish(kBarFill + (b & 3), smem + (size_t)lane_cell);
    }
    // the last blocks' completions (keeps every barrier balanced at exit)
    for (int b = nb > C::Ahead ? nb - C::Ahead : 0; b < nb; ++b) bar_sync(kBarDone + (b & 3), 32 + 32 * kNL);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
#ifdef GSL_TRACE
    if (lane == 0 && n < 8192) {
      g_gsl_trace[n][3] = tr_wait;
      g_gsl_trace[n][4] = tr_poll;
    }
#endif
    if (kNL > 1) bar_sync(11, 32 * kNL);  // every loader warp is done with the incoming slot
    if (has_up && lw == 0 && lane == 0) {
      // every read (and sentinel reset) of the incoming slot is done: release
      // it (the ticket is re-read: nothing long-lived stays in a register)
      const int nn = *(volatile int*)&s_ticket;
      __threadfence();
      atomicMax(p.done + (nn - 1 + kNumSlots) % kNumSlots, nn);
    }
  }
  if (p.blocks_done) {
    const int n = *(volatile int*)&s_ticket;
    // publish "CTAs 0..n finished" in ticket order (CTA n-1 started before n
    // and never waits on it: no deadlock); the drop-in path's download stream
    // waits on this count for the rows whose final values are written
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long t0 = clock64();
      for (;;) {
        unsigned seen;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.blocks_done) : "memory");
        if (seen >= (unsigned)n) break;
        if (clock64() - t0 > (1ll << 35)) __trap();
      }
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.blocks_done), "r"((unsigned)n + 1u) : "memory");
    }
  }
}

__global__ void gsl_sentinel_kernel(unsigned long long* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = gsl::kSent;
}

static unsigned gsl_mask(const tvs_stencil& st, double w[9]) {
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

constexpr unsigned kGslStar = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);

bool gs2d_lane_supported(const tvs_stencil& st) {
  double w[9];
  const unsigned m = gsl_mask(st, w);
  unsigned long long bb;
  std::memcpy(&bb, &st.boundary, sizeof(bb));
  return st.dim == 2 && (m == 0x1FFu || m == kGslStar) && bb != gsl::kSent;
}

template <unsigned MASK, bool REF, int LC>
static int gsl_launch(GslArgs a, int64_t steps, int64_t per, cudaStream_t s, const unsigned* rows_ready,
                      unsigned* blocks_done) {
  using namespace gsl;
  using C = Cfg<REF, LC>;
  auto kern = gs2d_lane_kernel<MASK, REF, LC>;
  TVS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::Smem));
#ifdef GSL_NOPACK
  a.lr = LC;
#else
  a.lr = (int)std::min<int64_t>((per + 1) / 2 * 2, LC);  // lanes in use per group (even: 16-byte hand-off pieces)
#endif
  // the last group's lanes reach column e1 (the boundary the consumer reads)
  const int m_need = a.e1 + kLam * (C::G - 1) + kSk * (a.lr - 1) + kB + 2;
  a.m_end = (m_need + kR - 1) / kR * kR;
  const size_t cells = (size_t)kNumSlots * a.m_end * C::RowCells;
  const size_t ctrl_bytes = sizeof(int) * 2 * kNumSlots + 64;
  a.gring = static_cast<double*>(scratch(sizeof(double) * cells, 4));
  char* ctrl = static_cast<char*>(scratch(ctrl_bytes, 5));
  if (!a.gring || !ctrl) return fail(TVS_ERR_CUDA, "gs2d_lane: scratch");
  a.done = reinterpret_cast<int*>(ctrl);
  a.epoch = a.done + kNumSlots;
  a.ticket = a.epoch + kNumSlots;
  // every ring cell unwritten.  Consumers reset every cell they read and
  // every written cell is read, so a ring stays clean after a launch: the
  // sentinel fill runs only when the buffer or its layout changes
  static thread_local uint64_t clean_gen = 0;
  static thread_local size_t clean_cells = 0;
  if (clean_gen != scratch_generation() || clean_cells != cells) {
    gsl_sentinel_kernel<<<1184, 256, 0, s>>>(reinterpret_cast<unsigned long long*>(a.gring), cells);
    TVS_LAUNCHED("gsl_sentinel_kernel");
    clean_gen = scratch_generation();
    clean_cells = cells;
  }
  if ((rows_ready || blocks_done) && per < steps) return fail(TVS_ERR_INVALID, "gs2d_lane: pipeline hooks need one pass");
  a.rows_ready = rows_ready;
  a.blocks_done = blocks_done;
  const int nthreads = ((C::G * a.lr + 31) / 32 + C::NL) * 32;  // packed compute warps + the loader warps
  for (int64_t done = 0; done < steps; done += per) {
    a.tp = (int)std::min<int64_t>(per, steps - done);
    const int ngroups = a.e0 + a.tp - 1;
    a.nctas = (ngroups + C::G - 1) / C::G;
    TVS_CUDA(cudaMemsetAsync(ctrl, 0, ctrl_bytes, s));
    kern<<<a.nctas, nthreads, C::Smem, s>>>(a);
    TVS_LAUNCHED("gs2d_lane_kernel");
  }
  return TVS_OK;
}

#ifdef GSL_TRACE
extern "C" int tvs_gsl_trace(unsigned long long* host, int n) {
  TVS_CUDA(cudaDeviceSynchronize());
  TVS_CUDA(cudaMemcpyFromSymbol(host, g_gsl_trace, sizeof(unsigned long long) * 8 * std::min(n, 8192)));
  return 0;
}
#endif

// A pass holds <= 128 sweeps; passes are balanced, and the lane capacity is
// the smallest instantiated one that holds a pass (T = 100: one pass, 102).
static void gsl_plan(int64_t steps, int64_t* per, int* lc) {
  const int64_t npass = (steps + 127) / 128;
  *per = (steps + npass - 1) / npass;
  *lc = *per <= 32 ? 32 : (*per <= 64 ? 64 : (*per <= 102 ? 102 : 128));
}
static int gsl_groups(int64_t steps, int order) {
  int64_t per;
  int lc;
  gsl_plan(std::max<int64_t>(steps, 1), &per, &lc);
  // the groups per CTA of exactly the instantiation gs2d_lane() launches
  const bool ref = order == TVS_GS_REFERENCE;
  switch (lc) {
    case 32: return ref ? gsl::Cfg<true, 32>::G : gsl::Cfg<false, 32>::G;
    case 64: return ref ? gsl::Cfg<true, 64>::G : gsl::Cfg<false, 64>::G;
    case 102: return ref ? gsl::Cfg<true, 102>::G : gsl::Cfg<false, 102>::G;
    default: return ref ? gsl::Cfg<true, 128>::G : gsl::Cfg<false, 128>::G;
  }
}
// Drop-in pipeline hooks (api.cu gs2d_pipelined): one pass of <= 128 sweeps;
// CTAs of that pass, and how many must have exited before row `row` holds
// its final value (the group row + steps - 1 writes it).
int gs2d_lane_max_sweeps() { return 128; }
int64_t gs2d_lane_ctas(int64_t rows, int64_t steps, int order) {
  const int G = gsl_groups(steps, order);
  return (rows + steps - 1 + G - 1) / G;
}
int64_t gs2d_lane_ctas_for_row(int64_t row, int64_t steps, int order) {
  return (row + steps - 1) / gsl_groups(steps, order) + 1;
}

int gs2d_lane(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, int order, cudaStream_t s,
              const unsigned* rows_ready, unsigned* blocks_done) {
  double w[9];
  const unsigned mask = gsl_mask(st, w);
  if (!gs2d_lane_supported(st)) return fail(TVS_ERR_UNSUPPORTED, "gs2d_lane: tap set / boundary");
  if (g.extents[0] >= (1ll << 30) || g.extents[1] >= (1ll << 28)) return fail(TVS_ERR_UNSUPPORTED, "gs2d_lane: extent");
  if (steps <= 0) return TVS_OK;
  GslArgs a{};
  a.a = grid + g.origin;
  a.s0 = g.strides[0];
  a.e0 = (int)g.extents[0];
  a.e1 = (int)g.extents[1];
  for (int k = 0; k < 9; ++k) a.w[k] = w[k];
  a.bnd = st.boundary;
  int64_t per;
  int lc;
  gsl_plan(steps, &per, &lc);
  const bool ref = order == TVS_GS_REFERENCE, box = mask == 0x1FFu;
  auto go = [&](auto m_tag, auto r_tag) -> int {
    constexpr unsigned M = decltype(m_tag)::value;
    constexpr bool R = decltype(r_tag)::value;
    if (lc == 32) return gsl_launch<M, R, 32>(a, steps, per, s, rows_ready, blocks_done);
    if (lc == 64) return gsl_launch<M, R, 64>(a, steps, per, s, rows_ready, blocks_done);
    if (lc == 102) return gsl_launch<M, R, 102>(a, steps, per, s, rows_ready, blocks_done);
    return gsl_launch<M, R, 128>(a, steps, per, s, rows_ready, blocks_done);
  };
  using Box = std::integral_constant<unsigned, 0x1FFu>;
  using Star = std::integral_constant<unsigned, kGslStar>;
  if (box) return ref ? go(Box{}, std::true_type{}) : go(Box{}, std::false_type{});
  return ref ? go(Star{}, std::true_type{}) : go(Star{}, std::false_type{});
}

}  // namespace tvs
