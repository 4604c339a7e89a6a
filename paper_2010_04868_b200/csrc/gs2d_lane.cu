// K6v2: 2D radius-1 Gauss-Seidel (9-point box / 5-point star) as time-lane
// groups advancing in per-iteration CTA lockstep.
//
// Replaces gs2d_temporal (reference kernels_nd.py:48-50, star-only there) for
// the row-major in-place sweep of BASELINE config 4, bit-exact with the
// oracle's lexicographic loop (oracle/stencil_oracle.c gs_lex; the reference
// loop test test_baselines.py:39-52) and, with order = reference, with the
// reference's anti-diagonal gather/scatter (baselines.py:83-107: the NE
// neighbour is read from the previous sweep).
//
// The paper's time lanes.  A "group" is WG warps = 32*WG lanes; lane l runs
// sweep t0 + l and group d owns the units {(sweep l, row d - l)} (a diagonal
// through (time, row) space), streaming left to right over the columns, one
// column per iteration.  Every input of unit (l, row r = d - l, column c) is
//   NW, N, NE  row r-1, sweep l    = group d-1, lane l     (smem ring)
//   W          row r,   sweep l    = my previous output    (register)
//   C, E       row r,   sweep l-1  = group d-1, lane l-1   (smem ring)
//   SW, S, SE  row r+1, sweep l-1  = group d,   lane l-1   (__shfl_up; a
//                                     warp's lane 0 reads the ring)
// (reference order: NE = row r-1, sweep l-1 = group d-2, lane l-1), where
// "lane -1" of group d is grid row d+1 as it was before the pass (loaded by
// the CTA's loader warp).  Lane l trails lane l-1 by 2 columns and group g
// trails group g-1 by 2 iterations (LAM): the hyperplane slope of the
// dependence graph (h = 2 row + column + 4 sweep), so the pipeline is no
// longer than the computation's critical path.  Taps are summed in sorted
// order (NW N NE W C E SW S SE), unfused: bit-exact.
//
// CTA = G groups (G*WG compute warps) + a loader warp, one CTA barrier per
// iteration: every warp does identical work per iteration, so lockstep costs
// only the barrier, and everything a warp reads from shared memory was
// written before the previous barrier.  The loader prefetches, ahead of use,
// the grid rows of every group's lane -1 (cp.async) and the previous CTA's
// last group(s) ("phantom" groups).  CTA-to-CTA hand-off is fence-free: the
// producer's last groups store every output to an L2 ring whose cells hold a
// signalling-NaN sentinel until written (arithmetic never yields a
// signalling NaN, and the boundary value is checked on the host), the
// consumer's loader polls the cells themselves (8-byte single-copy atomic)
// and puts the sentinel back after reading, so the ring is clean for its next
// use.  CTAs take tickets and only wait on lower tickets; a ring slot is
// reused only after its consumer has exited.  Units outside the grid output
// the boundary; lane Tp-1 (the pass's last sweep) writes its row's final
// values to the grid in place.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace tvs {
namespace gsl {
constexpr int kLam = 2;          // group lag (iterations)
constexpr int kB = 2;            // every lane starts >= 2 columns left of column 0
constexpr int kPre = 6;          // phantom / lane -1 rows read before iteration 0 (rows -6..-1)
constexpr int kLR = 128;         // lane -1 staging ring (iterations), power of two
#ifndef GSL_BATCH
#define GSL_BATCH 0  // 0: per order (Cfg::Batch)
#endif
constexpr int kAheadL = 64;      // lane -1 rows are requested this many iterations ahead (HBM latency)
constexpr int kNumSlots = 320;   // global ring slots (CTA boundaries in flight) >= resident CTAs
// sentinel of an unwritten global-ring cell: a signalling NaN (quiet bit
// clear), which no arithmetic result can be
constexpr unsigned long long kSent = 0x7FF4DEADBEEF0001ull;

template <bool REF, int WG>
struct Cfg {
#ifndef GSL_G
#define GSL_G 0
#endif
  // groups per CTA: 4, two CTAs per SM, in both orders (config 4 lex G 3 /
  // 4 / 7: 33.8 / 29.3 / 32.3 ms with the round-1 loader)
#ifndef GSL_GREF
#define GSL_GREF 0
#endif
#ifndef GSL_RREF
#define GSL_RREF 0
#endif
  static constexpr int G = REF ? (GSL_GREF > 0 ? GSL_GREF : 4) : (GSL_G > 0 ? GSL_G : 4);
  // smem ring rows (iterations, power of two; also the unroll of the
  // compute loop).  Reference order: 8, so that two CTAs of three rings
  // more fit one SM (config 4: G 7 R 16 one CTA/SM / G 7 R 8 / G 5 R 8 two /
  // G 4 R 8 two: 31.9 / 29.3 / 27.2 / 25.4 ms)
  static constexpr int R = REF ? (GSL_RREF > 0 ? GSL_RREF : 8) : 16;
  // rows per loader block (lane -1 staging batch, phantom poll block).
  // Config 4 lexicographic 8 / 4 / 2 / 1 rows: 44.3 / 33.8 / 26.1 / 28.7 ms;
  // reference order 2 / 1: 51.8 / 45.3 ms
  static constexpr int Batch = GSL_BATCH > 0 ? GSL_BATCH : (REF ? 1 : 2);
  static constexpr int Ph = REF ? 2 : 1;        // phantom groups (reads reach group d-2 in REF)
  static constexpr int L = 32 * WG;             // lanes per group
  static constexpr int S = L + 2;               // ring row: [pad][lane -1][lanes 0..L-1] (16-B aligned lanes)
  static constexpr int Rings = G + Ph;          // ring index = local group + Ph
  static constexpr int Compute = G * WG;        // compute warps
  // one loader warp (a second one, phantom blocks | lane -1 rows, measured
  // slower: 28.6 vs 23.6 ms at config 4 -- one more warp in every barrier)
  static constexpr int Threads = (Compute + 1) * 32;
#ifndef GSL_DIST
#define GSL_DIST 0
#endif
  // phantom blocks are requested Dist blocks ahead of their validation
  // (config 4 reference order, one-row blocks: Dist 1 / 2: 33.1 / 30.0 ms;
  // lexicographic two-row blocks: 19.6 / 22.0 ms)
  static constexpr int Dist = GSL_DIST > 0 ? GSL_DIST : (REF ? 2 : 1);
  static constexpr int StgBlocks = Dist < 2 ? 2 : 4;  // staging ring (power of two > Dist)
  static_assert(Dist <= 3, "staging ring");
  static constexpr int Stg = StgBlocks * Batch * Ph * L;  // phantom staging: blocks of Batch compact rows
  static constexpr size_t Smem = sizeof(double) * ((size_t)Rings * R * S + (size_t)Rings * kLR + Stg);
  static constexpr int Back = REF ? 2 * kLam + 1 : kLam + 1;  // deepest ring read behind m
  static_assert(R >= Back + Batch + 1, "ring too shallow for a phantom block written ahead");
  static_assert(kLR >= kAheadL + Batch + 8, "lane -1 staging ring too shallow");
  static_assert(kPre >= Back + 1, "prologue rows");
  static constexpr int ProRows = (kPre + Batch - 1) / Batch * Batch;  // phantom rows before iteration 0
  static_assert(R % Batch == 0 && kAheadL % Batch == 0, "block sizes");
};
}  // namespace gsl

#ifdef GSL_TRACE
// [cta][0] start ns, [1] first iteration ns, [2] end ns, [3] loader poll-spin cycles,
// [4] loader cp.async wait cycles, [5] compute warp 0 barrier-wait cycles, [6] loader barrier-wait cycles
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
  int tp;             // sweeps of this pass (<= 32 * WG)
  int nctas;
  int m_end;          // iterations per CTA (multiple of kR)
  double* gring;      // kNumSlots x m_end x Ph x L (sentinel until written)
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
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(double* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
__device__ __forceinline__ void cta_bar(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

#ifndef GSL_MINB
#define GSL_MINB 2
#endif
#ifndef GSL_MINB_REF
#define GSL_MINB_REF 2
#endif
template <unsigned MASK, bool REF, int WG>
__global__ void __launch_bounds__(gsl::Cfg<REF, WG>::Threads, REF ? GSL_MINB_REF : GSL_MINB) gs2d_lane_kernel(GslArgs p) {
  using namespace gsl;
  using C = Cfg<REF, WG>;
  constexpr int kG = C::G, kPh = C::Ph, kL = C::L, kS = C::S, kRings = C::Rings, kThreads = C::Threads;
  constexpr int kBatch = C::Batch;
  constexpr int kR = C::R;
  extern __shared__ __align__(16) double smem[];
  double* const lm1 = smem + (size_t)kRings * kR * kS;  // lane -1 staging [ring][kLR]
  double* const stg = lm1 + kRings * kLR;                 // phantom staging [StgBlocks][kBatch][kPh * kL]
  __shared__ int s_ticket;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const double bnd = p.bnd;
  // every ring cell starts as the boundary (iterations before 0 are columns
  // left of the grid)
  for (int i = threadIdx.x; i < kRings * (kR * kS + kLR); i += blockDim.x) smem[i] = bnd;
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1);
  __syncthreads();
  const int n = s_ticket;  // position in the CTA chain
#ifdef GSL_TRACE
  if (threadIdx.x == 0 && n < 8192) g_gsl_trace[n][0] = gsl_now();
  unsigned long long tr_bar = 0, tr_poll = 0, tr_cpw = 0;
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
  double* gin = p.gring + (size_t)slot_in * m_end * kPh * kL;
  double* gout = p.gring + (size_t)slot_out * m_end * kPh * kL;
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

  if (wi < C::Compute) {
    // ---------------- compute warp: group g, lanes l = 32 w + t ----------
    const int g = wi / WG, w = wi % WG, l = 32 * w + lane;
    const int d = d0 + g, row = d - l;
    const int col0 = -kLam * g - 2 * l - kB;  // my column at iteration 0
    double* const ring_me = smem + (size_t)(g + kPh) * kR * kS;
    const double* const ring_up = ring_me - kR * kS;
    const double* const ring_up2 = ring_me - 2 * kR * kS;
    const bool emit = l == p.tp - 1;  // last sweep of the pass: final values
    double* const arow = p.a + (long long)row * p.s0;
    const bool to_ring = has_down && g >= kG - kPh;  // phantom source of the next CTA
    double* const gdst = gout + (size_t)(g - (kG - kPh)) * kL + l;
    // this warp's lanes all inside the grid (rows, and columns for iterations
    // [m_in0, m_in1)): the steady body needs no selects
    const bool rows_in = d - 32 * w - 31 >= 0 && d - 32 * w <= e0 - 1;
    const int m_in0 = kLam * g + 64 * w + 62 + kB, m_in1 = kLam * g + 64 * w + kB + e1;
    const bool row_ok = row >= 0 && row < e0;
    double nw = bnd, nn = bnd, ne = bnd, ww = bnd, cc = bnd, ee = bnd, sw = bnd, ss = bnd, se = bnd;
    double out = bnd;
    cta_bar(kThreads);  // prologue rows landed
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
          const int r1 = ((u - 1) & (kR - 1)) * kS, r3 = ((u - kLam - 1) & (kR - 1)) * kS;
          const double ne_new = ring_up[r1 + 2 + l];  // group d-1, lane l, iteration m-1
          const double e_new = ring_up[r3 + 1 + l];   // group d-1, lane l-1, iteration m-3 (lane 0: grid row d)
          const double se_new = ring_me[r1 + 1 + l];  // my group, lane l-1, iteration m-1 (lane 0: grid row d+1)
          nw = nn; nn = ne; ne = ne_new;
          cc = ee; ee = e_new;
          sw = ss; ss = se; se = se_new;
          double ne_use = ne;
          if constexpr (REF) {
            // group d-2, lane l-1, iteration m-5 (lane 0: grid row d-1)
            const int r5 = ((u - 2 * kLam - 1) & (kR - 1)) * kS;
            ne_use = ring_up2[r5 + 1 + l];
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
          ring_me[(u & (kR - 1)) * kS + 2 + l] = out;
          if (to_ring && m >= ring_lo) st_relaxed_gpu(gdst + (size_t)m * kPh * kL, __double_as_longlong(out));
          if (emit && inside) arow[col0 + m] = out;
#ifdef GSL_TRACE
          const long long tb0 = clock64();
#endif
          cta_bar(kThreads);  // iteration m done everywhere; the loader's rows for m+1 landed
#ifdef GSL_TRACE
          tr_bar += clock64() - tb0;
#endif
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
      g_gsl_trace[n][5] = tr_bar;
    }
#endif
  } else {
    // ---------------- loader -----------------------------------------------
    //  * lane -1 of ring ri (local group g = ri - kPh, global d0 + g) at
    //    iteration i = grid row d0 + g + 1 at column i - LAM*g + 2 - B:
    //    cp.async batches of kBatch rows, kAheadL iterations ahead;
    //  * phantom rows (the previous CTA's last kPh groups at producer
    //    iteration i + LAM*G; its groups G-kPh.. are my -kPh..) in blocks of
    //    kBatch rows: a block is requested (cp.async from the L2 ring) one
    //    block ahead, then validated cell by cell (sentinel: re-polled until
    //    written), copied into the phantom rings and reset to the sentinel
    //    in the L2 ring.  One L2 round trip per block, not per row.
    //    Producer rows >= m_end are columns right of the grid: the boundary.
    constexpr int kRowCells = kPh * kL;            // cells of one phantom row
    constexpr int kPieces = kBatch * kRowCells / 2;  // 16-byte pieces per block
    constexpr int kPerLane = (kPieces + 31) / 32;  // pieces per loader lane (the last round partial)
    // lane -1 rows: loader lane t < kRings * kBatch owns ring t / kBatch,
    // iteration offset t % kBatch (grid row d0 + g + 1, g = ring - kPh)
    static_assert(kRings * kBatch <= 32, "one lane -1 cell per loader lane");
    const int lm_ri = lane / kBatch, lm_o = lane % kBatch, lm_g = lm_ri - kPh, lm_r = d0 + lm_g + 1;
    const bool lm_on = lane < kRings * kBatch, lm_row = lm_r >= 0 && lm_r < e0;
    const int lm_c0 = lm_o - kLam * lm_g + 2 - kB;  // grid column at i0 = 0
    double* const lm_dst = lm1 + lm_ri * kLR + lm_o;
    auto batch_lane_m1 = [&](int i0) {  // iterations [i0, i0 + kBatch), every ring
      if (lm_on) {
        const int c = i0 + lm_c0;
        double* dst = lm_dst + (i0 & (kLR - 1));
        if (lm_row && c >= 0 && c < e1)
          cp_async8(dst, p.a + (long long)lm_r * p.s0 + c);
        else
          *dst = bnd;
      }
    };
    auto slot1 = [&](int i) {  // lane -1 of every ring at iteration i -> ring slot 1
      if (lane < kRings) smem[((size_t)lane * kR + (i & (kR - 1))) * kS + 1] = lm1[lane * kLR + (i & (kLR - 1))];
    };
    auto in_ring = [&](int i) { return has_up && i + kLam * kG < m_end; };
    auto gcell = [&](int i, int e) -> double* { return gin + (size_t)(i + kLam * kG) * kRowCells + e; };
    auto request_block = [&](int i0) {  // phantom rows [i0, i0 + kBatch) -> staging
      double* sb = stg + ((i0 / kBatch) & (C::StgBlocks - 1)) * (kBatch * kRowCells);
#pragma unroll 4
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j, r = k / (kRowCells / 2), e = 2 * (k % (kRowCells / 2));
        if (k < kPieces && in_ring(i0 + r)) cp_async16g(sb + r * kRowCells + e, gcell(i0 + r, e));
      }
    };
    // lexicographic: the block's pieces loaded together, 16-byte smem and L2
    // accesses; reference order keeps the one-piece-at-a-time loop (faster
    // there: 45.3 vs 51.8 ms at config 4 size)
    auto finish_block_vec = [&](int i0) {
      const double* sb = stg + ((i0 / kBatch) & (C::StgBlocks - 1)) * (kBatch * kRowCells);
      double2 got[kPerLane];
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j, r = k / (kRowCells / 2), e = 2 * (k % (kRowCells / 2));
        if (kPieces % 32 == 0 || k < kPieces) got[j] = *reinterpret_cast<const double2*>(sb + r * kRowCells + e);
      }
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j, r = k / (kRowCells / 2), e = 2 * (k % (kRowCells / 2));
        if (kPieces % 32 != 0 && k >= kPieces) break;
        const int i = i0 + r;
        unsigned long long v0 = __double_as_longlong(bnd), v1 = v0;
        if (in_ring(i)) {
          v0 = __double_as_longlong(got[j].x);
          v1 = __double_as_longlong(got[j].y);
          if (v0 == kSent || v1 == kSent) {
            const long long t0 = clock64();
            while (v0 == kSent) {
              v0 = ld_relaxed_gpu(gcell(i, e));
              if (clock64() - t0 > (1ll << 34)) __trap();
            }
            while (v1 == kSent) {
              v1 = ld_relaxed_gpu(gcell(i, e + 1));
              if (clock64() - t0 > (1ll << 34)) __trap();
            }
          }
          asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(gcell(i, e)), "l"(kSent), "l"(kSent)
                       : "memory");
        }
        const int ph = e / kL, ll = e % kL;
        double* dst = smem + ((size_t)ph * kR + (i & (kR - 1))) * kS + 2 + ll;
        *reinterpret_cast<double2*>(dst) = make_double2(__longlong_as_double(v0), __longlong_as_double(v1));
      }
    };
    auto finish_block_one = [&](int i0) {
      const double* sb = stg + ((i0 / kBatch) & (C::StgBlocks - 1)) * (kBatch * kRowCells);
#pragma unroll 1
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j, r = k / (kRowCells / 2), e = 2 * (k % (kRowCells / 2));
        if (k >= kPieces) break;
        const int i = i0 + r;
        unsigned long long v0 = __double_as_longlong(bnd), v1 = v0;
        if (in_ring(i)) {
          v0 = __double_as_longlong(sb[r * kRowCells + e]);
          v1 = __double_as_longlong(sb[r * kRowCells + e + 1]);
          if (v0 == kSent || v1 == kSent) {
            const long long t0 = clock64();
            while (v0 == kSent) {
              v0 = ld_relaxed_gpu(gcell(i, e));
              if (clock64() - t0 > (1ll << 34)) __trap();
            }
            while (v1 == kSent) {
              v1 = ld_relaxed_gpu(gcell(i, e + 1));
              if (clock64() - t0 > (1ll << 34)) __trap();
            }
#ifdef GSL_TRACE
            tr_poll += clock64() - t0;
#endif
          }
#ifndef GSL_NO_RESET
          st_relaxed_gpu(gcell(i, e), kSent);
          st_relaxed_gpu(gcell(i, e + 1), kSent);
#endif
        }
        const int ph = e / kL, ll = e % kL;
        double* dst = smem + ((size_t)ph * kR + (i & (kR - 1))) * kS + 2 + ll;
        dst[0] = __longlong_as_double(v0);
        dst[1] = __longlong_as_double(v1);
      }
    };
    // blocks wholly inside the producer's rows (all but the first and last
    // few of a CTA with a producer): piece j of lane t is block cell pair
    // 2 (t + 32 j) in staging and in the L2 ring alike; one warp vote checks
    // the sentinels, late cells are re-polled out of line
    auto block_full = [&](int i0) { return has_up && i0 + kBatch - 1 + kLam * kG < m_end; };
    auto request_fast = [&](int i0) {
      double* sb = stg + ((i0 / kBatch) & (C::StgBlocks - 1)) * (kBatch * kRowCells);
      const double* gb = gin + (size_t)(i0 + kLam * kG) * kRowCells;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j;
        if (kPieces % 32 == 0 || k < kPieces) cp_async16g(sb + 2 * k, gb + 2 * k);
      }
    };
    auto finish_fast = [&](int i0) {
      const double* sb = stg + ((i0 / kBatch) & (C::StgBlocks - 1)) * (kBatch * kRowCells);
      double* const gb = gin + (size_t)(i0 + kLam * kG) * kRowCells;
      double2 got[kPerLane];
      bool bad = false;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j;
        if (kPieces % 32 == 0 || k < kPieces) {
          got[j] = *reinterpret_cast<const double2*>(sb + 2 * k);
          bad |= (__double_as_longlong(got[j].x) == kSent) | (__double_as_longlong(got[j].y) == kSent);
        }
      }
      if (__any_sync(0xffffffffu, bad)) {
        // late cells (the consumer caught up with its producer): re-read
        // every late pair at once until all have landed
        const long long t0 = clock64();
        do {
          bad = false;
#pragma unroll
          for (int j = 0; j < kPerLane; ++j) {
            const int k = lane + 32 * j;
            if ((kPieces % 32 == 0 || k < kPieces) &&
                ((__double_as_longlong(got[j].x) == kSent) | (__double_as_longlong(got[j].y) == kSent))) {
              got[j] = ld_relaxed_gpu2(gb + 2 * k);
              bad |= (__double_as_longlong(got[j].x) == kSent) | (__double_as_longlong(got[j].y) == kSent);
            }
          }
          if (clock64() - t0 > (1ll << 34)) __trap();
        } while (__any_sync(0xffffffffu, bad));
      }
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const int k = lane + 32 * j;
        if (kPieces % 32 == 0 || k < kPieces) {
#ifndef GSL_NO_RESET
          asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(gb + 2 * k), "l"(kSent), "l"(kSent)
                       : "memory");
#endif
          const int r = k / (kRowCells / 2), e = 2 * (k % (kRowCells / 2));
          const int ph = e / kL, ll = e % kL;
          *reinterpret_cast<double2*>(smem + ((size_t)ph * kR + ((i0 + r) & (kR - 1))) * kS + 2 + ll) = got[j];
        }
      }
    };
    auto finish_block = [&](int i0) {  // validate, copy into the rings, reset the L2 cells
      if constexpr (REF)
        finish_block_one(i0);
      else
        finish_block_vec(i0);
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
    // prologue: lane -1 rows [-kBatch, kAheadL) landed; phantom rows
    // [-kBatch, 0) in the rings, rows [0, kBatch) requested
    for (int i0 = -C::ProRows; i0 < kAheadL; i0 += kBatch) batch_lane_m1(i0);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    for (int i = -kPre; i <= 0; ++i) slot1(i);
    for (int i0 = -C::ProRows; i0 < 0; i0 += kBatch) {
      request_block(i0);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      finish_block(i0);
    }
    // blocks 0 .. Dist-1 in flight, each followed by an (empty) lane -1
    // group so that every block below commits the same pair
    for (int j = 0; j < C::Dist; ++j) {
      request_block(j * kBatch);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    __syncwarp();
    cta_bar(kThreads);
    for (int mb = 0; mb < m_end; mb += kR) {
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const int m = mb + u;
        // per block: group A = the phantom block Dist blocks ahead (first
        // iteration), group B = lane -1 rows kAheadL iterations ahead (the
        // second iteration, to even out the loader's work); waiting for all
        // but the newest 2 Dist groups (2 Dist + 1 with one-row blocks)
        // retires this block's request, committed Dist blocks ago
#ifdef GSL_LM_SAME
        constexpr int kLmU = 0;
#else
        constexpr int kLmU = kBatch > 1 ? 1 : 0;
#endif
        if (u % kBatch == 0) {
          const int iq = m + C::Dist * kBatch;
          if (block_full(iq))
            request_fast(iq);
          else
            request_block(iq);
          asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
        if (u % kBatch == kLmU) {
          batch_lane_m1(m - kLmU + kAheadL);
          asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
        if (u % kBatch == 0) {
#ifdef GSL_TRACE
          const long long tw0 = clock64();
#endif
          asm volatile("cp.async.wait_group %0;\n" ::"n"(2 * C::Dist + (kLmU > 0 ? 0 : 1)) : "memory");
#ifdef GSL_TRACE
          tr_cpw += clock64() - tw0;
#endif
          __syncwarp();
          // rows [m, m + kBatch): read from iteration m + 1 on
          if (block_full(m))
            finish_fast(m);
          else
            finish_block(m);
        }
        slot1(m + 1);  // read from iteration m + 2 on
        __syncwarp();
#ifdef GSL_TRACE
        const long long tb0 = clock64();
#endif
        cta_bar(kThreads);
#ifdef GSL_TRACE
        tr_bar += clock64() - tb0;
#endif
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
#ifdef GSL_TRACE
    if (lane == 0 && n < 8192) {
      g_gsl_trace[n][3] = tr_poll;
      g_gsl_trace[n][4] = tr_cpw;
      g_gsl_trace[n][6] = tr_bar;
    }
#endif
    if (has_up && lane == 0) {
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

template <unsigned MASK, bool REF, int WG>
static int gsl_launch(GslArgs a, int64_t steps, int64_t per, cudaStream_t s, const unsigned* rows_ready,
                      unsigned* blocks_done) {
  using namespace gsl;
  using C = Cfg<REF, WG>;
  auto kern = gs2d_lane_kernel<MASK, REF, WG>;
  TVS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::Smem));
  // the last group's lanes reach column e1 (the boundary the consumer reads)
  const int m_need = a.e1 + kLam * (C::G - 1) + 2 * (C::L - 1) + kB + 2;
  a.m_end = (m_need + C::R - 1) / C::R * C::R;
  const size_t cells = (size_t)kNumSlots * a.m_end * C::Ph * C::L;
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
  for (int64_t done = 0; done < steps; done += per) {
    a.tp = (int)std::min<int64_t>(per, steps - done);
    const int ngroups = a.e0 + a.tp - 1;
    a.nctas = (ngroups + C::G - 1) / C::G;
    TVS_CUDA(cudaMemsetAsync(ctrl, 0, ctrl_bytes, s));
    kern<<<a.nctas, C::Threads, C::Smem, s>>>(a);
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

// Drop-in pipeline hooks (api.cu gs2d_pipelined): one pass of <= 128 sweeps;
// CTAs of that pass, and how many must have exited before row `row` holds
// its final value (the group row + steps - 1 writes it).
static int gsl_groups(int64_t steps, int order) {
  (void)steps;
  return order == TVS_GS_REFERENCE ? gsl::Cfg<true, 4>::G : gsl::Cfg<false, 4>::G;
}
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
  // lanes per group = the smallest warp multiple holding a pass of <= 128
  // sweeps in balanced passes (T = 100: one pass on 4-warp groups)
  const int64_t npass = (steps + 127) / 128;
  const int64_t per = (steps + npass - 1) / npass;
  const int wg = per <= 32 ? 1 : (per <= 64 ? 2 : 4);
  const bool ref = order == TVS_GS_REFERENCE, box = mask == 0x1FFu;
  auto go = [&](auto m_tag, auto r_tag) -> int {
    constexpr unsigned M = decltype(m_tag)::value;
    constexpr bool R = decltype(r_tag)::value;
    if (wg == 1) return gsl_launch<M, R, 1>(a, steps, per, s, rows_ready, blocks_done);
    if (wg == 2) return gsl_launch<M, R, 2>(a, steps, per, s, rows_ready, blocks_done);
    return gsl_launch<M, R, 4>(a, steps, per, s, rows_ready, blocks_done);
  };
  using Box = std::integral_constant<unsigned, 0x1FFu>;
  using Star = std::integral_constant<unsigned, kGslStar>;
  if (box) return ref ? go(Box{}, std::true_type{}) : go(Box{}, std::false_type{});
  return ref ? go(Star{}, std::true_type{}) : go(Star{}, std::false_type{});
}

}  // namespace tvs
