// K3: 2D radius-1 Jacobi (5-point star / 9-point box), temporally blocked.
//
// Replaces jacobi2d_temporal / _JacobiNd (reference kernels_nd.py:38-40,
// 179-291).  Each warp owns a strip of 32*P contiguous columns and streams
// down a segment of rows; D time levels are advanced per pass over HBM with
// a one-row time skew between levels (level l works on row m-l while level 0
// loads row m) — the GPU form of the paper's time-skewed lanes.  Nothing
// leaves registers between levels:
//
//   * a lane holds P columns; the only cross-lane traffic per (level, row) is
//     its two edge values (__shfl_up/__shfl_down);
//   * instead of keeping a 3-row window per level, each level keeps two
//     partial sums per column.  When row q of level l-1 arrives it finishes
//     output q-1 with the +1-row taps, adds the 0-row taps to output q and
//     starts output q+1 with the -1-row taps.  Sorted tap order is
//     -1-row taps, 0-row taps, +1-row taps, each left to right, so the
//     accumulation order — and the rounding — is exactly the reference's
//     `acc = c*v + acc` chain (baselines.py:43-49).
//
// Ghost trapezoid: the outer D columns of a strip and the first/last D rows
// of a segment are recomputed by neighbouring warps; useful width is
// 32*P - 2*D.  HBM traffic per useful update ~ 16 B / D.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "common.cuh"

namespace tvs {

constexpr int kMaxD2 = 12;     // deepest temporal block instantiated (P = 4 / 3 / 2 columns per lane, see launch2d_one)
constexpr int kWarps2 = 1;     // warps per block (task = blockIdx.x: warp-uniform control flow)
#ifndef J2D_SEG
#define J2D_SEG 256
#endif
constexpr int kRowsSeg = J2D_SEG;
#ifndef J2D_RING
#define J2D_RING 4  // > 0: cp.async row ring depth (0: register prefetch); 4 measured best (config 3: 0 1733, 4 1754-1793, 8 1754, 16 1741 GSt/s)
#endif
#ifndef J2D_PF
#define J2D_PF 2
#endif  // output rows per warp task

constexpr unsigned kStar5 = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);
constexpr unsigned kBox9 = 0x1FFu;

template <unsigned MASK, int G>
__device__ __forceinline__ constexpr bool has_group() {
  return ((MASK >> (G * 3)) & 7u) != 0;
}

// acc[p] (+)= sum over taps of row-group G, columns dc = -1, 0, +1, in order.
// SC (scaled power-of-two taps): c holds c_k / c_first, all powers of two,
// and acc carries the partial sum divided by c_first: the first tap is the
// input itself, every other tap one DFMA whose product is exact — equal bit
// for bit to the reference's separately rounded c*v then +acc, because
// scaling by a power of two commutes with rounding (barring under/overflow).
template <unsigned MASK, int G, bool START, bool FMA, int kP2, bool SC = false>
__device__ __forceinline__ void add_group(double (&acc)[kP2], const double (&in)[kP2 + 2], const double (&c)[9]) {
#pragma unroll
  for (int p = 0; p < kP2; ++p) {
    bool fresh = START;
#pragma unroll
    for (int dc = 0; dc < 3; ++dc) {
      if ((MASK >> (G * 3 + dc)) & 1u) {
        const double v = in[p + dc];
        if (fresh) {
          if constexpr (SC)
            acc[p] = v;  // c_first / c_first = 1
          else
            acc[p] = tap_first(c[G * 3 + dc], v);
          fresh = false;
        } else {
          acc[p] = tap_next<FMA || SC>(c[G * 3 + dc], v, acc[p]);
        }
      }
    }
  }
}

struct Coeff9 {
  double c[9];
  // SC: values of level l are the true values / c_first^(l+1); pinned cells
  // of level l hold bnd / c_first^(l+1) (bl[l]); a stored level-D value is
  // multiplied by c_first^D (out_scale)
  double bl[13];
  double out_scale;
};

// One level update when row q of the level below arrives (see header):
// out(q-1) = F + taps(+1 row); N(q) = M + taps(0 row); M'(q+1) = taps(-1 row).
// F is finished in place (it becomes the fresh accumulator), so calling this
// with (F, M) and then (M, F) on the next row rotates roles without copies.
template <unsigned MASK, bool FMA, int kP2, bool SC>
__device__ __forceinline__ void level_row(double (&F)[kP2], double (&M)[kP2], const double (&in)[kP2 + 2],
                                          const double (&c)[9], double (&out)[kP2]) {
  constexpr bool G0 = has_group<MASK, 0>(), G1 = has_group<MASK, 1>(), G2 = has_group<MASK, 2>();
  if constexpr (G2) add_group<MASK, 2, !(G0 || G1), FMA, kP2, SC>(F, in, c);
#pragma unroll
  for (int p = 0; p < kP2; ++p) out[p] = F[p];
  if constexpr (G1) add_group<MASK, 1, !G0, FMA, kP2, SC>(M, in, c);
  if constexpr (G0) add_group<MASK, 0, true, FMA, kP2, SC>(F, in, c);
}

template <unsigned MASK, int D, bool FMA, int kP2, bool MIR, bool SC>
__global__ void __maxnreg__(192) jacobi2d_kernel(const double* __restrict__ src,
                                                                double* __restrict__ dst, Geo g, int64_t origin,
                                                                Coeff9 cf, double bnd, int64_t n_strips,
                                                                int64_t n_tasks, int64_t row_lo, int64_t row_hi, int seg_rows,
                                                                Mirror mir) {
  constexpr int U = 32 * kP2 - 2 * D;  // useful columns per strip
  const double(&c)[9] = cf.c;          // constant-bank operands

  const int lane = threadIdx.x & 31;
  const int64_t task = kWarps2 == 1 ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * kWarps2 + (threadIdx.x >> 5);
  if (task >= n_tasks) return;
  const int64_t strip = task % n_strips, seg = task / n_strips;
  const int col0 = (int)(-D + strip * U);  // first column of the strip
  const int cl = col0 + lane * kP2;        // this lane's first column
  const int r0 = (int)(row_lo + seg * seg_rows);  // first output row
  const int r1 = (int)(r0 + seg_rows < row_hi ? r0 + seg_rows : row_hi);
  const int e0 = (int)g.e0, e1 = (int)g.e1;
  const int a0 = (int)g.a0_off, ag = (int)g.a0_glob;

  unsigned col_out = 0;  // bit p: column cl+p outside the domain
#pragma unroll
  for (int p = 0; p < kP2; ++p) col_out |= (cl + p < 0 || cl + p >= e1 ? 1u : 0u) << p;
  const bool any_col_out = __any_sync(0xffffffffu, col_out != 0);
  unsigned store_mask = 0;  // bit p: column is a useful output of this strip
#pragma unroll
  for (int p = 0; p < kP2; ++p) {
    const int x = cl + p;
    store_mask |= (x >= col0 + D && x < col0 + D + U && x >= 0 && x < e1 ? 1u : 0u) << p;
  }

  double A[D][kP2], B[D][kP2];
#pragma unroll
  for (int l = 0; l < D; ++l)
#pragma unroll
    for (int p = 0; p < kP2; ++p) A[l][p] = B[l][p] = 0.0;

  const double* col_base = src + origin + cl;
  auto load_row = [&](int m, double (&r)[kP2]) {
    const bool row_ok = m >= 0 && m < e0 && m + a0 >= 0 && m + a0 < ag;
    const double* rp = col_base + (int64_t)m * g.s0;
#pragma unroll
    for (int p = 0; p < kP2; ++p) r[p] = (row_ok && !(col_out >> p & 1u)) ? __ldg(rp + p) : bnd;
  };
  const int m_begin = r0 - D, m_end = r1 + D;
  // One stream step: level-0 row m enters, level-D row m-D leaves.  EVEN
  // selects which accumulator set finishes (role swap every step).  The
  // interior/boundary choice is made once per step (warp-uniform), so the
  // interior body is straight-line code with no selects or merge copies.
  // IN (interior warp, see below): every row is known to be inside the
  // domain, so the per-step check is skipped.
  auto step = [&](int m, double (&row)[kP2], auto even_tag, auto in_tag) {
    constexpr bool EVEN = decltype(even_tag)::value;
    constexpr bool IN = decltype(in_tag)::value;
    auto body = [&](auto fast_tag) {
      constexpr bool FAST = decltype(fast_tag)::value;
      double in[kP2 + 2];
#pragma unroll
      for (int p = 0; p < kP2; ++p) in[p + 1] = row[p];
      in[0] = __shfl_up_sync(0xffffffffu, in[kP2], 1);
      in[kP2 + 1] = __shfl_down_sync(0xffffffffu, in[1], 1);
#pragma unroll
      for (int l = 0; l < D; ++l) {
        double out[kP2];
        if constexpr (EVEN)
          level_row<MASK, FMA, kP2, SC>(B[l], A[l], in, c, out);
        else
          level_row<MASK, FMA, kP2, SC>(A[l], B[l], in, c, out);
        if constexpr (FAST) {
#pragma unroll
          for (int p = 0; p < kP2; ++p) in[p + 1] = out[p];
        } else {
          const int gq = m - l - 1 + a0;
          const bool pin_row = gq < 0 || gq >= ag;
          const double pin = SC ? cf.bl[l] : bnd;  // the boundary at this level's scale
#pragma unroll
          for (int p = 0; p < kP2; ++p) in[p + 1] = (pin_row || (col_out >> p & 1u)) ? pin : out[p];
        }
        if (l + 1 < D) {
          in[0] = __shfl_up_sync(0xffffffffu, in[kP2], 1);
          in[kP2 + 1] = __shfl_down_sync(0xffffffffu, in[1], 1);
        }
      }
      const int q = m - D;  // level-D row leaving
      if (q >= r0 && q < r1) {
        if constexpr (SC) {
#pragma unroll
          for (int p = 0; p < kP2; ++p) in[p + 1] = __dmul_rn(in[p + 1], cf.out_scale);  // exact: a power of two
        }
        if constexpr (MIR) {
          // sharded pass: local row, plus the neighbour's ghost row
          for_each_dst(dst, mir, q, [&](double* base) {
            double* wp = base + origin + (int64_t)q * g.s0 + cl;
#pragma unroll
            for (int p = 0; p < kP2; ++p)
              if (store_mask >> p & 1u) wp[p] = in[p + 1];
          });
        } else {
          double* wp = dst + origin + (int64_t)q * g.s0 + cl;
#pragma unroll
          for (int p = 0; p < kP2; ++p)
            if (store_mask >> p & 1u) wp[p] = in[p + 1];
        }
      }
    };
    if constexpr (IN) {
      body(std::true_type{});
    } else {
      // rows m-1-l (l < D) produced this step; all inside the domain?
      const bool rows_in = m - D + a0 >= 0 && m - 1 + a0 < ag;
      if (rows_in && !any_col_out)
        body(std::true_type{});
      else
        body(std::false_type{});
    }
  };
  // Interior warp: no column of the strip outside the domain, and every row
  // the segment loads (m_begin .. m_end-1) and every level row it produces
  // (m-D .. m-1) inside the local and global row range — the row loop then
  // runs without per-row range checks, selects or boundary branches
  // (~15% of the loop's instructions in the ncu source view).
  const bool interior = !any_col_out && m_begin >= 0 && m_end <= e0 && m_begin - D + a0 >= 0 && m_end - 1 + a0 < ag;

  using T0 = std::true_type;
  using T1 = std::false_type;
#if J2D_RING > 0
  // rows staged NR-1 ahead by per-lane 8-byte cp.async into a per-warp shared
  // ring ([slot][p][lane]: conflict-free); each lane reads back only what it
  // copied itself, so cp.async.wait_group is the only synchronisation
  constexpr int NR = J2D_RING;
  static_assert((NR & (NR - 1)) == 0, "ring depth must be a power of two");
  __shared__ double ring[NR][kP2][32];
  auto row_ok_f = [&](int mm) { return mm >= 0 && mm < e0 && mm + a0 >= 0 && mm + a0 < ag; };
  auto run = [&](auto in_tag) {
    constexpr bool IN = decltype(in_tag)::value;
    auto issue_row = [&](int mm) {
      if (mm < m_end && (IN || row_ok_f(mm))) {
        const double* rp = col_base + (int64_t)mm * g.s0;
        const int slot = (mm - m_begin) & (NR - 1);
#pragma unroll
        for (int p = 0; p < kP2; ++p)
          if (IN || !(col_out >> p & 1u)) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&ring[slot][p][lane]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(rp + p));
          }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    auto read_row = [&](int mm, double (&r)[kP2]) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NR - 1) : "memory");
      const int slot = (mm - m_begin) & (NR - 1);
      if constexpr (IN) {
#pragma unroll
        for (int p = 0; p < kP2; ++p) r[p] = ring[slot][p][lane];
      } else {
        const bool ok = row_ok_f(mm);
#pragma unroll
        for (int p = 0; p < kP2; ++p) r[p] = (ok && !(col_out >> p & 1u)) ? ring[slot][p][lane] : bnd;
      }
    };
#pragma unroll
    for (int k = 0; k < NR - 1; ++k) issue_row(m_begin + k);
    int m = m_begin;
    for (; m + 2 <= m_end; m += 2) {
      double row[kP2];
      issue_row(m + NR - 1);
      read_row(m, row);
      step(m, row, T0{}, in_tag);
      issue_row(m + NR);
      read_row(m + 1, row);
      step(m + 1, row, T1{}, in_tag);
    }
    if (m < m_end) {
      double row[kP2];
      issue_row(m + NR - 1);
      read_row(m, row);
      step(m, row, T0{}, in_tag);
    }
  };
  if (interior)
    run(T0{});
  else
    run(T1{});
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

#else
  (void)interior;
  constexpr int PF = J2D_PF;  // rows prefetched ahead (registers, even)
  static_assert(PF % 2 == 0, "role swap alternates per step");
  double pre[PF][kP2];
#pragma unroll
  for (int k = 0; k < PF; ++k) load_row(m_begin + k, pre[k]);
  int m = m_begin;
  for (; m + PF <= m_end; m += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      double row[kP2];
#pragma unroll
      for (int p = 0; p < kP2; ++p) row[p] = pre[k][p];
      load_row(m + k + PF, pre[k]);
      if (k % 2 == 0)
        step(m + k, row, T0{}, T1{});
      else
        step(m + k, row, T1{}, T1{});
    }
  }
  // tail (fewer than PF rows left); parity continues from the unrolled loop
  for (; m < m_end; ++m) {
    double row[kP2];
#pragma unroll
    for (int p = 0; p < kP2; ++p) row[p] = pre[0][p];
#pragma unroll
    for (int kk = 0; kk + 1 < PF; ++kk)
#pragma unroll
      for (int p = 0; p < kP2; ++p) pre[kk][p] = pre[kk + 1][p];
    if (((m - m_begin) & 1) == 0)
      step(m, row, T0{}, T1{});
    else
      step(m, row, T1{}, T1{});
  }
}
#endif

// Coefficients by 3x3 position if the offsets are strictly sorted (the
// kernel's fixed order); returns the tap mask or 0.
static unsigned slots2d(const tvs_stencil& st, Coeff9& cf) {
  unsigned mask = 0;
  int last = -100;
  for (int k = 0; k < 9; ++k) cf.c[k] = 0.0;
  for (int k = 0; k < st.ntaps; ++k) {
    const int pos = (st.offsets[k][0] + 1) * 3 + (st.offsets[k][1] + 1);
    if (pos <= last) return 0;
    last = pos;
    mask |= 1u << pos;
    cf.c[pos] = st.coeffs[k];
  }
  return mask;
}

bool jacobi2d_blocked_supported(const tvs_stencil& st) {
  Coeff9 cf;
  const unsigned m = slots2d(st, cf);
  return m == kStar5 || m == kBox9;
}

int jacobi2d_max_depth() { return kMaxD2; }
int jacobi2d_default_depth() { return 8; }  // measured best (config 3, P = 3: D = 6 1392, 7 1593, 8 1723, 10 1576 GSt/s)

// mode 0: unfused taps, 1: fused (FMA), 2: scaled power-of-two taps (SC)
template <unsigned MASK, int D, int P>
static void launch2d_d(int mode, unsigned blocks, cudaStream_t s, const double* src, double* dst, const Geo& geo,
                       int64_t origin, const Coeff9& cf, double bnd, int64_t ns, int64_t nt, int64_t lo, int64_t hi,
                       int seg_rows, const Mirror& mir) {
  // the mirror-store form only for sharded passes: no cost on one GPU
  const bool mirrored = mir.p[0] != nullptr || mir.p[1] != nullptr;
  auto go = [&](auto kern) { kern<<<blocks, kWarps2 * 32, 0, s>>>(src, dst, geo, origin, cf, bnd, ns, nt, lo, hi, seg_rows, mir); };
  if (mode == 2) {
    if (mirrored) go(jacobi2d_kernel<MASK, D, true, P, true, true>);
    else go(jacobi2d_kernel<MASK, D, true, P, false, true>);
  } else if (mode == 1) {
    if (mirrored) go(jacobi2d_kernel<MASK, D, true, P, true, false>);
    else go(jacobi2d_kernel<MASK, D, true, P, false, false>);
  } else {
    if (mirrored) go(jacobi2d_kernel<MASK, D, false, P, true, false>);
    else go(jacobi2d_kernel<MASK, D, false, P, false, false>);
  }
}

// Rows per warp task when the caller does not fix it.  One-warp blocks are
// scheduled in waves of `resident` (occupancy x SMs); a launch of
// strips x segments tasks costs ~ ceil(tasks / resident) x (seg + 2D + c)
// row-steps (c: per-task prologue).  The segment count is chosen to fill the
// last wave: config 3 (16384 rows, 171 strips, 1776 resident at D = 8):
// 256-row segments give 10944 tasks = 6.2 waves (the 7th at 16%), 72
// segments of 228 rows 12312 = 6.9 waves.  TVS_J2D_SEG fixes it.  Rows
// shorter than 128 form one segment.
static int auto_seg(int64_t rows, int64_t strips, int depth, int64_t resident) {
  static const int fixed = [] {
    const char* e = getenv("TVS_J2D_SEG");
    return e ? atoi(e) : 0;
  }();
  if (fixed > 0) return fixed;
  if (resident <= 0) return kRowsSeg;
  double best = 1e300;
  int64_t best_seg = kRowsSeg;
  const int64_t max_nseg = std::max<int64_t>(1, rows / 32);
  for (int64_t nseg = 1; nseg <= max_nseg; ++nseg) {
    const int64_t seg = (rows + nseg - 1) / nseg;
    // 128..256 rows: the measured range (config 3 per MHz: 128 0.89, 192
    // 1.01, 228 1.01, 256 0.96 GSt/s/MHz); longer segments leave too little
    // slack for the uneven boundary / interior warps
    if (seg > 256 || (seg < 128 && rows >= 128)) continue;
    const int64_t tasks = strips * ((rows + seg - 1) / seg);
    const double cost = (double)((tasks + resident - 1) / resident) * (double)(seg + 2 * depth + 4);
    if (cost < best * 0.999) best = cost, best_seg = seg;
  }
  return (int)best_seg;
}

template <class K>
static int64_t resident_blocks(K kern) {
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kWarps2 * 32, 0) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (int64_t)per * sms;
}

// rows [row_lo, row_hi) of the grid (any band; the
// whole grid by default): one row band of the pipelined host path
template <unsigned MASK, int D>
static void launch2d_one(int mode, cudaStream_t s, const double* src, double* dst, const Geo& geo, int64_t origin,
                         const Coeff9& cf, double bnd, int64_t row_lo, int64_t row_hi, int seg_rows,
                         const Mirror& mir) {
  // columns per lane: registers grow as 2 * P * D accumulators; P = 3 at
  // D = 5..8 keeps 12 warps/SM at D = 8 (168 registers) where P = 4 held 9
  // (config 3: D = 8 P = 4 1596, P = 3 1723 GSt/s; D > 8 at P = 3 is slower)
#ifndef J2D_P4MAX
#define J2D_P4MAX 4
#endif
  constexpr int P = D <= J2D_P4MAX ? 4 : (D <= 8 ? 3 : 2);
  const int64_t U = 32 * P - 2 * D;
  const int64_t ns = (geo.e1 + U - 1) / U;
  if (seg_rows <= 0) {
    static const int64_t res[3] = {resident_blocks(jacobi2d_kernel<MASK, D, false, P, false, false>),
                                   resident_blocks(jacobi2d_kernel<MASK, D, true, P, false, false>),
                                   resident_blocks(jacobi2d_kernel<MASK, D, true, P, false, true>)};
    seg_rows = auto_seg(row_hi - row_lo, ns, D, res[mode]);
  }
  const int64_t nseg = (row_hi - row_lo + seg_rows - 1) / seg_rows;
  const int64_t nt = ns * nseg;
  const unsigned blocks = (unsigned)((nt + kWarps2 - 1) / kWarps2);
  launch2d_d<MASK, D, P>(mode, blocks, s, src, dst, geo, origin, cf, bnd, ns, nt, row_lo, row_hi, seg_rows, mir);
}

template <unsigned MASK>
static void launch2d(int depth, int mode, cudaStream_t s, const double* src, double* dst, const Geo& geo,
                     int64_t origin, const Coeff9& cf, double bnd, int64_t lo, int64_t hi, int seg, const Mirror& mir) {
  switch (depth) {
    case 1: launch2d_one<MASK, 1>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 2: launch2d_one<MASK, 2>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 3: launch2d_one<MASK, 3>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 4: launch2d_one<MASK, 4>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 5: launch2d_one<MASK, 5>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 6: launch2d_one<MASK, 6>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 7: launch2d_one<MASK, 7>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 8: launch2d_one<MASK, 8>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 9: launch2d_one<MASK, 9>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 10: launch2d_one<MASK, 10>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    case 11: launch2d_one<MASK, 11>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
    default: launch2d_one<MASK, 12>(mode, s, src, dst, geo, origin, cf, bnd, lo, hi, seg, mir); break;
  }
}

int jacobi2d_band_rows() { return kRowsSeg; }


// Scaled taps (SC) instead of DMUL + DFMAs when every coefficient is a power
// of two (the fused form is already exact then): one FP64 instruction less
// per update.  The carried values grow by 1/|c_first| per level (heat2d:
// 8^D, 2^24 at D = 8), so values must stay below 2^(1023 - D*log2(1/|c0|))
// — the same class of caveat as the fused-exact form's subnormal products;
// TVS_J2D_SCALED=0 disables it.
static bool scaled_ok(const tvs_stencil& st, const Coeff9& cf, int depth) {
  static const bool off = [] {
    const char* e = getenv("TVS_J2D_SCALED");
    return e && atoi(e) == 0;
  }();
  if (off || !coeffs_power_of_two(st)) return false;
  int first = -1;
  for (int k = 0; k < 9 && first < 0; ++k)
    if (cf.c[k] != 0.0) first = k;
  if (first < 0) return false;
  int ex0;
  std::frexp(cf.c[first], &ex0);
  for (int k = 0; k < 9; ++k) {
    if (cf.c[k] == 0.0) continue;
    int ex;
    std::frexp(cf.c[k], &ex);
    if (std::abs(ex - ex0) > 60) return false;
  }
  return std::abs(ex0 - 1) * depth <= 120;  // growth of the carried values
}

int jacobi2d_blocked(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, int depth,
                     bool fma, cudaStream_t s, int64_t row_lo, int64_t row_hi, int seg_rows, const Mirror* mir) {
  Coeff9 cf;
  const unsigned mask = slots2d(st, cf);
  if ((mask != kStar5 && mask != kBox9) || depth < 1 || depth > kMaxD2)
    return fail(TVS_ERR_UNSUPPORTED, "jacobi2d_blocked: tap set or depth");
  if (row_hi < 0) row_hi = g.extents[0];
  if (row_lo < 0 || row_hi > g.extents[0] || row_lo >= row_hi)
    return fail(TVS_ERR_INVALID, "jacobi2d_blocked: row band");
  const Geo geo = make_geo(g);
  const Mirror m = mir ? *mir : Mirror{};
  const int mode = fma ? (scaled_ok(st, cf, depth) ? 2 : 1) : 0;
  if (mode == 2) {
    // scaled taps: ratios to the first tap's coefficient, per-level pins
    const double c0 = cf.c[__builtin_ctz(mask)];
    for (int k = 0; k < 9; ++k) cf.c[k] /= c0;
    double sc = 1.0;
    for (int l = 0; l <= kMaxD2; ++l) {
      sc /= c0;
      cf.bl[l] = st.boundary * sc;
    }
    cf.out_scale = 1.0;
    for (int l = 0; l < depth; ++l) cf.out_scale *= c0;  // exact: powers of two
  }
  if (mask == kStar5)
    launch2d<kStar5>(depth, mode, s, src, dst, geo, g.origin, cf, st.boundary, row_lo, row_hi, seg_rows, m);
  else
    launch2d<kBox9>(depth, mode, s, src, dst, geo, g.origin, cf, st.boundary, row_lo, row_hi, seg_rows, m);
  TVS_LAUNCHED("jacobi2d_kernel");
  return TVS_OK;
}

}  // namespace tvs
