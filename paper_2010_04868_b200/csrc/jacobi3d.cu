// K4: 3D radius-1 Jacobi (27-point box / 7-point star), 2.5D plane streaming.
//
// Replaces jacobi3d_temporal (reference kernels_nd.py:43-45).  A block owns a
// (32 x 32) tile of axis-1 x axis-2 columns (4 outputs per thread) and streams
// along axis 0.  Each input plane is staged once in shared memory (16-byte
// cp.async, three buffers, one barrier per plane) and
// contributes to three outputs: it *finishes* output p-1 with the +1-plane
// taps, continues output p with the 0-plane taps and *starts* output p+1 with
// the -1-plane taps.  Sorted tap order is exactly plane -1, plane 0, plane +1
// (each row-major), so the per-point accumulation order equals the
// reference's `acc = c*v + acc` chain (baselines.py:43-49) — bit-exact.
//
// Unfused, a 27-point update costs 53 FP64 ops, so this kernel is FP64-issue
// bound (~351 GStencil/s at 1.965 GHz), below the single-step HBM roofline
// (~409); the FMA form (tolerance mode) halves the op count.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cuda.h>

#include "common.cuh"

namespace tvs {

constexpr int kTX3 = 32;              // tile width (axis 2) = threads in x
constexpr int kTYT = 8;               // threads in y
constexpr int kRY = 4;                // outputs per thread along axis 1
constexpr int kTY3 = kTYT * kRY;      // tile height (axis 1) = 32
constexpr int kSW = kTX3 + 4;         // smem row: x0-2 .. x0+33 (16-byte aligned start)
constexpr int kSH = kTY3 + 2;         // smem rows: y0-1 .. y0+32
constexpr int kChunks = kSH * kSW / 2;  // 16-byte copies per plane
constexpr int kThreads3 = kTX3 * kTYT;
constexpr int kSlots = (kChunks + kThreads3 - 1) / kThreads3;
constexpr int kBufs3 = 3;             // plane buffers (one barrier per plane)
constexpr int kPlanesSeg = 64;        // output planes per block

constexpr unsigned kBox27 = (1u << 27) - 1;
constexpr unsigned kStar7 = (1u << 4) | (1u << 10) | (1u << 12) | (1u << 13) | (1u << 14) | (1u << 16) | (1u << 22);

struct Coeff27 {
  double c[27];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// acc[r] (+)= taps of plane-group G (d0 = G-1) for the thread's kRY outputs.
template <unsigned MASK, int G, bool START, bool FMA>
__device__ __forceinline__ void add_plane(double (&acc)[kRY], const double (&v)[kRY + 2][3], const double* c) {
#pragma unroll
  for (int r = 0; r < kRY; ++r) {
    bool fresh = START;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int bit = G * 9 + k;
      if ((MASK >> bit) & 1u) {
        const double x = v[r + k / 3][k % 3];
        if (fresh) {
          acc[r] = tap_first(c[bit], x);
          fresh = false;
        } else {
          acc[r] = tap_next<FMA>(c[bit], x, acc[r]);
        }
      }
    }
  }
}

template <unsigned MASK>
__device__ __forceinline__ constexpr bool has_plane(int G) {
  return ((MASK >> (G * 9)) & 0x1FFu) != 0;
}

template <unsigned MASK, bool FMA>
__global__ void __launch_bounds__(kThreads3) jacobi3d_kernel(const double* __restrict__ src,
                                                            double* __restrict__ dst, Geo g, int64_t origin,
                                                            Coeff27 cf, double bnd, int64_t plo, int64_t phi,
                                                            int seg, Mirror mir) {
  constexpr bool G0 = has_plane<MASK>(0), G1 = has_plane<MASK>(1), G2 = has_plane<MASK>(2);
  __shared__ __align__(16) double tile[kBufs3][kSH][kSW];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * kTX3 + tx;
  const int64_t x0 = (int64_t)blockIdx.x * kTX3, y0 = (int64_t)blockIdx.y * kTY3;
  const int64_t p0 = plo + (int64_t)blockIdx.z * seg;
  const int64_t p1 = min(p0 + seg, phi);  // outputs [p0, p1)

  // per-thread staging slots, fixed for every plane: smem offset + global
  // offset relative to the plane base; rows beyond the halo are not read
  int soff[kSlots];
  int64_t goff[kSlots];
  bool sval[kSlots];
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int e = tid + k * kThreads3;
    const int r = e / (kSW / 2), c2 = e % (kSW / 2);
    const int64_t y = y0 + r - 1;
    soff[k] = r * kSW + 2 * c2;
    goff[k] = y * g.s1 + (x0 - 2 + 2 * c2);
    sval[k] = e < kChunks && y <= g.e1;
  }
  const double* base = src + origin;
  auto stage = [&](int64_t p, int buf) {
    const double* pb = base + p * g.s0;
    double* tb = &tile[buf][0][0];
#pragma unroll
    for (int k = 0; k < kSlots; ++k)
      if (sval[k]) cp_async16(tb + soff[k], pb + goff[k]);
    cp_async_commit();
  };

  double A[kRY], B[kRY];
#pragma unroll
  for (int r = 0; r < kRY; ++r) A[r] = B[r] = 0.0;

  const int64_t x = x0 + tx;
  const bool x_ok = x < g.e2;
  stage(p0 - 1, 0);
  for (int64_t p = p0 - 1; p <= p1; ++p) {
    const int buf = (int)((p - p0 + 1) % kBufs3);
    if (p + 1 <= p1) {
      // buffer of plane p-2: every thread finished reading it before the
      // previous iteration's barrier
      stage(p + 1, (int)((p - p0 + 2) % kBufs3));
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // plane p landed for everyone; plane p-2's buffer is free
    double v[kRY + 2][3];
#pragma unroll
    for (int rr = 0; rr < kRY + 2; ++rr)
#pragma unroll
      for (int k = 0; k < 3; ++k) v[rr][k] = tile[buf][ty * kRY + rr][tx + 1 + k];
    double out[kRY];
    if constexpr (G2) add_plane<MASK, 2, !(G0 || G1), FMA>(B, v, cf.c);
#pragma unroll
    for (int r = 0; r < kRY; ++r) out[r] = B[r];
#pragma unroll
    for (int r = 0; r < kRY; ++r) B[r] = A[r];
    if constexpr (G1) add_plane<MASK, 1, !G0, FMA>(B, v, cf.c);
    if constexpr (G0) add_plane<MASK, 0, true, FMA>(A, v, cf.c);
    // out = output plane p-1
    const int64_t q = p - 1;
    if (q >= p0 && q < p1 && x_ok) {
      const int64_t gq = q + g.a0_off;
      const bool pin = gq < 0 || gq >= g.a0_glob;
      // local plane, plus the neighbour's ghost plane when sharded
      for_each_dst(dst, mir, q, [&](double* b) {
        double* op = b + origin + q * g.s0 + x;
#pragma unroll
        for (int r = 0; r < kRY; ++r) {
          const int64_t y = y0 + ty * kRY + r;
          if (y < g.e1) op[y * g.s1] = pin ? bnd : out[r];
        }
      });
    }
  }
}

// ---- K4b: two time levels per HBM pass ---------------------------------
//
// Temporal blocking of K4 (north_star: "several time steps are advanced per
// HBM round-trip").  A block owns a 64 x 32 frame of axis-2 x axis-1
// positions (frame (i, j) = global (y0-1+i, x0-1+j)) and streams along axis
// 0.  Per input plane p (staged once in shared memory by 16-byte cp.async,
// 34 x 68 cells = the frame plus a 1-cell ring):
//   level 1: every frame position takes the plane's 3x3 taps (finishing
//            level-1 plane p-1, continuing p, starting p+1) — the K4 partial
//            sums — and the finished plane p-1 is written to a shared level-1
//            buffer (cells outside the domain pinned to the boundary, exactly
//            what a single step reads from the memory halo);
//   level 2: after one barrier, every frame position takes level-1 plane
//            p-1's 3x3 taps, finishing level-2 plane p-2, which is stored for
//            the inner 62 x 30 positions.
// Both levels use K4's accumulation order (sorted taps: plane -1, 0, +1,
// each row-major), so two levels equal two K4 launches bit for bit.  HBM
// traffic per update ~ (8 B x 34*68/(62*30) + 8 B) / 2 ~ 9 B instead of 16.
constexpr int kTBW = 64;               // frame width (2 columns per lane)
constexpr int kTBH = 32;               // frame height (8 warps x kRY rows)
constexpr int kTBOX = kTBW - 2;        // useful output columns per block
constexpr int kTBOY = kTBH - 2;        // useful output rows per block
constexpr int kTBP = 68;               // smem pitch (frame + ring, 16-byte rows)
constexpr int kTBR = kTBH + 2;         // smem rows
constexpr int kTBChunks = kTBR * (kTBP / 2);
constexpr int kTBSlots = (kTBChunks + kThreads3 - 1) / kThreads3;
#ifndef J3D_TBSEG
#define J3D_TBSEG 128  // measured (1024^3, T=20): 32 225 / 318, 64 235 / 332, 128 237 / 342, 256 232 / 339 GSt/s (exact / fma)
#endif
constexpr int kTBPlanesSeg = J3D_TBSEG;  // output planes per block
constexpr size_t kTBSmem = (size_t)(3 + 2) * kTBR * kTBP * sizeof(double);

template <unsigned MASK, bool FMA>
__device__ __forceinline__ void tb_level(const double* __restrict__ plane, int w, int lane, double (&A)[2][kRY],
                                         double (&B)[2][kRY], double (&out)[2][kRY], const double* c) {
  constexpr bool G0 = has_plane<MASK>(0), G1 = has_plane<MASK>(1), G2 = has_plane<MASK>(2);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double v[kRY + 2][3];
    const double* b = plane + (w * kRY) * kTBP + lane + 32 * h;
#pragma unroll
    for (int rr = 0; rr < kRY + 2; ++rr)
#pragma unroll
      for (int k = 0; k < 3; ++k) v[rr][k] = b[rr * kTBP + k];
    if constexpr (G2) add_plane<MASK, 2, !(G0 || G1), FMA>(B[h], v, c);
#pragma unroll
    for (int r = 0; r < kRY; ++r) out[h][r] = B[h][r];
#pragma unroll
    for (int r = 0; r < kRY; ++r) B[h][r] = A[h][r];
    if constexpr (G1) add_plane<MASK, 1, !G0, FMA>(B[h], v, c);
    if constexpr (G0) add_plane<MASK, 0, true, FMA>(A[h], v, c);
  }
}

template <unsigned MASK, bool FMA, bool MIR>
__global__ void __launch_bounds__(kThreads3, 2) jacobi3d_tb_kernel(const double* __restrict__ src,
                                                                   double* __restrict__ dst, Geo g, int64_t origin,
                                                                   Coeff27 cf, double bnd, int64_t plo,
                                                                   int64_t phi, int seg, Mirror mir) {
  extern __shared__ __align__(16) double tb_smem[];
  double* l0 = tb_smem;                       // 3 staged input planes
  double* l1 = tb_smem + 3 * kTBR * kTBP;     // 2 level-1 planes (frame at +1,+1)
  const int lane = threadIdx.x, w = threadIdx.y;
  const int tid = w * 32 + lane;
  const int64_t x0 = (int64_t)blockIdx.x * kTBOX, y0 = (int64_t)blockIdx.y * kTBOY;
  const int64_t p0 = plo + (int64_t)blockIdx.z * seg;
  const int64_t p1 = min(p0 + seg, phi);  // level-2 outputs [p0, p1)

  // staging slots: smem cell (row i, col 2c) <- global (y0-2+i, x0-2+2c);
  // rows/columns beyond the memory halo are never needed (their level-1
  // positions are pinned) and are not read
  int soff[kTBSlots];  // shared offset, -1: slot not read
  int goff[kTBSlots];    // element offset within the plane (host checks a plane fits 31 bits)
#pragma unroll
  for (int k = 0; k < kTBSlots; ++k) {
    const int e = tid + k * kThreads3;
    const int i = e / (kTBP / 2), c2 = e % (kTBP / 2);
    const int64_t y = y0 - 2 + i, x = x0 - 2 + 2 * c2;
    const bool ok = e < kTBChunks && y >= -1 && y <= g.e1 && x <= g.e2;
    soff[k] = ok ? i * kTBP + 2 * c2 : -1;
    goff[k] = (int)(y * g.s1 + x);
  }

  // per-thread frame positions: rows i = w*kRY + r, columns j = lane + 32h
  unsigned in_dom = 0;   // bit (h*kRY + r): level-1 position inside the domain (axes 1, 2)
  unsigned store_ok = 0; // bit (h*kRY + r): useful level-2 output
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < kRY; ++r) {
      const int i = w * kRY + r, j = lane + 32 * h;
      const int64_t y = y0 - 1 + i, x = x0 - 1 + j;
      const bool dom = y >= 0 && y < g.e1 && x >= 0 && x < g.e2;
      in_dom |= (dom ? 1u : 0u) << (h * kRY + r);
      store_ok |= (dom && i >= 1 && i < kTBH - 1 && j >= 1 && j < kTBW - 1 ? 1u : 0u) << (h * kRY + r);
    }
  const bool all_dom = in_dom == 0xFFu;

  double A1[2][kRY], B1[2][kRY], A2[2][kRY], B2[2][kRY], out[2][kRY];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < kRY; ++r) A1[h][r] = B1[h][r] = A2[h][r] = B2[h][r] = 0.0;

  // Iteration t handles input plane p = p0-2+t: level-1 plane q1 = p-1 and
  // level-2 plane q2 = p-2.  Every plane-range test is a 32-bit compare of t
  // against a bound fixed per block (seg <= 2^30 planes).
  const int np = (int)(p1 - p0);
  auto clampi = [](int64_t v) { return (int)max((int64_t)-4, min(v, (int64_t)1 << 30)); };
  const int ts_lo = clampi(1 - p0), ts_hi = clampi(g.e0 - p0 + 2);  // staged planes: t in [ts_lo, ts_hi]
  // level-1 plane q1 = p0-3+t is inside the (local and global) domain for t in [t1_lo, t1_hi)
  const int t1_lo = clampi(max(3 - p0, 3 - p0 - g.a0_off));
  const int t1_hi = clampi(min(g.e0 - p0 + 3, g.a0_glob - g.a0_off - p0 + 3));
  // level-2 plane q2 = p0-4+t inside the global domain for t in [t2_lo, t2_hi)
  const int t2_lo = clampi(4 - p0 - g.a0_off), t2_hi = clampi(g.a0_glob - g.a0_off - p0 + 4);

  constexpr int kPlane = kTBR * kTBP;
  const double* pb = src + origin + (p0 - 2) * g.s0;  // plane staged next
  // its ring slot as a shared-window byte address (the generic -> shared
  // conversion happens once, not per copy)
  const unsigned l0a = smaddr(l0);
  unsigned sba = l0a;
  auto stage = [&](int t) {
    if (t >= ts_lo && t <= ts_hi) {
#pragma unroll
      for (int k = 0; k < kTBSlots; ++k)
        if (soff[k] >= 0)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sba + 8u * (unsigned)soff[k]), "l"(pb + goff[k]));
    }
    cp_async_commit();
    pb += g.s0;
    sba = sba == l0a + 2u * kPlane * 8u ? l0a : sba + kPlane * 8u;
  };
  // the thread's first output cell of level-2 plane p0 (advanced per plane)
  int64_t ooff = origin + p0 * g.s0 + (y0 - 1 + w * kRY) * g.s1 + (x0 - 1 + lane);
  const int tpos = (w * kRY) * kTBP + lane;  // the thread's window origin in a plane
  const double* cur = l0;                    // staged plane of iteration t
  int l1sel = kPlane;                        // level-1 buffer of iteration t (t = 0: buffer 1)

  // One barrier per plane: level 2 runs one plane behind level 1 and reads
  // the level-1 plane written in the previous iteration (two level-1 buffers:
  // iteration t writes buffer t & 1, which iteration t-1's level 2 -- reading
  // buffer (t-2) & 1 -- released before this iteration's barrier).
#ifndef J3D_LAG
#define J3D_LAG 1
#endif
  constexpr int kLag = J3D_LAG;  // 0: level 2 in the same iteration (a second barrier per plane)
  stage(0);
  for (int t = 0; t <= np + 3 + kLag; ++t) {
    stage(t + 1);  // empty group past the end keeps the wait count uniform
    cp_async_wait<1>();
    __syncthreads();  // plane p visible; iteration t-1 finished everywhere
    // level 1: plane p -> finishes level-1 plane q1 = p-1
    tb_level<MASK, FMA>(cur, w, lane, A1, B1, out, cf.c);
    cur = cur == l0 + 2 * kPlane ? l0 : cur + kPlane;
    double* l1b = l1 + l1sel;
    l1sel ^= kPlane;
    {
      double* q = l1b + tpos + kTBP + 1;
      if (t >= t1_lo && t < t1_hi && all_dom) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int r = 0; r < kRY; ++r) q[r * kTBP + 32 * h] = out[h][r];
      } else {
        const bool plane_in = t >= t1_lo && t < t1_hi;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int r = 0; r < kRY; ++r)
            q[r * kTBP + 32 * h] = plane_in && (in_dom >> (h * kRY + r) & 1u) ? out[h][r] : bnd;
      }
    }
    if constexpr (kLag == 0) __syncthreads();  // level-1 plane q1 visible
    if (t >= 2 + kLag) {
      // level 2: level-1 plane q1 - kLag -> finishes level-2 plane q2 = q1 - kLag - 1
      tb_level<MASK, FMA>(kLag ? l1 + l1sel : l1b, w, lane, A2, B2, out, cf.c);
      if (t >= 4 + kLag) {
        if (t < t2_lo + kLag || t >= t2_hi + kLag) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < kRY; ++r) out[h][r] = bnd;
        }
        auto store = [&](double* b) {
          double* op = b + ooff;
#pragma unroll
          for (int r = 0; r < kRY; ++r) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (store_ok >> (h * kRY + r) & 1u) op[32 * h] = out[h][r];
            op += g.s1;
          }
        };
        if constexpr (MIR)
          for_each_dst(dst, mir, p0 - 4 - kLag + t, store);  // sharded: local plane + the neighbour's ghost plane
        else
          store(dst);
        ooff += g.s0;
      }
    }
  }
}

// ---- K4c: K4b staged by TMA, adjacent column pairs per lane --------------
//
// Same two-level scheme, frame and arithmetic as K4b (bit-identical), with the
// per-plane overhead cut (K4b in FMA mode issued ~300 non-FP64 instructions
// per 432 DFMAs and was issue-limited):
//   * the 34 x 66 input box of every plane is one 3D tensor-map copy
//     (cp.async.bulk.tensor, issued by one thread, completion on an mbarrier;
//     out-of-range rows / planes are zero-filled by the TMA unit and only ever
//     feed pinned or discarded positions) instead of five predicated 16-byte
//     cp.async per thread with their address arithmetic;
//   * a lane owns two ADJACENT frame columns (2 lane, 2 lane + 1): the 4-wide
//     window row both columns need is two LDS.128 (12 loads per level instead
//     of 36 LDS.64), consumed row by row so the window is never held whole;
//   * one CTA barrier per plane: level 2 runs one plane behind level 1.
constexpr int kPW = kTBW + 2;                 // staged box width (frame + ring)
// NW warps of kRY frame rows each: 8 (64 x 32 frame, two CTAs per SM, K4b's
// frame; the default) or 16 (64 x 64, one CTA per SM: 62 x 62 useful of
// 64 x 64 instead of 62 x 30 of 64 x 32; slower, see jacobi3d_blocked2)
template <int NW>
struct TmaCfg {
  static constexpr int H = NW * kRY;        // frame rows
  static constexpr int OY = H - 2;          // useful output rows per block
  static constexpr int R = H + 2;           // staged box rows
  static constexpr int Slot = (R * kPW * 8 + 127) / 128 * 128 / 8;  // slot pitch (elements), 128-byte multiple
  static constexpr unsigned Bytes = R * kPW * 8;                   // bytes one plane copy delivers
  static constexpr size_t Smem = (size_t)5 * Slot * sizeof(double) + 3 * sizeof(unsigned long long) + 128;
  static constexpr int Threads = 32 * NW;
  static constexpr int MinB = NW <= 8 ? 2 : 1;
};

template <unsigned MASK, int G>
constexpr int first_tap() {
  for (int k = 0; k < 9; ++k)
    if ((MASK >> (9 * G + k)) & 1u) return k;
  return -1;
}

// One level over the thread's 4 rows x 2 adjacent columns: `win` = window
// origin (plane cell of frame row 4w - 1, frame column 2 lane - 1).  Sorted
// tap order per accumulator (plane group, then window row, then column), as
// add_plane: finishes out = B + (+1-plane taps), B <- A + (0-plane taps),
// A <- (-1-plane taps).
template <unsigned MASK, bool FMA>
__device__ __forceinline__ void pair_level(const double* __restrict__ win, double (&A)[2][kRY], double (&B)[2][kRY],
                                           double (&out)[2][kRY], const double* c) {
  constexpr bool G0 = has_plane<MASK>(0), G1 = has_plane<MASK>(1), G2 = has_plane<MASK>(2);
  constexpr int f0 = first_tap<MASK, 0>(), f1 = first_tap<MASK, 1>(), f2 = first_tap<MASK, 2>();
  double An[2][kRY];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < kRY; ++r) {
      out[h][r] = B[h][r];
      B[h][r] = A[h][r];
      An[h][r] = 0.0;
    }
#pragma unroll
  for (int rr = 0; rr < kRY + 2; ++rr) {
    const double2 lo = *reinterpret_cast<const double2*>(win + rr * kPW);
    const double2 hi = *reinterpret_cast<const double2*>(win + rr * kPW + 2);
    const double v[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
    for (int dy = 2; dy >= 0; --dy) {  // the output closest to completion first
      const int r = rr - dy;
      if (r < 0 || r >= kRY) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int t9 = dy * 3 + k;
          const double x = v[h + k];
          if (G2 && ((MASK >> (18 + t9)) & 1u))
            out[h][r] = (!(G0 || G1) && t9 == f2) ? tap_first(c[18 + t9], x) : tap_next<FMA>(c[18 + t9], x, out[h][r]);
          if (G1 && ((MASK >> (9 + t9)) & 1u))
            B[h][r] = (!G0 && t9 == f1) ? tap_first(c[9 + t9], x) : tap_next<FMA>(c[9 + t9], x, B[h][r]);
          if (G0 && ((MASK >> t9) & 1u))
            An[h][r] = t9 == f0 ? tap_first(c[t9], x) : tap_next<FMA>(c[t9], x, An[h][r]);
        }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < kRY; ++r) A[h][r] = An[h][r];
}

template <unsigned MASK, bool FMA, bool MIR, int NW>
__global__ void __launch_bounds__(TmaCfg<NW>::Threads, TmaCfg<NW>::MinB) jacobi3d_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                    double* __restrict__ dst, Geo g, int64_t origin,
                                                                    Coeff27 cf, double bnd, int64_t plo,
                                                                    int64_t phi, int seg, Mirror mir) {
  constexpr int kPSlot = TmaCfg<NW>::Slot, kFH = TmaCfg<NW>::H, kFOY = TmaCfg<NW>::OY;
  constexpr unsigned kPBytes = TmaCfg<NW>::Bytes;
  extern __shared__ unsigned char tma_smem_raw[];
  // 128-byte aligned slots (TMA destination alignment)
  const unsigned raw = smaddr(tma_smem_raw);
  double* const l0 = reinterpret_cast<double*>(tma_smem_raw + ((128u - (raw & 127u)) & 127u));  // 3 staged planes
  double* const l1 = l0 + 3 * kPSlot;                                                              // 2 level-1 planes
  unsigned long long* const full = reinterpret_cast<unsigned long long*>(l1 + 2 * kPSlot);
  const int lane = threadIdx.x, w = threadIdx.y;
  const int tid = w * 32 + lane;
  const int64_t x0 = (int64_t)blockIdx.x * kTBOX, y0 = (int64_t)blockIdx.y * kFOY;
  const int64_t p0 = plo + (int64_t)blockIdx.z * seg;
  const int64_t p1 = min(p0 + seg, phi);  // level-2 outputs [p0, p1)
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) mbar_init(full + k, 1);
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  // frame (i, j) = global (y0-1+i, x0-1+j) = plane cell (i+1, j+1); the
  // thread owns rows i = 4w + r, columns j = 2 lane + h
  unsigned in_dom = 0;    // bit (h*kRY + r): level-1 position inside the domain (axes 1, 2)
  unsigned store_ok = 0;  // bit (h*kRY + r): useful level-2 output
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < kRY; ++r) {
      const int i = w * kRY + r, j = 2 * lane + h;
      const int64_t y = y0 - 1 + i, x = x0 - 1 + j;
      const bool dom = y >= 0 && y < g.e1 && x >= 0 && x < g.e2;
      in_dom |= (dom ? 1u : 0u) << (h * kRY + r);
      store_ok |= (dom && i >= 1 && i < kFH - 1 && j >= 1 && j < kTBW - 1 ? 1u : 0u) << (h * kRY + r);
    }
  const bool all_dom = in_dom == 0xFFu;

  double A1[2][kRY], B1[2][kRY], A2[2][kRY], B2[2][kRY], out[2][kRY];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < kRY; ++r) A1[h][r] = B1[h][r] = A2[h][r] = B2[h][r] = 0.0;

  // Iteration t: input plane p = p0-2+t lands (slot t % 3), level 1 finishes
  // level-1 plane p-1 into buffer t & 1, level 2 reads buffer (t-1) & 1
  // (level-1 plane p-2) and finishes level-2 plane p-3 = p0-5+t.
  const int np = (int)(p1 - p0);
  auto clampi = [](int64_t v) { return (int)max((int64_t)-4, min(v, (int64_t)1 << 30)); };
  const int t1_lo = clampi(max(3 - p0, 3 - p0 - g.a0_off));
  const int t1_hi = clampi(min(g.e0 - p0 + 3, g.a0_glob - g.a0_off - p0 + 3));
  const int t2_lo = clampi(5 - p0 - g.a0_off), t2_hi = clampi(g.a0_glob - g.a0_off - p0 + 5);
  const int t_last = np + 4;

  // tensor coordinates of the box of plane p0-2 (allocation-relative: the
  // pads / halo row / halo plane precede the interior origin)
  const int c0 = (int)(kPadLast + x0 - 2), c1 = (int)(y0 - 1);
  int c2 = (int)(p0 - 1);
  const unsigned l0a = smaddr(l0), fulla = smaddr(full);
  unsigned slot_a = l0a, bar_a = fulla;  // slot / barrier of the next plane to request
  auto request = [&]() {
    if (tid == 0) {
      asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(bar_a), "r"(kPBytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(slot_a), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_a)
          : "memory");
    }
    ++c2;
    const bool wrap = slot_a == l0a + 2u * kPSlot * 8u;
    slot_a = wrap ? l0a : slot_a + kPSlot * 8u;
    bar_a = wrap ? fulla : bar_a + 8u;
  };
  const int tpos = (w * kRY) * kPW + 2 * lane;  // the thread's window origin in a plane
  int64_t ooff = origin + p0 * g.s0 + (y0 - 1 + w * kRY) * g.s1 + (x0 - 1 + 2 * lane);
  const double* cur = l0;
  unsigned cur_bar = fulla, parity = 0;
  int l1sel = 0;

  __syncthreads();  // barriers initialised
  request();
  for (int t = 0; t <= t_last; ++t) {
    // plane t+1 -> slot (t+1) % 3, last read in iteration t-2: every thread
    // passed iteration t-1's barrier after that
    if (t < t_last) request();
    __syncthreads();  // iteration t-1 finished everywhere (level-1 buffers)
    mbar_wait_a(cur_bar, parity);
    // level 1: plane p -> finishes level-1 plane q1 = p-1
    pair_level<MASK, FMA>(cur + tpos, A1, B1, out, cf.c);
    if (cur == l0 + 2 * kPSlot) {
      cur = l0;
      cur_bar = fulla;
      parity ^= 1u;
    } else {
      cur += kPSlot;
      cur_bar += 8u;
    }
    double* const l1b = l1 + l1sel;
    l1sel ^= kPSlot;
    {
      double* q = l1b + tpos + kPW + 1;
      const bool plane_in = t >= t1_lo && t < t1_hi;
      if (plane_in && all_dom) {
#pragma unroll
        for (int r = 0; r < kRY; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) q[r * kPW + h] = out[h][r];
      } else {
#pragma unroll
        for (int r = 0; r < kRY; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) q[r * kPW + h] = plane_in && (in_dom >> (h * kRY + r) & 1u) ? out[h][r] : bnd;
      }
    }
    if (t >= 3) {
      // level 2: level-1 plane q1-1 (previous iteration's buffer) -> level-2 plane q1-2
      pair_level<MASK, FMA>(l1 + l1sel + tpos, A2, B2, out, cf.c);
      if (t >= 5) {
        if (t < t2_lo || t >= t2_hi) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < kRY; ++r) out[h][r] = bnd;
        }
        auto store = [&](double* b) {
          double* op = b + ooff;
#pragma unroll
          for (int r = 0; r < kRY; ++r) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (store_ok >> (h * kRY + r) & 1u) op[h] = out[h][r];
            op += g.s1;
          }
        };
        if constexpr (MIR)
          for_each_dst(dst, mir, p0 - 5 + t, store);  // sharded: local plane + the neighbour's ghost plane
        else
          store(dst);
        ooff += g.s0;
      }
    }
  }
}

static unsigned slots3d(const tvs_stencil& st, Coeff27& cf) {
  unsigned mask = 0;
  int last = -1;
  for (int k = 0; k < 27; ++k) cf.c[k] = 0.0;
  for (int k = 0; k < st.ntaps; ++k) {
    const int pos = (st.offsets[k][0] + 1) * 9 + (st.offsets[k][1] + 1) * 3 + (st.offsets[k][2] + 1);
    if (pos <= last) return 0;
    last = pos;
    mask |= 1u << pos;
    cf.c[pos] = st.coeffs[k];
  }
  return mask;
}

bool jacobi3d_streaming_supported(const tvs_stencil& st) {
  Coeff27 cf;
  const unsigned m = slots3d(st, cf);
  return m == kBox27 || m == kStar7;
}

int jacobi3d_max_depth() { return 2; }
int jacobi3d_default_depth() { return 2; }

template <unsigned MASK, bool FMA>
static int launch_tb(const Geo& geo, const tvs_geometry& g, const double* src, double* dst, const Coeff27& cf,
                     double bnd, cudaStream_t s, int64_t plo, int64_t phi, int seg, const Mirror& mir) {
  // per device context; a host-side attribute write, no synchronisation
  const bool mirrored = mir.p[0] != nullptr || mir.p[1] != nullptr;
  auto kern = mirrored ? jacobi3d_tb_kernel<MASK, FMA, true> : jacobi3d_tb_kernel<MASK, FMA, false>;
  TVS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTBSmem));
  const dim3 block(kTX3, kTYT);
  const dim3 grid((unsigned)((geo.e2 + kTBOX - 1) / kTBOX), (unsigned)((geo.e1 + kTBOY - 1) / kTBOY),
                  (unsigned)((phi - plo + seg - 1) / seg));
  kern<<<grid, block, kTBSmem, s>>>(src, dst, geo, g.origin, cf, bnd, plo, phi, seg, mir);
  TVS_LAUNCHED("jacobi3d_tb_kernel");
  return TVS_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point lookup (the
// library does not link libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// K4c applies when the block can be described to the TMA unit: 16-byte
// aligned base and pitches, 32-bit extents.  TVS_J3D=cpasync keeps K4b.
static bool tma_usable(const tvs_geometry& g, const double* src) {
  static const bool off = [] {
    const char* e = std::getenv("TVS_J3D");
    return e && std::strcmp(e, "cpasync") == 0;
  }();
  if (off || !encode_tiled_fn()) return false;
  const int64_t s0 = g.strides[0], s1 = g.strides[1];
  return (reinterpret_cast<uintptr_t>(src) & 15u) == 0 && s1 % 2 == 0 && s0 % s1 == 0 && g.alloc_elems % s0 == 0 &&
         s1 < ((int64_t)1 << 31) && s0 / s1 < ((int64_t)1 << 31) && g.alloc_elems / s0 < ((int64_t)1 << 31);
}

template <unsigned MASK, bool FMA, int NW>
static int launch_tma(const Geo& geo, const tvs_geometry& g, const double* src, double* dst, const Coeff27& cf,
                      double bnd, cudaStream_t s, int64_t plo, int64_t phi, int seg, const Mirror& mir) {
  using T = TmaCfg<NW>;
  // the whole allocation as a (pitch, rows, planes) tensor; one box = the
  // 66 x 34 cells a block needs of one plane
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)g.strides[1], (cuuint64_t)(g.strides[0] / g.strides[1]),
                              (cuuint64_t)(g.alloc_elems / g.strides[0])};
  const cuuint64_t strides[2] = {(cuuint64_t)g.strides[1] * 8, (cuuint64_t)g.strides[0] * 8};
  const cuuint32_t box[3] = {(cuuint32_t)kPW, (cuuint32_t)T::R, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult rc = encode_tiled_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(src), dims, strides,
                                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return fail(TVS_ERR_CUDA, "jacobi3d: cuTensorMapEncodeTiled failed");
  const bool mirrored = mir.p[0] != nullptr || mir.p[1] != nullptr;
  auto kern = mirrored ? jacobi3d_tma_kernel<MASK, FMA, true, NW> : jacobi3d_tma_kernel<MASK, FMA, false, NW>;
  TVS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::Smem));
  const dim3 block(kTX3, NW);
  const dim3 grid((unsigned)((geo.e2 + kTBOX - 1) / kTBOX), (unsigned)((geo.e1 + T::OY - 1) / T::OY),
                  (unsigned)((phi - plo + seg - 1) / seg));
  kern<<<grid, block, T::Smem, s>>>(tm, dst, geo, g.origin, cf, bnd, plo, phi, seg, mir);
  TVS_LAUNCHED("jacobi3d_tma_kernel");
  return TVS_OK;
}

// Two time levels in one pass (K4c, or K4b when the block cannot be a tensor
// map): src -> dst after 2 steps.
int jacobi3d_blocked2(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, bool fma,
                      cudaStream_t s, int64_t plo, int64_t phi, int seg, const Mirror* mir) {
  const Mirror m = mir ? *mir : Mirror{};
  Coeff27 cf;
  const unsigned mask = slots3d(st, cf);
  const Geo geo = make_geo(g);
  if (phi < 0) phi = geo.e0;
  if (seg <= 0) seg = kTBPlanesSeg;
  if (plo < 0 || phi > geo.e0 || plo >= phi) return fail(TVS_ERR_INVALID, "jacobi3d_blocked2: plane range");
  // the kernel keeps its staging offsets within a plane in 32 bits
  if (geo.s0 >= ((int64_t)1 << 31) - 4 * geo.s1) return fail(TVS_ERR_UNSUPPORTED, "jacobi3d_blocked2: plane of 2^31 elements");
  if (tma_usable(g, src)) {
    // frame rows: 32 (two 8-warp CTAs per SM); TVS_J3D_FRAME=64 selects the
    // 64 x 64 frame (one 16-warp CTA per SM, 11% instead of 14% overlap), which
    // measured slower -- config 5: 238.6 / 366.9 against 258.8 / 389.3 GSt/s
    // (bit-exact / fma allow): one CTA per SM leaves nothing to run while its
    // 16 warps meet at the plane barrier
    static const int frame_env = [] {
      const char* e = std::getenv("TVS_J3D_FRAME");
      return e ? std::atoi(e) : 0;
    }();
    const bool tall = frame_env == 64;
    auto go = [&](auto mask_tag, auto fma_tag) -> int {
      constexpr unsigned M = decltype(mask_tag)::value;
      constexpr bool F = decltype(fma_tag)::value;
      return tall ? launch_tma<M, F, 16>(geo, g, src, dst, cf, st.boundary, s, plo, phi, seg, m)
                  : launch_tma<M, F, 8>(geo, g, src, dst, cf, st.boundary, s, plo, phi, seg, m);
    };
    using Box = std::integral_constant<unsigned, kBox27>;
    using Star = std::integral_constant<unsigned, kStar7>;
    if (mask == kBox27) return fma ? go(Box{}, std::true_type{}) : go(Box{}, std::false_type{});
    if (mask == kStar7) return fma ? go(Star{}, std::true_type{}) : go(Star{}, std::false_type{});
  }
  if (mask == kBox27)
    return fma ? launch_tb<kBox27, true>(geo, g, src, dst, cf, st.boundary, s, plo, phi, seg, m)
               : launch_tb<kBox27, false>(geo, g, src, dst, cf, st.boundary, s, plo, phi, seg, m);
  if (mask == kStar7)
    return fma ? launch_tb<kStar7, true>(geo, g, src, dst, cf, st.boundary, s, plo, phi, seg, m)
               : launch_tb<kStar7, false>(geo, g, src, dst, cf, st.boundary, s, plo, phi, seg, m);
  return fail(TVS_ERR_UNSUPPORTED, "jacobi3d_blocked2: tap set");
}

int jacobi3d_streaming(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, bool fma,
                       cudaStream_t s, int64_t plo, int64_t phi, int seg, const Mirror* mir) {
  const Mirror m = mir ? *mir : Mirror{};
  Coeff27 cf;
  const unsigned mask = slots3d(st, cf);
  if (mask != kBox27 && mask != kStar7) return fail(TVS_ERR_UNSUPPORTED, "jacobi3d_streaming: tap set");
  const Geo geo = make_geo(g);
  if (phi < 0) phi = geo.e0;
  if (seg <= 0) seg = kPlanesSeg;
  if (plo < 0 || phi > geo.e0 || plo >= phi) return fail(TVS_ERR_INVALID, "jacobi3d_streaming: plane range");
  const dim3 block(kTX3, kTYT);
  const dim3 grid((unsigned)((geo.e2 + kTX3 - 1) / kTX3), (unsigned)((geo.e1 + kTY3 - 1) / kTY3),
                  (unsigned)((phi - plo + seg - 1) / seg));
  if (mask == kBox27) {
    if (fma)
      jacobi3d_kernel<kBox27, true><<<grid, block, 0, s>>>(src, dst, geo, g.origin, cf, st.boundary, plo, phi, seg, m);
    else
      jacobi3d_kernel<kBox27, false><<<grid, block, 0, s>>>(src, dst, geo, g.origin, cf, st.boundary, plo, phi, seg, m);
  } else {
    if (fma)
      jacobi3d_kernel<kStar7, true><<<grid, block, 0, s>>>(src, dst, geo, g.origin, cf, st.boundary, plo, phi, seg, m);
    else
      jacobi3d_kernel<kStar7, false><<<grid, block, 0, s>>>(src, dst, geo, g.origin, cf, st.boundary, plo, phi, seg, m);
  }
  TVS_LAUNCHED("jacobi3d_kernel");
  return TVS_OK;
}

}  // namespace tvs
