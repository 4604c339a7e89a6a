// K2: 1D radius-1 Jacobi, temporally blocked in registers.
//
// Replaces heat1d_temporal / _run_1d (reference kernels1d.py:89-93,
// 106-220).  The reference packs consecutive *time* levels into one CPU
// vector to dodge unaligned loads; on a B200 the same goal — touch memory
// once per many time steps, and make the neighbour exchange a fixed, tiny
// number of register moves per step — is met by giving each lane P = 32
// contiguous points in registers and advancing them `depth` (<= 64) steps
// per launch.  Per step a lane exchanges exactly two values with its
// neighbours (__shfl_up/__shfl_down of its edge points); each warp owns a
// 32*P-point tile whose outer `depth` points on each side are the ghost
// trapezoid (their values decay into garbage one point per step and are
// never stored).  No block barriers; shared memory only as a per-warp
// staging tile that turns fully coalesced 16-byte loads / stores of the
// warp's 1024-point tile into the lanes' contiguous runs (a lane's run lies
// 256 bytes from the next lane's: per-lane 8-byte accesses cost 4 requests
// per sector and 30% of the run time).
//
// Per launch: reads 32*P doubles and writes 32*P - 2*depth per warp; the
// data (2^20 points = 8 MiB) stays L2-resident between launches, so the
// kernel is FP64-issue bound: 5 DP ops / update unfused, 3 with the exact
// power-of-two FMA form (heat1d: 0.25/0.5/0.25), 2 with the scaled taps.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace tvs {

#ifndef J1D_P
#define J1D_P 32
#endif
#ifndef J1D_DEPTH
#define J1D_DEPTH 64
#endif
constexpr int kP1 = J1D_P;          // points per lane
constexpr int kMaxDepth1 = 2 * J1D_DEPTH;  // deepest block a launch accepts
constexpr int kWarps1 = 8;          // warps per block
// per-warp staging tile for coalesced loads / stores: a lane's run of kP1
// points starts (kP1 + 2) cells after the previous lane's (the 2-cell pad
// spreads the lanes' 16-byte accesses over all banks)
constexpr int kTile1 = 32 * (kP1 + 2);
constexpr size_t kSmem1 = (size_t)kWarps1 * kTile1 * sizeof(double);

// SC (scaled power-of-two taps, as K3's): w holds w_k / w_first, all powers of
// two, and the values of level s are carried divided by w_first^s: the first
// tap is the input itself and every other tap one DFMA whose product is exact
// -- bit for bit the reference's separately rounded w*v then +acc, because
// scaling by a power of two commutes with rounding (barring under/overflow).
// heat1d: 2 FP64 instructions per update instead of 3.
template <unsigned MASK, bool FMA, bool SC>
__device__ __forceinline__ double upd1(double l, double c, double r, const double w[3]) {
  double acc = 0.0;
  bool first = true;
  if constexpr (MASK & 1u) { acc = SC ? l : tap_first(w[0], l); first = false; }
  if constexpr (MASK & 2u) { acc = first ? (SC ? c : tap_first(w[1], c)) : tap_next<FMA || SC>(w[1], c, acc); first = false; }
  if constexpr (MASK & 4u) { acc = first ? (SC ? r : tap_first(w[2], r)) : tap_next<FMA || SC>(w[2], r, acc); }
  return acc;
}

template <unsigned MASK, bool FMA, bool SC>
__global__ void __launch_bounds__(kWarps1 * 32) jacobi1d_kernel(const double* __restrict__ src,
                                                                double* __restrict__ dst, int64_t n, int depth,
                                                                double w0, double w1, double w2, double bnd,
                                                                int64_t rlo, int64_t rhi, double inv_first,
                                                                double out_scale) {
  const double w[3] = {w0, w1, w2};
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * kWarps1 + (threadIdx.x >> 5);
  const int64_t useful = 32 * kP1 - 2 * depth;
  const int64_t x0 = rlo - depth + warp * useful;  // first point of the warp tile (outputs [rlo, rhi))
  if (x0 + depth >= rhi) return;                  // whole warp beyond the range
  const int64_t xl = x0 + lane * kP1;         // this lane's first point

  double v[kP1];
  unsigned out_mask = 0;  // bit m: point xl+m outside [0, n) -> pinned to bnd
  // a lane's points are contiguous (lanes 256 bytes apart): 16-byte loads /
  // stores halve the requests when the lane's run is aligned and inside
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(src + xl) | reinterpret_cast<uintptr_t>(dst + xl)) & 15u) == 0;
  // whole warp tile inside the domain: fully coalesced 16-byte loads (lane t
  // takes pairs t, t + 32, ...), transposed into the lanes' runs through the
  // staging tile (config 1: 2475 GSt/s with per-lane 8-byte loads, 2935 with
  // per-lane 16-byte loads)
  extern __shared__ __align__(16) double stage1[];
  double* const ws = stage1 + (threadIdx.x >> 5) * kTile1;
  const bool tile_ok = (reinterpret_cast<uintptr_t>(src + x0) & 15u) == 0 && (reinterpret_cast<uintptr_t>(dst + x0) & 15u) == 0;
  if (tile_ok && x0 >= 0 && x0 + 32 * kP1 <= n) {
    const double2* s2 = reinterpret_cast<const double2*>(src + x0);
#pragma unroll
    for (int k = 0; k < kP1 / 2; ++k) {
      const int i = 2 * (lane + 32 * k);  // first point of the pair within the tile
      *reinterpret_cast<double2*>(ws + i + 2 * (i / kP1)) = __ldg(s2 + lane + 32 * k);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < kP1; m += 2) {
      const double2 t = *reinterpret_cast<const double2*>(ws + (kP1 + 2) * lane + m);
      v[m] = t.x;
      v[m + 1] = t.y;
    }
    __syncwarp();
  } else if (vec_ok && xl >= 0 && xl + kP1 <= n) {
    const double2* s2 = reinterpret_cast<const double2*>(src + xl);
#pragma unroll
    for (int m = 0; m < kP1; m += 2) {
      const double2 t = __ldg(s2 + m / 2);
      v[m] = t.x;
      v[m + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int m = 0; m < kP1; ++m) {
      const int64_t x = xl + m;
      const bool in = x >= 0 && x < n;
      v[m] = in ? src[x] : bnd;
      out_mask |= (in ? 0u : 1u) << m;
    }
  }
  const bool any_out = __any_sync(0xffffffffu, out_mask != 0);

  double pin = bnd;  // the boundary at the current level's scale
  for (int s = 0; s < depth; ++s) {
    const double left = __shfl_up_sync(0xffffffffu, v[kP1 - 1], 1);
    const double right = __shfl_down_sync(0xffffffffu, v[0], 1);
    double prev = left;
#pragma unroll
    for (int m = 0; m < kP1; ++m) {
      const double cur = v[m];
      const double nxt = m + 1 < kP1 ? v[m + 1] : right;
      v[m] = upd1<MASK, FMA, SC>(prev, cur, nxt, w);
      prev = cur;
    }
    if constexpr (SC) pin = __dmul_rn(pin, inv_first);  // exact: a power of two
    if (any_out) {
#pragma unroll
      for (int m = 0; m < kP1; ++m)
        if (out_mask >> m & 1u) v[m] = pin;
    }
  }

  const int64_t lo = x0 + depth, hi = x0 + depth + useful;  // valid outputs
  const int64_t slo = lo > rlo ? lo : rlo, shi = hi < rhi ? hi : rhi;
  if (tile_ok && (depth & 1) == 0 && lo >= rlo && hi <= rhi) {
    // the warp's useful points [depth, depth + useful) of the tile, coalesced
#pragma unroll
    for (int m = 0; m < kP1; m += 2)
      *reinterpret_cast<double2*>(ws + (kP1 + 2) * lane + m) =
          SC ? make_double2(__dmul_rn(v[m], out_scale), __dmul_rn(v[m + 1], out_scale)) : make_double2(v[m], v[m + 1]);
    __syncwarp();
    double2* d2 = reinterpret_cast<double2*>(dst + x0);
#pragma unroll
    for (int k = 0; k < kP1 / 2; ++k) {
      const int i = 2 * (lane + 32 * k);
      if (i >= depth && i < 32 * kP1 - depth) d2[lane + 32 * k] = *reinterpret_cast<const double2*>(ws + i + 2 * (i / kP1));
    }
  } else if (vec_ok && xl >= slo && xl + kP1 <= shi) {
    double2* d2 = reinterpret_cast<double2*>(dst + xl);
#pragma unroll
    for (int m = 0; m < kP1; m += 2)
      d2[m / 2] = SC ? make_double2(__dmul_rn(v[m], out_scale), __dmul_rn(v[m + 1], out_scale)) : make_double2(v[m], v[m + 1]);
  } else {
#pragma unroll
    for (int m = 0; m < kP1; ++m) {
      const int64_t x = xl + m;
      if (x >= slo && x < shi) dst[x] = SC ? __dmul_rn(v[m], out_scale) : v[m];
    }
  }
}

// Tap slots of a 1D radius-1 stencil whose offsets are strictly sorted;
// -1 if the kernel's fixed (-1, 0, +1) order would not reproduce it.
static int slots1d(const tvs_stencil& st, double w[3]) {
  unsigned mask = 0;
  int last = -2;
  w[0] = w[1] = w[2] = 0.0;
  for (int k = 0; k < st.ntaps; ++k) {
    const int o = st.offsets[k][0];
    if (o <= last) return -1;
    last = o;
    mask |= 1u << (o + 1);
    w[o + 1] = st.coeffs[k];
  }
  return (int)mask;
}

// mode 0: unfused taps, 1: fused (FMA), 2: scaled power-of-two taps (SC)
template <unsigned MASK>
static void launch1d(int mode, unsigned blocks, cudaStream_t s, const double* src, double* dst, int64_t n, int depth,
                     const double w[3], double bnd, int64_t rlo, int64_t rhi, double inv_first, double out_scale) {
  // per device context; a host-side attribute write, no synchronisation
  auto go = [&](auto kern, double inv, double osc) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem1);
    kern<<<blocks, kWarps1 * 32, kSmem1, s>>>(src, dst, n, depth, w[0], w[1], w[2], bnd, rlo, rhi, inv, osc);
  };
  if (mode == 2)
    go(jacobi1d_kernel<MASK, true, true>, inv_first, out_scale);
  else if (mode == 1)
    go(jacobi1d_kernel<MASK, true, false>, 1.0, 1.0);
  else
    go(jacobi1d_kernel<MASK, false, false>, 1.0, 1.0);
}

int jacobi1d_default_depth() { return J1D_DEPTH; }
int jacobi1d_max_depth() { return std::min(kMaxDepth1, 16 * kP1 - 1); }

bool jacobi1d_blocked_supported(const tvs_stencil& st, const tvs_geometry& g) {
  double w[3];
  return slots1d(st, w) > 0 && g.axis0_offset == 0 && g.axis0_global == g.extents[0];
}

int jacobi1d_blocked(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, int depth,
                     bool fma, cudaStream_t s, int64_t rlo, int64_t rhi) {
  double w[3];
  const int mask = slots1d(st, w);
  if (mask <= 0 || depth < 1 || depth > kMaxDepth1 || 2 * depth >= 32 * kP1)
    return fail(TVS_ERR_UNSUPPORTED, "jacobi1d_blocked: unsorted taps or depth out of range");
  const int64_t n = g.extents[0];
  if (rhi < 0) rhi = n;
  if (rlo < 0 || rhi > n || rlo >= rhi) return fail(TVS_ERR_INVALID, "jacobi1d_blocked: range");
  const int64_t useful = 32 * kP1 - 2 * depth;
  const int64_t warps = (rhi - rlo + useful - 1) / useful;
  const unsigned blocks = (unsigned)((warps + kWarps1 - 1) / kWarps1);
  const double* s0 = src + g.origin;
  double* d0 = dst + g.origin;
  // Scaled taps when every coefficient is a power of two (the fused form is
  // already exact then).  The carried values grow by 1 / |w_first| per step
  // (heat1d: 4^depth, 2^128 at depth 64), so |values| must stay below
  // 2^(1023 - depth log2(1 / |w_first|)) -- the caveat of K3's scaled taps;
  // TVS_J1D_SCALED=0 disables it.
  static const bool sc_off = [] {
    const char* e = getenv("TVS_J1D_SCALED");
    return e && atoi(e) == 0;
  }();
  int mode = fma ? 1 : 0;
  double inv_first = 1.0, out_scale = 1.0;
  if (fma && !sc_off && coeffs_power_of_two(st)) {
    const double wf = w[__builtin_ctz((unsigned)mask)];
    int ex0;
    std::frexp(wf, &ex0);
    bool ok = std::abs(ex0 - 1) * depth <= 300;
    for (int k = 0; k < 3 && ok; ++k) {
      if (w[k] == 0.0) continue;
      int ex;
      std::frexp(w[k], &ex);
      ok = std::abs(ex - ex0) <= 60;
    }
    if (ok) {
      mode = 2;
      inv_first = 1.0 / wf;
      for (int k = 0; k < 3; ++k) w[k] /= wf;                   // exact: powers of two
      for (int l = 0; l < depth; ++l) out_scale *= wf;          // exact
    }
  }
  switch (mask) {
    case 1: launch1d<1>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
    case 2: launch1d<2>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
    case 3: launch1d<3>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
    case 4: launch1d<4>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
    case 5: launch1d<5>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
    case 6: launch1d<6>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
    default: launch1d<7>(mode, blocks, s, s0, d0, n, depth, w, st.boundary, rlo, rhi, inv_first, out_scale); break;
  }
  TVS_LAUNCHED("jacobi1d_kernel");
  return TVS_OK;
}

}  // namespace tvs
