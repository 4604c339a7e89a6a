// K1: generic one-step Jacobi update, any radius-1 tap set in 1D/2D/3D.
//
// Replaces jacobi_plane_update (reference baselines.py:43-49): every output
// is the caller's (sorted) tap chain over the previous time level, unfused
// unless the FMA policy allows.  It is the fallback for tap sets the
// specialised kernels do not instantiate, the `algo=naive` path, and the
// single-step ("untiled") HBM-roofline kernel: 8 B read + 8 B written per
// update, so it must run at HBM speed.
//
// Bandwidth design: a thread owns R outputs along the slowest in-block axis
// (rows in 2D, axis-1 rows in 3D, 256-element strides in 1D) and issues all
// R x NT tap loads before the first arithmetic, so every warp keeps R full
// 256-byte rows in flight; lanes run along the contiguous axis (coalesced
// 256 B per warp access), neighbour taps hit L1 (same warp) or L2 (adjacent
// blocks, which the launch order keeps resident).  Stores are 256 B per warp
// row.  Cells beyond a block edge read the memory halo (boundary value,
// tvs_fill_halo); axis-0 positions outside the global domain are pinned to
// the boundary.
#include <algorithm>

#include "common.cuh"

namespace tvs {

constexpr int kNR = 8;  // outputs per thread

// R outputs at idx + r*rstride; NT > 0: unrolled tap loop (all loads first)
template <int NT, bool FMA>
__device__ __forceinline__ void naive_points(const double* __restrict__ src, int64_t idx, int64_t rstride,
                                             const TapList& tl, double (&acc)[kNR]) {
  if constexpr (NT > 0) {
    double v[NT][kNR];
#pragma unroll
    for (int k = 0; k < NT; ++k)
#pragma unroll
      for (int r = 0; r < kNR; ++r) v[k][r] = __ldg(src + idx + r * rstride + tl.lin[k]);
#pragma unroll
    for (int r = 0; r < kNR; ++r) {
      acc[r] = tap_first(tl.c[0], v[0][r]);
#pragma unroll
      for (int k = 1; k < NT; ++k) acc[r] = tap_next<FMA>(tl.c[k], v[k][r], acc[r]);
    }
  } else {
#pragma unroll
    for (int r = 0; r < kNR; ++r) acc[r] = tap_first(tl.c[0], __ldg(src + idx + r * rstride + tl.lin[0]));
    for (int k = 1; k < tl.n; ++k) {
      double v[kNR];
#pragma unroll
      for (int r = 0; r < kNR; ++r) v[r] = __ldg(src + idx + r * rstride + tl.lin[k]);
#pragma unroll
      for (int r = 0; r < kNR; ++r) acc[r] = tap_next<FMA>(tl.c[k], v[r], acc[r]);
    }
  }
}

// same, bounds-checked tail (r < nr)
template <bool FMA>
__device__ __forceinline__ double naive_point(const double* __restrict__ src, int64_t idx, const TapList& tl) {
  double acc = tap_first(tl.c[0], __ldg(src + idx + tl.lin[0]));
  for (int k = 1; k < tl.n; ++k) acc = tap_next<FMA>(tl.c[k], __ldg(src + idx + tl.lin[k]), acc);
  return acc;
}

// Block (32, 8).  1D: tile = 8 warps x kNR x 32 consecutive elements
// (element = tile0 + (r*8 + ty)*32 + tx).  2D: tile = 32 columns x (8 kNR)
// rows, thread rows ty*kNR + r.  3D: tile = 32 x (8 kNR) on axes 2 x 1 of
// plane blockIdx.z.  Full tiles take the unrolled path; edge tiles the
// checked one.
template <int NT, bool FMA>
__global__ void __launch_bounds__(256) jacobi_naive_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                           Geo g, TapList tl, int64_t origin) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  double acc[kNR];
  if (g.dim == 1) {
    const int64_t i0 = (int64_t)blockIdx.x * (256 * kNR) + ty * 32 + tx;  // + r*256
    const int64_t last = i0 + (kNR - 1) * 256;
    if (last < g.e0 && g.a0_off == 0 && g.a0_glob == g.e0) {
      naive_points<NT, FMA>(src, origin + i0, 256, tl, acc);
#pragma unroll
      for (int r = 0; r < kNR; ++r) dst[origin + i0 + r * 256] = acc[r];
    } else {
      for (int r = 0; r < kNR; ++r) {
        const int64_t i = i0 + r * 256;
        if (i >= g.e0) break;
        const int64_t gi = i + g.a0_off;
        dst[origin + i] = (gi < 0 || gi >= g.a0_glob) ? tl.bnd : naive_point<FMA>(src, origin + i, tl);
      }
    }
    return;
  }
  // 2D: rows along axis 0 (stride s0), 3D: rows along axis 1 (stride s1) of plane p
  const bool d3 = g.dim == 3;
  const int64_t rows = d3 ? g.e1 : g.e0;
  const int64_t cols = d3 ? g.e2 : g.e1;
  const int64_t rs = d3 ? g.s1 : g.s0;
  const int64_t c = (int64_t)blockIdx.x * 32 + tx;
  const int64_t r0 = (int64_t)blockIdx.y * (8 * kNR) + ty * kNR;
  const int64_t p = d3 ? (int64_t)blockIdx.z : 0;
  const int64_t base = origin + (d3 ? p * g.s0 : 0) + c;
  if (c >= cols) return;
  // axis-0 pinning: 3D by plane, 2D by row
  if (d3) {
    const int64_t gp = p + g.a0_off;
    if (gp < 0 || gp >= g.a0_glob) {
      for (int r = 0; r < kNR && r0 + r < rows; ++r) dst[base + (r0 + r) * rs] = tl.bnd;
      return;
    }
  }
  const bool rows_ok = d3 || (r0 + g.a0_off >= 0 && r0 + kNR - 1 + g.a0_off < g.a0_glob);
  if (r0 + kNR <= rows && rows_ok) {
    naive_points<NT, FMA>(src, base + r0 * rs, rs, tl, acc);
#pragma unroll
    for (int r = 0; r < kNR; ++r) dst[base + (r0 + r) * rs] = acc[r];
  } else {
    for (int r = 0; r < kNR && r0 + r < rows; ++r) {
      const int64_t idx = base + (r0 + r) * rs;
      const int64_t gr = r0 + r + g.a0_off;
      dst[idx] = (!d3 && (gr < 0 || gr >= g.a0_glob)) ? tl.bnd : naive_point<FMA>(src, idx, tl);
    }
  }
}

static TapList make_taps(const tvs_stencil& st, const tvs_geometry& g, bool fma) {
  TapList tl{};
  tl.n = st.ntaps;
  tl.fma = fma;
  tl.bnd = st.boundary;
  const int64_t s0 = g.strides[0];
  const int64_t s1 = g.dim == 3 ? g.strides[1] : 1;
  for (int k = 0; k < st.ntaps; ++k) {
    const int* o = st.offsets[k];
    tl.c[k] = st.coeffs[k];
    for (int d = 0; d < 3; ++d) tl.off[k][d] = (int8_t)o[d];
    if (g.dim == 1)
      tl.lin[k] = o[0];
    else if (g.dim == 2)
      tl.lin[k] = o[0] * s0 + o[1];
    else
      tl.lin[k] = o[0] * s0 + o[1] * s1 + o[2];
  }
  return tl;
}

template <int NT>
static void launch_nt(const double* src, double* dst, const Geo& geo, const TapList& tl, int64_t origin, bool fma,
                      dim3 grid, cudaStream_t s) {
  const dim3 block(32, 8);
  if (fma)
    jacobi_naive_kernel<NT, true><<<grid, block, 0, s>>>(src, dst, geo, tl, origin);
  else
    jacobi_naive_kernel<NT, false><<<grid, block, 0, s>>>(src, dst, geo, tl, origin);
}

int jacobi_naive_step(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, bool fma,
                      cudaStream_t s) {
  const Geo geo = make_geo(g);
  const TapList tl = make_taps(st, g, fma);
  auto cdiv = [](int64_t a, int64_t b) { return (a + b - 1) / b; };
  int64_t gx, gy = 1, gz = 1;
  if (geo.dim == 1) {
    gx = cdiv(geo.e0, 256 * kNR);
  } else if (geo.dim == 2) {
    gx = cdiv(geo.e1, 32);
    gy = cdiv(geo.e0, 8 * kNR);
  } else {
    gx = cdiv(geo.e2, 32);
    gy = cdiv(geo.e1, 8 * kNR);
    gz = geo.e0;
  }
  if (gx >= (1ll << 31) || gy > 65535 || gz > 65535) return fail(TVS_ERR_SIZE, "jacobi_naive_step: grid too large");
  const dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)gz);
  switch (st.ntaps) {
    case 3: launch_nt<3>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 5: launch_nt<5>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 7: launch_nt<7>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 9: launch_nt<9>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    default: launch_nt<0>(src, dst, geo, tl, g.origin, fma, grid, s); break;
  }
  TVS_LAUNCHED("jacobi_naive_kernel");
  return TVS_OK;
}

}  // namespace tvs
