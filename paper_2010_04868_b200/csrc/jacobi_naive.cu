// K1: generic one-step Jacobi update, any radius-1 tap set in 1D/2D/3D.
//
// Replaces jacobi_plane_update (reference baselines.py:43-49): one thread
// per output point, taps read straight from global memory in the caller's
// (sorted) order, unfused unless the FMA policy allows.  It is the fallback
// for tap sets the specialised kernels do not instantiate, the `algo=naive`
// path, and the single-step HBM roofline baseline (16 B / update).
#include "common.cuh"

namespace tvs {

template <int NT, bool FMA>
__device__ __forceinline__ double naive_point(const double* __restrict__ src, int64_t idx, const TapList& tl) {
  double acc = tap_first(tl.c[0], __ldg(src + idx + tl.lin[0]));
#pragma unroll
  for (int k = 1; k < (NT > 0 ? NT : TVS_MAX_TAPS); ++k) {
    if (NT == 0 && k >= tl.n) break;
    acc = tap_next<FMA>(tl.c[k], __ldg(src + idx + tl.lin[k]), acc);
  }
  return acc;
}

// Block (32, 8): x runs along the contiguous axis, y along the next one,
// blockIdx.z (3D) along axis 0; grid-stride loops cover any extent.  Cells
// beyond a block edge read the memory halo (boundary value, tvs_fill_halo);
// axis-0 positions outside the global domain are pinned to the boundary.
template <int NT, bool FMA>
__global__ void __launch_bounds__(256) jacobi_naive_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                           Geo g, TapList tl, int64_t origin) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (g.dim == 1) {
    for (int64_t i = (blockIdx.x * 8 + ty) * 32ll + tx; i < g.e0; i += (int64_t)gridDim.x * 256) {
      const int64_t gi = i + g.a0_off;
      dst[origin + i] = (gi < 0 || gi >= g.a0_glob) ? tl.bnd : naive_point<NT, FMA>(src, origin + i, tl);
    }
  } else if (g.dim == 2) {
    for (int64_t r = blockIdx.y * 8ll + ty; r < g.e0; r += gridDim.y * 8ll) {
      const int64_t gr = r + g.a0_off;
      const bool pinned = gr < 0 || gr >= g.a0_glob;
      for (int64_t c = blockIdx.x * 32ll + tx; c < g.e1; c += gridDim.x * 32ll) {
        const int64_t idx = origin + r * g.s0 + c;
        dst[idx] = pinned ? tl.bnd : naive_point<NT, FMA>(src, idx, tl);
      }
    }
  } else {
    for (int64_t p = blockIdx.z; p < g.e0; p += gridDim.z) {
      const int64_t gp = p + g.a0_off;
      const bool pinned = gp < 0 || gp >= g.a0_glob;
      for (int64_t r = blockIdx.y * 8ll + ty; r < g.e1; r += gridDim.y * 8ll) {
        for (int64_t c = blockIdx.x * 32ll + tx; c < g.e2; c += gridDim.x * 32ll) {
          const int64_t idx = origin + p * g.s0 + r * g.s1 + c;
          dst[idx] = pinned ? tl.bnd : naive_point<NT, FMA>(src, idx, tl);
        }
      }
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
  dim3 grid;
  if (geo.dim == 1) {
    grid = dim3((unsigned)std::min<int64_t>(cdiv(geo.e0, 256), 148 * 64));
  } else if (geo.dim == 2) {
    grid = dim3((unsigned)std::min<int64_t>(cdiv(geo.e1, 32), 1 << 16), (unsigned)std::min<int64_t>(cdiv(geo.e0, 8), 65535));
  } else {
    grid = dim3((unsigned)std::min<int64_t>(cdiv(geo.e2, 32), 1 << 16), (unsigned)std::min<int64_t>(cdiv(geo.e1, 8), 65535),
                (unsigned)std::min<int64_t>(geo.e0, 65535));
  }
  switch (st.ntaps) {
    case 3: launch_nt<3>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 5: launch_nt<5>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 7: launch_nt<7>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 9: launch_nt<9>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    case 27: launch_nt<27>(src, dst, geo, tl, g.origin, fma, grid, s); break;
    default: launch_nt<0>(src, dst, geo, tl, g.origin, fma, grid, s); break;
  }
  TVS_LAUNCHED("jacobi_naive_kernel");
  return TVS_OK;
}

}  // namespace tvs
