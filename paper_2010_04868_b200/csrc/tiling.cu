// K9: wave executor for iteration-space tile schedules (reference
// tiling.py:347-406: execute_parallel / lcs_blocked).
//
// The reference runs the tiles of a wave on a CPU thread pool over a full
// time history (one padded plane per time level, tiling.py:331-344).  Here
// the history lives in HBM and each wave is ONE launch, one CTA per tile:
//   * Jacobi / Life: each time level of the tile's (moving, clipped) window
//     is a flat parallel loop reading plane t and writing plane t+1, with a
//     CTA barrier between levels;
//   * Gauss-Seidel (lexicographic in-place semantics: lexicographically
//     negative taps read the current sweep = plane t+1, the others plane t):
//     the window is swept by hyperplanes h = 2x0 + x1 (2D) / 4x0 + 2x1 + x2
//     (3D) / x0 (1D), on which no point reads another, barrier in between;
//   * LCS: rectangles of the (A index, B index) table by anti-diagonals.
// Every read outside the tile was produced by an earlier wave (the schedule's
// wave-order invariant, tiling.check_wave_order); reads outside the domain
// hit the planes' halo, filled with the boundary value.  Same arithmetic as
// the other kernels (tap_first / tap_next), so results are bit-identical to
// the unblocked path.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace tvs {

struct TileDev {
  int t0, t1;
  int lo[3], hi[3], slo[3], shi[3];
};
static_assert(sizeof(TileDev) == sizeof(tvs_tile), "tile layout");

struct TileGeo {
  int dim;
  int64_t ext[3];
  int64_t str[3];  // element strides (last = 1)
  int64_t origin;
  int64_t plane;   // elements per history plane
};

__device__ __forceinline__ bool tile_window(const TileDev& tl, int t, const TileGeo& g, int64_t (&a)[3],
                                            int64_t (&b)[3]) {
  const int dt = t - tl.t0;
  bool ok = true;
  for (int d = 0; d < 3; ++d) {
    if (d < g.dim) {
      a[d] = max((int64_t)tl.lo[d] + (int64_t)tl.slo[d] * dt, (int64_t)0);
      b[d] = min((int64_t)tl.hi[d] + (int64_t)tl.shi[d] * dt, g.ext[d]);
      ok = ok && b[d] > a[d];
    } else {
      a[d] = 0;
      b[d] = 1;
    }
  }
  return ok;
}

struct FpTaps {
  int n;
  int fma;
  int64_t lin[TVS_MAX_TAPS];
  double c[TVS_MAX_TAPS];
  unsigned newmask;  // bit k: tap k reads the current sweep (Gauss-Seidel)
};

__device__ __forceinline__ double fp_point(const double* cur, const double* nxt, int64_t idx, const FpTaps& t) {
  double acc = tap_first(t.c[0], (t.newmask & 1u) ? nxt[idx + t.lin[0]] : cur[idx + t.lin[0]]);
  for (int k = 1; k < t.n; ++k) {
    const double v = ((t.newmask >> k) & 1u) ? nxt[idx + t.lin[k]] : cur[idx + t.lin[k]];
    acc = t.fma ? tap_next<true>(t.c[k], v, acc) : tap_next<false>(t.c[k], v, acc);
  }
  return acc;
}

struct LifeT {
  int n, bmask, smask;
  int64_t lin[26];
};

__device__ __forceinline__ int64_t lin_index(const TileGeo& g, int64_t x0, int64_t x1, int64_t x2) {
  return g.origin + x0 * g.str[0] + (g.dim > 1 ? x1 * g.str[1] : 0) + (g.dim > 2 ? x2 * g.str[2] : 0);
}

// one CTA per tile of the wave; KIND 0 Jacobi fp64, 1 Gauss-Seidel fp64, 2 Life int32
template <int KIND>
__global__ void __maxnreg__(128) tile_wave_kernel(void* hist, TileGeo g, const TileDev* __restrict__ tiles,
                                                        FpTaps ft, LifeT lt) {
  const TileDev tl = tiles[blockIdx.x];
  for (int t = tl.t0; t < tl.t1; ++t) {
    int64_t a[3], b[3];
    if (!tile_window(tl, t, g, a, b)) continue;  // uniform over the CTA
    const int64_t n1 = b[1] - a[1], n2 = b[2] - a[2];
    if constexpr (KIND == 1) {
      const double* cur = static_cast<const double*>(hist) + (int64_t)t * g.plane;
      double* nxt = static_cast<double*>(hist) + (int64_t)(t + 1) * g.plane;
      const int64_t n0 = b[0] - a[0];
      // h = w . (x - a), w = (1) | (2, 1) | (4, 2, 1)
      const int64_t w0 = g.dim == 1 ? 1 : (g.dim == 2 ? 2 : 4), w1 = g.dim == 3 ? 2 : 1;
      const int64_t hmax = w0 * (n0 - 1) + (g.dim > 1 ? w1 * (n1 - 1) : 0) + (g.dim > 2 ? n2 - 1 : 0);
      for (int64_t h = 0; h <= hmax; ++h) {
        // enumerate (x0, x1) with the last coordinate solved from h
        const int64_t pairs = g.dim == 3 ? n0 * n1 : (g.dim == 2 ? n0 : 1);
        for (int64_t q = threadIdx.x; q < pairs; q += blockDim.x) {
          int64_t x0, x1 = 0, x2 = 0;
          bool ok;
          if (g.dim == 1) {
            x0 = h;
            ok = x0 < n0;
          } else if (g.dim == 2) {
            x0 = q;
            x1 = h - 2 * x0;
            ok = x1 >= 0 && x1 < n1;
          } else {
            x0 = q / n1;
            x1 = q % n1;
            x2 = h - 4 * x0 - 2 * x1;
            ok = x2 >= 0 && x2 < n2;
          }
          if (ok) {
            const int64_t idx = lin_index(g, a[0] + x0, a[1] + x1, a[2] + x2);
            nxt[idx] = fp_point(cur, nxt, idx, ft);
          }
        }
        __syncthreads();
      }
    } else {
      const int64_t vol = (b[0] - a[0]) * n1 * n2;
      for (int64_t q = threadIdx.x; q < vol; q += blockDim.x) {
        const int64_t x2 = q % n2, r = q / n2, x1 = r % n1, x0 = r / n1;
        const int64_t idx = lin_index(g, a[0] + x0, a[1] + x1, a[2] + x2);
        if constexpr (KIND == 0) {
          const double* cur = static_cast<const double*>(hist) + (int64_t)t * g.plane;
          double* nxt = static_cast<double*>(hist) + (int64_t)(t + 1) * g.plane;
          nxt[idx] = fp_point(cur, cur, idx, ft);
        } else {
          const int* cur = static_cast<const int*>(hist) + (int64_t)t * g.plane;
          int* nxt = static_cast<int*>(hist) + (int64_t)(t + 1) * g.plane;
          unsigned s = 0u;
          for (int k = 0; k < lt.n; ++k) s += (unsigned)cur[idx + lt.lin[k]];
          const int alive = cur[idx];
          nxt[idx] = (s <= 26u && ((lt.bmask >> s) & 1)) ? 1 : ((s <= 26u && ((lt.smask >> s) & 1)) ? alive : 0);
        }
      }
    }
    __syncthreads();
  }
}

__global__ void fill_planes_kernel(void* base, int64_t n, int elem, double vd, int vi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (elem == 8)
      static_cast<double*>(base)[i] = vd;
    else
      static_cast<int*>(base)[i] = vi;
  }
}

// LCS table (na+1) x (nb+1), row-major, row/column 0 zero; tile rows
// x in [t0+1, min(t1, na)+1), columns y in [lo+1, min(hi, nb)+1)
__global__ void __launch_bounds__(256) lcs_tile_kernel(int* __restrict__ table, const int* __restrict__ a,
                                                       const int* __restrict__ b, int na, int nb,
                                                       const TileDev* __restrict__ tiles) {
  const TileDev tl = tiles[blockIdx.x];
  const int x0 = tl.t0 + 1, x1 = min(tl.t1, na) + 1, y0 = tl.lo[0] + 1, y1 = min(tl.hi[0], nb) + 1;
  if (x1 <= x0 || y1 <= y0) return;
  const int64_t pitch = (int64_t)nb + 1;
  for (int d = x0 + y0; d <= x1 + y1 - 2; ++d) {
    const int i0 = max(x0, d - (y1 - 1)), i1 = min(x1 - 1, d - y0);
    for (int i = i0 + threadIdx.x; i <= i1; i += blockDim.x) {
      const int j = d - i;
      int* cell = table + i * pitch + j;
      *cell = a[i - 1] == b[j - 1] ? cell[-pitch - 1] + 1 : max(cell[-pitch], cell[-1]);
    }
    __syncthreads();
  }
}

static int check_waves(const tvs_tile* tiles, const int64_t* wave_start, int64_t nwaves) {
  if (nwaves < 0 || (nwaves > 0 && (!tiles || !wave_start))) return fail(TVS_ERR_INVALID, "bad tile schedule");
  if (nwaves > 0 && wave_start[0] != 0) return fail(TVS_ERR_INVALID, "wave_start[0] must be 0");
  for (int64_t w = 0; w < nwaves; ++w)
    if (wave_start[w + 1] < wave_start[w] || wave_start[w + 1] - wave_start[w] > 0x7fffffff)
      return fail(TVS_ERR_INVALID, "wave_start must be non-decreasing");
  return TVS_OK;
}

// shared driver: history in HBM, waves as launches, plane `steps` downloaded
static int tiled_driver(int kind, const tvs_geometry& g, const tvs_layout& lay, const void* in, void* out,
                        int64_t steps, const tvs_tile* tiles, const int64_t* wave_start, int64_t nwaves,
                        const FpTaps& ft, const LifeT& lt, double bndd, int bndi, int device) {
  const int elem = kind == 2 ? 4 : 8;
  const int64_t plane = g.alloc_elems;
  const int64_t ntiles = nwaves > 0 ? wave_start[nwaves] : 0;
  cudaStream_t s;
  TVS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  void* hist = nullptr;
  TileDev* dt = nullptr;
  auto done = [&](int code) {
    if (hist) cudaFreeAsync(hist, s);
    if (dt) cudaFreeAsync(dt, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return code;
  };
  (void)device;
  if (cudaMallocAsync(&hist, (size_t)elem * plane * (steps + 1), s) != cudaSuccess)
    return done(fail(TVS_ERR_SIZE, "tiled run: time history does not fit in device memory"));
  if (ntiles > 0 && cudaMallocAsync((void**)&dt, sizeof(TileDev) * ntiles, s) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "cudaMallocAsync"));
  fill_planes_kernel<<<148 * 8, 256, 0, s>>>(hist, plane * (steps + 1), elem, bndd, bndi);
  if (cudaGetLastError() != cudaSuccess) return done(cuda_fail(cudaGetLastError(), "fill_planes_kernel"));
  count_launch();
  if (ntiles > 0 && cudaMemcpyAsync(dt, tiles, sizeof(TileDev) * ntiles, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "tile upload"));
  // plane 0 <- the input interior (host Grid layout, re-pitched)
  {
    cudaMemcpy3DParms p;
    std::memset(&p, 0, sizeof(p));
    const int64_t rows = g.dim == 3 ? g.extents[1] : 1, planes = g.dim >= 2 ? g.extents[0] : 1;
    const int64_t hrow = lay.shape[g.dim - 1], hrows = g.dim == 3 ? lay.shape[1] : 1;
    const int64_t drow = g.dim == 1 ? g.alloc_elems : g.strides[g.dim - 2], drows = g.dim == 3 ? g.strides[0] / g.strides[1] : 1;
    p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(in), elem * hrow, hrow, hrows);
    p.dstPtr = make_cudaPitchedPtr(hist, elem * drow, drow, drows);
    p.srcPos = make_cudaPos(elem * lay.offset, g.dim == 3 ? lay.offset : 0, g.dim >= 2 ? lay.offset : 0);
    p.dstPos = make_cudaPos(elem * kPadLast, g.dim == 3 ? 1 : 0, g.dim >= 2 ? 1 : 0);
    p.extent = make_cudaExtent(elem * g.extents[g.dim - 1], rows, planes);
    p.kind = cudaMemcpyHostToDevice;
    if (cudaMemcpy3DAsync(&p, s) != cudaSuccess) return done(cuda_fail(cudaGetLastError(), "history upload"));
    TileGeo tg{};
    tg.dim = g.dim;
    for (int d = 0; d < 3; ++d) {
      tg.ext[d] = g.extents[d];
      tg.str[d] = d < g.dim ? g.strides[d] : 0;
    }
    tg.origin = g.origin;
    tg.plane = plane;
    for (int64_t w = 0; w < nwaves; ++w) {
      const int64_t n = wave_start[w + 1] - wave_start[w];
      if (n == 0) continue;
      const TileDev* wt = dt + wave_start[w];
      if (kind == 0)
        tile_wave_kernel<0><<<(unsigned)n, 256, 0, s>>>(hist, tg, wt, ft, lt);
      else if (kind == 1)
        tile_wave_kernel<1><<<(unsigned)n, 256, 0, s>>>(hist, tg, wt, ft, lt);
      else
        tile_wave_kernel<2><<<(unsigned)n, 256, 0, s>>>(hist, tg, wt, ft, lt);
      if (cudaGetLastError() != cudaSuccess) return done(cuda_fail(cudaGetLastError(), "tile_wave_kernel"));
      count_launch();
    }
    // plane `steps` -> out interior
    std::swap(p.srcPtr, p.dstPtr);
    std::swap(p.srcPos, p.dstPos);
    p.srcPtr.ptr = static_cast<char*>(hist) + (size_t)elem * plane * steps;
    p.dstPtr.ptr = out;
    p.kind = cudaMemcpyDeviceToHost;
    if (cudaMemcpy3DAsync(&p, s) != cudaSuccess) return done(cuda_fail(cudaGetLastError(), "history download"));
  }
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return done(cuda_fail(e, "tiled run"));
  return done(TVS_OK);
}

static bool lex_negative(const int* o, int dim) {
  for (int d = 0; d < dim; ++d) {
    if (o[d] < 0) return true;
    if (o[d] > 0) return false;
  }
  return false;
}

}  // namespace tvs

using namespace tvs;

extern "C" {

int tvs_tiled_run(const tvs_stencil* st, const tvs_layout* lay, const double* in, double* out, int64_t steps,
                  const tvs_tile* tiles, const int64_t* wave_start, int64_t nwaves, const tvs_exec* ex) {
  if (!st || !lay || !in || !out) return fail(TVS_ERR_INVALID, "null argument");
  int rc = validate_exec_api(ex);
  if (rc) return rc;
  if (st->dim < 1 || st->dim > 3 || st->ntaps < 1 || st->ntaps > TVS_MAX_TAPS || st->radius != 1)
    return fail(TVS_ERR_INVALID, "bad stencil");
  if (lay->dim != st->dim) return fail(TVS_ERR_SIZE, "grid/stencil dimension mismatch");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  if ((rc = check_waves(tiles, wave_start, nwaves))) return rc;
  if ((rc = set_device_api(ex->device))) return rc;
  tvs_geometry g;
  if ((rc = geometry_init_api(st->dim, lay->extents, 0, lay->extents[0], &g))) return rc;
  FpTaps ft{};
  ft.n = st->ntaps;
  ft.fma = use_fma(*st, *ex) ? 1 : 0;
  const bool gs = st->kind == TVS_GAUSS_SEIDEL;
  for (int k = 0; k < st->ntaps; ++k) {
    const int* o = st->offsets[k];
    ft.c[k] = st->coeffs[k];
    ft.lin[k] = st->dim == 1 ? o[0] : st->dim == 2 ? o[0] * g.strides[0] + o[1]
                                                   : o[0] * g.strides[0] + o[1] * g.strides[1] + o[2];
    if (gs && lex_negative(o, st->dim)) ft.newmask |= 1u << k;
  }
  LifeT lt{};
  return tiled_driver(gs ? 1 : 0, g, *lay, in, out, steps, tiles, wave_start, nwaves, ft, lt, st->boundary, 0,
                      ex->device);
}

int tvs_tiled_life(const tvs_life_rule* r, const tvs_layout* lay, const int32_t* in, int32_t* out, int64_t steps,
                   const tvs_tile* tiles, const int64_t* wave_start, int64_t nwaves, const tvs_exec* ex) {
  if (!r || !lay || !in || !out) return fail(TVS_ERR_INVALID, "null argument");
  int rc = validate_exec_api(ex);
  if (rc) return rc;
  if (r->dim < 1 || r->dim > 3 || r->ntaps < 1 || r->ntaps > 26) return fail(TVS_ERR_INVALID, "bad life rule");
  if (lay->dim != r->dim) return fail(TVS_ERR_SIZE, "grid/rule dimension mismatch");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  if ((rc = check_waves(tiles, wave_start, nwaves))) return rc;
  if ((rc = set_device_api(ex->device))) return rc;
  tvs_geometry g;
  if ((rc = geometry_init_api(r->dim, lay->extents, 0, lay->extents[0], &g))) return rc;
  LifeT lt{};
  lt.n = r->ntaps;
  lt.bmask = r->birth_mask;
  lt.smask = r->survive_mask;
  for (int k = 0; k < r->ntaps; ++k) {
    const int* o = r->offsets[k];
    lt.lin[k] = r->dim == 1 ? o[0] : r->dim == 2 ? o[0] * g.strides[0] + o[1]
                                                 : o[0] * g.strides[0] + o[1] * g.strides[1] + o[2];
  }
  FpTaps ft{};
  return tiled_driver(2, g, *lay, in, out, steps, tiles, wave_start, nwaves, ft, lt, 0.0, r->boundary, ex->device);
}

int tvs_lcs_tiled(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, const tvs_tile* tiles,
                  const int64_t* wave_start, int64_t nwaves, const tvs_exec* ex, int64_t* length) {
  int rc = validate_exec_api(ex);
  if (rc) return rc;
  if (!length || na < 0 || nb < 0 || (na > 0 && !a) || (nb > 0 && !b)) return fail(TVS_ERR_INVALID, "bad argument");
  if ((rc = check_waves(tiles, wave_start, nwaves))) return rc;
  *length = 0;
  if (na == 0 || nb == 0) return TVS_OK;
  if ((na + 1) * (nb + 1) > (1ll << 31)) return fail(TVS_ERR_SIZE, "lcs_blocked: DP table above 2^31 cells");
  if ((rc = set_device_api(ex->device))) return rc;
  cudaStream_t s;
  TVS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* buf = nullptr;
  TileDev* dt = nullptr;
  auto done = [&](int code) {
    if (buf) cudaFreeAsync(buf, s);
    if (dt) cudaFreeAsync(dt, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return code;
  };
  const int64_t cells = (na + 1) * (nb + 1);
  const int64_t ntiles = nwaves > 0 ? wave_start[nwaves] : 0;
  if (cudaMallocAsync((void**)&buf, sizeof(int) * (cells + na + nb), s) != cudaSuccess)
    return done(fail(TVS_ERR_SIZE, "lcs_blocked: DP table does not fit in device memory"));
  if (ntiles > 0 && cudaMallocAsync((void**)&dt, sizeof(TileDev) * ntiles, s) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "cudaMallocAsync"));
  int* table = buf;
  int* da = buf + cells;
  int* db = da + na;
  if (cudaMemsetAsync(table, 0, sizeof(int) * cells, s) != cudaSuccess ||
      cudaMemcpyAsync(da, a, sizeof(int) * na, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(db, b, sizeof(int) * nb, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      (ntiles > 0 && cudaMemcpyAsync(dt, tiles, sizeof(TileDev) * ntiles, cudaMemcpyHostToDevice, s) != cudaSuccess))
    return done(cuda_fail(cudaGetLastError(), "lcs_blocked upload"));
  for (int64_t w = 0; w < nwaves; ++w) {
    const int64_t n = wave_start[w + 1] - wave_start[w];
    if (n == 0) continue;
    lcs_tile_kernel<<<(unsigned)n, 256, 0, s>>>(table, da, db, (int)na, (int)nb, dt + wave_start[w]);
    if (cudaGetLastError() != cudaSuccess) return done(cuda_fail(cudaGetLastError(), "lcs_tile_kernel"));
    count_launch();
  }
  int res = 0;
  if (cudaMemcpyAsync(&res, table + cells - 1, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "lcs_blocked download"));
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return done(cuda_fail(e, "lcs_blocked"));
  *length = res;
  return done(TVS_OK);
}

}  // extern "C"
