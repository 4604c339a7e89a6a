// K6 (baseline form): Gauss-Seidel in 2D/3D as a hyperplane wavefront over
// (time, space), in place, any radius-1 tap set, both update orders.
//
// Replaces gs2d_temporal / gs3d_temporal (reference kernels_nd.py:48-55) and
// reproduces the oracle sweeps bit-exactly:
//   * TVS_GS_LEXICOGRAPHIC: the row-major in-place loop (model.py:150-156;
//     reference test test_baselines.py:39-52).  Hyperplane h = a.x + tau*t
//     with a = (2,1), tau = 4 (2D box) / a = (4,2,1), tau = 8 (3D box) /
//     a = 1, tau = 2 (stars): every dependence lies on an earlier hyperplane
//     and no two points of a hyperplane touch each other's cells.
//   * TVS_GS_REFERENCE: the oracle's anti-diagonal gather-then-scatter
//     (_gs_sweep_nd, baselines.py:93-107): a = 1, tau = dim + 1; taps with
//     coordinate sum 0 (NE/SW) read the previous sweep, so each hyperplane
//     gathers every point first and scatters after a grid barrier.
// All T sweeps are in flight at once (sweep t trails sweep t-1 by tau
// hyperplanes), so the number of grid-wide steps is ~ a.E + tau*T instead of
// T * a.E.  The (a, tau) choice is mirrored by model.gs_hyperplane().
//
// Persistent cooperative kernel; one software grid barrier per hyperplane.
#include <algorithm>

#include "common.cuh"

namespace tvs {

struct Wave {
  double* a;        // interior origin
  double* tmp;      // gather buffer (simultaneous mode)
  unsigned* bar;    // [0] arrival counter, [1] generation
  Geo g;
  TapList tl;
  int hx[3];        // hyperplane coefficients per axis (last = 1)
  int tau;
  int simultaneous;
  long long T;
  long long h_lo, h_hi;
  long long width;  // threads per (t, outer) slot
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      SpinGuard sg;
      while (*gen == g0) sg.tick();
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double gs_point(const double* __restrict__ a, long long idx, const TapList& tl) {
  double acc = tap_first(tl.c[0], __ldcg(a + idx + tl.lin[0]));
  for (int k = 1; k < tl.n; ++k) acc = tap_next<false>(tl.c[k], __ldcg(a + idx + tl.lin[k]), acc);
  return acc;
}

__device__ __forceinline__ long long floordiv(long long x, long long d) {
  return x >= 0 ? x / d : -((-x + d - 1) / d);
}

// Enumerate the points of hyperplane h: slot = (t, outer coords) x width,
// lane of the slot = position along the second-to-last axis (3D) or the
// first axis (2D); the last coordinate follows from h.
template <int DIM>
__device__ __forceinline__ bool wave_point(const Wave& w, long long h, long long tid, long long& idx) {
  const Geo& g = w.g;
  if constexpr (DIM == 1) {
    // x = h - tau*t; slot = t
    const long long t = tid;
    if (t >= w.T) return false;
    const long long x = h - w.tau * t;
    if (x < 0 || x >= g.e0) return false;
    idx = x;
    return true;
  } else if constexpr (DIM == 2) {
    const long long t = tid / w.width;
    const long long k = tid - t * w.width;
    if (t >= w.T) return false;
    const long long rem = h - w.tau * t;  // = hx0*i + j
    // smallest i with j = rem - hx0*i <= e1-1
    long long i_lo = rem - (g.e1 - 1) <= 0 ? 0 : (rem - (g.e1 - 1) + w.hx[0] - 1) / w.hx[0];
    const long long i = i_lo + k;
    if (i >= g.e0) return false;
    const long long j = rem - w.hx[0] * i;
    if (j < 0 || j >= g.e1) return false;
    idx = i * g.s0 + j;
    return true;
  } else {
    const long long slot = tid / w.width;
    const long long k = tid - slot * w.width;
    const long long t = slot / g.e0;
    const long long i = slot - t * g.e0;
    if (t >= w.T) return false;
    const long long rem = h - w.tau * t - (long long)w.hx[0] * i;  // = hx1*j + l
    long long j_lo = rem - (g.e2 - 1) <= 0 ? 0 : (rem - (g.e2 - 1) + w.hx[1] - 1) / w.hx[1];
    const long long j = j_lo + k;
    if (j >= g.e1) return false;
    const long long l = rem - (long long)w.hx[1] * j;
    if (l < 0 || l >= g.e2) return false;
    idx = i * g.s0 + j * g.s1 + l;
    return true;
  }
}

template <int DIM>
__global__ void __launch_bounds__(256) gs_wave_kernel(Wave w, long long total_threads) {
  const unsigned nblocks = gridDim.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long h = w.h_lo; h <= w.h_hi; ++h) {
    if (!w.simultaneous) {
      for (long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x; tid < total_threads; tid += stride) {
        long long idx;
        if (wave_point<DIM>(w, h, tid, idx)) w.a[idx] = gs_point(w.a, idx, w.tl);
      }
      grid_barrier(w.bar, nblocks);
    } else {
      for (long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x; tid < total_threads; tid += stride) {
        long long idx;
        if (wave_point<DIM>(w, h, tid, idx)) w.tmp[tid] = gs_point(w.a, idx, w.tl);
      }
      grid_barrier(w.bar, nblocks);
      for (long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x; tid < total_threads; tid += stride) {
        long long idx;
        if (wave_point<DIM>(w, h, tid, idx)) w.a[idx] = w.tmp[tid];
      }
      grid_barrier(w.bar, nblocks);
    }
  }
}

// Hyperplane (a, tau) per order — same search result as model.gs_hyperplane.
static bool pick_hyperplane(const tvs_stencil& st, int order, int hx[3], int& tau, int& simul) {
  // new-tap predicate per order
  auto is_new = [&](const int* o) {
    if (order == TVS_GS_REFERENCE) return o[0] + o[1] + o[2] < 0;
    for (int d = 0; d < st.dim; ++d)
      if (o[d]) return o[d] < 0;
    return false;
  };
  int best_key = 1 << 30;
  bool found = false;
  int a[3] = {1, 1, 1};
  const int lim = 8;
  for (a[0] = 1; a[0] <= lim; ++a[0])
    for (a[1] = 1; a[1] <= (st.dim > 1 ? lim : 1); ++a[1])
      for (a[2] = 1; a[2] <= (st.dim > 2 ? lim : 1); ++a[2]) {
        if (a[st.dim - 1] != 1) continue;  // last-axis coefficient 1 (enumeration assumes it)
        for (int tt = 1; tt < 40; ++tt) {
          bool ok = true, sim = false;
          for (int k = 0; k < st.ntaps && ok; ++k) {
            const int* o = st.offsets[k];
            if (!o[0] && !o[1] && !o[2]) continue;
            int ao = 0;
            for (int d = 0; d < st.dim; ++d) ao += a[d] * o[d];
            if (is_new(o)) {
              ok = 0 < -ao && -ao < tt;
            } else {
              ok = 0 <= ao && ao < tt;
              sim = sim || ao == 0;
            }
          }
          if (ok) {
            const int key = (sim ? 1 << 20 : 0) + tt * 64 + a[0] + a[1] + a[2];
            if (key < best_key) {
              best_key = key;
              found = true;
              hx[0] = a[0]; hx[1] = a[1]; hx[2] = a[2];
              tau = tt;
              simul = sim;
            }
            break;
          }
        }
      }
  return found;
}

int gs_wavefront(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, int order,
                 cudaStream_t s) {
  Wave w{};
  if (!pick_hyperplane(st, order, w.hx, w.tau, w.simultaneous))
    return fail(TVS_ERR_UNSUPPORTED, "no wavefront schedule for this Gauss-Seidel tap set");
  w.g = make_geo(g);
  w.a = grid + g.origin;
  w.T = steps;
  w.tl.n = st.ntaps;
  w.tl.bnd = st.boundary;
  const int64_t s0 = g.strides[0], s1 = g.dim == 3 ? g.strides[1] : 1;
  for (int k = 0; k < st.ntaps; ++k) {
    const int* o = st.offsets[k];
    w.tl.c[k] = st.coeffs[k];
    w.tl.lin[k] = g.dim == 1 ? o[0] : (g.dim == 2 ? o[0] * s0 + o[1] : o[0] * s0 + o[1] * s1 + o[2]);
  }
  const Geo& G = w.g;
  long long hmax = 0, total = 0;
  if (g.dim == 1) {
    hmax = (G.e0 - 1) + w.tau * (steps - 1);
    w.width = 1;
    total = steps;
  } else if (g.dim == 2) {
    hmax = w.hx[0] * (G.e0 - 1) + (G.e1 - 1) + w.tau * (steps - 1);
    w.width = std::min<long long>(G.e0, (G.e1 + w.hx[0] - 1) / w.hx[0] + 1);
    total = steps * w.width;
  } else {
    hmax = w.hx[0] * (G.e0 - 1) + w.hx[1] * (G.e1 - 1) + (G.e2 - 1) + w.tau * (steps - 1);
    w.width = std::min<long long>(G.e1, (G.e2 + w.hx[1] - 1) / w.hx[1] + 1);
    total = steps * G.e0 * w.width;
  }
  w.h_lo = 0;
  w.h_hi = hmax;
  unsigned* bar = static_cast<unsigned*>(scratch(64, 2));
  if (!bar) return fail(TVS_ERR_CUDA, "gs_wavefront: scratch");
  TVS_CUDA(cudaMemsetAsync(bar, 0, 64, s));
  w.bar = bar;
  if (w.simultaneous) {
    w.tmp = static_cast<double*>(scratch(sizeof(double) * std::max<long long>(total, 1), 3));
    if (!w.tmp) return fail(TVS_ERR_CUDA, "gs_wavefront: out of memory for the gather buffer");
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* fn = g.dim == 1 ? (void*)gs_wave_kernel<1> : (g.dim == 2 ? (void*)gs_wave_kernel<2> : (void*)gs_wave_kernel<3>);
  TVS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0));
  long long want = (total + 255) / 256;
  const int blocks = (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * std::max(occ, 1)));
  void* args[] = {&w, &total};
  TVS_CUDA(cudaLaunchCooperativeKernel(fn, blocks, 256, args, 0, s));
  count_launch();
  return TVS_OK;
}

}  // namespace tvs
