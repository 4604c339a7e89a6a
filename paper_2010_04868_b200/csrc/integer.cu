// Integer kernels of the reference catalog: Life-like
// cellular automata and the LCS dynamic programme, int32 throughout.
//
// K7 life_kernel — replaces life_plane_update (reference baselines.py:52-66)
// behind jacobi2d_temporal(kernel="life") (verify.py:60): one time step per
// launch over a padded int32 block (same geometry as the fp64 path, 4-byte
// cells).  n = wrapping int32 sum of the radius-1 box neighbours (the
// centre excluded, StencilSpec.offsets() for life, model.py); the
// B-then-S rule: n in birth -> 1, else n in survive -> the cell's own
// state, else 0.  Integer addition is exact mod 2^32, so any summation order
// is bit-identical to the reference's.  A thread owns 8 outputs along the
// slowest in-block axis and issues every neighbour load before the first
// add (the K1 bandwidth layout): 4 B read + 4 B written per cell update.
//
// K8 lcs_kernel — replaces lcs_temporal (reference kernels/lcs.py:32-108)
// and its oracle lcs_reference (baselines.py:128-150).  The paper's
// time lanes on a GPU: the A index is time; each lane owns 4 consecutive DP
// rows skewed by one column each (a 4-row time-lane vector in registers) and
// the 32 lanes of a warp continue the skew, so at every step
//   up   = lcs[x-1][y]   = the row above's output one step earlier,
//   diag = lcs[x-1][y-1] = its output two steps earlier,
//   left = lcs[x][y-1]   = the row's own previous output,
//   b[y-1] slides through the rows and lanes one position per step,
// out = a[x-1] == b[y-1] ? diag + 1 : max(up, left); only the lane's first
// row takes a shuffle (from lane k-1's last row).  Lane 0 reads row
// x0 + 128w from a boundary row written by warp w-1's lane 31, whose 64-bit
// entries carry their own column tag (value and validity in one
// single-copy-atomic store: no fences, no progress counters); warps take
// tickets in start order and only wait on lower tickets (deadlock-free).
// Passes of at most kLcsMaxWarps warps bound the boundary-row workspace.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace tvs {

// ---------------------------------------------------------------- Life ----
constexpr int kLifeNR = 8;

struct LifeTaps {
  int n;
  int bmask, smask;  // bit v: count v in birth / survive
  int bnd;
  int64_t lin[26];
};

__device__ __forceinline__ int life_rule(unsigned n, int alive, const LifeTaps& t) {
  if (n <= 26u && ((t.bmask >> n) & 1)) return 1;
  if (n <= 26u && ((t.smask >> n) & 1)) return alive;
  return 0;
}

template <int NT>
__device__ __forceinline__ void life_points(const int* __restrict__ src, int64_t idx, int64_t rs, const LifeTaps& t,
                                            int (&out)[kLifeNR]) {
  unsigned n[kLifeNR];
  int c[kLifeNR];
#pragma unroll
  for (int r = 0; r < kLifeNR; ++r) c[r] = __ldg(src + idx + r * rs);
  if constexpr (NT > 0) {
    int v[NT][kLifeNR];
#pragma unroll
    for (int k = 0; k < NT; ++k)
#pragma unroll
      for (int r = 0; r < kLifeNR; ++r) v[k][r] = __ldg(src + idx + r * rs + t.lin[k]);
#pragma unroll
    for (int r = 0; r < kLifeNR; ++r) {
      n[r] = (unsigned)v[0][r];
#pragma unroll
      for (int k = 1; k < NT; ++k) n[r] += (unsigned)v[k][r];
    }
  } else {
#pragma unroll
    for (int r = 0; r < kLifeNR; ++r) n[r] = 0u;
    for (int k = 0; k < t.n; ++k) {
      int v[kLifeNR];
#pragma unroll
      for (int r = 0; r < kLifeNR; ++r) v[r] = __ldg(src + idx + r * rs + t.lin[k]);
#pragma unroll
      for (int r = 0; r < kLifeNR; ++r) n[r] += (unsigned)v[r];
    }
  }
#pragma unroll
  for (int r = 0; r < kLifeNR; ++r) out[r] = life_rule(n[r], c[r], t);
}

__device__ __forceinline__ int life_point(const int* __restrict__ src, int64_t idx, const LifeTaps& t) {
  unsigned n = 0u;
  for (int k = 0; k < t.n; ++k) n += (unsigned)__ldg(src + idx + t.lin[k]);
  return life_rule(n, __ldg(src + idx), t);
}

// Block (32, 8), tiles as K1 (jacobi_naive.cu): 1D 2048 consecutive cells,
// 2D/3D 32 columns x 64 rows (of plane blockIdx.z in 3D).
template <int NT>
__global__ void __launch_bounds__(256) life_kernel(const int* __restrict__ src, int* __restrict__ dst, Geo g,
                                                   LifeTaps t, int64_t origin) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  int out[kLifeNR];
  if (g.dim == 1) {
    const int64_t i0 = (int64_t)blockIdx.x * (256 * kLifeNR) + ty * 32 + tx;
    if (i0 + (kLifeNR - 1) * 256 < g.e0 && g.a0_off == 0 && g.a0_glob == g.e0) {
      life_points<NT>(src, origin + i0, 256, t, out);
#pragma unroll
      for (int r = 0; r < kLifeNR; ++r) dst[origin + i0 + r * 256] = out[r];
    } else {
      for (int r = 0; r < kLifeNR; ++r) {
        const int64_t i = i0 + r * 256;
        if (i >= g.e0) break;
        const int64_t gi = i + g.a0_off;
        dst[origin + i] = (gi < 0 || gi >= g.a0_glob) ? t.bnd : life_point(src, origin + i, t);
      }
    }
    return;
  }
  const bool d3 = g.dim == 3;
  const int64_t rows = d3 ? g.e1 : g.e0, cols = d3 ? g.e2 : g.e1, rs = d3 ? g.s1 : g.s0;
  const int64_t c = (int64_t)blockIdx.x * 32 + tx;
  const int64_t r0 = (int64_t)blockIdx.y * (8 * kLifeNR) + ty * kLifeNR;
  const int64_t p = d3 ? (int64_t)blockIdx.z : 0;
  const int64_t base = origin + (d3 ? p * g.s0 : 0) + c;
  if (c >= cols) return;
  if (d3) {
    const int64_t gp = p + g.a0_off;
    if (gp < 0 || gp >= g.a0_glob) {
      for (int r = 0; r < kLifeNR && r0 + r < rows; ++r) dst[base + (r0 + r) * rs] = t.bnd;
      return;
    }
  }
  const bool rows_ok = d3 || (r0 + g.a0_off >= 0 && r0 + kLifeNR - 1 + g.a0_off < g.a0_glob);
  if (r0 + kLifeNR <= rows && rows_ok) {
    life_points<NT>(src, base + r0 * rs, rs, t, out);
#pragma unroll
    for (int r = 0; r < kLifeNR; ++r) dst[base + (r0 + r) * rs] = out[r];
  } else {
    for (int r = 0; r < kLifeNR && r0 + r < rows; ++r) {
      const int64_t idx = base + (r0 + r) * rs;
      const int64_t gr = r0 + r + g.a0_off;
      dst[idx] = (!d3 && (gr < 0 || gr >= g.a0_glob)) ? t.bnd : life_point(src, idx, t);
    }
  }
}

// 2D, all 8 box neighbours (the catalog's Life): a thread owns column c and
// kLifeNR rows; it loads the (kLifeNR + 2) x 3 window once (every load issued
// before the first add; the side columns hit L1) and forms
// n = rowsum(r-1) + rowsum(r) + rowsum(r+1) - centre, exact mod 2^32 like
// the reference's wrapping int32 sum in any order.
__global__ void __launch_bounds__(256) life2d_box_kernel(const int* __restrict__ src, int* __restrict__ dst, Geo g,
                                                         LifeTaps t, int64_t origin) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t c = (int64_t)blockIdx.x * 32 + tx;
  const int64_t r0 = (int64_t)blockIdx.y * (8 * kLifeNR) + ty * kLifeNR;
  if (c >= g.e1) return;
  const int64_t base = origin + c;
  const bool full = r0 + kLifeNR <= g.e0 && r0 + g.a0_off >= 0 && r0 + kLifeNR - 1 + g.a0_off < g.a0_glob;
  if (full) {
    unsigned v[kLifeNR + 2][3];
#pragma unroll
    for (int r = 0; r < kLifeNR + 2; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k) v[r][k] = (unsigned)__ldg(src + base + (r0 + r - 1) * g.s0 + (k - 1));
    unsigned h[kLifeNR + 2];
#pragma unroll
    for (int r = 0; r < kLifeNR + 2; ++r) h[r] = v[r][0] + v[r][1] + v[r][2];
#pragma unroll
    for (int r = 0; r < kLifeNR; ++r) {
      const unsigned n = h[r] + h[r + 1] + h[r + 2] - v[r + 1][1];
      dst[base + (r0 + r) * g.s0] = life_rule(n, (int)v[r + 1][1], t);
    }
  } else {
    for (int r = 0; r < kLifeNR && r0 + r < g.e0; ++r) {
      const int64_t idx = base + (r0 + r) * g.s0;
      const int64_t gr = r0 + r + g.a0_off;
      dst[idx] = (gr < 0 || gr >= g.a0_glob) ? t.bnd : life_point(src, idx, t);
    }
  }
}

// K7b: 2D box Life, D time levels per HBM pass (the K3 scheme in int32).
// One warp per block owns a strip of 32*kLP columns (kLP per lane) and
// streams a segment of rows; level l works one row behind level l-1.  Per
// level and column a lane keeps F = rowsum(q-1) + rowsum(q), M = rowsum(q)
// and the centre of row q; when row q+1 of level l-1 arrives (its edge
// columns by __shfl_up / __shfl_down) the count of row q is
// F + rowsum(q+1) - centre (exact mod 2^32) and the rule gives the level-l
// value of row q, which is what level l+1 consumes next.  Rows / columns
// outside the domain are pinned to the boundary at every level.  The outer
// D columns of a strip and D rows of a segment are recomputed by the
// neighbouring tasks, so each level of a task is exactly one Life step of
// its output cells: bit-identical to D single steps.
constexpr int kLP = 4;           // columns per lane
constexpr int kLifeSeg = 256;    // output rows per task

__device__ __forceinline__ int life_rule_u(unsigned n, int centre, unsigned bmask, unsigned smask) {
  const bool in = n < 27u;
  const bool born = in && ((bmask >> n) & 1u);
  const bool keep = in && ((smask >> n) & 1u);
  return born ? 1 : (keep ? centre : 0);
}

template <int D>
__global__ void __launch_bounds__(32) life2d_tb_kernel(const int* __restrict__ src, int* __restrict__ dst, Geo g,
                                                       int64_t origin, unsigned bmask, unsigned smask, int bnd,
                                                       int64_t n_strips, int64_t n_tasks) {
  constexpr int U = 32 * kLP - 2 * D;  // useful columns per strip
  const int lane = threadIdx.x;
  const int64_t task = blockIdx.x;
  if (task >= n_tasks) return;
  const int64_t strip = task % n_strips, seg = task / n_strips;
  const int col0 = (int)(-D + strip * U);
  const int cl = col0 + lane * kLP;
  const int r0 = (int)(seg * kLifeSeg);
  const int r1 = (int)min((int64_t)r0 + kLifeSeg, g.e0);
  const int e0 = (int)g.e0, e1 = (int)g.e1;
  const int a0 = (int)g.a0_off, ag = (int)g.a0_glob;
  unsigned col_out = 0, store_mask = 0;
#pragma unroll
  for (int p = 0; p < kLP; ++p) {
    const int x = cl + p;
    col_out |= (x < 0 || x >= e1 ? 1u : 0u) << p;
    store_mask |= (x >= col0 + D && x < col0 + D + U && x >= 0 && x < e1 ? 1u : 0u) << p;
  }
  unsigned F[D][kLP], M[D][kLP];
  int C[D][kLP];
#pragma unroll
  for (int l = 0; l < D; ++l)
#pragma unroll
    for (int p = 0; p < kLP; ++p) F[l][p] = M[l][p] = 0u, C[l][p] = bnd;
  const int* col_base = src + origin + cl;
  const int m_begin = r0 - D, m_end = r1 + D;
  // interior warp (no column outside, every loaded row and every produced
  // level row inside the local and global range): no per-row checks or
  // boundary selects (the same split as the fp64 2D kernel)
  const bool any_col_out = __any_sync(0xffffffffu, col_out != 0);
  const bool interior = !any_col_out && m_begin >= 0 && m_end + 2 <= e0 && m_begin - D + a0 >= 0 &&
                        m_end + 1 + a0 < ag;
  auto run = [&](auto in_tag) {
    constexpr bool IN = decltype(in_tag)::value;
    auto load_row = [&](int m, int (&r)[kLP]) {
      const int* rp = col_base + (int64_t)m * g.s0;
      if constexpr (IN) {
#pragma unroll
        for (int p = 0; p < kLP; ++p) r[p] = __ldg(rp + p);
      } else {
        const bool row_ok = m >= 0 && m < e0 && m + a0 >= 0 && m + a0 < ag;
#pragma unroll
        for (int p = 0; p < kLP; ++p) r[p] = (row_ok && !(col_out >> p & 1u)) ? __ldg(rp + p) : bnd;
      }
    };
    int pre[2][kLP];
    load_row(m_begin, pre[0]);
    load_row(m_begin + 1, pre[1]);
    for (int m = m_begin; m < m_end; ++m) {
      int in[kLP + 2];
#pragma unroll
      for (int p = 0; p < kLP; ++p) in[p + 1] = pre[0][p];
#pragma unroll
      for (int p = 0; p < kLP; ++p) pre[0][p] = pre[1][p];
      load_row(m + 2, pre[1]);
#pragma unroll
      for (int l = 0; l < D; ++l) {
        // row m - l of level l (its input) arrived: finish row m - l - 1 of level l+1
        in[0] = __shfl_up_sync(0xffffffffu, in[kLP], 1);
        in[kLP + 1] = __shfl_down_sync(0xffffffffu, in[1], 1);
        const int q = m - l - 1;  // row finished at level l+1
        const bool pin_row = !IN && (q + a0 < 0 || q + a0 >= ag);
        int out[kLP];
#pragma unroll
        for (int p = 0; p < kLP; ++p) {
          const unsigned rs = (unsigned)in[p] + (unsigned)in[p + 1] + (unsigned)in[p + 2];
          const unsigned nsum = F[l][p] + rs - (unsigned)C[l][p];
          const int v = life_rule_u(nsum, C[l][p], bmask, smask);
          if constexpr (IN)
            out[p] = v;
          else
            out[p] = (pin_row || (col_out >> p & 1u)) ? bnd : v;
          F[l][p] = M[l][p] + rs;
          M[l][p] = rs;
          C[l][p] = in[p + 1];
        }
#pragma unroll
        for (int p = 0; p < kLP; ++p) in[p + 1] = out[p];
      }
      const int q = m - D;  // level-D row leaving
      if (q >= r0 && q < r1) {
        int* wp = dst + origin + (int64_t)q * g.s0 + cl;
#pragma unroll
        for (int p = 0; p < kLP; ++p)
          if (store_mask >> p & 1u) wp[p] = in[p + 1];
      }
    }
  };
  if (interior)
    run(std::true_type{});
  else
    run(std::false_type{});
}

// halo fill touching only halo lines and pads (see fill_halo_kernel, api.cu)
__global__ void fill_halo_i32_kernel(int* base, tvs_geometry g, int value) {
  if (g.dim == 1) {
    const int64_t n = g.extents[0], pads = g.alloc_elems - n;  // kPadLast before, the rest after
    for (int64_t c = threadIdx.x; c < pads; c += blockDim.x) base[c < kPadLast ? c : c + n] = value;
    return;
  }
  const int64_t pitch = g.strides[g.dim - 2];
  const int64_t lines = g.alloc_elems / pitch;
  const int64_t ncols = g.extents[g.dim - 1];
  for (int64_t l = blockIdx.x; l < lines; l += gridDim.x) {
    bool inner;
    if (g.dim == 2) {
      inner = l - 1 >= 0 && l - 1 < g.extents[0];
    } else {
      const int64_t per = g.extents[1] + 2;
      const int64_t p = l / per - 1, r = l % per - 1;
      inner = p >= 0 && p < g.extents[0] && r >= 0 && r < g.extents[1];
    }
    int* line = base + l * pitch;
    if (!inner) {
      for (int64_t c = threadIdx.x; c < pitch; c += blockDim.x) line[c] = value;
    } else {
      const int64_t right = pitch - kPadLast - ncols;
      for (int64_t c = threadIdx.x; c < kPadLast + right; c += blockDim.x) line[c < kPadLast ? c : c + ncols] = value;
    }
  }
}

static int fill_halo_i32(const tvs_geometry& g, int* dev, int value, cudaStream_t s) {
  if (g.dim == 1) {
    fill_halo_i32_kernel<<<1, 256, 0, s>>>(dev, g, value);
  } else {
    const int64_t lines = g.alloc_elems / g.strides[g.dim - 2];
    fill_halo_i32_kernel<<<(int)std::min<int64_t>(lines, 148 * 32), 64, 0, s>>>(dev, g, value);
  }
  TVS_LAUNCHED("fill_halo_i32_kernel");
  return TVS_OK;
}

static int validate_life(const tvs_life_rule* r) {
  if (!r) return fail(TVS_ERR_INVALID, "null life rule");
  if (r->dim < 1 || r->dim > 3) return fail(TVS_ERR_INVALID, "dim must be 1..3");
  if (r->ntaps < 1 || r->ntaps > 26) return fail(TVS_ERR_INVALID, "life: ntaps must be 1..26");
  if ((r->birth_mask | r->survive_mask) & ~0x1FF) return fail(TVS_ERR_INVALID, "life rule sets must be subsets of 0..8");
  for (int k = 0; k < r->ntaps; ++k)
    for (int d = 0; d < 3; ++d) {
      const int o = r->offsets[k][d];
      if (o < -1 || o > 1) return fail(TVS_ERR_INVALID, "tap offset exceeds radius 1");
      if (d >= r->dim && o != 0) return fail(TVS_ERR_INVALID, "tap offset on a missing axis");
    }
  return TVS_OK;
}

static int life_step(const tvs_life_rule& r, const tvs_geometry& g, const int* src, int* dst, cudaStream_t s) {
  LifeTaps t{};
  t.n = r.ntaps;
  t.bmask = r.birth_mask;
  t.smask = r.survive_mask;
  t.bnd = r.boundary;
  const int64_t s0 = g.strides[0], s1 = g.dim == 3 ? g.strides[1] : 1;
  for (int k = 0; k < r.ntaps; ++k) {
    const int* o = r.offsets[k];
    t.lin[k] = g.dim == 1 ? o[0] : g.dim == 2 ? o[0] * s0 + o[1] : o[0] * s0 + o[1] * s1 + o[2];
  }
  const Geo geo = make_geo(g);
  auto cdiv = [](int64_t a, int64_t b) { return (a + b - 1) / b; };
  int64_t gx, gy = 1, gz = 1;
  if (geo.dim == 1) {
    gx = cdiv(geo.e0, 256 * kLifeNR);
  } else if (geo.dim == 2) {
    gx = cdiv(geo.e1, 32);
    gy = cdiv(geo.e0, 8 * kLifeNR);
  } else {
    gx = cdiv(geo.e2, 32);
    gy = cdiv(geo.e1, 8 * kLifeNR);
    gz = geo.e0;
  }
  if (gx >= (1ll << 31) || gy > 65535 || gz > 65535) return fail(TVS_ERR_SIZE, "life: grid too large");
  const dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)gz), block(32, 8);
  unsigned ring = 0;  // 3x3 positions named by the taps
  for (int k = 0; k < r.ntaps; ++k) ring |= 1u << ((r.offsets[k][0] + 1) * 3 + (r.offsets[k][1] + 1));
  if (geo.dim == 2 && r.ntaps == 8 && ring == 0x1EFu) {  // exactly the 8 box neighbours
    life2d_box_kernel<<<grid, block, 0, s>>>(src, dst, geo, t, g.origin);
    TVS_LAUNCHED("life2d_box_kernel");
    return TVS_OK;
  }
  if (r.ntaps == 8)
    life_kernel<8><<<grid, block, 0, s>>>(src, dst, geo, t, g.origin);
  else if (r.ntaps == 2)
    life_kernel<2><<<grid, block, 0, s>>>(src, dst, geo, t, g.origin);
  else
    life_kernel<0><<<grid, block, 0, s>>>(src, dst, geo, t, g.origin);
  TVS_LAUNCHED("life_kernel");
  return TVS_OK;
}

template <int D>
static int life2d_tb_launch(const tvs_life_rule& r, const tvs_geometry& g, const int* src, int* dst, cudaStream_t s) {
  const Geo geo = make_geo(g);
  constexpr int U = 32 * kLP - 2 * D;
  const int64_t ns = (geo.e1 + U - 1) / U;
  const int64_t nt = ns * ((geo.e0 + kLifeSeg - 1) / kLifeSeg);
  life2d_tb_kernel<D><<<(unsigned)nt, 32, 0, s>>>(src, dst, geo, g.origin, (unsigned)r.birth_mask,
                                                  (unsigned)r.survive_mask, r.boundary, ns, nt);
  TVS_LAUNCHED("life2d_tb_kernel");
  return TVS_OK;
}

static bool life_is_box2d(const tvs_life_rule& r) {
  unsigned ring = 0;
  for (int k = 0; k < r.ntaps; ++k) ring |= 1u << ((r.offsets[k][0] + 1) * 3 + (r.offsets[k][1] + 1));
  return r.dim == 2 && r.ntaps == 8 && ring == 0x1EFu;
}

static int life_device(const tvs_life_rule& r, const tvs_geometry& g, int* src, int* dst, int64_t steps,
                       cudaStream_t s, int32_t* in_dst, int depth = 0) {
  int* a = src;
  int* b = dst;
  static const int env_depth = [] {
    const char* e = getenv("TVS_LIFE_DEPTH");  // 16384^2 B2S23 x 20 (interior-warp loop): 2 971, 4 1231, 8 1243 GCellUpd/s
    return e ? atoi(e) : 4;
  }();
  const int D = depth > 0 ? depth : env_depth;
  const bool box2d = life_is_box2d(r);
  const int cap = D >= 8 ? 8 : (D >= 4 ? 4 : (D >= 2 ? 2 : 1));
  for (int64_t k = 0; k < steps;) {
    const int64_t left = steps - k;
    int done = box2d ? cap : 1;
    while (done > left) done >>= 1;  // 8, 4, 2 or 1 levels this pass
    const int rc = done == 8   ? life2d_tb_launch<8>(r, g, a, b, s)
                   : done == 4 ? life2d_tb_launch<4>(r, g, a, b, s)
                   : done == 2 ? life2d_tb_launch<2>(r, g, a, b, s)
                               : life_step(r, g, a, b, s);
    if (rc) return rc;
    std::swap(a, b);
    k += done;
  }
  if (in_dst) *in_dst = a == dst ? 1 : 0;
  return TVS_OK;
}

static int copy_interior_i32(const tvs_geometry& g, int* dev, const tvs_layout& lay, int* host, bool upload,
                             cudaStream_t s) {
  if (lay.dim != g.dim) return fail(TVS_ERR_SIZE, "layout/geometry dimension mismatch");
  for (int d = 0; d < g.dim; ++d) {
    if (lay.extents[d] != g.extents[d]) return fail(TVS_ERR_SIZE, "layout/geometry extents mismatch");
    if (lay.offset + lay.extents[d] > lay.shape[d]) return fail(TVS_ERR_INVALID, "layout shape too small");
  }
  const size_t E = sizeof(int);
  const auto kind = upload ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  int* d0 = dev + g.origin;
  if (g.dim == 1) {
    int* h0 = host + lay.offset;
    TVS_CUDA(cudaMemcpyAsync(upload ? (void*)d0 : (void*)h0, upload ? (void*)h0 : (void*)d0, E * g.extents[0], kind, s));
  } else if (g.dim == 2) {
    int* h0 = host + lay.offset * lay.shape[1] + lay.offset;
    const size_t hp = E * lay.shape[1], dp = E * g.strides[0], w = E * g.extents[1];
    if (upload)
      TVS_CUDA(cudaMemcpy2DAsync(d0, dp, h0, hp, w, g.extents[0], kind, s));
    else
      TVS_CUDA(cudaMemcpy2DAsync(h0, hp, d0, dp, w, g.extents[0], kind, s));
  } else {
    cudaMemcpy3DParms p;
    std::memset(&p, 0, sizeof(p));
    const cudaPitchedPtr hptr = make_cudaPitchedPtr(host, E * lay.shape[2], lay.shape[2], lay.shape[1]);
    const cudaPitchedPtr dptr = make_cudaPitchedPtr(dev, E * g.strides[1], g.strides[1], g.strides[0] / g.strides[1]);
    const cudaPos hpos = make_cudaPos(E * lay.offset, lay.offset, lay.offset);
    const cudaPos dpos = make_cudaPos(E * kPadLast, 1, 1);
    p.extent = make_cudaExtent(E * g.extents[2], g.extents[1], g.extents[0]);
    if (upload) {
      p.srcPtr = hptr; p.srcPos = hpos; p.dstPtr = dptr; p.dstPos = dpos;
    } else {
      p.srcPtr = dptr; p.srcPos = dpos; p.dstPtr = hptr; p.dstPos = hpos;
    }
    p.kind = kind;
    TVS_CUDA(cudaMemcpy3DAsync(&p, s));
  }
  return TVS_OK;
}

// ----------------------------------------------------------------- LCS ----
constexpr int kLcsMaxWarps = 4096;  // warps (128 DP rows each) per pass

struct LcsArgs {
  const int* a;   // device, na
  const int* b;   // device, nb
  int na, nb;
  int x0;         // DP rows x0+1 .. handled by this pass
  int nwarps;
  unsigned long long* rows;  // (nwarps + 1) x (nb + 1): row w = lcs[x0 + 128w][*], (y + 1) << 32 | value
  int* ticket;
  int* result;    // lcs[na][nb]
};

// Lane k owns kLcsRPL consecutive DP rows x_j = x0 + 32*kLcsRPL*w +
// kLcsRPL*k + j + 1; at step s its row j updates column c - j with
// c = s + 1 - kLcsRPL*k.  Every input of a step was produced in an earlier
// step: up_j / diag_j of row j > 0 are row j-1's outputs one / two steps
// back (registers), row 0's come from lane k-1's last row (one shuffle);
// the B window shifts through the rows and lanes the same way.  So the
// kLcsRPL updates of a step are independent and the loop-carried path is one
// shuffle plus one select per step.
constexpr int kLcsRPL = 4;
constexpr int kLcsWarpRows = 32 * kLcsRPL;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* q) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(q) : "memory");
  return v;
}
// predicated inside the asm: no branch, so the warp never diverges around the
// shuffles (a divergent region compiles them to the slow collective form)
__device__ __forceinline__ void st_relaxed_u64_if(bool pred, unsigned long long* q, unsigned long long v) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.relaxed.gpu.global.b64 [%0], %1; }"
               ::"l"(q), "l"(v), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ void st_i32_if(bool pred, int* q, int v) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.global.b32 [%0], %1; }"
               ::"l"(q), "r"(v), "r"((unsigned)pred) : "memory");
}

// Boundary rows carry (column + 1) in the high word of every 64-bit entry:
// one single-copy-atomic store publishes a value together with its own
// validity tag, so the hand-off needs no fence and no progress counter; the
// consumer re-reads an entry until its tag matches.
__global__ void __launch_bounds__(32) lcs_kernel(LcsArgs p) {
  __shared__ int s_w;
  const int lane = threadIdx.x;
  if (lane == 0) s_w = atomicAdd(p.ticket, 1);
  __syncwarp();
  const int w = s_w;
  if (w >= p.nwarps) return;
  const int nb = p.nb;
  const int xb = p.x0 + kLcsWarpRows * w + kLcsRPL * lane;  // row j of this lane is xb + j + 1
  int av[kLcsRPL];
#pragma unroll
  for (int j = 0; j < kLcsRPL; ++j) av[j] = xb + j + 1 <= p.na ? p.a[xb + j] : 0;
  const unsigned long long* rin = p.rows + (size_t)w * (nb + 1);
  unsigned long long* rout = p.rows + (size_t)(w + 1) * (nb + 1);
  int out[kLcsRPL], prev[kLcsRPL], bw[kLcsRPL];  // prev: outputs one step older than out
#pragma unroll
  for (int j = 0; j < kLcsRPL; ++j) out[j] = prev[j] = bw[j] = 0;
  int up0_prev = 0;  // row-0 `up` of the previous step = row-0 diag now
  // lane 0's inputs come in chunks of 32 columns, read half a chunk ahead and
  // validated (re-read until the tag matches) when the chunk starts
  int c_up = 0, c_b = 0, n_b = 0;
  unsigned long long n_raw = 0;
  SpinGuard guard;
  const int nsteps = nb + kLcsWarpRows - 1;
  // the lane/row holding DP row na (if any) meets column nb at step rstep
  const int rj = p.na - 1 - xb;
  const bool has_res = rj >= 0 && rj < kLcsRPL;
  const int rstep = has_res ? nb - 1 + kLcsRPL * lane + rj : -1;
  int res = 0;
  auto chunk_start = [&](int s) {
    const int y = s + 1 + lane;
    unsigned long long raw = s == 0 && y <= nb ? ld_relaxed_u64(rin + y) : n_raw;
    if (s == 0) n_b = lane < nb ? p.b[lane] : 0;
    // warp-uniform retry loop (lanes whose entry is not tagged yet re-read)
    bool bad = y <= nb && (int)(raw >> 32) != y + 1;
    while (__any_sync(0xffffffffu, bad)) {
      if (bad) raw = ld_relaxed_u64(rin + y);
      bad = y <= nb && (int)(raw >> 32) != y + 1;
      guard.tick();
    }
    c_up = y <= nb ? (int)(unsigned)raw : 0;
    c_b = n_b;
  };
  // one step; WARM: rows may still be left of column 1 (first 128 steps)
  auto step = [&](int s, int ph, auto warm_tag) {
    constexpr bool WARM = decltype(warm_tag)::value;
    // from lane k-1: its last row's output and its oldest B value (previous step)
    const int up_sh = __shfl_up_sync(0xffffffffu, out[kLcsRPL - 1], 1);
    const int b_sh = __shfl_up_sync(0xffffffffu, bw[kLcsRPL - 1], 1);
    const int up0_in = __shfl_sync(0xffffffffu, c_up, ph);
    const int b0_in = __shfl_sync(0xffffffffu, c_b, ph);
    const int up0 = lane == 0 ? up0_in : up_sh;
    const int c = s + 1 - kLcsRPL * lane;
    int nw[kLcsRPL];
#pragma unroll
    for (int j = kLcsRPL - 1; j >= 0; --j) {
      const int bj = j == 0 ? (lane == 0 ? b0_in : b_sh) : bw[j - 1];
      const int up = j == 0 ? up0 : out[j - 1];
      const int dg = j == 0 ? up0_prev : prev[j - 1];
      int v = av[j] == bj ? dg + 1 : max(up, out[j]);
      if (WARM && c - j < 1) v = 0;  // lcs[x][0] = 0 before the row's first column
      nw[j] = v;
      bw[j] = bj;
    }
    up0_prev = up0;
#pragma unroll
    for (int j = 0; j < kLcsRPL; ++j) {
      prev[j] = out[j];
      out[j] = nw[j];
    }
    const int ylast = c - (kLcsRPL - 1);  // column of this lane's last row
    st_relaxed_u64_if(lane == 31 && ylast >= 1 && ylast <= nb, rout + ylast,
                      ((unsigned long long)(ylast + 1) << 32) | (unsigned)out[kLcsRPL - 1]);
    if (s == rstep) res = rj == 0 ? out[0] : rj == 1 ? out[1] : rj == 2 ? out[2] : out[kLcsRPL - 1];
  };
  // chunks of 32 steps, the body unrolled so the chunk bookkeeping (start,
  // next-chunk prefetch at ph 16) costs no per-step branches
  const int nfull = nsteps / 32;
  for (int q = 0; q < nfull; ++q) {
    const int s0 = q * 32;
    chunk_start(s0);
    const bool pre = s0 + 32 < nsteps;
    if (s0 < kLcsWarpRows) {
#pragma unroll
      for (int ph = 0; ph < 32; ++ph) {
        if (ph == 16 && pre) {
          const int y = s0 + 33 + lane;  // next chunk
          n_raw = y <= nb ? ld_relaxed_u64(rin + y) : 0ull;
          n_b = s0 + 32 + lane < nb ? p.b[s0 + 32 + lane] : 0;
        }
        step(s0 + ph, ph, std::true_type{});
      }
    } else {
#pragma unroll
      for (int ph = 0; ph < 32; ++ph) {
        if (ph == 16 && pre) {
          const int y = s0 + 33 + lane;
          n_raw = y <= nb ? ld_relaxed_u64(rin + y) : 0ull;
          n_b = s0 + 32 + lane < nb ? p.b[s0 + 32 + lane] : 0;
        }
        step(s0 + ph, ph, std::false_type{});
      }
    }
  }
  if (nfull * 32 < nsteps) {  // ragged last chunk
    const int s0 = nfull * 32;
    chunk_start(s0);
    for (int ph = 0; s0 + ph < nsteps; ++ph) step(s0 + ph, ph, std::true_type{});
  }
  st_i32_if(has_res, p.result, res);
}

// row 0 of the first pass: lcs[0][y] = 0 for every column, tagged
__global__ void lcs_row0_kernel(unsigned long long* row, int nb) {
  for (int y = blockIdx.x * blockDim.x + threadIdx.x; y <= nb; y += gridDim.x * blockDim.x)
    row[y] = (unsigned long long)(y + 1) << 32;
}

struct LcsWork {
  int device = -1;
  int* buf = nullptr;
  size_t bytes = 0;
  ~LcsWork() {
    if (buf) cudaFree(buf);
  }
};
static thread_local LcsWork g_lcs;

// tvs_release_thread_cache: the calling thread's LCS workspace
void release_integer_cache() {
  if (g_lcs.buf) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g_lcs.device);
    cudaFree(g_lcs.buf);
    cudaSetDevice(cur);
  }
  g_lcs.buf = nullptr;
  g_lcs.bytes = 0;
  g_lcs.device = -1;
}

static int lcs_device(const int* a, int na, const int* b, int nb, int* result_dev, cudaStream_t s) {
  if (na == 0 || nb == 0) {
    TVS_CUDA(cudaMemsetAsync(result_dev, 0, sizeof(int), s));
    return TVS_OK;
  }
  const int total_warps = (na + kLcsWarpRows - 1) / kLcsWarpRows;
  // workspace budget ~512 MB of tagged boundary rows
  const int64_t row_bytes = (int64_t)(nb + 1) * sizeof(unsigned long long);
  const int cap = (int)std::max<int64_t>(1, std::min<int64_t>(kLcsMaxWarps, (512ll << 20) / row_bytes - 1));
  const int per = std::min(total_warps, cap);
  const size_t need = (size_t)(per + 1) * row_bytes + 256;
  int dev;
  TVS_CUDA(cudaGetDevice(&dev));
  if (g_lcs.bytes < need || g_lcs.device != dev) {
    if (g_lcs.buf) cudaFree(g_lcs.buf);
    g_lcs.buf = nullptr;
    g_lcs.bytes = 0;
    TVS_CUDA(cudaMalloc(&g_lcs.buf, need));
    g_lcs.bytes = need;
    g_lcs.device = dev;
  }
  unsigned long long* rows = reinterpret_cast<unsigned long long*>(g_lcs.buf);
  int* ticket = reinterpret_cast<int*>(rows + (size_t)(per + 1) * (nb + 1));
  lcs_row0_kernel<<<64, 256, 0, s>>>(rows, nb);
  TVS_LAUNCHED("lcs_row0_kernel");
  for (int x0 = 0, first = 1; x0 < na; x0 += kLcsWarpRows * per, first = 0) {
    const int nw = std::min(per, (na - x0 + kLcsWarpRows - 1) / kLcsWarpRows);
    if (!first)  // the previous pass's last row (tags intact) becomes row 0
      TVS_CUDA(cudaMemcpyAsync(rows, rows + (size_t)per * (nb + 1), row_bytes, cudaMemcpyDeviceToDevice, s));
    // stale tags of the previous pass must not validate: clear rows 1..nw
    TVS_CUDA(cudaMemsetAsync(rows + (nb + 1), 0, (size_t)nw * row_bytes, s));
    TVS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), s));
    LcsArgs p{a, b, na, nb, x0, nw, rows, ticket, result_dev};
    lcs_kernel<<<nw, 32, 0, s>>>(p);
    TVS_LAUNCHED("lcs_kernel");
    if (nw < per) break;
  }
  return TVS_OK;
}

}  // namespace tvs

using namespace tvs;

extern "C" {

int tvs_fill_halo_i32(const tvs_geometry* g, int32_t* dev, int32_t value, void* stream) {
  if (!g || !dev) return fail(TVS_ERR_INVALID, "null argument");
  return fill_halo_i32(*g, dev, value, (cudaStream_t)stream);
}

int tvs_upload_i32(const tvs_geometry* g, int32_t* dev, const tvs_layout* lay, const int32_t* host, void* stream) {
  if (!g || !dev || !lay || !host) return fail(TVS_ERR_INVALID, "null argument");
  return copy_interior_i32(*g, dev, *lay, const_cast<int*>(host), true, (cudaStream_t)stream);
}

int tvs_download_i32(const tvs_geometry* g, const int32_t* dev, const tvs_layout* lay, int32_t* host, void* stream) {
  if (!g || !dev || !lay || !host) return fail(TVS_ERR_INVALID, "null argument");
  return copy_interior_i32(*g, const_cast<int*>(dev), *lay, host, false, (cudaStream_t)stream);
}

int tvs_life_device(const tvs_life_rule* r, const tvs_geometry* g, int32_t* src, int32_t* dst, int64_t steps,
                    const tvs_exec* ex, void* stream, int32_t* result_in_dst) {
  int rc = validate_life(r);
  if (rc) return rc;
  if ((rc = validate_exec_api(ex))) return rc;
  if (!g || !src || !dst) return fail(TVS_ERR_INVALID, "null argument");
  if (g->dim != r->dim) return fail(TVS_ERR_SIZE, "grid/rule dimension mismatch");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  return life_device(*r, *g, src, dst, steps, (cudaStream_t)stream, result_in_dst, ex->temporal_depth);
}

int tvs_life_run(const tvs_life_rule* r, const tvs_layout* lay, const int32_t* in, int32_t* out, int64_t steps,
                 const tvs_exec* ex) {
  int rc = validate_life(r);
  if (rc) return rc;
  if ((rc = validate_exec_api(ex))) return rc;
  if (!lay || !in || !out) return fail(TVS_ERR_INVALID, "null argument");
  if ((rc = validate_layout_api(lay, r->dim))) return rc;
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  if ((rc = set_device_api(ex->device))) return rc;
  tvs_geometry g;
  if ((rc = geometry_init_api(r->dim, lay->extents, 0, lay->extents[0], &g))) return rc;
  int* buf[2] = {nullptr, nullptr};
  cudaStream_t s;
  TVS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  auto done = [&](int code) {
    for (int* b : buf)
      if (b) cudaFreeAsync(b, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return code;
  };
  for (int k = 0; k < 2; ++k) {
    if (cudaMallocAsync(&buf[k], sizeof(int) * g.alloc_elems, s) != cudaSuccess)
      return done(cuda_fail(cudaGetLastError(), "cudaMallocAsync"));
    if ((rc = fill_halo_i32(g, buf[k], r->boundary, s))) return done(rc);
  }
  if ((rc = copy_interior_i32(g, buf[0], *lay, const_cast<int*>(in), true, s))) return done(rc);
  int32_t in_dst = 0;
  if ((rc = life_device(*r, g, buf[0], buf[1], steps, s, &in_dst, ex->temporal_depth))) return done(rc);
  if ((rc = copy_interior_i32(g, in_dst ? buf[1] : buf[0], *lay, out, false, s))) return done(rc);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return done(cuda_fail(e, "tvs_life_run"));
  return done(TVS_OK);
}

int tvs_lcs_device(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, int32_t* result, void* stream) {
  if (na < 0 || nb < 0) return fail(TVS_ERR_INVALID, "negative length");
  if (na > INT32_MAX - 64 || nb > INT32_MAX - 64) return fail(TVS_ERR_SIZE, "lcs: sequence too long");
  if (!result || (na > 0 && !a) || (nb > 0 && !b)) return fail(TVS_ERR_INVALID, "null argument");
  return lcs_device(a, (int)na, b, (int)nb, result, (cudaStream_t)stream);
}

int tvs_lcs(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, const tvs_exec* ex, int64_t* length) {
  int rc = validate_exec_api(ex);
  if (rc) return rc;
  if (!length || na < 0 || nb < 0 || (na > 0 && !a) || (nb > 0 && !b)) return fail(TVS_ERR_INVALID, "bad argument");
  if (na > INT32_MAX - 64 || nb > INT32_MAX - 64) return fail(TVS_ERR_SIZE, "lcs: sequence too long");
  *length = 0;
  if (na == 0 || nb == 0) return TVS_OK;
  if ((rc = set_device_api(ex->device))) return rc;
  cudaStream_t s;
  TVS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* d = nullptr;
  auto done = [&](int code) {
    if (d) cudaFreeAsync(d, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return code;
  };
  const size_t bytes = sizeof(int) * (size_t)(na + nb + 1);
  if (cudaMallocAsync(&d, bytes, s) != cudaSuccess) return done(cuda_fail(cudaGetLastError(), "cudaMallocAsync"));
  if (cudaMemcpyAsync(d, a, sizeof(int) * na, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(d + na, b, sizeof(int) * nb, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "tvs_lcs upload"));
  if ((rc = lcs_device(d, (int)na, d + na, (int)nb, d + na + nb, s))) return done(rc);
  int res = 0;
  if (cudaMemcpyAsync(&res, d + na + nb, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "tvs_lcs download"));
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return done(cuda_fail(e, "tvs_lcs"));
  *length = res;
  return done(TVS_OK);
}

}  // extern "C"
