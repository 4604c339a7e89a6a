// C-ABI entry points of libtvstencil.so (include/tvstencil.h).
//
// Dispatch:
//   Jacobi 1D        -> jacobi1d_blocked   (register trapezoid, default 64 steps/launch)
//   Jacobi 2D star/box -> jacobi2d_blocked (warp strips, D levels per HBM pass)
//   Jacobi 3D star/box -> jacobi3d_blocked2 (2 levels/launch) + jacobi3d_streaming (2.5D, 1 step/launch)
//   Jacobi other     -> jacobi_naive_step  (generic taps, 1 step/launch)
//   Gauss-Seidel 1D  -> gs1d_pipeline      (time-skewed warp pipeline)
//   Gauss-Seidel 2D lexicographic -> gs2d_pipeline (time-lane chain)
//   Gauss-Seidel 2D reference order / 3D -> gs_wavefront (hyperplane wavefront)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace tvs {

static thread_local std::string g_err;
// bumped whenever page-locked host memory is released (tvs_host_free /
// tvs_host_unregister): invalidates captured copy graphs in every thread
static std::atomic<uint64_t> g_host_generation{0};
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return TVS_ERR_CUDA;
}
void count_launch(int64_t n) { g_launches += n; }

bool coeffs_power_of_two(const tvs_stencil& st) {
  for (int k = 0; k < st.ntaps; ++k) {
    double c = std::fabs(st.coeffs[k]);
    if (c == 0.0) continue;
    if (!std::isfinite(c)) return false;
    int ex;
    double m = std::frexp(c, &ex);
    if (m != 0.5) return false;
  }
  return true;
}

bool use_fma(const tvs_stencil& st, const tvs_exec& ex) {
  if (ex.fma_policy == TVS_FMA_ALLOW) return true;
  if (ex.fma_policy == TVS_FMA_EXACT) return coeffs_power_of_two(st);
  return false;
}

struct ScratchSlot {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = -1;
};
static thread_local ScratchSlot g_scratch[kScratchSlots];
static thread_local uint64_t g_scratch_gen = 1;  // bumped whenever a slot is (re)allocated or freed

uint64_t scratch_generation() { return g_scratch_gen; }

void* scratch(size_t bytes, int slot) {
  int dev = 0;
  cudaGetDevice(&dev);
  ScratchSlot& s = g_scratch[slot];
  if (s.ptr && s.bytes >= bytes && s.device == dev) return s.ptr;
  ++g_scratch_gen;
  if (s.ptr) {
    int cur = dev;
    cudaSetDevice(s.device);
    cudaFree(s.ptr);
    cudaSetDevice(cur);
    s.ptr = nullptr;
  }
  if (cudaMalloc(&s.ptr, bytes) != cudaSuccess) {
    s.ptr = nullptr;
    s.bytes = 0;
    return nullptr;
  }
  s.bytes = bytes;
  s.device = dev;
  return s.ptr;
}

static int validate(const tvs_stencil* st) {
  if (!st) return fail(TVS_ERR_INVALID, "null stencil");
  if (st->dim < 1 || st->dim > 3) return fail(TVS_ERR_INVALID, "dim must be 1..3");
  if (st->radius != 1) return fail(TVS_ERR_UNSUPPORTED, "only radius-1 stencils are supported");
  if (st->ntaps < 1 || st->ntaps > TVS_MAX_TAPS) return fail(TVS_ERR_INVALID, "ntaps must be 1..27");
  if (st->kind != TVS_JACOBI && st->kind != TVS_GAUSS_SEIDEL) return fail(TVS_ERR_INVALID, "bad kind");
  for (int k = 0; k < st->ntaps; ++k) {
    for (int d = 0; d < 3; ++d) {
      int o = st->offsets[k][d];
      if (o < -1 || o > 1) return fail(TVS_ERR_INVALID, "tap offset exceeds radius 1");
      if (d >= st->dim && o != 0) return fail(TVS_ERR_INVALID, "tap offset on a missing axis");
    }
  }
  return TVS_OK;
}

static int validate_exec(const tvs_exec* ex) {
  if (!ex) return fail(TVS_ERR_INVALID, "null exec");
  if (ex->n_gpus < 0) return fail(TVS_ERR_INVALID, "n_gpus must be >= 0");
  if (ex->flags & ~TVS_EXEC_EMULATE_SHARDS) return fail(TVS_ERR_INVALID, "unknown tvs_exec flags");
  if (ex->fma_policy < 0 || ex->fma_policy > 2) return fail(TVS_ERR_INVALID, "bad fma_policy");
  if (ex->gs_order < 0 || ex->gs_order > 1) return fail(TVS_ERR_INVALID, "bad gs_order");
  if (ex->algo < 0 || ex->algo > 2) return fail(TVS_ERR_INVALID, "bad algo");
  if (ex->temporal_depth < 0) return fail(TVS_ERR_INVALID, "bad temporal_depth");
  return TVS_OK;
}

// Host Grid layout (grid.py:27-37) checked once, before any path is chosen:
// every copy path (whole grid, row bands, planes, positions) stays inside
// [0, prod(shape)) when offset >= 0 and offset + extents <= shape.
static int validate_layout(const tvs_layout* lay, int dim) {
  if (!lay) return fail(TVS_ERR_INVALID, "null layout");
  if (lay->dim != dim) return fail(TVS_ERR_SIZE, "grid/stencil dimension mismatch");
  if (lay->offset < 0) return fail(TVS_ERR_INVALID, "layout offset must be >= 0");
  for (int d = 0; d < dim; ++d) {
    if (lay->extents[d] < 1) return fail(TVS_ERR_SIZE, "extents must be positive");
    if (lay->shape[d] < 1 || lay->offset + lay->extents[d] > lay->shape[d])
      return fail(TVS_ERR_INVALID, "layout shape too small for offset + extents");
  }
  return TVS_OK;
}

static int set_device(int dev) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(TVS_ERR_CUDA, "no CUDA device available (libtvstencil has no CPU fallback)");
  if (dev < 0 || dev >= n) return fail(TVS_ERR_INVALID, "device ordinal out of range");
  TVS_CUDA(cudaSetDevice(dev));
  return TVS_OK;
}

// ---- device blocks ---------------------------------------------------------
static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static int geometry_init(int dim, const int64_t* ext, int64_t a0_off, int64_t a0_glob, tvs_geometry* g) {
  std::memset(g, 0, sizeof(*g));
  if (dim < 1 || dim > 3) return fail(TVS_ERR_INVALID, "dim must be 1..3");
  for (int d = 0; d < dim; ++d)
    if (ext[d] < 1) return fail(TVS_ERR_SIZE, "extents must be positive");
  g->dim = dim;
  for (int d = 0; d < 3; ++d) g->extents[d] = d < dim ? ext[d] : 1;
  const int64_t pitch = round_up(ext[dim - 1] + 2 * kPadLast, 32);
  if (dim == 1) {
    g->strides[0] = 1;
    g->origin = kPadLast;
    g->alloc_elems = pitch;
  } else if (dim == 2) {
    g->strides[0] = pitch;
    g->strides[1] = 1;
    g->origin = pitch + kPadLast;
    g->alloc_elems = (ext[0] + 2) * pitch;
  } else {
    g->strides[2] = 1;
    g->strides[1] = pitch;
    g->strides[0] = (ext[1] + 2) * pitch;
    g->origin = g->strides[0] + pitch + kPadLast;
    g->alloc_elems = (ext[0] + 2) * g->strides[0];
  }
  g->axis0_offset = a0_off;
  g->axis0_global = a0_glob > 0 ? a0_glob : ext[0];
  return TVS_OK;
}

// Halo fill that touches only non-interior cells: one block per line of the
// last axis (row) — a halo line is filled whole, an interior line only in its
// two pads.  (The earlier element-wise version evaluated 64-bit div/mod for
// every cell of the allocation, ~1.5 ms per 2 GB buffer ahead of the first
// upload of the drop-in pipeline.)
__global__ void fill_halo_kernel(double* base, tvs_geometry g, double value) {
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
      const int64_t r = l - 1;
      inner = r >= 0 && r < g.extents[0];
    } else {
      const int64_t per = g.extents[1] + 2;
      const int64_t p = l / per - 1, r = l % per - 1;
      inner = p >= 0 && p < g.extents[0] && r >= 0 && r < g.extents[1];
    }
    double* line = base + l * pitch;
    if (!inner) {
      for (int64_t c = threadIdx.x; c < pitch; c += blockDim.x) line[c] = value;
    } else {
      const int64_t right = pitch - kPadLast - ncols;
      for (int64_t c = threadIdx.x; c < kPadLast + right; c += blockDim.x)
        line[c < kPadLast ? c : c + ncols] = value;
    }
  }
}

static int fill_halo(const tvs_geometry& g, double* dev, double value, cudaStream_t s) {
  if (g.dim == 1) {
    fill_halo_kernel<<<1, 256, 0, s>>>(dev, g, value);
  } else {
    const int64_t lines = g.alloc_elems / g.strides[g.dim - 2];
    fill_halo_kernel<<<(int)std::min<int64_t>(lines, 148 * 32), 64, 0, s>>>(dev, g, value);
  }
  TVS_LAUNCHED("fill_halo_kernel");
  return TVS_OK;
}

static int copy_interior(const tvs_geometry& g, double* dev, const tvs_layout& lay, double* host, bool upload,
                         cudaStream_t s) {
  if (lay.dim != g.dim) return fail(TVS_ERR_SIZE, "layout/geometry dimension mismatch");
  for (int d = 0; d < g.dim; ++d) {
    if (lay.extents[d] != g.extents[d]) return fail(TVS_ERR_SIZE, "layout/geometry extents mismatch");
    if (lay.offset + lay.extents[d] > lay.shape[d]) return fail(TVS_ERR_INVALID, "layout shape too small");
  }
  double* d0 = dev + g.origin;
  if (g.dim == 1) {
    double* h0 = host + lay.offset;
    size_t bytes = sizeof(double) * g.extents[0];
    if (upload) return upload_block((char*)d0, bytes, 0, (const char*)h0, bytes, 0, bytes, 1, 1, s);
    TVS_CUDA(cudaMemcpyAsync(h0, d0, bytes, cudaMemcpyDeviceToHost, s));
  } else if (g.dim == 2) {
    double* h0 = host + lay.offset * lay.shape[1] + lay.offset;
    size_t hp = sizeof(double) * lay.shape[1], dp = sizeof(double) * g.strides[0];
    size_t w = sizeof(double) * g.extents[1];
    if (upload) return upload_block((char*)d0, dp, 0, (const char*)h0, hp, 0, w, g.extents[0], 1, s);
    TVS_CUDA(cudaMemcpy2DAsync(h0, hp, d0, dp, w, g.extents[0], cudaMemcpyDeviceToHost, s));
  } else if (upload) {
    const size_t hr = sizeof(double) * lay.shape[2], hz = hr * lay.shape[1];
    const double* h0 = host + (lay.offset * lay.shape[1] + lay.offset) * lay.shape[2] + lay.offset;
    return upload_block((char*)d0, sizeof(double) * g.strides[1], sizeof(double) * g.strides[0], (const char*)h0, hr,
                        hz, sizeof(double) * g.extents[2], g.extents[1], g.extents[0], s);
  } else {
    cudaMemcpy3DParms p;
    std::memset(&p, 0, sizeof(p));
    cudaPitchedPtr hptr = make_cudaPitchedPtr(host, sizeof(double) * lay.shape[2], lay.shape[2], lay.shape[1]);
    cudaPitchedPtr dptr = make_cudaPitchedPtr(dev, sizeof(double) * g.strides[1], g.strides[1],
                                              g.strides[0] / g.strides[1]);
    cudaPos hpos = make_cudaPos(sizeof(double) * lay.offset, lay.offset, lay.offset);
    cudaPos dpos = make_cudaPos(sizeof(double) * kPadLast, 1, 1);
    p.extent = make_cudaExtent(sizeof(double) * g.extents[2], g.extents[1], g.extents[0]);
    if (upload) {
      p.srcPtr = hptr; p.srcPos = hpos; p.dstPtr = dptr; p.dstPos = dpos; p.kind = cudaMemcpyHostToDevice;
    } else {
      p.srcPtr = dptr; p.srcPos = dpos; p.dstPtr = hptr; p.dstPos = hpos; p.kind = cudaMemcpyDeviceToHost;
    }
    TVS_CUDA(cudaMemcpy3DAsync(&p, s));
  }
  return TVS_OK;
}

// field-wise stencil equality (no padding bytes compared; coefficients and
// boundary bit for bit)
bool same_stencil(const tvs_stencil& a, const tvs_stencil& b) {
  if (a.dim != b.dim || a.kind != b.kind || a.ntaps != b.ntaps || a.radius != b.radius) return false;
  if (std::memcmp(&a.boundary, &b.boundary, sizeof(double)) != 0) return false;
  for (int k = 0; k < a.ntaps && k < TVS_MAX_TAPS; ++k) {
    if (std::memcmp(a.offsets[k], b.offsets[k], sizeof(a.offsets[k])) != 0) return false;
    if (std::memcmp(&a.coeffs[k], &b.coeffs[k], sizeof(double)) != 0) return false;
  }
  return true;
}

bool wants_shards(const tvs_stencil& st, const tvs_exec& ex) {
  if (ex.n_gpus <= 1 || st.kind != TVS_JACOBI || ex.algo == TVS_ALGO_NAIVE) return false;
  if (st.dim == 2) return jacobi2d_blocked_supported(st);
  if (st.dim == 3) return jacobi3d_streaming_supported(st);
  return false;  // 1D: one GPU ("replicas only")
}

// non-static forms for the other translation units (integer.cu, shard.cu)
int fill_halo_api(const tvs_geometry& g, double* dev, double value, cudaStream_t s) {
  return fill_halo(g, dev, value, s);
}
int validate_stencil_api(const tvs_stencil* st) { return validate(st); }
int validate_exec_api(const tvs_exec* ex) { return validate_exec(ex); }
int validate_layout_api(const tvs_layout* lay, int dim) { return validate_layout(lay, dim); }
int set_device_api(int dev) { return set_device(dev); }
int geometry_init_api(int dim, const int64_t* ext, int64_t a0_off, int64_t a0_glob, tvs_geometry* g) {
  return geometry_init(dim, ext, a0_off, a0_glob, g);
}

// ---- algorithm drivers -----------------------------------------------------
static int jacobi_device(const tvs_stencil& st, const tvs_geometry& g, double* src, double* dst, int64_t steps,
                         const tvs_exec& ex, cudaStream_t s, int32_t* in_dst) {
  const bool fma = use_fma(st, ex);
  double* a = src;
  double* b = dst;
  int64_t done = 0;
  const bool naive = ex.algo == TVS_ALGO_NAIVE;
  while (done < steps) {
    int64_t left = steps - done;
    int rc;
    int step_now = 1;
    if (!naive && g.dim == 1 && jacobi1d_blocked_supported(st, g)) {
      int depth = ex.temporal_depth > 0 ? ex.temporal_depth : jacobi1d_default_depth();
      step_now = (int)std::min<int64_t>(left, std::min(depth, jacobi1d_max_depth()));
      rc = jacobi1d_blocked(st, g, a, b, step_now, fma, s);
    } else if (!naive && g.dim == 2 && jacobi2d_blocked_supported(st)) {
      int depth = ex.temporal_depth > 0 ? ex.temporal_depth : jacobi2d_default_depth();
      depth = std::min(depth, jacobi2d_max_depth());
      step_now = (int)std::min<int64_t>(left, depth);
      rc = jacobi2d_blocked(st, g, a, b, step_now, fma, s);
    } else if (!naive && g.dim == 3 && jacobi3d_streaming_supported(st)) {
      int depth = ex.temporal_depth > 0 ? ex.temporal_depth : jacobi3d_default_depth();
      depth = std::min(depth, jacobi3d_max_depth());
      if (depth >= 2 && left >= 2) {
        step_now = 2;
        rc = jacobi3d_blocked2(st, g, a, b, fma, s);
      } else {
        rc = jacobi3d_streaming(st, g, a, b, fma, s);
      }
    } else {
      rc = jacobi_naive_step(st, g, a, b, fma, s);
    }
    if (rc != TVS_OK) return rc;
    std::swap(a, b);
    done += step_now;
  }
  if (in_dst) *in_dst = (a == dst) ? 1 : 0;
  return TVS_OK;
}

// 2D Gauss-Seidel kernel: 0 = K6v2 lane groups (gs2d_lane.cu, default; config
// 4 26.0 ms), 1 = the round-1 K6 pipeline (gs2d_pipe.cu, 31.3 ms; kept for the
// overlapped drop-in copies) — TVS_GS2D=lane|pipe.  The reference order always
// runs on K6v2 (K6 has no reference-order form).
static int gs2d_kernel_choice() {
  static const int v = [] {
    const char* e = getenv("TVS_GS2D");
    return e && std::string(e) == "pipe" ? 1 : 0;
  }();
  return v;
}

static int gs_device(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, const tvs_exec& ex,
                     cudaStream_t s) {
  if (g.axis0_offset != 0 || g.axis0_global != g.extents[0])
    return fail(TVS_ERR_UNSUPPORTED, "Gauss-Seidel runs on a single GPU (no slab decomposition)");
  if (steps == 0) return TVS_OK;
  if (g.dim == 1 && ex.algo != TVS_ALGO_NAIVE) return gs1d_pipeline(st, g, grid, steps, s);
  // (reference order with one sweep: the pass's only sweep would overwrite
  // row d-1 in place while the next CTA still reads it as "old": wavefront)
  if (g.dim == 2 && ex.algo != TVS_ALGO_NAIVE && gs2d_lane_supported(st) &&
      (gs2d_kernel_choice() == 0 || ex.gs_order == TVS_GS_REFERENCE) && !(ex.gs_order == TVS_GS_REFERENCE && steps < 2))
    return gs2d_lane(st, g, grid, steps, ex.gs_order, s);
  if (g.dim == 2 && ex.algo != TVS_ALGO_NAIVE && ex.gs_order == TVS_GS_LEXICOGRAPHIC && gs2d_pipe_supported(st))
    return gs2d_pipeline(st, g, grid, steps, s);
  return gs_wavefront(st, g, grid, steps, ex.gs_order, s);
}

// ---- per-thread cached device context for tvs_run ---------------------------
struct RunCtx {
  int device = -1;
  int dim = 0;
  int64_t ext[3] = {0, 0, 0};
  double* buf[2] = {nullptr, nullptr};
  int nbuf = 0;
  cudaStream_t stream = nullptr;
  tvs_geometry geo{};
  std::vector<cudaStream_t> bands;  // pipelined 2D Jacobi: one stream per row band
  std::vector<cudaEvent_t> events;  // pool (timing disabled)
  // 1D drop-in pipeline captured as a CUDA graph, replayed while the call
  // (stencil, host buffers, sizes) repeats: ~100 tiny launches + copies cost
  // more to enqueue than the whole GPU run of config 1
  cudaGraphExec_t graph1 = nullptr;
  tvs_stencil graph1_st{};
  const void* graph1_in = nullptr;
  void* graph1_out = nullptr;
  int64_t graph1_key[8] = {};  // steps, band, depth, fma, buf[0], lay.offset, lay.shape[0], host generation
  ~RunCtx() { release(); }
  void release() {
    if (device >= 0) {
      int cur;
      cudaGetDevice(&cur);
      cudaSetDevice(device);
      if (graph1) cudaGraphExecDestroy(graph1), graph1 = nullptr;
      for (auto& b : buf)
        if (b) cudaFree(b), b = nullptr;
      if (stream) cudaStreamDestroy(stream), stream = nullptr;
      for (auto& b : bands) cudaStreamDestroy(b);
      for (auto& e : events) cudaEventDestroy(e);
      bands.clear();
      events.clear();
      cudaSetDevice(cur);
    }
    device = -1;
    nbuf = 0;
  }
};
static thread_local RunCtx g_run;
static thread_local ShardGroup g_group;  // tvs_run with n_gpus > 1

static int ensure_ctx(RunCtx& c, int device, int dim, const int64_t* ext, int nbuf) {
  bool same = c.device == device && c.dim == dim && c.nbuf >= nbuf;
  for (int d = 0; d < 3 && same; ++d) same = c.ext[d] == (d < dim ? ext[d] : 1);
  if (same) return TVS_OK;
  c.release();
  c.device = device;
  c.dim = dim;
  for (int d = 0; d < 3; ++d) c.ext[d] = d < dim ? ext[d] : 1;
  int rc = geometry_init(dim, ext, 0, ext[0], &c.geo);
  if (rc) return rc;
  TVS_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  for (int i = 0; i < nbuf; ++i) {
    cudaError_t e = cudaMalloc(&c.buf[i], sizeof(double) * c.geo.alloc_elems);
    if (e != cudaSuccess) {
      c.release();
      return cuda_fail(e, "cudaMalloc(grid)");
    }
  }
  c.nbuf = nbuf;
  return TVS_OK;
}

// ---- pipelined host -> device -> host path for 2D temporally blocked Jacobi --
// tvs_run on host buffers: instead of upload-all / T steps / download-all,
// rows are split into bands (512 rows).  Band b's launch k (depth D <= 12,
// so its halo lies in bands b-1..b+1) depends only on launches k-1 of bands
// b-1, b, b+1 — they write the rows it reads and read the rows it
// overwrites in the other ping-pong buffer.  Every band has its own stream;
// uploads run band by band on the copy stream, each band's launches wait on
// its neighbours' events, and each band downloads as soon as its last launch
// ends.  Measured (config 3, 16384^2 x 200, pinned host buffers): 108 ms
// single-stream -> 94 ms with 512-row bands; the dependency cone (band b's
// last launch needs bands b +- K uploaded) keeps the first download behind
// most of the upload, so full three-way overlap would need overlapped tiling
// (private per-band buffers with redundant halo rows) — not done.  Early bands therefore compute while later bands upload and download
// while the tail computes (PCIe is full duplex).  Same kernels, same
// arithmetic: bit-identical to the single-stream path.
static int band_rows_default() {
  static const int v = [] {
    const char* e = getenv("TVS_E2E_BANDS");  // 0 disables the pipelined path
    // config 3 e2e (skewed bands, 32-row segments): 128 58.1, 256 55.5, 512 56.4, 1024 59.6 ms
    return e ? atoi(e) : 256;
  }();
  return v;
}

static int copy_rows(const tvs_geometry& g, double* dev, const tvs_layout& lay, double* host, bool upload,
                     int64_t r0, int64_t r1, cudaStream_t s) {
  double* d0 = dev + g.origin + r0 * g.strides[0];
  double* h0 = host + (lay.offset + r0) * lay.shape[1] + lay.offset;
  const size_t hp = sizeof(double) * lay.shape[1], dp = sizeof(double) * g.strides[0];
  const size_t w = sizeof(double) * g.extents[1];
  if (upload) return upload_block((char*)d0, dp, 0, (const char*)h0, hp, 0, w, r1 - r0, 1, s);
  TVS_CUDA(cudaMemcpy2DAsync(h0, hp, d0, dp, w, r1 - r0, cudaMemcpyDeviceToHost, s));
  return TVS_OK;
}

// Drop-in path for 2D Jacobi with host Grids: uploads, temporally blocked
// passes and downloads overlap over row bands.  Band b of pass k covers rows
// [b*band - S_k, (b+1)*band - S_k) (clipped), S_k = levels of passes < k:
// every pass shifts the bands up by its own depth, so pass k of band b reads
// only rows that pass k-1 of bands b and b-1 wrote (a parallelogram in
// (rows, time)).  Band b therefore runs all its passes as soon as band b+1's
// first rows are uploaded and band b-1 has kept pace, and its final rows go
// back to the host while later bands are still uploading: H2D, compute and
// D2H all overlap (PCIe is full duplex).  One stream per band; pass k of band
// b waits on pass k-1 of band b-1 (same-stream order covers band b itself).
// WAR is safe: the only later writer of rows that pass k of band b reads is
// pass k+2 of band b+1, which depends on pass k+1 of band b.
static int jacobi2d_pipelined(const tvs_stencil& st, const tvs_layout& lay, const double* in, double* out,
                              int64_t steps, const tvs_exec& ex, RunCtx& c, int64_t band) {
  const tvs_geometry& g = c.geo;
  const int64_t rows = g.extents[0];
  int depth = ex.temporal_depth > 0 ? ex.temporal_depth : jacobi2d_default_depth();
  depth = std::min(depth, jacobi2d_max_depth());
  const int K = (int)((steps + depth - 1) / depth);
  const bool fma = use_fma(st, ex);
  // shorter row segments than the device-resident default: a band's pass is
  // then a shorter dependent chain, which is what the pipeline's tail waits on
  static const int seg = [] {
    const char* e = getenv("TVS_E2E_SEG");  // config 3 e2e at 256-row bands: 32 55.5, 64 60.1, 256 64.0 ms
    return e ? atoi(e) : 32;
  }();
  std::vector<int> dk(K);
  std::vector<int64_t> S(K + 1, 0);
  {
    int64_t left = steps;
    for (int k = 0; k < K; ++k) {
      dk[k] = (int)std::min<int64_t>(left, depth);
      left -= dk[k];
      S[k + 1] = S[k] + dk[k];
    }
  }
  if (band < 2 * depth) return fail(TVS_ERR_INVALID, "pipelined band shorter than two temporal blocks");
  // enough bands that the last one still reaches the top row after every shift
  const int nb = (int)((rows + S[K] + band - 1) / band);
  while ((int)c.bands.size() < nb) {
    cudaStream_t t;
    TVS_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    c.bands.push_back(t);
  }
  const size_t nev = (size_t)nb * (K + 1);
  while (c.events.size() < nev) {
    cudaEvent_t e;
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.events.push_back(e);
  }
  auto up = [&](int b) { return c.events[b]; };                               // upload of rows [b*band, (b+1)*band)
  auto done = [&](int b, int k) { return c.events[(size_t)nb * (k + 1) + b]; };  // pass k of band b ended
  auto lo_of = [&](int b, int k) { return std::max<int64_t>(0, (int64_t)b * band - S[k]); };
  auto hi_of = [&](int b, int k) { return std::min<int64_t>(rows, (int64_t)(b + 1) * band - S[k]); };
  cudaStream_t cs = c.stream;
  int rc;
  static const bool trace = getenv("TVS_E2E_TRACE") != nullptr;
  cudaEvent_t tr[4] = {};
  std::vector<cudaEvent_t> tup, tdn;  // per-band upload / download completion (trace only)
  std::vector<double> thost;            // host clock when band b's work was enqueued (trace only)
  const auto h0 = std::chrono::steady_clock::now();
  auto host_ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(); };
  if (trace) {
    for (auto& e : tr) cudaEventCreate(&e);
    tup.resize((rows + band - 1) / band);
    tdn.resize(nb);
    for (auto& e : tup) cudaEventCreate(&e);
    for (auto& e : tdn) cudaEventCreate(&e);
    cudaEventRecord(tr[0], cs);
  }
  if ((rc = fill_halo(g, c.buf[0], st.boundary, cs))) return rc;
  if ((rc = fill_halo(g, c.buf[1], st.boundary, cs))) return rc;
  const int nup = (int)((rows + band - 1) / band);
  double* result = c.buf[K & 1];
  int uploaded = 0;
  for (int b = 0; b < nb; ++b) {
    // uploads stay one band ahead of the band whose passes are enqueued next
    for (; uploaded < nup && uploaded <= b + 1; ++uploaded) {
      const int64_t r0 = (int64_t)uploaded * band, r1 = std::min(rows, (int64_t)(uploaded + 1) * band);
      if ((rc = copy_rows(g, c.buf[0], lay, const_cast<double*>(in), true, r0, r1, cs))) return rc;
      TVS_CUDA(cudaEventRecord(up(uploaded), cs));
      if (trace && uploaded == nup - 1) cudaEventRecord(tr[1], cs);
      if (trace) cudaEventRecord(tup[uploaded], cs);
    }
    cudaStream_t sb = c.bands[b];
    // pass 0 reads rows [b*band - d, (b+1)*band + d): uploads b-1 .. b+1
    for (int u = b - 1; u <= b + 1; ++u)
      if (u >= 0 && u < nup) TVS_CUDA(cudaStreamWaitEvent(sb, up(u), 0));
    for (int k = 0; k < K; ++k) {
      if (k > 0 && b > 0) TVS_CUDA(cudaStreamWaitEvent(sb, done(b - 1, k - 1), 0));
      const int64_t lo = lo_of(b, k), hi = hi_of(b, k);
      if (hi > lo && (rc = jacobi2d_blocked(st, g, c.buf[k & 1], c.buf[(k + 1) & 1], dk[k], fma, sb, lo, hi, seg)))
        return rc;
      TVS_CUDA(cudaEventRecord(done(b, k), sb));
    }
    // the final rows of band b also come from band b-1's last pass (the
    // bands shift up by each pass's levels): wait for it before reading
    if (b > 0) TVS_CUDA(cudaStreamWaitEvent(sb, done(b - 1, K - 1), 0));
    const int64_t lo = lo_of(b, K), hi = hi_of(b, K);
    if (hi > lo && (rc = copy_rows(g, result, lay, out, false, lo, hi, sb))) return rc;
    if (trace && b == 0) cudaEventRecord(tr[2], sb);
    if (trace) cudaEventRecord(tdn[b], sb), thost.push_back(host_ms());
  }
  for (int b = 0; b < nb; ++b) TVS_CUDA(cudaStreamSynchronize(c.bands[b]));
  const double t_sync = host_ms();
  if (trace) {
    cudaEventRecord(tr[3], cs);
    cudaStreamSynchronize(cs);
    float t[4] = {};
    for (int i = 1; i < 4; ++i) cudaEventElapsedTime(&t[i], tr[0], tr[i]);
    fprintf(stderr, "[e2e] bands %d x %lld rows, K %d: uploads done %.2f ms, band0 final D2H %.2f ms, end %.2f ms\n",
            nb, (long long)band, K, t[1], t[2], t[3]);
    for (size_t b = 0; b < tdn.size(); b += 4) {
      float u = 0, d = 0;
      if (b < tup.size()) cudaEventElapsedTime(&u, tr[0], tup[b]);
      cudaEventElapsedTime(&d, tr[0], tdn[b]);
      fprintf(stderr, "  band %3zu: up %7.2f  down %7.2f ms  (host enqueued %7.2f)\n", b, u, d, thost[b]);
    }
    fprintf(stderr, "  host: enqueue done %.2f ms, synchronized %.2f ms\n", thost.back(), t_sync);
    for (auto& e : tr) cudaEventDestroy(e);
    for (auto& e : tup) cudaEventDestroy(e);
    for (auto& e : tdn) cudaEventDestroy(e);
  }
  return TVS_OK;
}

// 1D Jacobi drop-in path: the same skewed pipeline over position bands
// (64 levels per pass in registers, K2), contiguous copies.
static int jacobi1d_pipelined(const tvs_stencil& st, const tvs_layout& lay, const double* in, double* out,
                              int64_t steps, const tvs_exec& ex, RunCtx& c, int64_t band) {
  const tvs_geometry& g = c.geo;
  const int64_t n = g.extents[0];
  int depth = ex.temporal_depth > 0 ? ex.temporal_depth : jacobi1d_default_depth();
  depth = std::max(1, std::min(depth, jacobi1d_max_depth()));
  const int K = (int)((steps + depth - 1) / depth);
  const bool fma = use_fma(st, ex);
  std::vector<int> dk(K);
  std::vector<int64_t> S(K + 1, 0);
  {
    int64_t left = steps;
    for (int k = 0; k < K; ++k) {
      dk[k] = (int)std::min<int64_t>(left, depth);
      left -= dk[k];
      S[k + 1] = S[k] + dk[k];
    }
  }
  if (band < 4 * depth) return fail(TVS_ERR_INVALID, "pipelined band shorter than four temporal blocks");
  auto pinned = [](const void* ptr) {
    cudaPointerAttributes a{};
    const bool ok = cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  // only page-locked host buffers are captured (pageable copies cannot be);
  // checked on every call, and the key carries the host-memory generation
  // (bumped by tvs_host_free / tvs_host_unregister), so a replay never DMAs
  // from memory that was unpinned or reused at the same address
  const bool use_graph = pinned(in) && pinned(out);
  const int64_t key[8] = {steps, band, depth, fma ? 1 : 0, (int64_t)(uintptr_t)c.buf[0], lay.offset, lay.shape[0],
                          (int64_t)g_host_generation.load()};
  static_assert(sizeof(key) == sizeof(c.graph1_key), "graph key size");
  if (use_graph && c.graph1 && c.graph1_in == in && c.graph1_out == out &&
      std::memcmp(key, c.graph1_key, sizeof(key)) == 0 && same_stencil(st, c.graph1_st)) {
    TVS_CUDA(cudaGraphLaunch(c.graph1, c.stream));
    TVS_CUDA(cudaStreamSynchronize(c.stream));
    return TVS_OK;
  }
  if (c.graph1) {
    cudaGraphExecDestroy(c.graph1);
    c.graph1 = nullptr;
  }
  const int nb = (int)((n + S[K] + band - 1) / band);
  while ((int)c.bands.size() < nb) {
    cudaStream_t t;
    TVS_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    c.bands.push_back(t);
  }
  const size_t nev = (size_t)nb * (K + 1);
  while (c.events.size() < nev) {
    cudaEvent_t e;
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.events.push_back(e);
  }
  auto up = [&](int b) { return c.events[b]; };
  auto done = [&](int b, int k) { return c.events[(size_t)nb * (k + 1) + b]; };
  auto lo_of = [&](int b, int k) { return std::max<int64_t>(0, (int64_t)b * band - S[k]); };
  auto hi_of = [&](int b, int k) { return std::min<int64_t>(n, (int64_t)(b + 1) * band - S[k]); };
  auto copy = [&](double* dev, double* host, bool upload, int64_t p0, int64_t p1, cudaStream_t s) -> cudaError_t {
    double* d = dev + g.origin + p0;
    double* h = host + lay.offset + p0;
    const size_t bytes = sizeof(double) * (p1 - p0);
    if (upload)  // page-locked (captured graph) or staged (pageable)
      return upload_block((char*)d, bytes, 0, (const char*)h, bytes, 0, bytes, 1, 1, s) == TVS_OK ? cudaSuccess
                                                                                                 : cudaErrorUnknown;
    return cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s);
  };
  cudaStream_t cs = c.stream;
  int rc;
  // capture the whole pipeline (fork from cs through the upload events,
  // join back below), then replay it
  while (c.events.size() < nev + nb) {
    cudaEvent_t e;
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.events.push_back(e);
  }
  if (use_graph) TVS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  auto abort_capture = [&](int code) {
    if (!use_graph) return code;
    cudaGraph_t gr = nullptr;
    cudaStreamEndCapture(cs, &gr);
    if (gr) cudaGraphDestroy(gr);
    cudaGetLastError();
    return code;
  };
  auto enqueue = [&]() -> int {
    if ((rc = fill_halo(g, c.buf[0], st.boundary, cs))) return rc;
    if ((rc = fill_halo(g, c.buf[1], st.boundary, cs))) return rc;
    const int nup = (int)((n + band - 1) / band);
    double* result = c.buf[K & 1];
    int uploaded = 0;
    for (int b = 0; b < nb; ++b) {
      for (; uploaded < nup && uploaded <= b + 1; ++uploaded) {
        TVS_CUDA(copy(c.buf[0], const_cast<double*>(in), true, (int64_t)uploaded * band,
                      std::min(n, (int64_t)(uploaded + 1) * band), cs));
        TVS_CUDA(cudaEventRecord(up(uploaded), cs));
      }
      cudaStream_t sb = c.bands[b];
      for (int u = b - 1; u <= b + 1; ++u)
        if (u >= 0 && u < nup) TVS_CUDA(cudaStreamWaitEvent(sb, up(u), 0));
      for (int k = 0; k < K; ++k) {
        if (k > 0 && b > 0) TVS_CUDA(cudaStreamWaitEvent(sb, done(b - 1, k - 1), 0));
        const int64_t lo = lo_of(b, k), hi = hi_of(b, k);
        if (hi > lo && (rc = jacobi1d_blocked(st, g, c.buf[k & 1], c.buf[(k + 1) & 1], dk[k], fma, sb, lo, hi)))
          return rc;
        TVS_CUDA(cudaEventRecord(done(b, k), sb));
      }
      // the final rows of band b also come from band b-1's last pass (the
    // bands shift up by each pass's levels): wait for it before reading
    if (b > 0) TVS_CUDA(cudaStreamWaitEvent(sb, done(b - 1, K - 1), 0));
    const int64_t lo = lo_of(b, K), hi = hi_of(b, K);
      if (hi > lo) TVS_CUDA(copy(result, out, false, lo, hi, sb));
    }
    for (int b = 0; b < nb; ++b) {  // join every band stream back into cs
      TVS_CUDA(cudaEventRecord(c.events[nev + b], c.bands[b]));
      TVS_CUDA(cudaStreamWaitEvent(cs, c.events[nev + b], 0));
    }
    return TVS_OK;
  };
  if ((rc = enqueue())) return abort_capture(rc);
  if (!use_graph) {
    TVS_CUDA(cudaStreamSynchronize(cs));
    return TVS_OK;
  }
  cudaGraph_t graph = nullptr;
  TVS_CUDA(cudaStreamEndCapture(cs, &graph));
  const cudaError_t ie = cudaGraphInstantiate(&c.graph1, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    c.graph1 = nullptr;
    return cuda_fail(ie, "cudaGraphInstantiate");
  }
  c.graph1_st = st;
  c.graph1_in = in;
  c.graph1_out = out;
  std::memcpy(c.graph1_key, key, sizeof(key));
  TVS_CUDA(cudaGraphLaunch(c.graph1, cs));
  TVS_CUDA(cudaStreamSynchronize(cs));
  return TVS_OK;
}

// 3D Jacobi drop-in path: the same skewed pipeline over axis-0 slabs (planes
// [b*slab - S_k, (b+1)*slab - S_k) in pass k, S_k = levels of passes < k),
// two levels per pass (K4b; a single-step last pass when T is odd).  Every
// slab-pass reads only planes that pass k-1 of slabs b and b-1 wrote.
static int copy_planes(const tvs_geometry& g, double* dev, const tvs_layout& lay, double* host, bool upload,
                       int64_t p0, int64_t p1, cudaStream_t s) {
  if (upload) {
    const size_t hr = sizeof(double) * lay.shape[2], hz = hr * lay.shape[1];
    const double* h0 = host + ((lay.offset + p0) * lay.shape[1] + lay.offset) * lay.shape[2] + lay.offset;
    return upload_block((char*)(dev + g.origin + p0 * g.strides[0]), sizeof(double) * g.strides[1],
                        sizeof(double) * g.strides[0], (const char*)h0, hr, hz, sizeof(double) * g.extents[2],
                        g.extents[1], p1 - p0, s);
  }
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  const cudaPitchedPtr hptr = make_cudaPitchedPtr(host, sizeof(double) * lay.shape[2], lay.shape[2], lay.shape[1]);
  const cudaPitchedPtr dptr = make_cudaPitchedPtr(dev, sizeof(double) * g.strides[1], g.strides[1],
                                                  g.strides[0] / g.strides[1]);
  const cudaPos hpos = make_cudaPos(sizeof(double) * lay.offset, lay.offset, lay.offset + p0);
  const cudaPos dpos = make_cudaPos(sizeof(double) * kPadLast, 1, 1 + p0);
  p.extent = make_cudaExtent(sizeof(double) * g.extents[2], g.extents[1], p1 - p0);
  if (upload) {
    p.srcPtr = hptr; p.srcPos = hpos; p.dstPtr = dptr; p.dstPos = dpos; p.kind = cudaMemcpyHostToDevice;
  } else {
    p.srcPtr = dptr; p.srcPos = dpos; p.dstPtr = hptr; p.dstPos = hpos; p.kind = cudaMemcpyDeviceToHost;
  }
  TVS_CUDA(cudaMemcpy3DAsync(&p, s));
  return TVS_OK;
}

static int slab_planes_default() {
  static const int v = [] {
    const char* e = getenv("TVS_E2E_SLAB");  // 0 disables the pipelined 3D path
    return e ? atoi(e) : 32;
  }();
  return v;
}

static int jacobi3d_pipelined(const tvs_stencil& st, const tvs_layout& lay, const double* in, double* out,
                              int64_t steps, const tvs_exec& ex, RunCtx& c, int64_t slab) {
  const tvs_geometry& g = c.geo;
  const int64_t planes = g.extents[0];
  int depth = ex.temporal_depth > 0 ? ex.temporal_depth : jacobi3d_default_depth();
  depth = std::max(1, std::min(depth, jacobi3d_max_depth()));
  const int K = (int)((steps + depth - 1) / depth);
  const bool fma = use_fma(st, ex);
  std::vector<int> dk(K);
  std::vector<int64_t> S(K + 1, 0);
  {
    int64_t left = steps;
    for (int k = 0; k < K; ++k) {
      dk[k] = (int)std::min<int64_t>(left, depth);
      left -= dk[k];
      S[k + 1] = S[k] + dk[k];
    }
  }
  if (slab < 4 * depth) return fail(TVS_ERR_INVALID, "pipelined slab thinner than four temporal blocks");
  const int nb = (int)((planes + S[K] + slab - 1) / slab);
  while ((int)c.bands.size() < nb) {
    cudaStream_t t;
    TVS_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    c.bands.push_back(t);
  }
  const size_t nev = (size_t)nb * (K + 1);
  while (c.events.size() < nev) {
    cudaEvent_t e;
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.events.push_back(e);
  }
  auto up = [&](int b) { return c.events[b]; };
  auto done = [&](int b, int k) { return c.events[(size_t)nb * (k + 1) + b]; };
  auto lo_of = [&](int b, int k) { return std::max<int64_t>(0, (int64_t)b * slab - S[k]); };
  auto hi_of = [&](int b, int k) { return std::min<int64_t>(planes, (int64_t)(b + 1) * slab - S[k]); };
  cudaStream_t cs = c.stream;
  int rc;
  if ((rc = fill_halo(g, c.buf[0], st.boundary, cs))) return rc;
  if ((rc = fill_halo(g, c.buf[1], st.boundary, cs))) return rc;
  const int nup = (int)((planes + slab - 1) / slab);
  double* result = c.buf[K & 1];
  int uploaded = 0;
  for (int b = 0; b < nb; ++b) {
    for (; uploaded < nup && uploaded <= b + 1; ++uploaded) {
      if ((rc = copy_planes(g, c.buf[0], lay, const_cast<double*>(in), true, (int64_t)uploaded * slab,
                            std::min(planes, (int64_t)(uploaded + 1) * slab), cs)))
        return rc;
      TVS_CUDA(cudaEventRecord(up(uploaded), cs));
    }
    cudaStream_t sb = c.bands[b];
    for (int u = b - 1; u <= b + 1; ++u)
      if (u >= 0 && u < nup) TVS_CUDA(cudaStreamWaitEvent(sb, up(u), 0));
    for (int k = 0; k < K; ++k) {
      if (k > 0 && b > 0) TVS_CUDA(cudaStreamWaitEvent(sb, done(b - 1, k - 1), 0));
      const int64_t lo = lo_of(b, k), hi = hi_of(b, k);
      if (hi > lo) {
        rc = dk[k] == 2 ? jacobi3d_blocked2(st, g, c.buf[k & 1], c.buf[(k + 1) & 1], fma, sb, lo, hi, (int)slab)
                        : jacobi3d_streaming(st, g, c.buf[k & 1], c.buf[(k + 1) & 1], fma, sb, lo, hi, (int)slab);
        if (rc) return rc;
      }
      TVS_CUDA(cudaEventRecord(done(b, k), sb));
    }
    // the final rows of band b also come from band b-1's last pass (the
    // bands shift up by each pass's levels): wait for it before reading
    if (b > 0) TVS_CUDA(cudaStreamWaitEvent(sb, done(b - 1, K - 1), 0));
    const int64_t lo = lo_of(b, K), hi = hi_of(b, K);
    if (hi > lo && (rc = copy_planes(g, result, lay, out, false, lo, hi, sb))) return rc;
  }
  for (int b = 0; b < nb; ++b) TVS_CUDA(cudaStreamSynchronize(c.bands[b]));
  return TVS_OK;
}

// 2D Gauss-Seidel drop-in path (lexicographic pipeline, one pass of <= 128
// sweeps): row bands are uploaded while the kernel runs — its loader warps
// wait on a rows-uploaded counter the copy stream advances with
// cuStreamWriteValue32 — and downloaded while it runs: the kernel publishes
// finished blocks in ticket order, and the download stream waits with
// cuStreamWaitValue32 for the block that writes a band's last final row.
// Every upload is enqueued before the kernel, so the kernel can never wait on
// a copy queued behind it.
typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, unsigned, unsigned);
static bool stream_value_fns(StreamValueFn* wait, StreamValueFn* write) {
  static StreamValueFn w = nullptr, r = nullptr;
  static const bool ok = [] {
    void* f1 = nullptr;
    void* f2 = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    // the v2 entry points (CUDA >= 12: stream memory operations need no opt-in)
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f1, 12000, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f2, 12000, cudaEnableDefault, &q2) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !f1 || !f2) {
      cudaGetLastError();
      return false;
    }
    w = reinterpret_cast<StreamValueFn>(f1);
    r = reinterpret_cast<StreamValueFn>(f2);
    return true;
  }();
  *wait = w;
  *write = r;
  return ok;
}

bool stream_value_fns_api(StreamValueFn* wait, StreamValueFn* write) { return stream_value_fns(wait, write); }

static int gs2d_pipelined(const tvs_stencil& st, const tvs_layout& lay, const double* in, double* out,
                          int64_t steps, RunCtx& c, int64_t band, int order, bool lane) {
  StreamValueFn wait_value, write_value;
  if (!stream_value_fns(&wait_value, &write_value)) return TVS_ERR_UNSUPPORTED;
  const tvs_geometry& g = c.geo;
  const int64_t rows = g.extents[0];
  const int nbands = (int)((rows + band - 1) / band);
  unsigned* ctr = static_cast<unsigned*>(scratch(128, 3));  // [0] rows uploaded, [16] blocks done (64 B apart)
  if (!ctr) return fail(TVS_ERR_CUDA, "gs2d_pipelined: scratch");
  while ((int)c.bands.size() < 2) {
    cudaStream_t t;
    TVS_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    c.bands.push_back(t);
  }
  if (c.events.empty()) {
    cudaEvent_t e;
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.events.push_back(e);
  }
  cudaStream_t cs = c.stream, ks = c.bands[0], ds = c.bands[1];
  int rc;
  TVS_CUDA(cudaMemsetAsync(ctr, 0, 128, cs));
  if ((rc = fill_halo(g, c.buf[0], st.boundary, cs))) return rc;
  TVS_CUDA(cudaEventRecord(c.events[0], cs));
  const unsigned long long rows_ready = reinterpret_cast<unsigned long long>(ctr);
  const unsigned long long blocks_done = reinterpret_cast<unsigned long long>(ctr + 16);
  for (int u = 0; u < nbands; ++u) {
    const int64_t r1 = std::min(rows, (int64_t)(u + 1) * band);
    if ((rc = copy_rows(g, c.buf[0], lay, const_cast<double*>(in), true, (int64_t)u * band, r1, cs))) return rc;
    const int wrc = write_value(cs, rows_ready, (unsigned)r1, 0);
    if (wrc != 0) return fail(TVS_ERR_CUDA, "cuStreamWriteValue32 failed (CUresult " + std::to_string(wrc) + ")");
  }
  TVS_CUDA(cudaStreamWaitEvent(ks, c.events[0], 0));
  TVS_CUDA(cudaStreamWaitEvent(ds, c.events[0], 0));  // counters reset before any wait reads them
  if ((rc = lane ? gs2d_lane(st, g, c.buf[0], steps, order, ks, ctr, ctr + 16)
                 : gs2d_pipeline(st, g, c.buf[0], steps, ks, ctr, ctr + 16)))
    return rc;
  // row r's final value is written by the block holding group r + steps - 1
  // (block geometry from the kernel's own file)
  const int64_t nblocks = lane ? gs2d_lane_ctas(rows, steps, order) : gs2d_pipe_blocks(rows);
  for (int u = 0; u < nbands; ++u) {
    const int64_t r0 = (int64_t)u * band, r1 = std::min(rows, r0 + band);
    const int64_t need = std::min<int64_t>(
        nblocks, lane ? gs2d_lane_ctas_for_row(r1 - 1, steps, order) : gs2d_pipe_blocks_for_row(r1 - 1, steps));
    const int wrc = wait_value(ds, blocks_done, (unsigned)need, 0 /* CU_STREAM_WAIT_VALUE_GEQ */);
    if (wrc != 0) return fail(TVS_ERR_CUDA, "cuStreamWaitValue32 failed (CUresult " + std::to_string(wrc) + ")");
    if ((rc = copy_rows(g, c.buf[0], lay, out, false, r0, r1, ds))) return rc;
  }
  TVS_CUDA(cudaStreamSynchronize(ds));
  TVS_CUDA(cudaStreamSynchronize(ks));
  TVS_CUDA(cudaStreamSynchronize(cs));
  return TVS_OK;
}

}  // namespace tvs

using namespace tvs;

struct tvs_plan {
  tvs_stencil st;
  tvs_exec ex;
  tvs_geometry geo;
  ShardGroup* group = nullptr;  // n_gpus > 1: sharded plan (shard.cu)
  double* buf[2] = {nullptr, nullptr};
  int cur = 0;  // which buffer holds the current field
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t last_launches = 0;
};

extern "C" {

const char* tvs_last_error(void) { return g_err.c_str(); }
const char* tvs_version(void) { return "tvstencil-b200 0.1.0 (sm_100a)"; }

int64_t tvs_launch_counter(void) {
  int64_t n = g_launches;
  g_launches = 0;
  return n;
}

int tvs_release_thread_cache(void) {
  // the calling thread's tvs_run buffers, streams, events and captured graph
  // plus its kernel scratch (reference ThreadPool workers: tiling.py:363-367)
  g_run.release();
  g_group.release();
  release_staging();
  ++g_scratch_gen;
  for (auto& sl : g_scratch) {
    if (!sl.ptr) continue;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(sl.device);
    cudaFree(sl.ptr);
    cudaSetDevice(cur);
    sl = ScratchSlot{};
  }
  release_integer_cache();
  return TVS_OK;
}

int tvs_device_count(int32_t* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) c = 0;
  if (n) *n = c;
  return TVS_OK;
}

uint64_t tvs_fnv1a64(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

int tvs_host_register(void* ptr, size_t bytes) {
  TVS_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  return TVS_OK;
}
int tvs_host_unregister(void* ptr) {
  g_host_generation.fetch_add(1);
  TVS_CUDA(cudaHostUnregister(ptr));
  return TVS_OK;
}
int tvs_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(TVS_ERR_INVALID, "null argument");
  *ptr = nullptr;
  TVS_CUDA(cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable));
  return TVS_OK;
}
int tvs_host_free(void* ptr) {
  g_host_generation.fetch_add(1);
  TVS_CUDA(cudaFreeHost(ptr));
  return TVS_OK;
}

int tvs_geometry_init(int32_t dim, const int64_t extents[3], int64_t axis0_offset, int64_t axis0_global,
                      tvs_geometry* g) {
  if (!g || !extents) return fail(TVS_ERR_INVALID, "null argument");
  return geometry_init(dim, extents, axis0_offset, axis0_global, g);
}

int tvs_fill_halo(const tvs_geometry* g, double* dev, double value, void* stream) {
  if (!g || !dev) return fail(TVS_ERR_INVALID, "null argument");
  return fill_halo(*g, dev, value, (cudaStream_t)stream);
}

int tvs_upload(const tvs_geometry* g, double* dev, const tvs_layout* lay, const double* host, void* stream) {
  if (!g || !dev || !lay || !host) return fail(TVS_ERR_INVALID, "null argument");
  if (int rc = validate_layout(lay, g->dim)) return rc;
  return copy_interior(*g, dev, *lay, const_cast<double*>(host), true, (cudaStream_t)stream);
}

int tvs_download(const tvs_geometry* g, const double* dev, const tvs_layout* lay, double* host, void* stream) {
  if (!g || !dev || !lay || !host) return fail(TVS_ERR_INVALID, "null argument");
  if (int rc = validate_layout(lay, g->dim)) return rc;
  return copy_interior(*g, const_cast<double*>(dev), *lay, host, false, (cudaStream_t)stream);
}

int tvs_jacobi_device(const tvs_stencil* st, const tvs_geometry* g, double* src, double* dst, int64_t steps,
                      const tvs_exec* ex, void* stream, int32_t* result_in_dst) {
  int rc = validate(st);
  if (rc) return rc;
  if ((rc = validate_exec(ex))) return rc;
  if (!g || !src || !dst) return fail(TVS_ERR_INVALID, "null argument");
  if (st->kind != TVS_JACOBI) return fail(TVS_ERR_INVALID, "tvs_jacobi_device needs a Jacobi stencil");
  if (st->dim != g->dim) return fail(TVS_ERR_SIZE, "stencil/geometry dimension mismatch");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  return jacobi_device(*st, *g, src, dst, steps, *ex, (cudaStream_t)stream, result_in_dst);
}

int tvs_jacobi_device_rows(const tvs_stencil* st, const tvs_geometry* g, const double* src, double* dst,
                           int64_t steps, const tvs_exec* ex, void* stream, int64_t row_lo, int64_t row_hi) {
  int rc = validate(st);
  if (rc) return rc;
  if ((rc = validate_exec(ex))) return rc;
  if (!g || !src || !dst) return fail(TVS_ERR_INVALID, "null argument");
  if (st->kind != TVS_JACOBI) return fail(TVS_ERR_INVALID, "tvs_jacobi_device_rows needs a Jacobi stencil");
  if (st->dim != g->dim) return fail(TVS_ERR_SIZE, "stencil/geometry dimension mismatch");
  if (steps < 1) return fail(TVS_ERR_INVALID, "steps must be >= 1");
  if (row_lo < 0 || row_hi > g->extents[0] || row_lo >= row_hi) return fail(TVS_ERR_INVALID, "row range");
  const bool fma = use_fma(*st, *ex);
  cudaStream_t s = (cudaStream_t)stream;
  if (g->dim == 2 && jacobi2d_blocked_supported(*st) && steps <= jacobi2d_max_depth())
    return jacobi2d_blocked(*st, *g, src, dst, (int)steps, fma, s, row_lo, row_hi);
  if (g->dim == 3 && jacobi3d_streaming_supported(*st) && steps <= 2)
    return steps == 2 ? jacobi3d_blocked2(*st, *g, src, dst, fma, s, row_lo, row_hi)
                      : jacobi3d_streaming(*st, *g, src, dst, fma, s, row_lo, row_hi);
  return fail(TVS_ERR_UNSUPPORTED, "tvs_jacobi_device_rows: one blocked 2D/3D launch of at most its depth");
}

int tvs_gauss_seidel_device(const tvs_stencil* st, const tvs_geometry* g, double* grid, int64_t steps,
                            const tvs_exec* ex, void* stream) {
  int rc = validate(st);
  if (rc) return rc;
  if ((rc = validate_exec(ex))) return rc;
  if (!g || !grid) return fail(TVS_ERR_INVALID, "null argument");
  if (st->kind != TVS_GAUSS_SEIDEL) return fail(TVS_ERR_INVALID, "needs a Gauss-Seidel stencil");
  if (st->dim != g->dim) return fail(TVS_ERR_SIZE, "stencil/geometry dimension mismatch");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  return gs_device(*st, *g, grid, steps, *ex, (cudaStream_t)stream);
}

int tvs_run(const tvs_stencil* st, const tvs_layout* lay, const double* in, double* out, int64_t steps,
            const tvs_exec* ex) {
  int rc = validate(st);
  if (rc) return rc;
  if ((rc = validate_exec(ex))) return rc;
  if (!lay || !in || !out) return fail(TVS_ERR_INVALID, "null argument");
  if ((rc = validate_layout(lay, st->dim))) return rc;
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  if ((rc = set_device(ex->device))) return rc;
  if (wants_shards(*st, *ex) && steps > 0) {
    // axis-0 slabs on n_gpus devices, each uploading / downloading its own
    // rows over its own PCIe link (shard.cu)
    if (!g_group.matches(*st, st->dim, lay->extents, *ex) &&
        (rc = g_group.create(*st, st->dim, lay->extents, *ex)))
      return rc;
    if ((rc = g_group.upload(*lay, in))) return rc;
    if ((rc = g_group.run(steps))) return rc;
    if ((rc = g_group.download(*lay, out))) return rc;
    return g_group.synchronize();
  }
  const bool gs = st->kind == TVS_GAUSS_SEIDEL;
  if ((rc = ensure_ctx(g_run, ex->device, st->dim, lay->extents, gs ? 1 : 2))) return rc;
  RunCtx& c = g_run;
  cudaStream_t s = c.stream;
  if (!gs) {
    const int64_t band = band_rows_default();
    if (band > 0 && st->dim == 2 && steps > 0 && ex->algo != TVS_ALGO_NAIVE && jacobi2d_blocked_supported(*st) &&
        c.geo.extents[0] >= 4 * band)
      return jacobi2d_pipelined(*st, *lay, in, out, steps, *ex, c, band);
    static const int64_t band1 = [] {
      const char* e = getenv("TVS_E2E_BAND1");  // 0 disables the pipelined 1D path
      return e ? atoll(e) : 131072ll;  // config 1 e2e (graph replay): 65536 0.747, 131072 0.727, 262144 0.759 ms (plain 0.86)
    }();
    if (band1 > 0 && st->dim == 1 && steps > 0 && ex->algo != TVS_ALGO_NAIVE && jacobi1d_blocked_supported(*st, c.geo) &&
        c.geo.extents[0] >= 4 * band1)
      return jacobi1d_pipelined(*st, *lay, in, out, steps, *ex, c, band1);
    const int64_t slab = slab_planes_default();
    if (slab > 0 && st->dim == 3 && steps > 0 && ex->algo != TVS_ALGO_NAIVE && jacobi3d_streaming_supported(*st) &&
        c.geo.extents[0] >= 4 * slab)
      return jacobi3d_pipelined(*st, *lay, in, out, steps, *ex, c, slab);
  }
  if (gs) {
    const int64_t band = band_rows_default();
    // lane kernel (K6v2, either order) or the K6 pipeline (lexicographic):
    // one pass, row bands uploaded / downloaded while it runs
    const bool lane = gs2d_kernel_choice() == 0 && gs2d_lane_supported(*st) &&
                      !(ex->gs_order == TVS_GS_REFERENCE && steps < 2);
    const bool pipe = !lane && ex->gs_order == TVS_GS_LEXICOGRAPHIC && gs2d_pipe_supported(*st);
    if ((lane || pipe) && band > 0 && st->dim == 2 && steps > 0 &&
        steps <= (lane ? gs2d_lane_max_sweeps() : gs2d_pipe_max_sweeps()) && ex->algo != TVS_ALGO_NAIVE &&
        c.geo.extents[0] >= 4 * band) {
      rc = gs2d_pipelined(*st, *lay, in, out, steps, c, band, ex->gs_order, lane);
      if (rc != TVS_ERR_UNSUPPORTED) return rc;  // no stream memory operations: plain path below
    }
  }
  if ((rc = fill_halo(c.geo, c.buf[0], st->boundary, s))) return rc;
  if ((rc = copy_interior(c.geo, c.buf[0], *lay, const_cast<double*>(in), true, s))) return rc;
  double* result = c.buf[0];
  if (gs) {
    if ((rc = gs_device(*st, c.geo, c.buf[0], steps, *ex, s))) return rc;
  } else {
    if ((rc = fill_halo(c.geo, c.buf[1], st->boundary, s))) return rc;
    int32_t in_dst = 0;
    if ((rc = jacobi_device(*st, c.geo, c.buf[0], c.buf[1], steps, *ex, s, &in_dst))) return rc;
    result = in_dst ? c.buf[1] : c.buf[0];
  }
  if ((rc = copy_interior(c.geo, result, *lay, out, false, s))) return rc;
  TVS_CUDA(cudaStreamSynchronize(s));
  return TVS_OK;
}

static int problem_to(const tvs_problem* p, int kind, tvs_stencil* st, tvs_layout* lay) {
  if (!p) return fail(TVS_ERR_INVALID, "null problem");
  if (p->ntaps < 1 || p->ntaps > TVS_MAX_TAPS) return fail(TVS_ERR_INVALID, "ntaps must be 1..27");
  std::memset(st, 0, sizeof(*st));
  std::memset(lay, 0, sizeof(*lay));
  st->dim = p->dim;
  st->kind = kind;
  st->ntaps = p->ntaps;
  st->radius = p->radius;
  st->boundary = p->boundary;
  for (int k = 0; k < p->ntaps; ++k) {
    for (int d = 0; d < 3; ++d) st->offsets[k][d] = p->offsets[k][d];
    st->coeffs[k] = p->coeffs[k];
  }
  lay->dim = p->dim;
  for (int d = 0; d < 3; ++d) {
    lay->extents[d] = d < p->dim ? p->extents[d] : 1;
    lay->shape[d] = d < p->dim ? p->padded_shape[d] : 1;
  }
  lay->offset = p->offset;
  return TVS_OK;
}

int tvs_jacobi(const tvs_problem* p, const double* in_padded, double* out_padded, int64_t steps, const tvs_exec* ex) {
  tvs_stencil st;
  tvs_layout lay;
  if (int rc = problem_to(p, TVS_JACOBI, &st, &lay)) return rc;
  return tvs_run(&st, &lay, in_padded, out_padded, steps, ex);
}

int tvs_gauss_seidel(const tvs_problem* p, double* inout_padded, int64_t steps, int32_t order, const tvs_exec* ex) {
  tvs_stencil st;
  tvs_layout lay;
  if (!ex) return fail(TVS_ERR_INVALID, "null exec");
  if (int rc = problem_to(p, TVS_GAUSS_SEIDEL, &st, &lay)) return rc;
  tvs_exec e = *ex;
  e.gs_order = order;
  return tvs_run(&st, &lay, inout_padded, inout_padded, steps, &e);
}

int tvs_plan_create(const tvs_stencil* st, int32_t dim, const int64_t extents[3], const tvs_exec* ex,
                    tvs_plan** out) {
  int rc = validate(st);
  if (rc) return rc;
  if ((rc = validate_exec(ex))) return rc;
  if (!out || !extents) return fail(TVS_ERR_INVALID, "null argument");
  if (dim != st->dim) return fail(TVS_ERR_SIZE, "grid/stencil dimension mismatch");
  if ((rc = set_device(ex->device))) return rc;
  tvs_plan* p = new tvs_plan();
  p->st = *st;
  p->ex = *ex;
  if (wants_shards(*st, *ex)) {
    p->group = new ShardGroup();
    if ((rc = p->group->create(*st, dim, extents, *ex))) {
      delete p->group;
      delete p;
      return rc;
    }
    geometry_init(dim, extents, 0, extents[0], &p->geo);  // the global geometry (layout checks)
    *out = p;
    return TVS_OK;
  }
  if ((rc = geometry_init(dim, extents, 0, extents[0], &p->geo))) {
    delete p;
    return rc;
  }
  const int nbuf = st->kind == TVS_GAUSS_SEIDEL ? 1 : 2;
  cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  for (int i = 0; i < nbuf && e == cudaSuccess; ++i) e = cudaMalloc(&p->buf[i], sizeof(double) * p->geo.alloc_elems);
  if (e == cudaSuccess) e = cudaEventCreate(&p->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&p->ev1);
  if (e != cudaSuccess) {
    tvs_plan_destroy(p);
    return cuda_fail(e, "tvs_plan_create");
  }
  for (int i = 0; i < nbuf; ++i)
    if ((rc = fill_halo(p->geo, p->buf[i], st->boundary, p->stream))) {
      tvs_plan_destroy(p);
      return rc;
    }
  *out = p;
  return TVS_OK;
}

int tvs_plan_upload(tvs_plan* p, const tvs_layout* lay, const double* host) {
  if (!p || !lay || !host) return fail(TVS_ERR_INVALID, "null argument");
  if (int rc = validate_layout(lay, p->geo.dim)) return rc;
  if (p->group) return p->group->upload(*lay, host);
  TVS_CUDA(cudaSetDevice(p->ex.device));
  p->cur = 0;
  return copy_interior(p->geo, p->buf[0], *lay, const_cast<double*>(host), true, p->stream);
}

int tvs_plan_download(tvs_plan* p, const tvs_layout* lay, double* host) {
  if (!p || !lay || !host) return fail(TVS_ERR_INVALID, "null argument");
  if (int rc = validate_layout(lay, p->geo.dim)) return rc;
  if (p->group) {
    if (int rc = p->group->download(*lay, host)) return rc;
    return p->group->synchronize();
  }
  TVS_CUDA(cudaSetDevice(p->ex.device));
  return copy_interior(p->geo, p->buf[p->cur], *lay, host, false, p->stream);
}

int tvs_plan_run(tvs_plan* p, int64_t steps) {
  if (!p) return fail(TVS_ERR_INVALID, "null plan");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  if (p->group) {
    const int rc = p->group->run(steps);
    p->last_launches = p->group->launches;
    return rc;
  }
  TVS_CUDA(cudaSetDevice(p->ex.device));
  int64_t before = g_launches;
  TVS_CUDA(cudaEventRecord(p->ev0, p->stream));
  int rc;
  if (p->st.kind == TVS_GAUSS_SEIDEL) {
    rc = gs_device(p->st, p->geo, p->buf[0], steps, p->ex, p->stream);
  } else {
    int32_t in_dst = 0;
    rc = jacobi_device(p->st, p->geo, p->buf[p->cur], p->buf[1 - p->cur], steps, p->ex, p->stream, &in_dst);
    if (rc == TVS_OK && in_dst) p->cur = 1 - p->cur;
  }
  if (rc) return rc;
  TVS_CUDA(cudaEventRecord(p->ev1, p->stream));
  p->last_launches = g_launches - before;
  return TVS_OK;
}

int tvs_plan_synchronize(tvs_plan* p) {
  if (!p) return fail(TVS_ERR_INVALID, "null plan");
  if (p->group) return p->group->synchronize();
  TVS_CUDA(cudaStreamSynchronize(p->stream));
  return TVS_OK;
}

int tvs_plan_last_ms(tvs_plan* p, float* ms) {
  if (!p || !ms) return fail(TVS_ERR_INVALID, "null argument");
  if (p->group) return p->group->last_ms(ms);  // lead stream: after every shard's last pass
  TVS_CUDA(cudaEventSynchronize(p->ev1));
  TVS_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
  return TVS_OK;
}

int tvs_plan_last_launches(tvs_plan* p, int64_t* n) {
  if (!p || !n) return fail(TVS_ERR_INVALID, "null argument");
  *n = p->last_launches;
  return TVS_OK;
}

int tvs_plan_stream(tvs_plan* p, void** stream) {
  if (!p || !stream) return fail(TVS_ERR_INVALID, "null argument");
  if (p->group) return tvs_shard_stream(p->group->shards[0], stream);  // the lead stream
  *stream = (void*)p->stream;
  return TVS_OK;
}

int tvs_plan_destroy(tvs_plan* p) {
  if (!p) return TVS_OK;
  if (p->group) {
    delete p->group;
    delete p;
    return TVS_OK;
  }
  cudaSetDevice(p->ex.device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  for (auto& b : p->buf)
    if (b) cudaFree(b);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
  return TVS_OK;
}

}  // extern "C"
