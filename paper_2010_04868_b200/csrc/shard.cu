// Sharded 2D/3D Jacobi over axis-0 slabs across GPUs.
//
// The reference has no distributed path; BASELINE configs 3 and
// 5 split the grid into row slabs (2D) / z-slabs (3D) across the GPUs of one
// node, with a halo as wide as the temporal block depth.  Design:
//
//  * shard i owns global axis-0 rows [r0, r1) (balanced split, the first
//    n % N shards one row more) and keeps G = depth ghost rows on each side:
//    its device block is rows [r0 - G, r1 + G) in the library layout
//    (tvs_geometry with axis0_offset = r0 - G), two ping-pong buffers;
//  * one pass advances d <= G levels of the owned rows with the temporally
//    blocked kernel (K3 / K4b).  The rows of the result that are a
//    neighbour's ghost rows (owned rows [G, 2G) for the left neighbour,
//    [n, n + G) for the right one) are stored by the same kernel straight
//    into the neighbour's next-input buffer through peer memory (NVLink P2P
//    stores; Mirror in common.cuh) — the halo exchange is fused into the
//    compute, row by row, with no copy, collective or packing step;
//  * passes are ordered by pass counters: after pass p a one-thread signal
//    kernel writes p into both neighbours' flag words (st.release.sys, after
//    the pass kernel completed), and pass p + 1 of a shard starts after a
//    stream wait (cuStreamWaitValue32) for both neighbours' counters >= p.
//    That single condition covers both hazards: the neighbours have written
//    this shard's ghost rows for level p, and they have finished reading the
//    buffer this pass writes their ghosts into (they read it in pass p).
//    No host synchronisation between passes, no spinning kernel;
//  * in one process, shards are connected by pointer
//    (tvs_shard_connect_local, peer access enabled between devices); with one
//    process per GPU, by CUDA IPC handles (tvs_shard_export /
//    tvs_shard_connect) that the caller exchanges (torch.distributed).
//
// Every point is computed by the same kernel expression whatever the shard
// count, so the result is bit-identical to the unsharded run for any N
// (tests/test_shard.py).  Several shards may share one device
// (TVS_EXEC_EMULATE_SHARDS): the path that the tests drive on one GPU.
//
// Enqueue order (in-process groups): pass p of every shard is enqueued
// before pass p + 1 of any shard, so every stream wait is pushed after the
// signals it waits for — no deadlock even when several shard streams share a
// hardware queue on one device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace tvs {

int fill_halo_api(const tvs_geometry& g, double* dev, double value, cudaStream_t s);
int validate_stencil_api(const tvs_stencil* st);

typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, unsigned, unsigned);
bool stream_value_fns_api(StreamValueFn* wait, StreamValueFn* write);

__global__ void shard_signal_kernel(unsigned* a, unsigned* b, unsigned v) {
  // the pass kernel before this one on the stream has completed (its peer
  // stores included); publish the pass count system-wide
  __threadfence_system();
  if (a) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
  if (b) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(b), "r"(v) : "memory");
}

__global__ void shard_fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

static void split_rows(int64_t n, int parts, int i, int64_t* r0, int64_t* r1) {
  const int64_t base = n / parts, extra = n % parts;
  *r0 = i * base + std::min<int64_t>(i, extra);
  *r1 = *r0 + base + (i < extra ? 1 : 0);
}

// flag words: [0] pass count written by the left neighbour, [kFlagR] by the
// right one (separate 128-byte lines)
constexpr int kFlagR = 32;
constexpr size_t kFlagBytes = 256;

struct ShardWire {  // the bytes behind tvs_shard_handle
  cudaIpcMemHandle_t buf[2];
  cudaIpcMemHandle_t flags;
  int32_t index, n_shards, ghost, device;
  int64_t r0, r1, pitch;
};
static_assert(sizeof(ShardWire) <= sizeof(tvs_shard_handle), "shard handle size");

}  // namespace tvs

using namespace tvs;

struct tvs_shard {
  tvs_stencil st{};
  tvs_exec ex{};
  int index = 0, n_shards = 1, device = 0, ghost = 1, depth = 1;
  int64_t r0 = 0, r1 = 0, e0 = 0;
  tvs_geometry geo{};
  double* buf[2] = {nullptr, nullptr};
  unsigned* flags = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // neighbours: [0] left (index - 1), [1] right (index + 1)
  bool has[2] = {false, false};
  double* peer_buf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  unsigned* peer_flag[2] = {nullptr, nullptr};  // my slot in the neighbour's flags
  int64_t peer_rows[2] = {0, 0};                // neighbour's owned row count
  bool ipc[2] = {false, false};                 // opened through CUDA IPC
  void* ipc_ptr[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  int cur = 0;
  uint32_t passes = 0;  // passes enqueued since creation (the flag epoch)
  int64_t last_launches = 0;
  bool timing = false;
};

namespace tvs {

static int shard_pass(tvs_shard* s, int d, StreamValueFn wait_value) {
  const uint32_t p = ++s->passes;
  if (p > 1) {
    // neighbours finished pass p-1: my ghost rows hold level p-1 data, and
    // they no longer read the buffer this pass writes their ghosts into
    for (int k = 0; k < 2; ++k) {
      if (!s->has[k]) continue;
      const unsigned long long addr = reinterpret_cast<unsigned long long>(s->flags + (k == 0 ? 0 : kFlagR));
      const int rc = wait_value(s->stream, addr, p - 1, 0 /* CU_STREAM_WAIT_VALUE_GEQ */);
      if (rc != 0) return fail(TVS_ERR_CUDA, "cuStreamWaitValue32 failed (CUresult " + std::to_string(rc) + ")");
    }
  }
  const int G = s->ghost;
  const int64_t n = s->r1 - s->r0;
  const int src = s->cur, dst = 1 - s->cur;
  Mirror m{};
  const int64_t s0 = s->geo.strides[0];
  if (s->has[0]) {  // owned rows [G, 2G) -> left neighbour's rows [nL + G, nL + 2G)
    m.p[0] = s->peer_buf[0][dst];
    m.lo[0] = G;
    m.hi[0] = 2 * G;
    m.shift[0] = s->peer_rows[0] * s0;
  }
  if (s->has[1]) {  // owned rows [n, n + G) -> right neighbour's rows [0, G)
    m.p[1] = s->peer_buf[1][dst];
    m.lo[1] = n;
    m.hi[1] = n + G;
    m.shift[1] = -n * s0;
  }
  const bool fma = use_fma(s->st, s->ex);
  int rc;
  if (s->geo.dim == 2) {
    // segment rows chosen by the kernel to fill its last wave (jacobi2d.cu auto_seg)
    rc = jacobi2d_blocked(s->st, s->geo, s->buf[src], s->buf[dst], d, fma, s->stream, G, G + n, 0, &m);
  } else {
    rc = d == 2 ? jacobi3d_blocked2(s->st, s->geo, s->buf[src], s->buf[dst], fma, s->stream, G, G + n, 0, &m)
                : jacobi3d_streaming(s->st, s->geo, s->buf[src], s->buf[dst], fma, s->stream, G, G + n, 0, &m);
  }
  if (rc) return rc;
  s->last_launches += 1;
  if (s->has[0] || s->has[1]) {
    shard_signal_kernel<<<1, 1, 0, s->stream>>>(s->peer_flag[0], s->peer_flag[1], p);
    TVS_LAUNCHED("shard_signal_kernel");
    s->last_launches += 1;
  }
  s->cur = dst;
  return TVS_OK;
}

// level counts of the passes of a `steps` run (all d <= ghost)
static std::vector<int> pass_depths(const tvs_shard* s, int64_t steps) {
  std::vector<int> d;
  for (int64_t left = steps; left > 0;) {
    const int k = (int)std::min<int64_t>(left, s->depth);
    d.push_back(k);
    left -= k;
  }
  return d;
}

// host rows [g0, g1) of the global grid <-> local rows [g0 - (r0 - G), ...)
static int shard_copy(tvs_shard* s, const tvs_layout& lay, double* host, bool upload, int64_t g0, int64_t g1) {
  if (g1 <= g0) return TVS_OK;
  const tvs_geometry& g = s->geo;
  const int64_t l0 = g0 - (s->r0 - s->ghost);  // local row of global row g0
  if (g.dim == 2) {
    double* d0 = s->buf[s->cur] + g.origin + l0 * g.strides[0];
    double* h0 = host + (lay.offset + g0) * lay.shape[1] + lay.offset;
    const size_t hp = sizeof(double) * lay.shape[1], dp = sizeof(double) * g.strides[0];
    const size_t w = sizeof(double) * g.extents[1];
    if (upload) return upload_block((char*)d0, dp, 0, (const char*)h0, hp, 0, w, g1 - g0, 1, s->stream);
    TVS_CUDA(cudaMemcpy2DAsync(h0, hp, d0, dp, w, g1 - g0, cudaMemcpyDeviceToHost, s->stream));
    return TVS_OK;
  }
  if (upload) {
    const size_t hr = sizeof(double) * lay.shape[2], hz = hr * lay.shape[1];
    const double* h0 = host + ((lay.offset + g0) * lay.shape[1] + lay.offset) * lay.shape[2] + lay.offset;
    return upload_block((char*)(s->buf[s->cur] + g.origin + l0 * g.strides[0]), sizeof(double) * g.strides[1],
                        sizeof(double) * g.strides[0], (const char*)h0, hr, hz, sizeof(double) * g.extents[2],
                        g.extents[1], g1 - g0, s->stream);
  }
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  const cudaPitchedPtr hptr = make_cudaPitchedPtr(host, sizeof(double) * lay.shape[2], lay.shape[2], lay.shape[1]);
  const cudaPitchedPtr dptr = make_cudaPitchedPtr(s->buf[s->cur], sizeof(double) * g.strides[1], g.strides[1],
                                                  g.strides[0] / g.strides[1]);
  const cudaPos hpos = make_cudaPos(sizeof(double) * lay.offset, lay.offset, lay.offset + g0);
  const cudaPos dpos = make_cudaPos(sizeof(double) * kPadLast, 1, 1 + l0);
  p.extent = make_cudaExtent(sizeof(double) * g.extents[2], g.extents[1], g1 - g0);
  if (upload) {
    p.srcPtr = hptr; p.srcPos = hpos; p.dstPtr = dptr; p.dstPos = dpos; p.kind = cudaMemcpyHostToDevice;
  } else {
    p.srcPtr = dptr; p.srcPos = dpos; p.dstPtr = hptr; p.dstPos = hpos; p.kind = cudaMemcpyDeviceToHost;
  }
  TVS_CUDA(cudaMemcpy3DAsync(&p, s->stream));
  return TVS_OK;
}

static int check_global_layout(const tvs_shard* s, const tvs_layout* lay) {
  if (!lay) return fail(TVS_ERR_INVALID, "null layout");
  if (lay->dim != s->geo.dim) return fail(TVS_ERR_SIZE, "layout/shard dimension mismatch");
  if (lay->offset < 0) return fail(TVS_ERR_INVALID, "layout offset must be >= 0");
  for (int d = 0; d < lay->dim; ++d) {
    const int64_t want = d == 0 ? s->e0 : s->geo.extents[d];
    if (lay->extents[d] != want) return fail(TVS_ERR_SIZE, "layout extents differ from the sharded grid's");
    if (lay->offset + lay->extents[d] > lay->shape[d]) return fail(TVS_ERR_INVALID, "layout shape too small");
  }
  return TVS_OK;
}

static int enable_peer(int dev, int peer) {
  if (dev == peer) return TVS_OK;
  int ok = 0;
  TVS_CUDA(cudaDeviceCanAccessPeer(&ok, dev, peer));
  if (!ok) return fail(TVS_ERR_UNSUPPORTED, "sharded Jacobi needs peer access between neighbouring GPUs");
  int cur = 0;
  TVS_CUDA(cudaGetDevice(&cur));
  TVS_CUDA(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  cudaSetDevice(cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return TVS_OK;
}

}  // namespace tvs

extern "C" {

int tvs_shard_create(const tvs_stencil* st, int32_t dim, const int64_t global_extents[3], int32_t n_shards,
                     int32_t index, const tvs_exec* ex, tvs_shard** out) {
  int rc = validate_stencil_api(st);
  if (rc) return rc;
  if ((rc = validate_exec_api(ex))) return rc;
  if (!out || !global_extents) return fail(TVS_ERR_INVALID, "null argument");
  *out = nullptr;
  if (st->kind != TVS_JACOBI) return fail(TVS_ERR_UNSUPPORTED, "sharding is for Jacobi stencils (Gauss-Seidel runs on one GPU)");
  if (dim != st->dim || (dim != 2 && dim != 3)) return fail(TVS_ERR_UNSUPPORTED, "sharding needs a 2D or 3D grid");
  if (dim == 2 ? !jacobi2d_blocked_supported(*st) : !jacobi3d_streaming_supported(*st))
    return fail(TVS_ERR_UNSUPPORTED, "sharding needs a star or box tap set (temporally blocked kernels)");
  if (n_shards < 1 || index < 0 || index >= n_shards) return fail(TVS_ERR_INVALID, "shard index / count");
  for (int d = 0; d < dim; ++d)
    if (global_extents[d] < 1) return fail(TVS_ERR_SIZE, "extents must be positive");
  if ((rc = set_device_api(ex->device))) return rc;
  tvs_shard* s = new tvs_shard();
  s->st = *st;
  s->ex = *ex;
  s->index = index;
  s->n_shards = n_shards;
  s->device = ex->device;
  s->depth = dim == 2 ? (ex->temporal_depth > 0 ? std::min(ex->temporal_depth, jacobi2d_max_depth())
                                                : jacobi2d_default_depth())
                      : std::max(1, std::min(ex->temporal_depth > 0 ? ex->temporal_depth : jacobi3d_default_depth(),
                                             jacobi3d_max_depth()));
  s->ghost = s->depth;
  s->e0 = global_extents[0];
  split_rows(s->e0, n_shards, index, &s->r0, &s->r1);
  if (n_shards > 1 && s->r1 - s->r0 < s->ghost) {
    delete s;
    return fail(TVS_ERR_SIZE, "a shard owns fewer axis-0 rows than the ghost depth: use fewer shards or a smaller depth");
  }
  int64_t ext[3] = {s->r1 - s->r0 + 2 * s->ghost, dim > 1 ? global_extents[1] : 1, dim > 2 ? global_extents[2] : 1};
  if ((rc = geometry_init_api(dim, ext, s->r0 - s->ghost, s->e0, &s->geo))) {
    delete s;
    return rc;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&s->buf[i], sizeof(double) * s->geo.alloc_elems);
  if (e == cudaSuccess) e = cudaMalloc(&s->flags, kFlagBytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->flags, 0, kFlagBytes, s->stream);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev1);
  if (e != cudaSuccess) {
    tvs_shard_destroy(s);
    return cuda_fail(e, "tvs_shard_create");
  }
  for (int i = 0; i < 2; ++i) {
    if ((rc = fill_halo_api(s->geo, s->buf[i], st->boundary, s->stream))) {
      tvs_shard_destroy(s);
      return rc;
    }
    // ghost rows outside the global domain (first / last shard) hold the
    // Dirichlet value like the memory halo of an unsharded block: the 3D
    // kernels stage input planes without a global range check
    const int64_t s0 = s->geo.strides[0];
    const int64_t lo_out = std::max<int64_t>(0, s->ghost - s->r0);              // local rows [0, lo_out)
    const int64_t hi_out = std::max<int64_t>(0, s->r1 + s->ghost - s->e0);     // last hi_out local rows
    const int64_t e0l = s->geo.extents[0];
    if (lo_out > 0) {
      shard_fill_kernel<<<64, 256, 0, s->stream>>>(s->buf[i] + s0, lo_out * s0, st->boundary);
      TVS_LAUNCHED("shard_fill_kernel");
    }
    if (hi_out > 0) {
      shard_fill_kernel<<<64, 256, 0, s->stream>>>(s->buf[i] + (e0l - hi_out + 1) * s0, hi_out * s0, st->boundary);
      TVS_LAUNCHED("shard_fill_kernel");
    }
  }
  // neighbours may write into these buffers as soon as they are connected
  if ((e = cudaStreamSynchronize(s->stream)) != cudaSuccess) {
    tvs_shard_destroy(s);
    return cuda_fail(e, "tvs_shard_create");
  }
  *out = s;
  return TVS_OK;
}

int tvs_shard_info(const tvs_shard* s, int64_t* row_begin, int64_t* row_end, int32_t* ghost, int32_t* device) {
  if (!s) return fail(TVS_ERR_INVALID, "null shard");
  if (row_begin) *row_begin = s->r0;
  if (row_end) *row_end = s->r1;
  if (ghost) *ghost = s->ghost;
  if (device) *device = s->device;
  return TVS_OK;
}

int tvs_shard_export(tvs_shard* s, tvs_shard_handle* h) {
  if (!s || !h) return fail(TVS_ERR_INVALID, "null argument");
  std::memset(h, 0, sizeof(*h));
  ShardWire w{};
  TVS_CUDA(cudaSetDevice(s->device));
  TVS_CUDA(cudaIpcGetMemHandle(&w.buf[0], s->buf[0]));
  TVS_CUDA(cudaIpcGetMemHandle(&w.buf[1], s->buf[1]));
  TVS_CUDA(cudaIpcGetMemHandle(&w.flags, s->flags));
  w.index = s->index;
  w.n_shards = s->n_shards;
  w.ghost = s->ghost;
  w.device = s->device;
  w.r0 = s->r0;
  w.r1 = s->r1;
  w.pitch = s->geo.strides[0];
  std::memcpy(h->bytes, &w, sizeof(w));
  return TVS_OK;
}

static int check_neighbour(const tvs_shard* s, int side, int index, int n_shards, int ghost, int64_t pitch) {
  if (index != s->index + (side == 0 ? -1 : 1) || n_shards != s->n_shards)
    return fail(TVS_ERR_INVALID, "shard connect: not the neighbour of this shard");
  if (ghost != s->ghost || pitch != s->geo.strides[0])
    return fail(TVS_ERR_INVALID, "shard connect: neighbour has a different ghost depth or row pitch");
  return TVS_OK;
}

int tvs_shard_connect(tvs_shard* s, const tvs_shard_handle* left, const tvs_shard_handle* right) {
  if (!s) return fail(TVS_ERR_INVALID, "null shard");
  if ((s->index > 0) != (left != nullptr) || (s->index + 1 < s->n_shards) != (right != nullptr))
    return fail(TVS_ERR_INVALID, "shard connect: pass exactly the existing neighbours");
  TVS_CUDA(cudaSetDevice(s->device));
  const tvs_shard_handle* hs[2] = {left, right};
  for (int k = 0; k < 2; ++k) {
    if (!hs[k]) continue;
    ShardWire w;
    std::memcpy(&w, hs[k]->bytes, sizeof(w));
    if (int rc = check_neighbour(s, k, w.index, w.n_shards, w.ghost, w.pitch)) return rc;
    // the neighbour's ordinal is from its own process (its CUDA_VISIBLE_DEVICES
    // may differ): peer access comes from cudaIpcMemLazyEnablePeerAccess
    for (int b = 0; b < 2; ++b)
      TVS_CUDA(cudaIpcOpenMemHandle(&s->ipc_ptr[k][b], w.buf[b], cudaIpcMemLazyEnablePeerAccess));
    TVS_CUDA(cudaIpcOpenMemHandle(&s->ipc_ptr[k][2], w.flags, cudaIpcMemLazyEnablePeerAccess));
    s->ipc[k] = true;
    s->has[k] = true;
    s->peer_buf[k][0] = static_cast<double*>(s->ipc_ptr[k][0]);
    s->peer_buf[k][1] = static_cast<double*>(s->ipc_ptr[k][1]);
    s->peer_flag[k] = static_cast<unsigned*>(s->ipc_ptr[k][2]) + (k == 0 ? kFlagR : 0);
    s->peer_rows[k] = w.r1 - w.r0;
  }
  return TVS_OK;
}

int tvs_shard_connect_local(tvs_shard* s, tvs_shard* left, tvs_shard* right) {
  if (!s) return fail(TVS_ERR_INVALID, "null shard");
  if ((s->index > 0) != (left != nullptr) || (s->index + 1 < s->n_shards) != (right != nullptr))
    return fail(TVS_ERR_INVALID, "shard connect: pass exactly the existing neighbours");
  tvs_shard* ns[2] = {left, right};
  for (int k = 0; k < 2; ++k) {
    tvs_shard* o = ns[k];
    if (!o) continue;
    if (int rc = check_neighbour(s, k, o->index, o->n_shards, o->ghost, o->geo.strides[0])) return rc;
    if (o->device != s->device)
      if (int rc = enable_peer(s->device, o->device)) return rc;
    s->has[k] = true;
    s->peer_buf[k][0] = o->buf[0];
    s->peer_buf[k][1] = o->buf[1];
    s->peer_flag[k] = o->flags + (k == 0 ? kFlagR : 0);  // left writes my [0]; I write its [kFlagR]
    s->peer_rows[k] = o->r1 - o->r0;
  }
  return TVS_OK;
}

int tvs_shard_upload(tvs_shard* s, const tvs_layout* lay, const double* host) {
  if (!s || !host) return fail(TVS_ERR_INVALID, "null argument");
  if (int rc = check_global_layout(s, lay)) return rc;
  TVS_CUDA(cudaSetDevice(s->device));
  s->cur = 0;
  // owned rows plus the ghost rows that lie inside the domain
  const int64_t g0 = std::max<int64_t>(0, s->r0 - s->ghost), g1 = std::min(s->e0, s->r1 + s->ghost);
  return shard_copy(s, *lay, const_cast<double*>(host), true, g0, g1);
}

int tvs_shard_download(tvs_shard* s, const tvs_layout* lay, double* host) {
  if (!s || !host) return fail(TVS_ERR_INVALID, "null argument");
  if (int rc = check_global_layout(s, lay)) return rc;
  TVS_CUDA(cudaSetDevice(s->device));
  return shard_copy(s, *lay, host, false, s->r0, s->r1);
}

int tvs_shard_run(tvs_shard* s, int64_t steps) {
  if (!s) return fail(TVS_ERR_INVALID, "null shard");
  if (steps < 0) return fail(TVS_ERR_INVALID, "steps must be >= 0");
  StreamValueFn wait_value = nullptr, write_value = nullptr;
  if ((s->has[0] || s->has[1]) && !stream_value_fns_api(&wait_value, &write_value))
    return fail(TVS_ERR_UNSUPPORTED, "sharded Jacobi needs CUDA stream memory operations");
  TVS_CUDA(cudaSetDevice(s->device));
  s->last_launches = 0;
  TVS_CUDA(cudaEventRecord(s->ev0, s->stream));
  for (int d : pass_depths(s, steps))
    if (int rc = shard_pass(s, d, wait_value)) return rc;
  TVS_CUDA(cudaEventRecord(s->ev1, s->stream));
  return TVS_OK;
}

int tvs_shard_synchronize(tvs_shard* s) {
  if (!s) return fail(TVS_ERR_INVALID, "null shard");
  TVS_CUDA(cudaSetDevice(s->device));
  TVS_CUDA(cudaStreamSynchronize(s->stream));
  return TVS_OK;
}

int tvs_shard_last_ms(tvs_shard* s, float* ms) {
  if (!s || !ms) return fail(TVS_ERR_INVALID, "null argument");
  TVS_CUDA(cudaSetDevice(s->device));
  TVS_CUDA(cudaEventSynchronize(s->ev1));
  TVS_CUDA(cudaEventElapsedTime(ms, s->ev0, s->ev1));
  return TVS_OK;
}

int tvs_shard_last_launches(tvs_shard* s, int64_t* n) {
  if (!s || !n) return fail(TVS_ERR_INVALID, "null argument");
  *n = s->last_launches;
  return TVS_OK;
}

int tvs_shard_stream(tvs_shard* s, void** stream) {
  if (!s || !stream) return fail(TVS_ERR_INVALID, "null argument");
  *stream = (void*)s->stream;
  return TVS_OK;
}

int tvs_shard_destroy(tvs_shard* s) {
  if (!s) return TVS_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (int k = 0; k < 2; ++k)
    if (s->ipc[k])
      for (void* p : s->ipc_ptr[k])
        if (p) cudaIpcCloseMemHandle(p);
  for (double* b : s->buf)
    if (b) cudaFree(b);
  if (s->flags) cudaFree(s->flags);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->stream) cudaStreamDestroy(s->stream);
  cudaSetDevice(cur);
  delete s;
  return TVS_OK;
}

}  // extern "C"

namespace tvs {

// ---- in-process groups: tvs_run / tvs_plan with tvs_exec.n_gpus > 1 -------
ShardGroup::~ShardGroup() { release(); }

void ShardGroup::release() {
  for (tvs_shard* s : shards) tvs_shard_destroy(s);
  shards.clear();
  if (lead_ev0) cudaSetDevice(lead_device), cudaEventDestroy(lead_ev0), lead_ev0 = nullptr;
  if (lead_ev1) cudaSetDevice(lead_device), cudaEventDestroy(lead_ev1), lead_ev1 = nullptr;
  for (size_t i = 0; i < done_ev.size(); ++i) {
    cudaSetDevice(shards_dev[i]);
    cudaEventDestroy(done_ev[i]);
  }
  done_ev.clear();
  shards_dev.clear();
}

int ShardGroup::create(const tvs_stencil& st, int dim, const int64_t* ext, const tvs_exec& ex) {
  release();
  int ndev = 0;
  TVS_CUDA(cudaGetDeviceCount(&ndev));
  const int n = ex.n_gpus;
  const bool emulate = (ex.flags & TVS_EXEC_EMULATE_SHARDS) != 0;
  if (!emulate && ex.device + n > ndev)
    return fail(TVS_ERR_INVALID, "n_gpus = " + std::to_string(n) + " from device " + std::to_string(ex.device) +
                                     " exceeds the " + std::to_string(ndev) + " visible devices");
  for (int i = 0; i < n; ++i) {
    tvs_exec e = ex;
    e.device = (ex.device + i) % ndev;
    e.n_gpus = 1;
    tvs_shard* s = nullptr;
    if (int rc = tvs_shard_create(&st, dim, ext, n, i, &e, &s)) {
      release();
      return rc;
    }
    shards.push_back(s);
    shards_dev.push_back(e.device);
  }
  for (int i = 0; i < n; ++i)
    if (int rc = tvs_shard_connect_local(shards[i], i > 0 ? shards[i - 1] : nullptr, i + 1 < n ? shards[i + 1] : nullptr)) {
      release();
      return rc;
    }
  lead_device = shards_dev[0];
  TVS_CUDA(cudaSetDevice(lead_device));
  TVS_CUDA(cudaEventCreate(&lead_ev0));
  TVS_CUDA(cudaEventCreate(&lead_ev1));
  for (int i = 0; i < n; ++i) {
    cudaEvent_t e;
    TVS_CUDA(cudaSetDevice(shards_dev[i]));
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    done_ev.push_back(e);
  }
  st_ = st;
  ex_ = ex;
  dim_ = dim;
  for (int d = 0; d < 3; ++d) ext_[d] = d < dim ? ext[d] : 1;
  return TVS_OK;
}

bool ShardGroup::matches(const tvs_stencil& st, int dim, const int64_t* ext, const tvs_exec& ex) const {
  if (shards.empty() || dim != dim_ || std::memcmp(&st, &st_, sizeof(st)) != 0 ||
      std::memcmp(&ex, &ex_, sizeof(ex)) != 0)
    return false;
  for (int d = 0; d < dim; ++d)
    if (ext[d] != ext_[d]) return false;
  return true;
}

int ShardGroup::upload(const tvs_layout& lay, const double* host) {
  for (tvs_shard* s : shards)
    if (int rc = tvs_shard_upload(s, &lay, host)) return rc;
  return synchronize();  // every shard quiescent before any pass writes a neighbour
}

int ShardGroup::download(const tvs_layout& lay, double* host) {
  for (tvs_shard* s : shards)
    if (int rc = tvs_shard_download(s, &lay, host)) return rc;
  return TVS_OK;
}

int ShardGroup::run(int64_t steps) {
  StreamValueFn wait_value = nullptr, write_value = nullptr;
  if (shards.size() > 1 && !stream_value_fns_api(&wait_value, &write_value))
    return fail(TVS_ERR_UNSUPPORTED, "sharded Jacobi needs CUDA stream memory operations");
  launches = 0;
  // every shard starts after the lead event; the lead stream ends after all
  TVS_CUDA(cudaSetDevice(lead_device));
  TVS_CUDA(cudaEventRecord(lead_ev0, shards[0]->stream));
  for (size_t i = 1; i < shards.size(); ++i) {
    TVS_CUDA(cudaSetDevice(shards_dev[i]));
    TVS_CUDA(cudaStreamWaitEvent(shards[i]->stream, lead_ev0, 0));
  }
  const std::vector<int> depths = pass_depths(shards[0], steps);
  // pass p of every shard before pass p+1 of any (see the header: waits are
  // always pushed after the signals they wait for)
  for (int d : depths)
    for (size_t i = 0; i < shards.size(); ++i) {
      TVS_CUDA(cudaSetDevice(shards_dev[i]));
      shards[i]->last_launches = 0;
      if (int rc = shard_pass(shards[i], d, wait_value)) return rc;
      launches += shards[i]->last_launches;
    }
  for (size_t i = 0; i < shards.size(); ++i) {
    TVS_CUDA(cudaSetDevice(shards_dev[i]));
    TVS_CUDA(cudaEventRecord(done_ev[i], shards[i]->stream));
  }
  TVS_CUDA(cudaSetDevice(lead_device));
  for (size_t i = 1; i < shards.size(); ++i) TVS_CUDA(cudaStreamWaitEvent(shards[0]->stream, done_ev[i], 0));
  TVS_CUDA(cudaEventRecord(lead_ev1, shards[0]->stream));
  return TVS_OK;
}

int ShardGroup::synchronize() {
  for (size_t i = 0; i < shards.size(); ++i) {
    TVS_CUDA(cudaSetDevice(shards_dev[i]));
    TVS_CUDA(cudaStreamSynchronize(shards[i]->stream));
  }
  return TVS_OK;
}

int ShardGroup::last_ms(float* ms) {
  TVS_CUDA(cudaSetDevice(lead_device));
  TVS_CUDA(cudaEventSynchronize(lead_ev1));
  TVS_CUDA(cudaEventElapsedTime(ms, lead_ev0, lead_ev1));
  return TVS_OK;
}

int ShardGroup::cur_all() const { return shards.empty() ? 0 : shards[0]->cur; }

}  // namespace tvs
