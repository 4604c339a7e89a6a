// Shared device/host helpers for libtvstencil.so (sm_100a).
//
// Arithmetic contract (reference baselines.py:43-49, vec.py:296-298): taps in
// the caller's (sorted) order, first tap a multiply, every further tap a
// separately rounded multiply and add.  `tap_first` / `tap_next` below are
// the only places arithmetic is emitted; __dmul_rn/__dadd_rn are never
// contracted by nvcc, and the FMA form is opt-in (TVS_FMA_*).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/tvstencil.h"

namespace tvs {

constexpr int kPadLast = 32;  // elements of pad on each side of the contiguous axis

// Per-kernel view of a device block (see tvs_geometry).
struct Geo {
  int dim;
  int64_t e0, e1, e2;  // local extents (unused axes = 1)
  int64_t s0, s1;      // element strides of axes 0,1 (last axis stride 1)
  int64_t a0_off;      // global index of local axis-0 position 0
  int64_t a0_glob;     // global axis-0 extent
};

inline Geo make_geo(const tvs_geometry& g) {
  Geo o{};
  o.dim = g.dim;
  o.e0 = g.extents[0];
  o.e1 = g.dim > 1 ? g.extents[1] : 1;
  o.e2 = g.dim > 2 ? g.extents[2] : 1;
  o.s0 = g.strides[0];
  o.s1 = g.dim > 2 ? g.strides[1] : 1;
  o.a0_off = g.axis0_offset;
  o.a0_glob = g.axis0_global;
  return o;
}

// Sharded Jacobi (shard.cu): a pass also stores the output
// axis-0 rows that are a neighbour shard's ghost rows straight into that
// shard's next-input buffer — peer memory over NVLink (the same device when
// shards are emulated on one GPU).  The halo exchange therefore happens
// inside the compute kernel, row by row as rows are finished, with no
// separate copy or collective.  Neighbours share strides and origin, so a
// row's element offset in the peer buffer is its local offset + shift.
struct Mirror {
  double* p[2];          // neighbour's destination buffer (nullptr = none)
  int64_t lo[2], hi[2];  // local axis-0 rows [lo, hi) that are its ghosts
  int64_t shift[2];      // element offset (peer row - local row) * stride
};
// f(base) for the local destination and for every neighbour buffer whose
// ghost range holds local row q (base + the row's local element offset is
// the target).  Not unrolled: the caller's store code exists once, so the
// mirror adds no live registers to the kernel's main loop.
template <class F>
__device__ __forceinline__ void for_each_dst(double* dst, const Mirror& m, int64_t q, F&& f) {
#pragma unroll 1
  for (int k = -1; k < 2; ++k) {
    double* b = dst;
    if (k >= 0) {
      if (m.p[k] == nullptr || q < m.lo[k] || q >= m.hi[k]) continue;
      b = m.p[k] + m.shift[k];
    }
    f(b);
  }
}

// Tap list in evaluation order, with linear element offsets precomputed for
// the block's strides.
struct TapList {
  int n;
  int fma;  // 1: fused multiply-add after the first tap
  double bnd;
  int64_t lin[TVS_MAX_TAPS];
  double c[TVS_MAX_TAPS];
  int8_t off[TVS_MAX_TAPS][3];
};

// Spin-wait watchdog: a pipeline kernel that waits ~2^28 times on one flag
// is deadlocked; trap (CUDA error) instead of hanging the device.
struct SpinGuard {
  unsigned n = 0;
  __device__ __forceinline__ void tick() {
    if (++n > (1u << 28)) __trap();
  }
};

template <bool FMA>
__device__ __forceinline__ double tap_next(double c, double v, double acc) {
  if constexpr (FMA) {
    return __fma_rn(c, v, acc);
  } else {
    return __dadd_rn(__dmul_rn(c, v), acc);
  }
}
__device__ __forceinline__ double tap_first(double c, double v) { return __dmul_rn(c, v); }

// ---- mbarriers and bulk (TMA) copies -------------------------------------
#ifndef TVS_MBAR_SLEEP
#define TVS_MBAR_SLEEP 0
#endif
__device__ __forceinline__ unsigned smaddr(const void* q) { return (unsigned)__cvta_generic_to_shared(q); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smaddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smaddr(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  // no suspend-time hint: a bare TRYWAIT suspends in hardware until the phase
  // completes or a system time limit passes (a hint expands to a
  // NANOSLEEP.SYNCS loop that every mbarrier event in the CTA wakes up)
  unsigned ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(smaddr(b)), "r"(parity) : "memory");
  return ok != 0;
}
// address form (shared::cta address precomputed by the caller)
__device__ __forceinline__ bool mbar_try_a(unsigned a, unsigned parity) {
  unsigned ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  return ok != 0;
}
static __device__ __noinline__ void mbar_wait_slow(unsigned a, unsigned parity) {
  const long long t0 = clock64();
  for (unsigned n = 1;; ++n) {
    if (mbar_try_a(a, parity)) return;
    if ((n & 63u) == 0 && clock64() - t0 > (1ll << 34)) __trap();
  }
}
__device__ __forceinline__ void mbar_wait_a(unsigned a, unsigned parity) {
  if (!mbar_try_a(a, parity)) mbar_wait_slow(a, parity);
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  if (mbar_try(b, parity)) return;
  // retry loop kept lean: waiting warps share the SMSP with computing ones.
  // Optional back-off (TVS_MBAR_SLEEP ns) frees issue slots while waiting;
  // the watchdog reads the clock once per 64 tries (trap after ~2^34 cycles)
  const long long t0 = clock64();
  for (unsigned n = 1;; ++n) {
#if TVS_MBAR_SLEEP > 0
    __nanosleep(TVS_MBAR_SLEEP);
#endif
    if (mbar_try(b, parity)) return;
    if ((n & 63u) == 0 && clock64() - t0 > (1ll << 34)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smaddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// global -> shared bulk copy (16-byte aligned, bytes % 16 == 0), completion
// counted as transaction bytes on mbarrier `b`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smaddr(dst)), "l"(src), "r"(bytes), "r"(smaddr(b)) : "memory");
}

// Variants whose control flow stays inside the asm, so the compiler's
// divergence analysis still sees warp-uniform code (keeps shuffles free of
// BRA.DIV scaffolding).  `leader`: only that thread issues.
__device__ __forceinline__ void mbar_wait_uniform(unsigned long long* b, unsigned parity) {
  // hardware-suspending TRYWAIT loop (no hint, see mbar_try); the watchdog
  // clock is read once per 8 tries: trap after ~2^34 cycles (~9 s)
  asm volatile(
      "{ .reg .pred p; .reg .u64 t0, t1; mov.u64 t0, %%clock64;\n"
      "TVS_WAIT: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @p bra TVS_DONE;\n"
      "mov.u64 t1, %%clock64; sub.u64 t1, t1, t0; setp.lt.u64 p, t1, 17179869184;\n"
      "@p bra TVS_WAIT; trap;\n"
      "TVS_DONE: }" ::"r"(smaddr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s_leader(bool leader, void* dst, const void* src, unsigned bytes,
                                                unsigned long long* b) {
  asm volatile(
      "{ .reg .pred p; setp.ne.u32 p, %4, 0;\n"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3]; }"
      ::"r"(smaddr(dst)), "l"(src), "r"(bytes), "r"(smaddr(b)), "r"((unsigned)leader) : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(bool leader, unsigned long long* b) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p mbarrier.arrive.shared::cta.b64 _, [%0]; }"
               ::"r"(smaddr(b)), "r"((unsigned)leader) : "memory");
}

// ---- error plumbing (host) -------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int64_t n = 1);

#define TVS_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return ::tvs::cuda_fail(e_, #call); \
  } while (0)

#define TVS_LAUNCHED(name)                                          \
  do {                                                              \
    cudaError_t e_ = cudaGetLastError();                            \
    if (e_ != cudaSuccess) return ::tvs::cuda_fail(e_, name);        \
    ::tvs::count_launch();                                          \
  } while (0)

// api.cu helpers shared with integer.cu
int validate_exec_api(const tvs_exec* ex);
int validate_layout_api(const tvs_layout* lay, int dim);
void release_integer_cache();
int set_device_api(int dev);
int geometry_init_api(int dim, const int64_t* ext, int64_t a0_off, int64_t a0_glob, tvs_geometry* g);

// Fused-multiply-add decision (TVS_FMA_EXACT: all coefficients 0 or +-2^k).
bool coeffs_power_of_two(const tvs_stencil& st);
bool use_fma(const tvs_stencil& st, const tvs_exec& ex);

// Kernel-family entry points (each returns a TVS status code).
int jacobi_naive_step(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst,
                      bool fma, cudaStream_t s);
bool jacobi1d_blocked_supported(const tvs_stencil& st, const tvs_geometry& g);
int jacobi1d_blocked(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst,
                     int depth, bool fma, cudaStream_t s, int64_t rlo = 0, int64_t rhi = -1);
int jacobi1d_default_depth();
int jacobi1d_max_depth();
bool jacobi2d_blocked_supported(const tvs_stencil& st);
// rows [row_lo, row_hi) only when given (any band): one band of the
// pipelined host path
int jacobi2d_blocked(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst,
                     int depth, bool fma, cudaStream_t s, int64_t row_lo = 0, int64_t row_hi = -1,
                     int seg_rows = 0, const Mirror* mir = nullptr);
int jacobi2d_band_rows();
int jacobi2d_max_depth();
int jacobi2d_default_depth();
bool jacobi3d_streaming_supported(const tvs_stencil& st);
int jacobi3d_max_depth();
int jacobi3d_default_depth();
// axis-0 planes [plo, phi) only when given, `seg` output planes per block
int jacobi3d_blocked2(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, bool fma,
                      cudaStream_t s, int64_t plo = 0, int64_t phi = -1, int seg = 0, const Mirror* mir = nullptr);
int jacobi3d_streaming(const tvs_stencil& st, const tvs_geometry& g, const double* src, double* dst, bool fma,
                       cudaStream_t s, int64_t plo = 0, int64_t phi = -1, int seg = 0, const Mirror* mir = nullptr);
int gs1d_pipeline(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, cudaStream_t s);
bool gs2d_pipe_supported(const tvs_stencil& st);
// rows_ready / blocks_done: drop-in pipeline hooks (see api.cu), single pass only
int gs2d_pipeline(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, cudaStream_t s,
                  const unsigned* rows_ready = nullptr, unsigned* blocks_done = nullptr);
int64_t gs2d_pipe_blocks(int64_t rows);
int64_t gs2d_pipe_blocks_for_row(int64_t row, int64_t steps);
int gs2d_pipe_max_sweeps();
// K6v2 (gs2d_lane.cu): one-warp time-lane groups, both update orders
bool gs2d_lane_supported(const tvs_stencil& st);
int gs2d_lane(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, int order, cudaStream_t s,
              const unsigned* rows_ready = nullptr, unsigned* blocks_done = nullptr);
int gs2d_lane_max_sweeps();
int64_t gs2d_lane_ctas(int64_t rows, int64_t steps, int order);
int64_t gs2d_lane_ctas_for_row(int64_t row, int64_t steps, int order);
int gs_wavefront(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, int order,
                 cudaStream_t s);

// In-process group of shards (shard.cu): tvs_run / tvs_plan with n_gpus > 1.
struct ShardGroup {
  std::vector<tvs_shard*> shards;
  std::vector<int> shards_dev;
  std::vector<cudaEvent_t> done_ev;
  cudaEvent_t lead_ev0 = nullptr, lead_ev1 = nullptr;
  int lead_device = 0;
  int64_t launches = 0;
  tvs_stencil st_{};
  tvs_exec ex_{};
  int dim_ = 0;
  int64_t ext_[3] = {0, 0, 0};
  ~ShardGroup();
  void release();
  int create(const tvs_stencil& st, int dim, const int64_t* ext, const tvs_exec& ex);
  bool matches(const tvs_stencil& st, int dim, const int64_t* ext, const tvs_exec& ex) const;
  int upload(const tvs_layout& lay, const double* host);
  int download(const tvs_layout& lay, double* host);
  int run(int64_t steps);
  int synchronize();
  int last_ms(float* ms);
  int cur_all() const;
};
// does tvs_exec ask for (and the stencil allow) a sharded run?
bool wants_shards(const tvs_stencil& st, const tvs_exec& ex);

// Host -> device block copy (hostcopy.cu): nplanes x nrows rows of `width`
// bytes with row / plane pitches on both sides; pageable sources are staged
// through page-locked slots by a pool of host threads, page-locked ones DMA'd
// directly.  release_staging frees the calling thread's slots.
int upload_block(char* dst, size_t drow, size_t dplane, const char* src, size_t srow, size_t splane, size_t width,
                 int64_t nrows, int64_t nplanes, cudaStream_t s);
void release_staging();

// scratch device memory owned by the calling thread (grown on demand).
// Slots: 0, 1 GS-1D / GS-2D pipeline rings and control words, 2 small
// constants, 3 drop-in pipeline counters, 4, 5 GS-2D lane ring and control.
constexpr int kScratchSlots = 6;
void* scratch(size_t bytes, int slot);
// changes whenever this thread's scratch memory is (re)allocated or freed
uint64_t scratch_generation();

}  // namespace tvs
