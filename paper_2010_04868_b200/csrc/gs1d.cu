// K5: 1D Gauss-Seidel as a time-skewed warp pipeline.
//
// Replaces gs1d_temporal (reference kernels1d.py:96-103) and reproduces the
// oracle's in-place lexicographic sweep (_gs_sweep_1d, baselines.py:73-80)
// bit-exactly:  a[i] = ((w0*a_new[i-1]) + w1*a_old[i]) + w2*a_old[i+1].
//
// The paper's temporal vectorisation puts consecutive sweeps in the lanes of
// one vector, lane k trailing lane k-1 by a space stride s > max dx/dt
// (min_space_stride = 2, model.py:171-193).  Here a lane *is* a sweep:
//
//   lane k of global warp g runs sweep q = 32*g + k and, at local step j,
//   updates position i = j - 3*(k+1)   (lag 3 = min stride 2 + 1, so the
//   value received by __shfl_up is consumed one step later and the 24-cycle
//   shuffle stays off the critical path).
//
// Per step each lane does one update (its new left neighbour is its own
// previous result — the serial GS dependence — and its two old values are
// what lane k-1 produced two and one steps earlier).  The only critical
// path is DMUL->DADD->DADD = 3 x 8 cycles per position, so one sweep's worth
// of positions streams through all T lanes with an (N + ~4T) step latency.
//
// Lane 31 of a warp feeds lane 0 of the next warp through a shared-memory
// ring guarded by release/acquire progress counters; the last warp of a block
// publishes its sweep to a global buffer (release/acquire at GPU scope) that
// the next block's first warp streams in.  Blocks take tickets in start
// order and only wait on lower tickets, so the launch is deadlock-free for
// any grid size.  Sweeps beyond T are identity lanes (they forward their
// old value), so the last lane always emits sweep T.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace tvs {

constexpr int kGsLag = 3;            // position lag between adjacent lanes
constexpr int kGsRing = 512;         // per-warp input ring (positions)
constexpr int kGsMaxBlocks = 64;     // sweeps per launch <= 64 * 128
constexpr int kGsPubChunks = 4;      // cross-block publication every 4 x 32 positions
constexpr int kGsPrefetch = 4;       // warp-0 input prefetch distance (chunks)
static_assert(kGsLag * 32 % 32 == 0, "lane-31 output chunks must align");

__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ long long ld_acquire_gpu(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(long long* p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Gs1dArgs {
  double* a;          // interior origin of the in-place grid
  double* gbuf;       // (nblocks-1) * n inter-block sweep buffers
  long long* gprog;   // nblocks progress counters (zeroed per launch)
  int* ticket;        // zeroed per launch
  long long n;
  long long sweeps;   // real sweeps in this launch
  int nblocks;
  double w0, w1, w2, bnd;
};

template <unsigned MASK>
__device__ __forceinline__ double gs_taps(double L, double C, double R, double w0, double w1, double w2) {
  double acc = 0.0;
  bool first = true;
  if constexpr (MASK & 1u) { acc = tap_first(w0, L); first = false; }
  if constexpr (MASK & 2u) { acc = first ? tap_first(w1, C) : tap_next<false>(w1, C, acc); first = false; }
  if constexpr (MASK & 4u) { acc = first ? tap_first(w2, R) : tap_next<false>(w2, R, acc); }
  return acc;
}

template <unsigned MASK, int kGsWarps>
__global__ void __launch_bounds__(kGsWarps * 32, 1) gs1d_kernel(Gs1dArgs p) {
  // ring[w]: input positions of warp w; ring[kGsWarps]: staging of the last
  // warp's sweep before it is flushed to global memory.
  __shared__ double ring[kGsWarps + 1][kGsRing];
  __shared__ int prod[kGsWarps], cons[kGsWarps + 1];
  __shared__ int s_ticket;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1);
  if (threadIdx.x < kGsWarps) prod[threadIdx.x] = 0;
  if (threadIdx.x <= kGsWarps) cons[threadIdx.x] = 0;
  __syncthreads();
  const int b = s_ticket;
  const int n = (int)p.n;  // host guarantees n < 2^30
  const double bnd = p.bnd;
  const long long q = ((long long)b * kGsWarps + w) * 32 + lane;  // this lane's sweep
  const bool real = q < p.sweeps;
  const bool last_block = b == p.nblocks - 1;
  const double* lsrc = b == 0 ? p.a : p.gbuf + (long long)(b - 1) * p.n;
  double* odst = last_block ? p.a : p.gbuf + (long long)b * p.n;
  const int nch = (n + 31) / 32 + kGsLag + 1;
  const int lane_off = kGsLag * (lane + 1);
  const double* rin = ring[w];
  double* rout = ring[w + 1];
  const bool writer = lane == 31;
  const bool warp_real = __all_sync(0xffffffffu, real);

  auto wait_upstream = [&](int need) {  // block b-1 published >= need positions
    if (b == 0) return;
    if (lane == 0) {
      long long want = need;
      SpinGuard sg;
      while (ld_acquire_gpu(p.gprog + b - 1) < want) {
        __nanosleep(32);
        sg.tick();
      }
    }
    __syncwarp();
  };

  double L = bnd, u0 = bnd, u1 = bnd, out = bnd;
  // warp 0 streams its input (the grid, or block b-1's sweep) into ring[0]
  // with cp.async, kGsPrefetch chunks ahead of consumption
  auto load_chunk = [&](int c) {
    const int x = c * 32 + lane;
    wait_upstream(min(((c * 32) / (32 * kGsPubChunks) + 1) * 32 * kGsPubChunks, n));
    double* slot = &ring[0][x & (kGsRing - 1)];
    if (x < n) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(slot);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(lsrc + x));
    } else {
      *slot = bnd;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if (w == 0) {
#pragma unroll 1
    for (int c = 0; c < kGsPrefetch; ++c) load_chunk(c);
  }

  for (int ch = 0; ch < nch; ++ch) {
    const int jb = ch * 32;
    if (w == 0) {
      load_chunk(ch + kGsPrefetch);  // (chunks past n just store bnd)
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kGsPrefetch));  // chunk ch landed
      __syncwarp();
    } else {
      const int need = min(jb + 31, n);
      SpinGuard sg;
      while (ld_acquire_cta(&prod[w]) < need) sg.tick();
    }
    {  // ring space in the consumer of my lane-31 stream: positions up to jb-65
      const int lim = jb - 65 - kGsRing;
      SpinGuard sg;
      while (ld_acquire_cta(&cons[w + 1]) <= lim) sg.tick();
    }
    // steady chunk: every lane real and every position of the chunk inside
    // [0, n) — no selects on the DMUL->DADD->DADD chain
    const bool steady = warp_real && jb - kGsLag * 32 >= 0 && jb + 31 - kGsLag < n;
    if (steady && MASK == 7u) {
      // full 3-tap stencil: the products w1*C and w2*R are formed as soon as
      // their operands arrive, so the loop-carried chain is exactly
      // L -> DMUL -> DADD -> DADD (bit-identical: same products, same adds)
      double pa = __dmul_rn(p.w1, u0), pb = __dmul_rn(p.w2, u1);
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int j = jb + u;
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const double rv = rin[(j - 1) & (kGsRing - 1)];  // same address for all lanes: broadcast
        const double sv = lane == 0 ? rv : sh;
        out = __dadd_rn(pb, __dadd_rn(pa, __dmul_rn(p.w0, L)));
        pa = __dmul_rn(p.w1, u1);  // next iteration's C is this iteration's R
        pb = __dmul_rn(p.w2, sv);  // next iteration's R just arrived
        L = out;
        u0 = u1;
        u1 = sv;
        const int po = j - kGsLag * 32;
        if (writer) rout[po & (kGsRing - 1)] = out;
      }
    } else if (steady) {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int j = jb + u;
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const double rv = rin[(j - 1) & (kGsRing - 1)];  // same address for all lanes: broadcast
        const double sv = lane == 0 ? rv : sh;
        out = gs_taps<MASK>(L, u0, u1, p.w0, p.w1, p.w2);
        L = out;
        u0 = u1;
        u1 = sv;
        const int po = j - kGsLag * 32;
        if (writer) rout[po & (kGsRing - 1)] = out;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int j = jb + u;
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const int pos = j - 1;
        const double rv = rin[pos & (kGsRing - 1)];
        const double up = (unsigned)pos < (unsigned)n ? rv : bnd;
        const double sv = lane == 0 ? up : sh;
        const int i = j - lane_off;
        const double v = gs_taps<MASK>(L, u0, u1, p.w0, p.w1, p.w2);
        out = (unsigned)i < (unsigned)n ? (real ? v : u0) : bnd;
        L = out;
        u0 = u1;
        u1 = sv;
        const int po = j - kGsLag * 32;
        if (writer && (unsigned)po < (unsigned)n) rout[po & (kGsRing - 1)] = out;
      }
    }
    __syncwarp();
    if (writer && w + 1 < kGsWarps) st_release_cta(&prod[w + 1], max(0, min(jb + 32 - kGsLag * 32, n)));
    if (lane == 0 && w > 0) st_release_cta(&cons[w], jb + 31);
    if (w == kGsWarps - 1) {
      const int pc = ch - kGsLag;  // position chunk completed by lane 31
      if (pc >= 0 && pc * 32 < n) {
        const int x = pc * 32 + lane;
        if (x < n) odst[x] = rout[x & (kGsRing - 1)];
        __syncwarp();
        if (lane == 0) st_release_cta(&cons[kGsWarps], x + 1 - lane);  // staging slots consumed
        const bool batch_end = ((pc + 1) % kGsPubChunks == 0) || (pc + 1) * 32 >= n;
        if (!last_block && batch_end) {
          __threadfence();
          __syncwarp();
          if (lane == 0) st_release_gpu(p.gprog + b, min((pc + 1) * 32, n));
        }
      }
      __syncwarp();
    }
  }
}

static unsigned gs_mask1d(const tvs_stencil& st, double w[3]) {
  unsigned mask = 0;
  int last = -2;
  w[0] = w[1] = w[2] = 0.0;
  for (int k = 0; k < st.ntaps; ++k) {
    const int o = st.offsets[k][0];
    if (o <= last) return 0;
    last = o;
    mask |= 1u << (o + 1);
    w[o + 1] = st.coeffs[k];
  }
  return mask;
}

int gs1d_pipeline(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, cudaStream_t s) {
  double w[3];
  const unsigned mask = gs_mask1d(st, w);
  if (mask == 0) return gs_wavefront(st, g, grid, steps, TVS_GS_LEXICOGRAPHIC, s);
  const long long n = g.extents[0];
  if (n >= (1ll << 30)) return fail(TVS_ERR_UNSUPPORTED, "gs1d_pipeline: N >= 2^30");
  static const int warps = [] {
    const char* e = getenv("TVS_GS1D_WARPS");
    const int v = e ? atoi(e) : 4;
    return (v == 1 || v == 2 || v == 4) ? v : 4;
  }();
  const long long per_launch = (long long)kGsMaxBlocks * warps * 32;
  const int max_blocks = (int)std::min<long long>((steps + warps * 32 - 1) / (warps * 32), kGsMaxBlocks);
  const size_t gbuf_bytes = sizeof(double) * (size_t)std::max(1, max_blocks - 1) * (size_t)n;
  const size_t ctrl_bytes = sizeof(long long) * (kGsMaxBlocks + 2);
  double* gbuf = static_cast<double*>(scratch(gbuf_bytes, 0));
  char* ctrl = static_cast<char*>(scratch(ctrl_bytes, 1));
  if (!gbuf || !ctrl) return fail(TVS_ERR_CUDA, "gs1d_pipeline: out of device memory for sweep buffers");
  Gs1dArgs a;
  a.a = grid + g.origin;
  a.gbuf = gbuf;
  a.gprog = reinterpret_cast<long long*>(ctrl);
  a.ticket = reinterpret_cast<int*>(ctrl + sizeof(long long) * kGsMaxBlocks);
  a.n = n;
  a.w0 = w[0];
  a.w1 = w[1];
  a.w2 = w[2];
  a.bnd = st.boundary;
  auto launch = [&](auto warps_tag) {
    constexpr int W = decltype(warps_tag)::value;
    switch (mask) {
      case 1: gs1d_kernel<1, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
      case 2: gs1d_kernel<2, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
      case 3: gs1d_kernel<3, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
      case 4: gs1d_kernel<4, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
      case 5: gs1d_kernel<5, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
      case 6: gs1d_kernel<6, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
      default: gs1d_kernel<7, W><<<a.nblocks, W * 32, 0, s>>>(a); break;
    }
  };
  for (long long done = 0; done < steps; done += per_launch) {
    a.sweeps = std::min<long long>(steps - done, per_launch);
    a.nblocks = (int)((a.sweeps + warps * 32 - 1) / (warps * 32));
    TVS_CUDA(cudaMemsetAsync(ctrl, 0, ctrl_bytes, s));
    if (warps == 1)
      launch(std::integral_constant<int, 1>{});
    else if (warps == 2)
      launch(std::integral_constant<int, 2>{});
    else
      launch(std::integral_constant<int, 4>{});
    TVS_LAUNCHED("gs1d_kernel");
  }
  return TVS_OK;
}

}  // namespace tvs
