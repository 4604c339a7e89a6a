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
//   updates position i = j - 4*(k+1)   (lag 4 = min stride 2 + 2: the value
//   received by __shfl_up is old(i+3), first used as a product operand two
//   steps later, so the 24-cycle shuffle can never land on the chain
//   whatever order the compiler issues the step in).
//
// Per step each lane does one update (its new left neighbour is its own
// previous result — the serial GS dependence — and its two old values are
// what lane k-1 produced three and two steps earlier).  The only critical
// path is DMUL->DADD->DADD = 3 x 8 cycles per position, so one sweep's worth
// of positions streams through all T lanes with an (N + ~4T) step latency.
//
// Data movement and synchronisation are kept off the compute warps:
//
//   * a LOADER warp streams the block's input (the grid for block 0, block
//     b-1's published sweep otherwise) into compute warp 0's ring;
//   * compute warp w's lane 31 writes its sweep into warp w+1's ring (the
//     last compute warp into a staging ring);
//   * a FLUSHER warp copies the staging ring to global memory and publishes
//     progress (GPU-scope release) for block b+1's loader.
//
// Everything advances in chunks of kCH = 256 positions.  Completion of chunk
// k by warp X is phase k / kNB of mbarrier bar[X][k % kNB] (hardware-suspended
// waits; no fences or acquire spins on the compute warps).  Ring bounds
// (R = 4 chunks of positions per ring; lane 31 lags S = 128 positions):
//   compute w at chunk c needs positions < min(n, (c+1)*kCH - 1), complete
//     once warp w-1 finished chunk ceil((need + S) / kCH) - 1 <= c + 1;
//   writing positions up to (c+1)*kCH - 1 - S into a ring overwrites position
//     p - R, consumed once the reader finished chunk c - 4  (4 * kCH < R + S);
//   the loader's chunk k overwrites chunk k - 4, consumed once warp 0 finished
//     chunk k - 3.
// A waiter is never more than 5 chunks away from the phase it waits for, so
// kNB = 8 barrier slots never alias.  Blocks take tickets in start order and
// only wait on lower tickets, so the launch is deadlock-free for any grid
// size.  The last block runs only as many warps as it has sweeps, and its last
// warp emits sweep T from lane (T-1) % 32 (lag 4 * (lane+1) <= S, so every
// bound above stays conservative; its staging writes are reused once the
// flusher finished chunk c - 3).  No lane ever selects between sweep and
// identity, so the loop-carried chain is the same in every warp.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace tvs {

constexpr int kGsLag = 4;                 // position lag between adjacent lanes
#ifndef GS1D_CH
#define GS1D_CH 256
#endif
constexpr int kCH = GS1D_CH;              // positions per chunk
#ifndef GS1D_SUB
#define GS1D_SUB 128  // measured (config 2): 32 -> 58.0, 64 -> 62.6, 128 -> 65.5, 256 -> 58.5 GSt/s
#endif
constexpr int kSubLen = GS1D_SUB;          // positions per unrolled sub-chunk
constexpr int kSub = kCH / kSubLen;       // unrolled sub-chunks per chunk
static_assert(kSubLen % 32 == 0 && kCH % kSubLen == 0, "sub-chunk length");
// the emitting lane's stores use one base per 128 positions of a sub-chunk:
// (wlag - woff) is a multiple of 128 (wlag of a full block is kGsLag * 32),
// so each 128-store run stays inside the ring (constant offsets)
constexpr int kWRun = kSubLen < 128 ? kSubLen : 128;
constexpr int kWRuns = kSubLen / kWRun;
static_assert(kSubLen <= 128 || kSubLen % 128 == 0, "sub-chunk length");
constexpr int kRingCh = 4;                // ring = 4 chunks
constexpr int kGsRing = kCH * kRingCh;    // ring positions (power of two)
constexpr int kNB = 8;                    // mbarrier ring per warp
constexpr int kWar = 4;                   // ring reuse: reader finished chunk c - kWar
constexpr int kGsMaxBlocks = 64;          // sweeps per launch <= 64 * 32 * kGsWarps
constexpr int kShiftLane31 = kGsLag * 32; // lane 31's position lag S (128)
static_assert((kGsRing & (kGsRing - 1)) == 0, "ring must be a power of two");
static_assert(kWar * kCH < kGsRing + kShiftLane31, "ring reuse bound");
static_assert(kCH >= kShiftLane31, "consumer waits at most one chunk ahead");
static_assert((kWar - 1) * kCH < kGsRing + 1, "staging reuse bound (writer lag >= 0)");

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
__global__ void __launch_bounds__((kGsWarps + 2) * 32, 1) gs1d_kernel(Gs1dArgs p) {
  constexpr int kLoader = kGsWarps, kFlusher = kGsWarps + 1;
  // ring[w]: input positions of compute warp w; ring[kGsWarps]: staging of
  // the last compute warp's sweep before the flusher writes it out.
  // (dynamic: (kGsWarps + 1) * kGsRing doubles, over 48 KB for long chunks)
  extern __shared__ __align__(16) double gs_dyn[];
  double(*ring)[kGsRing] = reinterpret_cast<double(*)[kGsRing]>(gs_dyn);
  // bar[x][k % kNB]: chunk k done by compute warp x (x < kGsWarps), loaded
  // (x = kLoader) or flushed (x = kFlusher)
  __shared__ __align__(8) unsigned long long bar[kGsWarps + 2][kNB];
  __shared__ int s_ticket;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_ticket = atomicAdd(p.ticket, 1);
    for (int x = 0; x < kGsWarps + 2; ++x)
      for (int k = 0; k < kNB; ++k) mbar_init(&bar[x][k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int b = s_ticket;
  const int n = (int)p.n;  // host guarantees n < 2^30
  const double bnd = p.bnd;
  const bool last_block = b == p.nblocks - 1;
  const int nch = (n + kShiftLane31 + kCH - 1) / kCH;  // lane 31 finishes position n-1 in chunk nch-1
  // compute warps with sweeps in this block; the last one feeds the flusher
  const int nw = last_block ? (int)((p.sweeps - (long long)b * kGsWarps * 32 + 31) / 32) : kGsWarps;
  // the staging ring stores position x at (x + soff) & (R-1) so that the
  // emitting lane's stores (runs of kWRun) never wrap (constant offsets)
  const int soff = last_block ? (kGsLag * ((int)((p.sweeps - 1) % 32) + 1)) & (kWRun - 1) : 0;
  auto done = [&](int x, int k) { mbar_wait_uniform(&bar[x][k % kNB], (unsigned)(k / kNB) & 1u); };
  auto signal = [&](int x, int k) {  // all lanes past their work on chunk k
    __syncwarp();
    mbar_arrive_leader(lane == 0, &bar[x][k % kNB]);
  };

  if (w == kLoader) {
    // block b-1's published prefix (or the grid) -> ring[0]
    const double* src = b == 0 ? p.a : p.gbuf + (long long)(b - 1) * p.n;
    for (int k = 0; k < nch; ++k) {
      if (k >= kWar - 1) done(0, k - (kWar - 1));
      const int lo = k * kCH, hi = min(n, lo + kCH);
      if (b > 0 && lo < n) {
        if (lane == 0) {
          SpinGuard sg;
          while (ld_acquire_gpu(p.gprog + b - 1) < hi) {
            __nanosleep(64);
            sg.tick();
          }
        }
        __syncwarp();
      }
      double v[kCH / 32];
#pragma unroll
      for (int s = 0; s < kCH / 32; ++s) {
        const int x = lo + s * 32 + lane;
        v[s] = x < hi ? __ldcg(src + x) : bnd;
      }
#pragma unroll
      for (int s = 0; s < kCH / 32; ++s) ring[0][(lo + s * 32 + lane) & (kGsRing - 1)] = v[s];
      signal(kLoader, k);
    }
    return;
  }
  if (w == kFlusher) {
    // staging ring -> grid (last block) or this block's sweep buffer
    double* dst = last_block ? p.a : p.gbuf + (long long)b * p.n;
    for (int k = 0; k < nch; ++k) {
      done(nw - 1, k);
      const int lo = max(0, k * kCH - kShiftLane31), hi = min(n, (k + 1) * kCH - kShiftLane31);
      for (int x = lo + lane; x < hi; x += 32) dst[x] = ring[kGsWarps][(x + soff) & (kGsRing - 1)];
      if (!last_block) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(p.gprog + b, hi);
      }
      signal(kFlusher, k);
    }
    return;
  }

  // ---- compute warps: lane k of warp w runs sweep 32 * (b * kGsWarps + w) + k ----
  if (w >= nw) return;
  const bool to_staging = w == nw - 1;
  const int wlane = last_block && to_staging ? (int)((p.sweeps - 1) % 32) : 31;  // emits this warp's sweep
  const int wlag = kGsLag * (wlane + 1);
  const int lane_off = kGsLag * (lane + 1);
  const double* rin = ring[w];
  double* rout = to_staging ? ring[kGsWarps] : ring[w + 1];
  const int woff = to_staging ? soff : 0;  // (wlag - woff) % kWRun == 0
  const bool writer = lane == wlane;
  // L: own previous result (new value at i-1); u0, u1, u2: old values at
  // i, i+1, i+2 (C, R, and next step's R); out: this step's result
  double L = bnd, u0 = bnd, u1 = bnd, u2 = bnd, out = bnd;

  for (int ch = 0; ch < nch; ++ch) {
    const int jb0 = ch * kCH;
    // inputs: positions < min(n, jb0 + kCH - 1)
    if (w == 0) {
      done(kLoader, ch);
    } else {
      const int need = min(n, jb0 + kCH - 1);
      done(w - 1, (need + kShiftLane31 + kCH - 1) / kCH - 1);
    }
    // ring space for the positions this chunk writes
    if (to_staging) {
      if (ch >= kWar - 1) done(kFlusher, ch - (kWar - 1));
    } else if (ch >= kWar) {
      done(w + 1, ch - kWar);
    }
    // first input of the next sub-chunk, loaded a sub-chunk ahead (inside the
    // chunk only: position jb0 + kCH - 1 is not yet guaranteed)
    double r0n = rin[(jb0 - 1) & (kGsRing - 1)];
    // ALL: every sub-chunk of this chunk is steady — a separate copy of the
    // sub-chunk loop holding only the steady body (its own register
    // allocation: no per-sub-chunk variant branch or constant reloads)
    auto sub_loop = [&](auto all_tag) {
      constexpr bool ALL = decltype(all_tag)::value;
#pragma unroll 1
      for (int sub = 0; sub < kSub; ++sub) {
        const int jb = jb0 + sub * kSubLen;
        const double r0v = r0n;
        if (sub + 1 < kSub) r0n = rin[(jb + kSubLen - 1) & (kGsRing - 1)];
        // steady sub-chunk: every lane's position (j - 4*(lane+1)) inside
        // [0, n) for the whole sub-chunk — no selects on the chain
        const bool steady = ALL || (jb - kShiftLane31 >= 0 && jb + kSubLen - 1 - kGsLag < n);
        // sub-chunk bases: lane 0 reads position j-1 (only u = 0 can wrap), the
        // emitting lane writes position j - wlag (never wraps, see woff)
        const double* rb = rin + (jb & (kGsRing - 1)) - 1;
        double* wb[kWRuns];
#pragma unroll
        for (int r = 0; r < kWRuns; ++r) wb[r] = rout + ((jb + r * kWRun - wlag + woff) & (kGsRing - 1));
        if (steady && MASK == 7u) {
          // full 3-tap stencil: products w1*C and w2*R are formed a step ahead
          // from values already in registers, so the loop-carried chain is
          // exactly L -> DMUL -> DADD -> DADD (same products, same adds)
          double pa = __dmul_rn(p.w1, u0), pb = __dmul_rn(p.w2, u1);
#pragma unroll
          for (int u = 0; u < kSubLen; ++u) {
            const double sh = __shfl_up_sync(0xffffffffu, out, 1);
            const double rv = u == 0 ? r0v : rb[u];  // same address for all lanes: broadcast
            const double sv = lane == 0 ? rv : sh;    // old(i+3)
            out = __dadd_rn(pb, __dadd_rn(pa, __dmul_rn(p.w0, L)));
            pa = __dmul_rn(p.w1, u1);  // next step's C
            pb = __dmul_rn(p.w2, u2);  // next step's R
            L = out;
            u0 = u1;
            u1 = u2;
            u2 = sv;
            if (writer) wb[u / kWRun][u % kWRun] = out;
          }
        } else if (steady) {
#pragma unroll 32
          for (int u = 0; u < kSubLen; ++u) {
            const double sh = __shfl_up_sync(0xffffffffu, out, 1);
            const double rv = u == 0 ? r0v : rb[u];
            const double sv = lane == 0 ? rv : sh;
            out = gs_taps<MASK>(L, u0, u1, p.w0, p.w1, p.w2);
            L = out;
            u0 = u1;
            u1 = u2;
            u2 = sv;
            if (writer) rout[(jb + u - wlag + woff) & (kGsRing - 1)] = out;
          }
        } else if constexpr (!ALL) {
#pragma unroll 32
          for (int u = 0; u < kSubLen; ++u) {
            const int j = jb + u;
            const double sh = __shfl_up_sync(0xffffffffu, out, 1);
            const int pos = j - 1;
            const double rv = rin[pos & (kGsRing - 1)];
            const double up = (unsigned)pos < (unsigned)n ? rv : bnd;
            const double sv = lane == 0 ? up : sh;
            const int i = j - lane_off;
            const double v = gs_taps<MASK>(L, u0, u1, p.w0, p.w1, p.w2);
            out = (unsigned)i < (unsigned)n ? v : bnd;
            L = out;
            u0 = u1;
            u1 = u2;
            u2 = sv;
            const int po = j - wlag;
            if (writer && (unsigned)po < (unsigned)n) rout[(po + woff) & (kGsRing - 1)] = out;
          }
        }
      }
    };
    if (jb0 - kShiftLane31 >= 0 && jb0 + kCH - 1 - kGsLag < n)
      sub_loop(std::true_type{});
    else
      sub_loop(std::false_type{});
    signal(w, ch);
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
    const int v = e ? atoi(e) : 2;  // measured: 2 compute warps/block >= 4 (config 2)
    return (v == 1 || v == 2 || v == 4) ? v : 2;
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
    constexpr size_t smem = sizeof(double) * (W + 1) * kGsRing;
    auto go = [&](auto kern) {
      // (over 48 KB with the static barriers included)
      if (smem > 40 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<a.nblocks, (W + 2) * 32, smem, s>>>(a);
    };
    switch (mask) {
      case 1: go(gs1d_kernel<1, W>); break;
      case 2: go(gs1d_kernel<2, W>); break;
      case 3: go(gs1d_kernel<3, W>); break;
      case 4: go(gs1d_kernel<4, W>); break;
      case 5: go(gs1d_kernel<5, W>); break;
      case 6: go(gs1d_kernel<6, W>); break;
      default: go(gs1d_kernel<7, W>); break;
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
