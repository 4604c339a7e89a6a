// K6: 2D radius-1 Gauss-Seidel (lexicographic order) as a time-lane pipeline.
//
// Replaces gs2d_temporal (reference kernels_nd.py:48-50, star-only there) for
// the row-major in-place sweep of BASELINE config 4 (9-point box), bit-exact
// with the oracle's lexicographic loop (oracle/oracle.py gs_sweep_loop; the
// reference loop test test_baselines.py:39-52).
//
// The paper's time lanes, on a GPU: lane t of a "group" runs sweep t, and
// group d owns the units {(sweep t, row d - t)}: a diagonal through
// (time, row) space.  With a lexicographic sweep every input of unit
// (t, i) comes from exactly three places:
//   * row i-1, sweep t   (NW, N, NE: new)      = group d-1, lane t
//   * row i,   sweep t-1 (C, E: old)           = group d-1, lane t-1
//   * row i+1, sweep t-1 (SW, S, SE: old)      = group d,   lane t-1
// plus W = the lane's own previous output.  So data only ever flows from
// group d-1 to group d and from lane t-1 to lane t: a one-directional chain.
//
//   * lanes:  lane t trails lane t-1 by lambda = 2 columns (its SE input is
//             what lane t-1 produced one step earlier: __shfl_up);
//   * warps:  a group is 4 warps (128 lanes = 128 sweeps); warp w trails
//             warp w-1 by mu extra columns (its lane 0 reads lane 31 of the
//             previous warp from shared memory);
//   * groups: group g of a block trails group g-1 by Lambda columns and
//             reads its outputs from a shared-memory ring indexed by
//             *iteration* (not column), so the 254-column lane skew inside a
//             group costs no ring space;
//   * blocks: G = 4 groups per block; one IO warp per block streams in the
//             previous block's last group (a tagged global ring, L2-resident)
//             and the grid rows the chain starts from, and drains this
//             block's last group to the next block.  Blocks take tickets and
//             only wait on lower tickets (plus bounded back-pressure), so the
//             launch is deadlock-free.
// "Virtual lane -1" of group g (ring slot 0) is grid row d_g + 1 at sweep
// t0 - 1: lane 0 reads its old own row / row below from there.  Lanes past
// the requested sweep count are identity lanes.  Lane 127 writes the final
// sweep of row d - 127 back to the grid in place.
#include <algorithm>
#include <climits>

#include "common.cuh"

namespace tvs {

namespace gs2p {
constexpr int kLanes = 128;          // sweeps per pass (4 warps)
constexpr int kWarpsG = 4;
constexpr int kG = 4;                // groups per block
constexpr int kC = 4;                // iterations per chunk (sync granularity)
constexpr int kR = 32;               // ring depth (iterations), power of two
constexpr int kSlots = kLanes + 2;   // [0] virtual lane -1, [1] pad, [2 + t] lane t (16-B aligned pairs)
constexpr int kLam = 2;              // column lag lane t-1 -> t
constexpr int kMu = 3;               // extra lag warp w-1 -> w (>= kC + 1 - kLam)
constexpr int kBig = 5;              // lag group g-1 -> g (>= kC + 1)
constexpr int kBase = 10;            // every producer starts left of column 0 (>= kLam + kBig + 2)
constexpr int kRG = 256;             // global ring depth (iterations)
constexpr int kK = 256;              // global ring slots (boundaries in flight)
constexpr int kPub = 8;              // IO warp publishes downstream every kPub chunks
constexpr int kComputeWarps = kG * kWarpsG;
constexpr int kThreads = (kComputeWarps + 2) * 32;  // + loader warp + drainer warp
constexpr size_t kSmem = sizeof(double) * (size_t)(kG + 1) * kR * kSlots;
static_assert(kMu >= kC + 1 - kLam && kBig >= kC + 1, "lags too small for chunked sync");
}  // namespace gs2p

struct Gs2pArgs {
  double* a;                 // interior origin (in place)
  long long s0;              // row pitch (elements)
  int e0, e1;                // rows, columns
  int sweeps;                // real sweeps this pass (<= 128)
  int nctas;
  int c_end;                 // iterations per warp (multiple of kC)
  double* gring;             // kK * kRG * 128
  unsigned long long* gprod; // kK tagged counters: (boundary+1) << 32 | iterations written
  unsigned long long* gcons; // kK tagged counters: (boundary+1) << 32 | iterations consumed
  int* ticket;
  double w[9];
  double bnd;
};

__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Wait until a shared-memory progress counter reaches `v`; back off so the
// spinning warps do not starve the IO warp of issue slots.
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  if (ld_acq_cta(p) >= v) return;
  SpinGuard sg;
  while (ld_acq_cta(p) < v) {
    __nanosleep(40);
    sg.tick();
  }
}

// taps in sorted order: NW N NE W C E SW S SE (mask bit k = position k)
template <unsigned MASK>
__device__ __forceinline__ double gs9(const double* w, double nw, double n, double ne, double ww, double c, double e,
                                      double sw, double s, double se) {
  const double v[9] = {nw, n, ne, ww, c, e, sw, s, se};
  double acc = 0.0;
  bool first = true;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if ((MASK >> k) & 1u) {
      acc = first ? tap_first(w[k], v[k]) : tap_next<false>(w[k], v[k], acc);
      first = false;
    }
  }
  return acc;
}

template <unsigned MASK>
__global__ void __launch_bounds__(gs2p::kThreads, 1) gs2d_pipe_kernel(Gs2pArgs p) {
  using namespace gs2p;
  extern __shared__ __align__(16) double smem[];
  // rings[0] = phantom (previous block's last group), rings[g+1] = group g
  auto ring = [&](int gi, int it, int slot) -> double& {
    return smem[((size_t)gi * kR + (it & (kR - 1))) * kSlots + (slot == 0 ? 0 : slot + 1)];
  };
  auto ring_lane0 = [&](int gi, int it) -> double* { return &smem[((size_t)gi * kR + (it & (kR - 1))) * kSlots + 2]; };
  __shared__ int prog[kComputeWarps];
  __shared__ int io_load, io_store;
  __shared__ int s_ticket;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1);
  if (threadIdx.x < kComputeWarps) prog[threadIdx.x] = 0;
  if (threadIdx.x == 0) io_load = io_store = 0;
  __syncthreads();
  const int n = s_ticket;           // block index along the chain
  const int d0 = n * kG;            // first group (diagonal) of this block
  const int nch = p.c_end / kC;
  const double bnd = p.bnd;
  const int e0 = p.e0, e1 = p.e1;

  const bool has_up = n > 0, has_down = n + 1 < p.nctas;
  const int up_slot = (n + kK - 1) % kK, dn_slot = n % kK;
  const unsigned long long up_tag = (unsigned long long)n << 32;        // boundary n-1 -> tag n
  const unsigned long long dn_tag = (unsigned long long)(n + 1) << 32;  // boundary n -> tag n+1
  if (wi == kComputeWarps) {
    // ============ loader warp: grid rows (slot 0) + previous block's last group ============
    const double* up_ring = p.gring + (size_t)up_slot * kRG * kLanes;
    unsigned long long up_seen = 0;
    SpinGuard guard;
    for (int kl = 0; kl < nch; ++kl) {
      const int it_lo = kl * kC, it_hi = it_lo + kC;
      // WAR: every compute warp finished chunk kl-5 (ring chunk kl-8 reusable)
      const int need = (kl - 4) * kC;
      // upstream data for producer iterations up to it_hi + Lambda*G
      const int up_need = min(it_hi + kBig * kG, p.c_end);
      for (;;) {
        const int mine = lane < kComputeWarps ? ld_acq_cta(&prog[lane]) : INT_MAX;
        bool ok = __reduce_min_sync(0xffffffffu, mine) >= need;
        if (ok && has_up && ((up_seen >> 32) != (up_tag >> 32) || (up_seen & 0xffffffffull) < (unsigned long long)up_need)) {
          up_seen = lane == 0 ? ld_acq_gpu(p.gprod + up_slot) : 0ull;
          up_seen = __shfl_sync(0xffffffffu, up_seen, 0);
          ok = (up_seen >> 32) == (up_tag >> 32) && (up_seen & 0xffffffffull) >= (unsigned long long)up_need;
        }
        if (ok) break;
        __nanosleep(20);
        guard.tick();
      }
      // slot 0 of rings -1..G-1: grid row d0+g+1 at column it + lam - Lambda*g - base
      if (lane < (kG + 1) * kC) {
        const int g = lane / kC - 1, it = it_lo + lane % kC;
        const int row = d0 + g + 1, col = it + kLam - kBig * g - kBase;
        double* dst = &ring(g + 1, it, 0);
        if (row >= 0 && row < e0 && col >= 0 && col < e1) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(p.a + (long long)row * p.s0 + col));
        } else {
          *dst = bnd;
        }
      }
      // phantom lanes: 4 iterations x 64 pairs, 16-byte copies (L2 only: the
      // global ring is rewritten every kRG iterations)
#pragma unroll
      for (int q = 0; q < kC * kLanes / 64; ++q) {
        const int e = lane + 32 * q;  // pair index
        const int it = it_lo + e / (kLanes / 2), t = 2 * (e % (kLanes / 2));
        const int pit = it + kBig * kG;
        double* dst = ring_lane0(0, it) + t;
        if (has_up && pit < p.c_end) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(up_ring + (size_t)(pit % kRG) * kLanes + t));
        } else {
          dst[0] = bnd;
          dst[1] = bnd;
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
      // publish the previous chunk once its copies landed (two chunks in flight)
      if (kl > 0) {
        asm volatile("cp.async.wait_group 1;\n" ::);
        __syncwarp();
        if (lane == 0) st_rel_cta(&io_load, it_lo);
      }
      if (has_up && ((kl + 1) % kPub == 0 || kl + 1 == nch)) {
        // everything below producer iteration it_hi + Lambda*G is staged in
        // smem; the global slots it came from may be rewritten
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncwarp();
        if (lane == 0) st_rel_gpu(p.gcons + up_slot, up_tag | (unsigned long long)min(it_hi + kBig * kG, p.c_end));
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();
    if (lane == 0) st_rel_cta(&io_load, p.c_end);
    return;
  }
  if (wi == kComputeWarps + 1) {
    // ============ drainer warp: last group -> next block (global ring) ============
    double* dn_ring = p.gring + (size_t)dn_slot * kRG * kLanes;
    bool slot_ok = !has_down || n < kK;
    unsigned long long dn_cons_seen = 0;
    SpinGuard guard;
    for (int ks = 0; ks < nch; ++ks) {
      const int lo = ks * kC;
      for (;;) {
        const int mine = lane < kWarpsG ? ld_acq_cta(&prog[(kG - 1) * kWarpsG + lane]) : INT_MAX;
        bool ok = __reduce_min_sync(0xffffffffu, mine) >= lo + kC;
        if (ok && has_down && !slot_ok) {  // previous user of this global slot fully consumed
          unsigned long long v = lane == 0 ? ld_acq_gpu(p.gcons + dn_slot) : 0ull;
          v = __shfl_sync(0xffffffffu, v, 0);
          slot_ok = v >= (((unsigned long long)(n + 1 - kK) << 32) | (unsigned long long)p.c_end);
          ok = slot_ok;
        }
        if (ok && has_down && lo + kC > kRG) {  // global back-pressure
          const unsigned long long need = dn_tag | (unsigned long long)(lo + kC - kRG);
          if (dn_cons_seen < need) {
            unsigned long long v = lane == 0 ? ld_acq_gpu(p.gcons + dn_slot) : 0ull;
            dn_cons_seen = __shfl_sync(0xffffffffu, v, 0);
          }
          ok = dn_cons_seen >= need;
        }
        if (ok) break;
        __nanosleep(20);
        guard.tick();
      }
      if (has_down) {
#pragma unroll
        for (int q = 0; q < kC * kLanes / 64; ++q) {
          const int e = lane + 32 * q;
          const int it = lo + e / (kLanes / 2), t = 2 * (e % (kLanes / 2));
          const double2 v = *reinterpret_cast<const double2*>(ring_lane0(kG, it) + t);
          *reinterpret_cast<double2*>(dn_ring + (size_t)(it % kRG) * kLanes + t) = v;
        }
      }
      __syncwarp();
      if (lane == 0) st_rel_cta(&io_store, lo + kC);
      if (has_down && ((ks + 1) % kPub == 0 || ks + 1 == nch)) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_rel_gpu(p.gprod + dn_slot, dn_tag | (unsigned long long)(lo + kC));
      }
    }
    return;
  }

  // ======================= compute warps =======================
  const int g = wi / kWarpsG, w = wi % kWarpsG;
  const int t = w * 32 + lane;           // lane index in the group = sweep offset
  const int d = d0 + g;                  // diagonal of this group
  const int row = d - t;
  const bool row_ok = row >= 0 && row < e0;
  const bool real = t < p.sweeps;
  const int col_off = kBase + kLam * t + kMu * w + kBig * g;  // column = iteration - col_off
  const int offE = 1 - kLam - kBig - ((lane == 0 && w > 0) ? kMu : 0);
  const int offSE = 1 - kLam - (w > 0 ? kMu : 0);   // lane 0 only
  const int slotE = t;                               // lane t-1 (or virtual lane -1)
  const int slotSE = w * 32;
  const int gi_prev = g, gi_cur = g + 1;
  const bool last_lane = t == kLanes - 1;
  double* out_row = p.a + (long long)(row_ok ? row : 0) * p.s0;
  double wk[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) wk[k] = p.w[k];
  const bool warp_rows_ok = __all_sync(0xffffffffu, row_ok && real);
  // progress of the warps I read from / that read me
  const int* dep_prev = g > 0 ? &prog[(g - 1) * kWarpsG + w] : &io_load;
  const int* dep_prev2 = g > 0 ? &prog[(g - 1) * kWarpsG + (w > 0 ? w - 1 : 0)] : &io_load;
  const int* dep_left = w > 0 ? &prog[g * kWarpsG + w - 1] : &io_load;
  const int* war0 = g + 1 < kG ? &prog[(g + 1) * kWarpsG + w] : &io_store;
  const int* war1 = g + 1 < kG ? &prog[(g + 1) * kWarpsG + (w + 1 < kWarpsG ? w + 1 : w)] : &io_store;
  const int* war2 = w + 1 < kWarpsG ? &prog[g * kWarpsG + w + 1] : war0;

  double nw = bnd, nn = bnd, ne = bnd, cc = bnd, ee = bnd, sw = bnd, ss = bnd, se = bnd, ww = bnd, out = bnd;

  for (int k = 0; k < nch; ++k) {
    const int cb = k * kC;
    // RAW: producers finished chunk k-1 (lags >= chunk + dependency distance);
    // WAR: readers of my ring slots finished chunk k-5.  All counters are
    // read with independent loads, one round trip per poll.
    {
      const int need = (k - 4) * kC;
      SpinGuard sg;
      for (;;) {
        const int v0 = ld_acq_cta(dep_prev), v1 = ld_acq_cta(dep_prev2), v2 = ld_acq_cta(dep_left);
        const int v3 = (g == 0 || w == 0) ? ld_acq_cta(&io_load) : INT_MAX;
        const int v4 = ld_acq_cta(war0), v5 = ld_acq_cta(war1), v6 = ld_acq_cta(war2);
        const bool raw_ok = v0 >= cb && v1 >= cb && v2 >= cb && v3 >= cb + kC;
        const bool war_ok = need <= 0 || (v4 >= need && v5 >= need && v6 >= need);
        if (raw_ok && war_ok) break;
        __nanosleep(32);
        sg.tick();
      }
    }
    // steady chunk: all columns of the chunk inside [0, e1), every lane real
    // and on a grid row, and no negative ring iterations
    const int jmin = cb - (kBase + kLam * (w * 32 + 31) + kMu * w + kBig * g);
    const int jmax = cb + kC - 1 - (kBase + kLam * (w * 32) + kMu * w + kBig * g);
    const bool steady = warp_rows_ok && jmin >= 0 && jmax < e1 && cb + offE - kMu >= 0;
    if (steady) {
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        const int c = cb + u;
        const double ne_new = ring(gi_prev, c + 1 - kBig, t + 1);
        const double e_new = ring(gi_prev, c + offE, slotE);
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const double sl = ring(gi_cur, c + offSE, slotSE);
        const double se_new = lane == 0 ? sl : sh;
        nw = nn; nn = ne; ne = ne_new;
        cc = ee; ee = e_new;
        sw = ss; ss = se; se = se_new;
        out = gs9<MASK>(wk, nw, nn, ne, ww, cc, ee, sw, ss, se);
        ww = out;
        ring(gi_cur, c, t + 1) = out;
        if (last_lane) out_row[c - col_off] = out;
      }
    } else {
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        const int c = cb + u;
        const int j = c - col_off;
        const int i1 = c + 1 - kBig, i2 = c + offE, i3 = c + offSE;
        const double ne_new = i1 >= 0 ? ring(gi_prev, i1, t + 1) : bnd;
        const double e_new = i2 >= 0 ? ring(gi_prev, i2, slotE) : bnd;
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const double sl = i3 >= 0 ? ring(gi_cur, i3, slotSE) : bnd;
        const double se_new = lane == 0 ? sl : sh;
        nw = nn; nn = ne; ne = ne_new;
        cc = ee; ee = e_new;
        sw = ss; ss = se; se = se_new;
        const double v = gs9<MASK>(wk, nw, nn, ne, ww, cc, ee, sw, ss, se);
        const bool inside = row_ok && j >= 0 && j < e1;
        out = inside ? (real ? v : cc) : bnd;
        ww = out;
        ring(gi_cur, c, t + 1) = out;
        if (last_lane && inside) out_row[j] = out;
      }
    }
    __syncwarp();
    if (lane == 0) st_rel_cta(&prog[wi], cb + kC);
  }
}

static unsigned gs_mask2d(const tvs_stencil& st, double w[9]) {
  unsigned mask = 0;
  int last = -1;
  for (int k = 0; k < 9; ++k) w[k] = 0.0;
  for (int k = 0; k < st.ntaps; ++k) {
    const int pos = (st.offsets[k][0] + 1) * 3 + (st.offsets[k][1] + 1);
    if (pos <= last) return 0;
    last = pos;
    mask |= 1u << pos;
    w[pos] = st.coeffs[k];
  }
  return mask;
}

bool gs2d_pipe_supported(const tvs_stencil& st) {
  double w[9];
  const unsigned m = gs_mask2d(st, w);
  constexpr unsigned kStar = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);
  return m == 0x1FFu || m == kStar;
}

int gs2d_pipeline(const tvs_stencil& st, const tvs_geometry& g, double* grid, int64_t steps, cudaStream_t s) {
  using namespace gs2p;
  double w[9];
  const unsigned mask = gs_mask2d(st, w);
  constexpr unsigned kStar = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);
  if (mask != 0x1FFu && mask != kStar) return fail(TVS_ERR_UNSUPPORTED, "gs2d_pipeline: tap set");
  if (g.extents[0] >= (1ll << 30) || g.extents[1] >= (1ll << 30)) return fail(TVS_ERR_UNSUPPORTED, "gs2d_pipeline: extent");
  Gs2pArgs a{};
  a.a = grid + g.origin;
  a.s0 = g.strides[0];
  a.e0 = (int)g.extents[0];
  a.e1 = (int)g.extents[1];
  const int ngroups = a.e0 + kLanes - 1;
  a.nctas = (ngroups + kG - 1) / kG;
  const int skew = kLam * (kLanes - 1) + kMu * (kWarpsG - 1) + kBig * (kG - 1);
  a.c_end = ((a.e1 + 2 + kBase + skew + kBig * kG + kC - 1) / kC) * kC;
  for (int k = 0; k < 9; ++k) a.w[k] = w[k];
  a.bnd = st.boundary;
  const size_t ring_bytes = sizeof(double) * (size_t)kK * kRG * kLanes;
  const size_t ctrl_bytes = sizeof(unsigned long long) * 2 * kK + 64;
  a.gring = static_cast<double*>(scratch(ring_bytes, 0));
  char* ctrl = static_cast<char*>(scratch(ctrl_bytes, 1));
  if (!a.gring || !ctrl) return fail(TVS_ERR_CUDA, "gs2d_pipeline: scratch");
  a.gprod = reinterpret_cast<unsigned long long*>(ctrl);
  a.gcons = a.gprod + kK;
  a.ticket = reinterpret_cast<int*>(a.gcons + kK);
  auto kern = mask == 0x1FFu ? gs2d_pipe_kernel<0x1FFu> : gs2d_pipe_kernel<kStar>;
  TVS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
  for (int64_t done = 0; done < steps; done += kLanes) {
    a.sweeps = (int)std::min<int64_t>(kLanes, steps - done);
    TVS_CUDA(cudaMemsetAsync(ctrl, 0, ctrl_bytes, s));
    kern<<<a.nctas, kThreads, kSmem, s>>>(a);
    TVS_LAUNCHED("gs2d_pipe_kernel");
  }
  return TVS_OK;
}

}  // namespace tvs
