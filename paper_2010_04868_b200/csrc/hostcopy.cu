// Host -> device copies of the drop-in path from pageable host memory.
//
// The reference's stencil-run functions take and return ordinary NumPy
// arrays (kernels_nd.py:38-40,91: grid.copy()), i.e. pageable memory.  A
// cudaMemcpy from pageable memory is staged by the driver through a small
// internal buffer with one host thread: ~10 GB/s on the B200 box against ~55
// GB/s of PCIe (config 3: 211 ms vs 54 ms end to end, tools/stock_probe.py).
// Here the library stages instead: the rows are copied by a pool of host
// threads into page-locked staging slots (32 MiB each, reused round robin),
// and each slot is DMA'd to the device as soon as it is filled, while the
// next one fills.  Page-locked sources skip all of this (direct DMA).
//
// The unit is a 3-D block of rows: nplanes x nrows rows of `width` bytes,
// with independent row / plane pitches on the host and on the device (2-D
// grids are one plane, 1-D grids one row).
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tvs {
namespace {

// Persistent worker threads for parallel host memcpy (one job at a time per
// caller; callers serialise on the pool mutex).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();  // never destroyed: workers live for the process
    return *p;
  }
  int size() const { return (int)workers_.size() + 1; }
  // fn(k) for k in [0, n): the caller runs share 0 itself
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> job(job_mu_);
    if (n <= 1 || workers_.empty()) {
      for (int k = 0; k < n; ++k) fn(k);
      return;
    }
    {
      std::unique_lock<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_ = 1;
      pending_ = (int)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    for (int k = 0; k < n; k += size()) fn(k);  // my share
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  CopyPool() {
    const char* e = getenv("TVS_COPY_THREADS");
    int t = e ? atoi(e) : (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    for (int i = 1; i < t; ++i) workers_.emplace_back([this, i] { loop(i); });
    for (auto& w : workers_) w.detach();
  }
  void loop(int me) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* fn;
      int n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        fn = fn_;
        n = n_;
      }
      for (int k = me; k < n; k += size()) (*fn)(k);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

constexpr size_t kSlotBytes = 32ull << 20;
constexpr int kSlots = 4;

// per-thread page-locked staging slots (the drop-in calls of one thread
// stage through them in order)
struct Staging {
  char* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  int device[kSlots] = {-1, -1, -1, -1};
  int next = 0;
  ~Staging() { release(); }
  void release() {
    for (int i = 0; i < kSlots; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]), ev[i] = nullptr;
      if (slot[i]) cudaFreeHost(slot[i]), slot[i] = nullptr;
    }
    next = 0;
  }
};
thread_local Staging g_stage;

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
  cudaGetLastError();
  return ok;
}

}  // namespace

void release_staging() { g_stage.release(); }

int upload_block(char* dst, size_t drow, size_t dplane, const char* src, size_t srow, size_t splane, size_t width,
                 int64_t nrows, int64_t nplanes, cudaStream_t s) {
  if (nrows <= 0 || nplanes <= 0 || width == 0) return TVS_OK;
  static const bool never = getenv("TVS_NO_STAGING") != nullptr;  // A/B switch: driver-staged pageable copies
  if (never || is_pinned(src)) {
    if (nplanes == 1) {
      TVS_CUDA(cudaMemcpy2DAsync(dst, drow, src, srow, width, nrows, cudaMemcpyHostToDevice, s));
    } else {
      for (int64_t z = 0; z < nplanes; ++z)
        TVS_CUDA(cudaMemcpy2DAsync(dst + z * dplane, drow, src + z * splane, srow, width, nrows,
                                   cudaMemcpyHostToDevice, s));
    }
    return TVS_OK;
  }
  int dev = 0;
  TVS_CUDA(cudaGetDevice(&dev));
  Staging& st = g_stage;
  const int64_t per = std::max<int64_t>(1, (int64_t)(kSlotBytes / width));  // rows per slot
  const int64_t total = nrows * nplanes;
  CopyPool& pool = CopyPool::get();
  for (int64_t q0 = 0; q0 < total; q0 += per) {
    const int64_t q1 = std::min(total, q0 + per);
    const int k = st.next;
    st.next = (st.next + 1) % kSlots;
    if (!st.slot[k] || st.device[k] != dev) {
      if (st.ev[k]) cudaEventDestroy(st.ev[k]), st.ev[k] = nullptr;
      if (st.slot[k]) cudaFreeHost(st.slot[k]), st.slot[k] = nullptr;
      TVS_CUDA(cudaHostAlloc((void**)&st.slot[k], std::max(kSlotBytes, width), cudaHostAllocPortable));
      TVS_CUDA(cudaEventCreateWithFlags(&st.ev[k], cudaEventDisableTiming));
      st.device[k] = dev;
    } else {
      TVS_CUDA(cudaEventSynchronize(st.ev[k]));  // the slot's previous DMA has read it
    }
    char* slot = st.slot[k];
    // fill: rows q0 .. q1-1 (row q = plane q / nrows, row q % nrows), compact
    const int64_t n = q1 - q0;
    const int parts = (int)std::min<int64_t>(n, (int64_t)pool.size() * 2);
    pool.run(parts, [&](int part) {
      const int64_t a = q0 + n * part / parts, b = q0 + n * (part + 1) / parts;
      for (int64_t q = a; q < b; ++q)
        std::memcpy(slot + (q - q0) * width, src + (q / nrows) * splane + (q % nrows) * srow, width);
    });
    // DMA: one 2-D copy per plane segment of the chunk
    for (int64_t q = q0; q < q1;) {
      const int64_t z = q / nrows, r = q % nrows;
      const int64_t cnt = std::min(q1 - q, nrows - r);
      TVS_CUDA(cudaMemcpy2DAsync(dst + z * dplane + r * drow, drow, slot + (q - q0) * width, width, width, cnt,
                                 cudaMemcpyHostToDevice, s));
      q += cnt;
    }
    TVS_CUDA(cudaEventRecord(st.ev[k], s));
  }
  return TVS_OK;
}

}  // namespace tvs
