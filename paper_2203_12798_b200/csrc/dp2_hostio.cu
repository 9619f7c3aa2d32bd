// Host side of large device -> host readbacks (the Q factor of a fit):
// dp2_d2h_staged streams a device buffer into pageable host memory at PCIe
// speed.  Chunks go by cudaMemcpyAsync into a ring of pinned staging buffers
// (allocated once: pinning costs ~0.5 ms/MB, far more than the copy), and a
// persistent pool of host threads copies each landed chunk out while the
// following chunks are in flight.  (Per-chunk thread dispatch from Python
// measured ~28 GB/s against the link's ~56 GB/s.)
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "dp2_internal.h"

namespace {

// Persistent copy team: run() splits one memcpy over the workers and the
// calling thread and returns when every slice is done.
class CopyTeam {
 public:
  explicit CopyTeam(int workers) {
    for (int i = 0; i < workers; ++i) threads_.emplace_back([this, i] { loop(i); });
  }
  ~CopyTeam() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  void run(char* dst, const char* src, size_t n) {
    const int parts = (int)threads_.size() + 1;
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = dst;
      src_ = src;
      n_ = n;
      parts_ = parts;
      pending_ = (int)threads_.size();
      ++gen_;
    }
    cv_.notify_all();
    slice(parts - 1);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  void slice(int i) {
    // 4 KB-aligned slices (whole pages per thread)
    const size_t per = ((n_ + parts_ - 1) / parts_ + 4095) & ~size_t(4095);
    const size_t a = std::min(n_, per * i), b = std::min(n_, a + per);
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(int i) {
    int seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      slice(i);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  int gen_ = 0, pending_ = 0, parts_ = 1;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
};

constexpr size_t kChunk = 32u << 20;
constexpr int kRing = 4;

struct Staging {
  char* buf[kRing] = {};
  cudaEvent_t ev[kRing] = {};
  CopyTeam* team = nullptr;
  int device = -1;
};
std::mutex g_stage_mu;
Staging g_stage;

cudaError_t ensure_staging(int dev) {
  if (g_stage.device == dev) return cudaSuccess;
  // the ring's last copies may still be landing (an earlier call that
  // returned on an error): finish them before the buffers go away
  for (int i = 0; i < kRing; ++i)
    if (g_stage.ev[i]) cudaEventSynchronize(g_stage.ev[i]);
  for (int i = 0; i < kRing; ++i) {
    if (g_stage.buf[i]) cudaFreeHost(g_stage.buf[i]);
    if (g_stage.ev[i]) cudaEventDestroy(g_stage.ev[i]);
    g_stage.buf[i] = nullptr;
    g_stage.ev[i] = nullptr;
  }
  g_stage.device = -1;
  for (int i = 0; i < kRing; ++i) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&g_stage.buf[i]), kChunk, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    e = cudaEventCreateWithFlags(&g_stage.ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  if (!g_stage.team) {
    const int hw = (int)std::thread::hardware_concurrency();
    g_stage.team = new CopyTeam(std::max(0, std::min(8, hw) - 1));
  }
  g_stage.device = dev;
  return cudaSuccess;
}

}  // namespace

namespace dp2 {

cudaError_t d2h_staged(void* dst, const void* src, size_t n, cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_stage_mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = ensure_staging(dev);
  if (e != cudaSuccess) return e;
  const size_t nch = (n + kChunk - 1) / kChunk;
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  auto issue = [&](size_t i) {
    const size_t o = i * kChunk, nb = std::min(kChunk, n - o);
    cudaError_t ei = cudaMemcpyAsync(g_stage.buf[i % kRing], s + o, nb, cudaMemcpyDeviceToHost, st);
    if (ei == cudaSuccess) ei = cudaEventRecord(g_stage.ev[i % kRing], st);
    return ei;
  };
  // on any error, drain the stream before returning: chunk copies already
  // issued into the pinned ring must not land after the next call reuses it
  auto bail = [&](cudaError_t err) {
    cudaStreamSynchronize(st);
    return err;
  };
  for (size_t i = 0; i < std::min<size_t>(kRing, nch); ++i)
    if ((e = issue(i)) != cudaSuccess) return bail(e);
  for (size_t i = 0; i < nch; ++i) {
    if ((e = cudaEventSynchronize(g_stage.ev[i % kRing])) != cudaSuccess) return bail(e);
    const size_t o = i * kChunk, nb = std::min(kChunk, n - o);
    g_stage.team->run(d + o, g_stage.buf[i % kRing], nb);
    if (i + kRing < nch && (e = issue(i + kRing)) != cudaSuccess) return bail(e);
  }
  return cudaSuccess;
}

}  // namespace dp2
