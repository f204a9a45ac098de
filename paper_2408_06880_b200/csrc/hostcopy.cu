// Host <-> device copies for the reference-facing calls that take or return
// plain NumPy arrays (init_canonical, canonical_state, macroscopic_fields:
// sparse.py:199-222, :308-331).  Those arrays are ordinary pageable memory;
// a cudaMemcpy from pageable memory goes through the driver's own
// single-threaded bounce buffer (measured: 4.3 GB of macroscopic fields
// in 0.9-1.2 s on the B200 box, vs 0.08 s of DMA).
//
// Here the transfer is split into T contiguous slices, one host thread per
// slice; each thread streams its slice through two pinned chunks of its own
// on its own CUDA stream, so T DMAs run against T host memcpys at once.
// Pinned destinations/sources (cudaHostAlloc / torch pin_memory) skip the
// staging and go straight to one cudaMemcpyAsync.
#include <sys/mman.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.cuh"

namespace slbm {
namespace {

constexpr int kMaxLanes = 16;
constexpr size_t kMinStaged = size_t(4) << 20;  // below this: plain copy
size_t g_chunk = size_t(4) << 20;  // bytes per pinned chunk (tuning knob 10, MiB)
int g_max_threads = 16;            // lanes used per transfer (tuning knob 11; capped by cores)

struct Lane {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};
  char* buf[2] = {nullptr, nullptr};
};

std::mutex g_mu;            // one staged transfer at a time per process
std::vector<Lane> g_lanes;  // kMaxLanes lanes, created for the current device

void drop_lanes() {
  for (Lane& l : g_lanes) {
    cudaSetDevice(l.device);
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(l.done[k]);
      cudaFreeHost(l.buf[k]);
    }
    cudaStreamDestroy(l.stream);
  }
  g_lanes.clear();
}

int lanes_for(int device) {
  if (!g_lanes.empty() && g_lanes[0].device == device) return SLBM_OK;
  drop_lanes();
  g_lanes.assign(kMaxLanes, Lane{});
  cudaSetDevice(device);
  for (Lane& l : g_lanes) {
    l.device = device;
    SLBM_CUDA_TRY(cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      SLBM_CUDA_TRY(cudaEventCreateWithFlags(&l.done[k], cudaEventDisableTiming));
      SLBM_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&l.buf[k]), g_chunk, 0));
    }
  }
  return SLBM_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged;
}

// first-touch page faults on a fresh destination are 2 MB instead of 4 KB
// when transparent huge pages are enabled in "madvise" mode
void advise_huge(void* p, size_t bytes) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~((size_t(2) << 20) - 1);
  if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
}

int threads_for(size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t by_size = (bytes + 4 * g_chunk - 1) / (4 * g_chunk);
  return int(std::max<size_t>(1, std::min<size_t>({size_t(g_max_threads), size_t(hw), by_size})));
}

// dir 0: device -> host, 1: host -> device.  `after` orders the lanes after
// everything already queued on the caller's stream.
int staged(int dir, void* host, void* dev, size_t bytes, int device, cudaStream_t after) {
  std::lock_guard<std::mutex> lock(g_mu);
  SLBM_TRY(lanes_for(device));
  cudaEvent_t ready;
  SLBM_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  SLBM_CUDA_TRY(cudaEventRecord(ready, after));
  const int T = threads_for(bytes);
  const size_t per = (bytes + T - 1) / T;
  std::vector<cudaError_t> err(T, cudaSuccess);
  auto work = [&](int t) {
    cudaSetDevice(device);
    Lane& l = g_lanes[t];
    const size_t lo = std::min(bytes, per * t), hi = std::min(bytes, lo + per);
    char* h = static_cast<char*>(host);
    char* d = static_cast<char*>(dev);
    cudaError_t e = cudaStreamWaitEvent(l.stream, ready, 0);
    if (dir == 0) {
      // DMA chunk k+1 while the host copies chunk k out of the other buffer
      size_t off = lo;
      int k = 0;
      if (off < hi) {
        const size_t n = std::min(g_chunk, hi - off);
        e = e ? e : cudaMemcpyAsync(l.buf[0], d + off, n, cudaMemcpyDeviceToHost, l.stream);
        e = e ? e : cudaEventRecord(l.done[0], l.stream);
      }
      while (off < hi && !e) {
        const size_t n = std::min(g_chunk, hi - off);
        const size_t nxt = off + n;
        if (nxt < hi) {
          const size_t m = std::min(g_chunk, hi - nxt);
          e = cudaMemcpyAsync(l.buf[k ^ 1], d + nxt, m, cudaMemcpyDeviceToHost, l.stream);
          e = e ? e : cudaEventRecord(l.done[k ^ 1], l.stream);
        }
        e = e ? e : cudaEventSynchronize(l.done[k]);
        if (!e) std::memcpy(h + off, l.buf[k], n);
        off = nxt;
        k ^= 1;
      }
    } else {
      // host copies chunk k into a buffer while chunk k-1 is in flight
      int k = 0;
      bool used[2] = {false, false};
      for (size_t off = lo; off < hi && !e; off += g_chunk, k ^= 1) {
        const size_t n = std::min(g_chunk, hi - off);
        if (used[k]) e = cudaEventSynchronize(l.done[k]);
        if (e) break;
        std::memcpy(l.buf[k], h + off, n);
        e = cudaMemcpyAsync(d + off, l.buf[k], n, cudaMemcpyHostToDevice, l.stream);
        e = e ? e : cudaEventRecord(l.done[k], l.stream);
        used[k] = true;
      }
      e = e ? e : cudaStreamSynchronize(l.stream);
    }
    err[t] = e;
  };
  if (dir == 0) advise_huge(host, bytes);
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  cudaEventDestroy(ready);
  for (cudaError_t e : err) SLBM_CUDA_TRY(e);
  return SLBM_OK;
}

}  // namespace

// allocate the pinned lanes ahead of the first large transfer (engine
// creation does this for blocks whose state is large)
int hostcopy_reserve(int device) {
  std::lock_guard<std::mutex> lock(g_mu);
  return lanes_for(device);
}

// knob 12: fields for pinned destinations written by the field kernel
// straight into mapped host memory (1) or staged in HBM and copied by the
// DMA engine (0, default).  Mapped writes measured 50 GB/s on most boxes
// but 5.6 GB/s on one (round 1); the DMA copy runs at the link rate on all.
int g_mapped_out = 0;

bool mapped_out_enabled() { return g_mapped_out != 0; }

int hostcopy_tune(int knob, int value) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (knob == 12) {
    g_mapped_out = value;
    return SLBM_OK;
  }
  if (value <= 0) return fail(SLBM_ECONFIG, "host copy tuning value must be positive");
  if (knob == 10) {
    drop_lanes();
    g_chunk = size_t(value) << 20;
  } else {
    g_max_threads = std::min(value, kMaxLanes);
  }
  return SLBM_OK;
}

// device-visible address of a pinned (page-locked, mapped) host buffer, or
// nullptr for pageable memory
void* mapped_device_ptr(void* host) {
  if (!is_pinned(host)) return nullptr;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, host, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return d;
}

int copy_d2h(void* host, const void* dev, size_t bytes, int device, cudaStream_t s) {
  if (!bytes) return SLBM_OK;
  if (bytes < kMinStaged || is_pinned(host)) {
    SLBM_CUDA_TRY(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
    SLBM_CUDA_TRY(cudaStreamSynchronize(s));
    return SLBM_OK;
  }
  return staged(0, host, const_cast<void*>(dev), bytes, device, s);
}

int copy_h2d(void* dev, const void* host, size_t bytes, int device, cudaStream_t s) {
  if (!bytes) return SLBM_OK;
  if (bytes < kMinStaged || is_pinned(host)) {
    SLBM_CUDA_TRY(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
    SLBM_CUDA_TRY(cudaStreamSynchronize(s));
    return SLBM_OK;
  }
  // the caller's stream must not run ahead into the destination before the
  // lanes have written it: lanes finish synchronously, so nothing to join
  return staged(1, const_cast<void*>(host), dev, bytes, device, s);
}

}  // namespace slbm
