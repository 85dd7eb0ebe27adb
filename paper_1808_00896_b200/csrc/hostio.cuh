// Host <-> device copies of the host-buffer entry points (so3_fsoft_host / so3_ifsoft_host).
//
// The reference's callers pass ordinary numpy arrays: pageable memory.  A cudaMemcpy from or
// to pageable memory is staged by the driver through its own pinned buffers on one host thread
// (measured 6.5 GB/s for the B = 512 round trip with fresh outputs, whose first-touch page
// faults that one thread also pays).  Here pageable transfers are split into fixed chunks
// spread over W worker threads; each worker owns two pinned bounce buffers and a stream, so it
// copies chunk k on the CPU while the DMA of chunk k - 1 is in flight, and the W workers'
// memcpys (and page faults) run in parallel.  Pinned (page-locked or registered) buffers are
// copied directly.  The bounce buffers belong to the plan and are allocated on the first
// pageable transfer, never on a device-only path.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace so3host {

// pinned / registered host memory can be handed to the DMA engines as it is
inline bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

struct Staging {
  int workers = 0;
  size_t chunk = 0;
  std::vector<void*> buf;             // 2 per worker
  std::vector<cudaStream_t> stream;   // 1 per worker
  std::vector<cudaEvent_t> ev;        // 2 per worker

  bool ready() const { return workers > 0; }

  cudaError_t init(int device, int nworkers, size_t chunk_bytes) {
    if (ready()) return cudaSuccess;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaError_t e = cudaSuccess;
    buf.assign(2 * nworkers, nullptr);
    stream.assign(nworkers, nullptr);
    ev.assign(2 * nworkers, nullptr);
    for (int i = 0; i < 2 * nworkers && e == cudaSuccess; ++i) e = cudaHostAlloc(&buf[i], chunk_bytes, cudaHostAllocPortable);
    for (int w = 0; w < nworkers && e == cudaSuccess; ++w) e = cudaStreamCreateWithFlags(&stream[w], cudaStreamNonBlocking);
    for (int i = 0; i < 2 * nworkers && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      release();
      return e;
    }
    workers = nworkers;
    chunk = chunk_bytes;
    return cudaSuccess;
  }

  void release() {
    for (void* p : buf)
      if (p) cudaFreeHost(p);
    for (cudaStream_t s : stream)
      if (s) cudaStreamDestroy(s);
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    buf.clear();
    stream.clear();
    ev.clear();
    workers = 0;
  }

  // worker w moves chunks w, w + W, w + 2W, ... of [0, bytes); dir > 0: host -> device
  template <int DIR>
  cudaError_t run(int device, void* dev, void* host, size_t bytes) {
    const size_t nch = (bytes + chunk - 1) / chunk;
    const int W = (int)std::min<size_t>(workers, nch);
    std::atomic<int> err{0};
    auto body = [&](int w) {
      cudaSetDevice(device);
      cudaStream_t s = stream[w];
      void* b[2] = {buf[2 * w], buf[2 * w + 1]};
      cudaEvent_t e[2] = {ev[2 * w], ev[2 * w + 1]};
      size_t prev_off = 0, prev_len = 0;
      int k = 0;
      for (size_t c = w; c < nch && !err.load(std::memory_order_relaxed); c += W, ++k) {
        const size_t off = c * chunk, len = std::min(chunk, bytes - off);
        const int i = k & 1;
        cudaError_t r;
        if constexpr (DIR > 0) {
          // the DMA of chunk k - 2 read this buffer: wait for it, fill, send
          if (k >= 2 && (r = cudaEventSynchronize(e[i])) != cudaSuccess) { err = (int)r; break; }
          memcpy(b[i], static_cast<const char*>(host) + off, len);
          r = cudaMemcpyAsync(static_cast<char*>(dev) + off, b[i], len, cudaMemcpyHostToDevice, s);
          if (r == cudaSuccess) r = cudaEventRecord(e[i], s);
        } else {
          // fetch chunk k into this buffer (its previous contents were copied out in step k - 1),
          // then copy chunk k - 1 out of the other buffer once its DMA is done
          r = cudaMemcpyAsync(b[i], static_cast<const char*>(dev) + off, len, cudaMemcpyDeviceToHost, s);
          if (r == cudaSuccess) r = cudaEventRecord(e[i], s);
          if (r == cudaSuccess && k >= 1) {
            r = cudaEventSynchronize(e[i ^ 1]);
            if (r == cudaSuccess) memcpy(static_cast<char*>(host) + prev_off, b[i ^ 1], prev_len);
          }
        }
        if (r != cudaSuccess) { err = (int)r; break; }
        prev_off = off;
        prev_len = len;
      }
      if (err.load()) return;
      cudaError_t r = cudaStreamSynchronize(s);
      if (r == cudaSuccess && DIR < 0 && k >= 1) memcpy(static_cast<char*>(host) + prev_off, b[(k - 1) & 1], prev_len);
      if (r != cudaSuccess) err = (int)r;
    };
    std::vector<std::thread> th;
    th.reserve(W);
    for (int w = 0; w < W; ++w) th.emplace_back(body, w);
    for (auto& t : th) t.join();
    return (cudaError_t)err.load();
  }
};

// default staging: one worker per host core up to 16, 16 MB chunks (2 x 16 x 16 MB pinned)
inline int default_workers() {
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(16u, hc ? hc : 4u));
}
constexpr size_t kChunk = size_t(16) << 20;

}  // namespace so3host
