// Scheduler ticket counters for the persistent kernels (dynamic work
// distribution: each CTA pulls its next unit / tile chunk with atomicAdd).
//
// One device ring per device of `blocks` × kWidth counters.  A launch
// acquires one block (≤ kWidth counters: one per pass), zeroes it on its
// stream and, after its kernels are queued, releases it by recording an
// event on that stream.  A block is handed out again only after the ring has
// wrapped, and the new user's stream first waits for the event of the block's
// previous user — so a counter is never re-zeroed under a kernel that is
// still pulling tickets from it, whatever streams the two launches use.
#pragma once
#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "host_util.h"

namespace cim {

class CounterRing {
 public:
  static constexpr int kWidth = 64;  // ≥ the largest pass count (k ≤ 64)

  // Lazily allocates the ring; returns CIM_OK or a CIM_ECUDA error.
  int init(int blocks) {
    std::lock_guard<std::mutex> lk(mu_);
    if (base_) return CIM_OK;
    cudaError_t e = cudaMalloc(&base_, (size_t)blocks * kWidth * sizeof(unsigned int));
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("counter ring: ") + cudaGetErrorString(e));
    ev_.assign(blocks, nullptr);
    busy_.assign(blocks, false);
    blocks_ = blocks;
    return CIM_OK;
  }

  // n ≤ kWidth counters, zeroed on `stream` after the block's previous user finished.
  int acquire(cudaStream_t stream, int n, unsigned int **out, int *block) {
    if (n < 1 || n > kWidth) return set_error(CIM_EINVAL, "counter ring: bad counter count");
    std::lock_guard<std::mutex> lk(mu_);
    int b = -1;
    for (int tries = 0; tries < blocks_; ++tries) {
      const int c = pos_;
      pos_ = (pos_ + 1) % blocks_;
      if (!busy_[c]) {
        b = c;
        break;
      }
    }
    if (b < 0) return set_error(CIM_ECUDA, "counter ring: every block is in use");
    cudaError_t e = cudaSuccess;
    if (ev_[b]) e = cudaStreamWaitEvent(stream, ev_[b], 0);
    if (e == cudaSuccess) e = cudaMemsetAsync(base_ + (size_t)b * kWidth, 0, (size_t)n * sizeof(unsigned int), stream);
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("counter ring: ") + cudaGetErrorString(e));
    busy_[b] = true;
    *out = base_ + (size_t)b * kWidth;
    *block = b;
    return CIM_OK;
  }

  // After the launches that use block b are queued on `stream`.
  int release(int b, cudaStream_t stream) {
    std::lock_guard<std::mutex> lk(mu_);
    cudaError_t e = cudaSuccess;
    if (!ev_[b]) e = cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev_[b], stream);
    busy_[b] = false;
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("counter ring event: ") + cudaGetErrorString(e));
    return CIM_OK;
  }

 private:
  std::mutex mu_;
  unsigned int *base_ = nullptr;
  std::vector<cudaEvent_t> ev_;
  std::vector<bool> busy_;
  int blocks_ = 0, pos_ = 0;
};

// RAII holder: releases the block on scope exit (also on error paths).
struct CounterLease {
  CounterRing *ring = nullptr;
  int block = -1;
  cudaStream_t stream = nullptr;
  unsigned int *ctr = nullptr;
  int take(CounterRing &r, cudaStream_t s, int n) {
    ring = &r;
    stream = s;
    return r.acquire(s, n, &ctr, &block);
  }
  ~CounterLease() {
    if (ring && block >= 0) ring->release(block, stream);
  }
};

}  // namespace cim
