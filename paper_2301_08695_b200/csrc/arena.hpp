// Host-side plumbing shared by the C ABI translation units: a bump layout
// over one device pool, host<->device copy records, and the per-thread
// arena the one-shot entry points (bx_place, bx_simulate, bx_schedulable_time,
// bx_critical_path_us, ...) reuse across calls, so a call in steady state
// does no cudaMalloc / cudaHostAlloc / stream or event creation.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>

namespace bx {

// Bump allocator over one device pool (256-byte aligned sub-arrays).
struct Layout {
  size_t off = 0;
  size_t align = 256;
  template <typename T>
  size_t take(size_t count) {
    off = (off + align - 1) & ~(align - 1);
    size_t at = off;
    off += std::max<size_t>(count, 1) * sizeof(T);
    return at;
  }
};

template <typename T>
T *at(void *pool, size_t off) {
  return reinterpret_cast<T *>(static_cast<char *>(pool) + off);
}

struct HostCopy {  // one H2D or D2H copy
  void *dst;
  const void *src;
  size_t bytes;
};

// Grow-only buffers of one host thread on one CUDA device. Buffers handed
// out stay valid until the next request of the same kind on this thread.
class Arena {
 public:
  struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
  };
  // Device slots: 0 = one-shot analysis calls, 1 = plan pool, 2 = simulator
  // pool, 3 = sort scratch, 4 / 5 = plan / simulator fill tables.
  // Pinned slots: 0 = plan inputs, 1 = plan outputs.
  cudaError_t device(size_t bytes, char **out, int slot = 0) {
    Buf &b = dev_[slot];
    if (b.bytes < bytes) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      b.bytes = 0;
      const size_t want = std::max(bytes + bytes / 4, size_t(1) << 20);
      cudaError_t e = cudaMalloc(&b.p, want);
      if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(&b.p, bytes);
        if (e != cudaSuccess) return e;
        b.bytes = bytes;
      } else {
        b.bytes = want;
      }
    }
    *out = static_cast<char *>(b.p);
    return cudaSuccess;
  }
  cudaError_t pinned(size_t bytes, void **out, int slot) {
    Buf &b = host_[slot];
    if (b.bytes < bytes) {
      if (b.p) cudaFreeHost(b.p);
      b.p = nullptr;
      b.bytes = 0;
      const size_t want = std::max(bytes + bytes / 4, size_t(1) << 16);
      cudaError_t e = cudaHostAlloc(&b.p, want, cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
      b.bytes = want;
    }
    *out = b.p;
    return cudaSuccess;
  }
  cudaStream_t stream() {
    if (!s_) cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking);
    return s_;
  }
  cudaStream_t side_stream() {
    if (!s2_) cudaStreamCreateWithFlags(&s2_, cudaStreamNonBlocking);
    return s2_;
  }
  cudaEvent_t event(int i, bool timing) {
    if (!ev_[i]) {
      if (timing) cudaEventCreate(&ev_[i]);
      else cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming);
    }
    return ev_[i];
  }
  int device_id = -1;

 private:
  Buf dev_[6];
  Buf host_[2];
  cudaStream_t s_ = nullptr, s2_ = nullptr;
  cudaEvent_t ev_[4] = {nullptr, nullptr, nullptr, nullptr};
};

// The calling thread's arena for the current CUDA device. Arenas live until
// the thread exits (the CUDA context outlives them at process exit, so their
// buffers are left to the driver rather than freed from a destructor).
Arena &thread_arena();

}  // namespace bx
