// device_util.hpp -- CUDA helpers shared by the engine's translation units
// (sources.cpp, runtime.cpp): status checks, the device guard, device /
// stream-ordered / pinned allocations as shared_ptr with their frees.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>
#include <string>

#include "dpb200/core.hpp"
#include "dpcuda.h"

namespace datapipe::b200::detail {

inline void CudaCheck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline void KCheck(int status, const char* what) {
  if (status != DP_OK) {
    if (status == DP_ERR_CUDA || status == DP_ERR_OUT_OF_MEMORY)
      throw DeviceError(std::string(what) + ": " + dp_last_error());
    throw PipelineError(static_cast<ErrorCode>(status - 1), std::string(what) + ": " + dp_last_error());
  }
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CudaCheck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

inline std::shared_ptr<void> DeviceAlloc(size_t bytes, int device) {
  DeviceGuard g(device);
  void* p = nullptr;
  CudaCheck(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc");
  return std::shared_ptr<void>(p, [device](void* q) {
    DeviceGuard g2(device);
    cudaFree(q);
  });
}

// Stream-ordered allocation for per-epoch plan buffers: allocated on the plan
// stream, returned with cudaFreeAsync on the batch stream (after the last
// batch kernel that reads them), so an epoch transition never blocks the
// host the way cudaMalloc / cudaFree do.  The device's default pool keeps
// freed memory cached for reuse.
inline std::shared_ptr<void> DeviceAllocAsync(size_t bytes, int device, cudaStream_t alloc_stream, cudaStream_t free_stream) {
  DeviceGuard g(device);
  static std::once_flag once[64];
  std::call_once(once[device & 63], [device] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  });
  void* p = nullptr;
  CudaCheck(cudaMallocAsync(&p, bytes ? bytes : 16, alloc_stream), "cudaMallocAsync");
  return std::shared_ptr<void>(p, [device, free_stream](void* q) {
    DeviceGuard g2(device);
    cudaFreeAsync(q, free_stream);
  });
}

inline std::shared_ptr<void> PinnedAlloc(size_t bytes) {
  void* p = nullptr;
  CudaCheck(cudaHostAlloc(&p, bytes ? bytes : 16, cudaHostAllocPortable | cudaHostAllocMapped), "cudaHostAlloc");
  return std::shared_ptr<void>(p, [](void* q) { cudaFreeHost(q); });
}

template <typename T>
T* P(const std::shared_ptr<void>& p) {
  return static_cast<T*>(p.get());
}

// Small-block recycling for the per-batch control blocks GetNext creates
// (slot leases, Tensor views): a per-thread free list per 64-byte size
// class, capped, falling back to operator new / delete.  Blocks freed on
// another thread join that thread's list.  A thread's lists are returned to
// the heap when the thread exits; blocks freed during or after that teardown
// (a lease dropped by a thread_local destructor) go straight to the heap.
struct BlockPool {
  static constexpr int kClasses = 4, kCap = 4096;
  struct Lists {
    std::vector<void*> l[kClasses];
    ~Lists() {
      Dead() = true;
      for (auto& v : l)
        for (void* p : v) ::operator delete(p);
    }
  };
  // trivially destructible, so still readable while the thread tears down
  static bool& Dead() {
    thread_local bool dead = false;
    return dead;
  }
  static std::vector<void*>* ThreadLists() {
    if (Dead()) return nullptr;
    thread_local Lists lists;
    return lists.l;
  }
  static void* Get(size_t bytes) {
    const size_t c = (bytes + 63) / 64 - 1;
    if (c < kClasses) {
      if (auto* lists = ThreadLists(); lists && !lists[c].empty()) {
        void* p = lists[c].back();
        lists[c].pop_back();
        return p;
      }
      return ::operator new((c + 1) * 64);
    }
    return ::operator new(bytes);
  }
  static void Put(void* p, size_t bytes) {
    const size_t c = (bytes + 63) / 64 - 1;
    if (c < kClasses) {
      if (auto* lists = ThreadLists(); lists && lists[c].size() < kCap) {
        lists[c].push_back(p);
        return;
      }
    }
    ::operator delete(p);
  }
};
template <class T>
struct PoolAllocator {
  using value_type = T;
  PoolAllocator() = default;
  template <class U>
  PoolAllocator(const PoolAllocator<U>&) {}
  T* allocate(size_t n) { return static_cast<T*>(BlockPool::Get(n * sizeof(T))); }
  void deallocate(T* p, size_t n) { BlockPool::Put(p, n * sizeof(T)); }
  template <class U>
  bool operator==(const PoolAllocator<U>&) const { return true; }
};

}  // namespace datapipe::b200::detail
