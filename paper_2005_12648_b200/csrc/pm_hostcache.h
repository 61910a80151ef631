// Host-side memo of per-device kernel attributes and occupancy answers.
// cudaFuncSetAttribute and cudaOccupancyMaxActiveBlocksPerMultiprocessor cost a
// few microseconds of host time each; on the launch path of a small or medium
// merge (tens of microseconds of GPU work) they are the critical path, since the
// GPU idles until the first kernel is enqueued.  Attributes belong to each
// device's context, so both memos are keyed by the current device.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace pm {

struct HostCache {
  std::mutex mu;
  std::map<std::pair<int, const void*>, size_t> smem;               // (device, kernel) -> limit set
  std::map<std::tuple<int, const void*, int, size_t>, int> occ;     // (device, kernel, block, smem) -> CTAs/SM
  static HostCache& get() {
    static HostCache c;
    return c;
  }
};

// Raise the kernel's dynamic shared memory limit on the current device to >= bytes
// (the runtime is called only when the limit grows; it never shrinks).
inline cudaError_t ensure_smem_attr(const void* func, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  HostCache& c = HostCache::get();
  std::lock_guard<std::mutex> lk(c.mu);
  size_t& cur = c.smem[{dev, func}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// Resident CTAs per SM for (kernel, block, smem) on the current device, memoised.
inline cudaError_t cached_occupancy(int* bps, const void* func, int block, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  HostCache& c = HostCache::get();
  std::lock_guard<std::mutex> lk(c.mu);
  auto key = std::make_tuple(dev, func, block, smem);
  auto it = c.occ.find(key);
  if (it != c.occ.end()) {
    *bps = it->second;
    return cudaSuccess;
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, func, block, smem);
  if (e == cudaSuccess) c.occ.emplace(key, *bps);
  return e;
}

}  // namespace pm
