// pm_rotate.cu -- in-place block exchange A|B -> B|A by three reversals
// (reverse A, reverse B, reverse A|B): two streaming passes over the records,
// every pass a perfectly parallel swap of mirrored records (coalesced on both
// sides), no bookkeeping.  Replaces _kernels.linear_shift / circular_shift
// (_kernels.py:92-197) behind pm_shift; the result is the same array (the
// reference's instrumented move counts are computed on the host, shift.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "pm_launch.h"

namespace pm {

// Swap row x and row y of the payload (w bytes per row).
__device__ __forceinline__ void swap_rows(uint8_t* pay, int64_t w, bool w4, int64_t x, int64_t y) {
  if (w4) {
    uint32_t* a = reinterpret_cast<uint32_t*>(pay + x * w);
    uint32_t* b = reinterpret_cast<uint32_t*>(pay + y * w);
    for (int64_t c = 0; c < (w >> 2); ++c) {
      const uint32_t t = a[c];
      a[c] = b[c];
      b[c] = t;
    }
  } else {
    uint8_t* a = pay + x * w;
    uint8_t* b = pay + y * w;
    for (int64_t c = 0; c < w; ++c) {
      const uint8_t t = a[c];
      a[c] = b[c];
      b[c] = t;
    }
  }
}

// Reverse [lo0, lo0+len0) and [lo1, lo1+len1) in place (len1 may be 0).
// Consecutive threads take consecutive pairs: the left records ascend and the
// mirrored ones descend, both coalesced.  Four pairs per thread per round keep
// eight loads in flight.
template <typename KT>
__global__ void __launch_bounds__(256) k_reverse(KT* keys, uint8_t* pay, int64_t w, int64_t lo0, int64_t len0,
                                                 int64_t lo1, int64_t len1) {
  const int64_t p0 = len0 >> 1, np = p0 + (len1 >> 1);
  const bool w4 = w && (w & 3) == 0 && (((uintptr_t)pay) & 3) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < np; base += stride * U) {
    int64_t xl[U], xr[U];
    KT vl[U], vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = base + u * stride;
      if (p < np) {
        const bool s0 = p < p0;
        const int64_t i = s0 ? p : p - p0;
        const int64_t lo = s0 ? lo0 : lo1, len = s0 ? len0 : len1;
        xl[u] = lo + i;
        xr[u] = lo + len - 1 - i;
        vl[u] = keys[xl[u]];
        vr[u] = keys[xr[u]];
      } else {
        xl[u] = -1;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (xl[u] >= 0) {
        keys[xl[u]] = vr[u];
        keys[xr[u]] = vl[u];
        if (w) swap_rows(pay, w, w4, xl[u], xr[u]);
      }
    }
  }
}

template <typename KT>
cudaError_t launch_rotate(void* keys, void* payload, int64_t w, int64_t lo, int64_t la, int64_t lb, int num_sms,
                          cudaStream_t st) {
  KT* k = static_cast<KT*>(keys);
  uint8_t* p = static_cast<uint8_t*>(payload);
  const int64_t pairs = (la >> 1) + (lb >> 1);
  const int64_t all = (la + lb) >> 1;
  auto grid_for = [&](int64_t np) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((np + 1023) / 1024, (int64_t)num_sms * 8));
  };
  if (pairs > 0) k_reverse<KT><<<grid_for(pairs), 256, 0, st>>>(k, p, w, lo, la, lo + la, lb);
  if (all > 0) k_reverse<KT><<<grid_for(all), 256, 0, st>>>(k, p, w, lo, la + lb, 0, 0);
  return cudaGetLastError();
}
template cudaError_t launch_rotate<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);
template cudaError_t launch_rotate<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);

}  // namespace pm
