// pm_small.cu -- small in-place merges in one CTA.
//
// When both runs fit in shared memory (keys + payload rows <= kSmallBytes), a
// single CTA stages A|B on chip (16-byte bulk loads), each thread finds its
// output range's stable merge-path split (A wins ties, as the reference's
// buffered_merge, _kernels.py:227-313) and merges it straight back into the
// caller's arrays -- everything was read before anything is written, so the
// in-place semantics hold with no scratch.  One launch, a few microseconds:
// the persistent engine's plan + ticket machinery costs ~50 us at these sizes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "pm_launch.h"

namespace pm {

namespace {

constexpr int kSmallThreads = 1024;

// stable merge-path split: number of A records among the first d outputs
template <typename KT>
__device__ __forceinline__ int split_smem(const KT* A, int la, const KT* B, int lb, int d) {
  int lo = max(0, d - lb), hi = min(d, la);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// copy `bytes` between 16-byte-aligned (dst, src) pairs cooperatively; the
// caller picks the widest word both addresses allow
template <typename W>
__device__ __forceinline__ void block_copy(void* dst, const void* src, int64_t bytes) {
  W* d = static_cast<W*>(dst);
  const W* s = static_cast<const W*>(src);
  for (int64_t i = threadIdx.x; i < bytes / (int64_t)sizeof(W); i += blockDim.x) d[i] = s[i];
}

template <typename KT>
__global__ void __launch_bounds__(kSmallThreads) k_merge_small(KT* keys, uint8_t* pay, int64_t w, int la, int lb) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int n = la + lb;
  KT* sk = reinterpret_cast<KT*>(sm);
  uint8_t* sp = sm + ((n * sizeof(KT) + 15) & ~(size_t)15);
  // stage keys (and payload rows) -- word size chosen by alignment
  if ((((uintptr_t)keys) & 15) == 0 && ((n * sizeof(KT)) & 15) == 0) block_copy<uint4>(sk, keys, n * sizeof(KT));
  else block_copy<KT>(sk, keys, n * sizeof(KT));
  const bool w4 = w && ((((uintptr_t)pay) | (uintptr_t)w) & 3) == 0;
  if (w) {
    if (((((uintptr_t)pay) | (uintptr_t)(n * w)) & 15) == 0) block_copy<uint4>(sp, pay, n * w);
    else if (w4) block_copy<uint32_t>(sp, pay, n * w);
    else block_copy<uint8_t>(sp, pay, n * w);
  }
  __syncthreads();
  const KT* A = sk;
  const KT* B = sk + la;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int d0 = min(n, (int)threadIdx.x * per), d1 = min(n, d0 + per);
  if (d0 >= d1) return;
  int i = split_smem(A, la, B, lb, d0), j = d0 - i;
  for (int d = d0; d < d1; ++d) {
    const bool ta = j >= lb || (i < la && A[i] <= B[j]);
    const int src = ta ? i : la + j;
    keys[d] = sk[src];
    if (w) {
      if (w4) {
        const uint32_t* s = reinterpret_cast<const uint32_t*>(sp + (int64_t)src * w);
        uint32_t* o = reinterpret_cast<uint32_t*>(pay + (int64_t)d * w);
        for (int64_t c = 0; c < (w >> 2); ++c) o[c] = s[c];
      } else {
        for (int64_t c = 0; c < w; ++c) pay[(int64_t)d * w + c] = sp[(int64_t)src * w + c];
      }
    }
    if (ta) ++i;
    else ++j;
  }
}

}  // namespace

int64_t small_merge_smem(int ks, int64_t w, int64_t n) { return ((n * ks + 15) & ~15ll) + n * w; }

template <typename KT>
cudaError_t launch_merge_small(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                               cudaStream_t st) {
  const int64_t n = e - s;
  const size_t smem = (size_t)small_merge_smem(sizeof(KT), w, n);
  cudaError_t ce = cudaFuncSetAttribute(k_merge_small<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (ce != cudaSuccess) return ce;
  k_merge_small<KT><<<1, kSmallThreads, smem, st>>>(static_cast<KT*>(keys) + s,
                                                    w ? static_cast<uint8_t*>(payload) + s * w : nullptr, w,
                                                    (int)(m - s), (int)(e - m));
  count_launches(1);
  return cudaGetLastError();
}
template cudaError_t launch_merge_small<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);
template cudaError_t launch_merge_small<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);

}  // namespace pm
