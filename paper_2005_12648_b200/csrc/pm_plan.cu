// pm_plan.cu -- split-point kernels behind find_median / plan_intervals /
// find_splits (sm_100a).
//
// k_find_median    : exact Alg. 1 (median.py:23-60), one thread -- API parity.
// k_find_splits    : stable merge-path splits at arbitrary diagonals, one warp
//                    per split (the GPU's partition search; A wins ties).
// k_plan_intervals : plan_intervals (soptmov.py:93-123): log2(t) levels of
//                    Alg. 1 over RunPairs, one thread per node, one CTA.
#include <cuda_runtime.h>

#include "pm_common.cuh"
#include "pm_launch.h"
#include "pm_search.cuh"

namespace pm {

template <typename KT>
__global__ void k_find_median(const KT* a, const KT* b, int64_t la, int64_t lb, int64_t* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) find_median_dev<KT>(a, la, b, lb, out, out + 1);
}

template <typename KT>
__global__ void k_find_splits(const KT* A, const KT* B, int64_t la, int64_t lb, const int64_t* diags, int64_t nd,
                              int64_t* out_a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nd; i += nwarps) {
    int64_t d = diags[i];
    d = d < 0 ? 0 : (d > la + lb ? la + lb : d);
    int64_t a = merge_path_warp<KT>(A, la, B, lb, d, lane);
    if (lane == 0) out_a[i] = a;
  }
}

// nodes: level-order RunPairs (a_start, a_end, b_start, b_end), 2t-1 of them
template <typename KT>
__global__ void k_plan_intervals(const KT* keys, int64_t s, int64_t m, int64_t e, int32_t levels, int64_t* nodes) {
  if (threadIdx.x == 0) {
    nodes[0] = s;
    nodes[1] = m;
    nodes[2] = m;
    nodes[3] = e;
  }
  __syncthreads();
  int64_t first = 0;  // index of the first node of the current level
  for (int32_t lv = 0; lv < levels; ++lv) {
    const int64_t width = 1ll << lv, nfirst = first + width;
    for (int64_t i = threadIdx.x; i < width; i += blockDim.x) {
      const int64_t* pr = nodes + 4 * (first + i);
      int64_t a0 = pr[0], a1 = pr[1], b0 = pr[2], b1 = pr[3], pa, pb;
      find_median_dev<KT>(keys + a0, a1 - a0, keys + b0, b1 - b0, &pa, &pb);
      int64_t* l = nodes + 4 * (nfirst + 2 * i);
      int64_t* r = l + 4;
      l[0] = a0;      l[1] = a0 + pa; l[2] = b0;      l[3] = b0 + pb;
      r[0] = a0 + pa; r[1] = a1;      r[2] = b0 + pb; r[3] = b1;
    }
    __syncthreads();
    first = nfirst;
  }
}

// ---- host launchers ---------------------------------------------------------
template <typename KT>
cudaError_t launch_find_median(const void* a, const void* b, int64_t la, int64_t lb, int64_t* out, cudaStream_t st) {
  k_find_median<KT><<<1, 32, 0, st>>>(reinterpret_cast<const KT*>(a), reinterpret_cast<const KT*>(b), la, lb, out);
  count_launches(1);
  return cudaGetLastError();
}
template <typename KT>
cudaError_t launch_find_splits(const void* a, const void* b, int64_t la, int64_t lb, const int64_t* diags, int64_t nd,
                               int64_t* out_a, int grid, cudaStream_t st) {
  k_find_splits<KT><<<grid, 256, 0, st>>>(reinterpret_cast<const KT*>(a), reinterpret_cast<const KT*>(b), la, lb,
                                          diags, nd, out_a);
  count_launches(1);
  return cudaGetLastError();
}
template <typename KT>
cudaError_t launch_plan_intervals(const void* keys, int64_t s, int64_t m, int64_t e, int32_t levels, int64_t* nodes,
                                  cudaStream_t st) {
  int block = levels >= 8 ? 256 : (1 << (levels > 5 ? levels : 5));
  k_plan_intervals<KT><<<1, block, 0, st>>>(reinterpret_cast<const KT*>(keys), s, m, e, levels, nodes);
  count_launches(1);
  return cudaGetLastError();
}
template cudaError_t launch_find_median<int32_t>(const void*, const void*, int64_t, int64_t, int64_t*, cudaStream_t);
template cudaError_t launch_find_median<int64_t>(const void*, const void*, int64_t, int64_t, int64_t*, cudaStream_t);
template cudaError_t launch_find_splits<int32_t>(const void*, const void*, int64_t, int64_t, const int64_t*, int64_t, int64_t*, int, cudaStream_t);
template cudaError_t launch_find_splits<int64_t>(const void*, const void*, int64_t, int64_t, const int64_t*, int64_t, int64_t*, int, cudaStream_t);
template cudaError_t launch_plan_intervals<int32_t>(const void*, int64_t, int64_t, int64_t, int32_t, int64_t*, cudaStream_t);
template cudaError_t launch_plan_intervals<int64_t>(const void*, int64_t, int64_t, int64_t, int32_t, int64_t*, cudaStream_t);

}  // namespace pm
