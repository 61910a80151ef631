// pm_search.cuh -- split-point searches shared by the plan kernels.
//
// merge_path_warp : stable merge-path split (A wins ties) of diagonal d, one
//                   warp, 33-ary search with ballots (~6 dependent probes at 2^29).
// find_median_dev : the reference's Alg. 1 double binary search, exact
//                   (median.py:23-60), one thread.
#pragma once
#include <cstdint>

namespace pm {

// largest a in [lo, hi] such that A[i] <= B[d-1-i] for every i < a (A wins ties);
// the caller guarantees the answer lies in [lo, hi].
template <typename KT>
__device__ __forceinline__ int64_t merge_path_warp_in(const KT* A, const KT* B, int64_t d, int64_t lo, int64_t hi,
                                                      int lane) {
  while (hi - lo > 32) {
    int64_t span = hi - lo;
    int64_t p = lo + ((int64_t)(lane + 1) * span) / 33;  // p in [lo, hi)
    bool f = A[p] <= B[d - 1 - p];
    unsigned fb = __ballot_sync(0xffffffffu, !f);
    if (fb == 0) {
      lo = lo + (32 * span) / 33 + 1;
    } else {
      int fl = __ffs(fb) - 1;
      int64_t pfl = lo + ((int64_t)(fl + 1) * span) / 33;
      int64_t pprev = fl == 0 ? lo - 1 : lo + ((int64_t)fl * span) / 33;
      hi = pfl;
      lo = pprev + 1;
    }
  }
  int64_t p = lo + lane;
  bool f = p < hi ? (A[p] <= B[d - 1 - p]) : false;
  unsigned fb = __ballot_sync(0xffffffffu, !f && p < hi);
  return fb == 0 ? hi : lo + (__ffs(fb) - 1);
}

// stable merge-path split of diagonal d over the full feasible range
template <typename KT>
__device__ __forceinline__ int64_t merge_path_warp(const KT* A, int64_t la, const KT* B, int64_t lb, int64_t d,
                                                   int lane) {
  const int64_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
  return merge_path_warp_in<KT>(A, B, d, lo, hi, lane);
}

// one thread: stable merge-path split of diagonal d (A wins ties)
template <typename KT>
__device__ __forceinline__ int64_t merge_path_thread(const KT* A, int64_t la, const KT* B, int64_t lb, int64_t d) {
  int64_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(A + mid) <= __ldg(B + d - 1 - mid)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <typename KT>
__device__ void find_median_dev(const KT* a, int64_t la, const KT* b, int64_t lb, int64_t* pa_out, int64_t* pb_out) {
  if (la == 0 || lb == 0 || a[la - 1] <= b[0]) {  // median.py:33-34
    *pa_out = la;
    *pb_out = 0;
    return;
  }
  if (!(a[0] <= b[lb - 1])) {  // median.py:35-36
    *pa_out = 0;
    *pb_out = lb;
    return;
  }
  int64_t left_a = 0, limit_a = la, left_b = 0, limit_b = lb;
  while (left_a < limit_a && left_b < limit_b) {  // median.py:40-57
    int64_t pa = (limit_a - left_a) / 2 + left_a;
    int64_t pb = (limit_b - left_b) / 2 + left_b;
    KT va = a[pa], vb = b[pb];
    if (va == vb) break;
    if (va < vb) {
      if (pa + pb < (la - pa) + (lb - pb)) left_a = pa + 1;
      else limit_b = pb;
    } else {
      if (pa + pb < (la - pa) + (lb - pb)) left_b = pb + 1;
      else limit_a = pa;
    }
  }
  *pa_out = (limit_a - left_a) / 2 + left_a;  // median.py:58-60
  *pb_out = (limit_b - left_b) / 2 + left_b;
}

}  // namespace pm
