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
// Narrow a stable merge-path bracket by interpolation.  f(x) = A[x] - B[d-1-x]
// rises with x; the split is the first x with f(x) > 0.  On entry the split is in
// [*lo, *hi], f(*lo - 1) = fl <= 0 and f(*hi) = fh > 0.  Each probe lands where the
// line through the bracket values crosses zero (a few records from the split when
// the keys are spread like the bracket ends) and replaces one end; the Illinois
// rule halves a retained end's value so the bracket cannot creep.  At most
// `probes` probes (the caller finishes with a binary search, so the worst case is
// logarithmic plus `probes`); each probe is one random DRAM line per run instead of
// the ~log2(window / 32) distinct lines a binary search touches.
template <typename KT>
__device__ __forceinline__ void interp_bracket(const KT* A, const KT* B, int64_t d, int64_t* lo, int64_t* hi, double fl,
                                               double fh, int probes) {
  int64_t wlo = *lo, whi = *hi;
  int side = 0;
  for (int it = 0; it < probes && whi - wlo > 8; ++it) {
    const int64_t xl = wlo - 1, xh = whi;
    int64_t x = xl + (int64_t)((-fl) / (fh - fl) * (double)(xh - xl));
    x = x < xl + 1 ? xl + 1 : (x > xh - 1 ? xh - 1 : x);
    const KT av = __ldg(A + x), bv = __ldg(B + d - 1 - x);
    const int s_now = av <= bv ? -1 : 1;
    if (s_now < 0) {
      wlo = x + 1;
      fl = (double)av - (double)bv;
    } else {
      whi = x;
      fh = (double)av - (double)bv;
    }
    if (s_now == side) {
      if (s_now < 0) fh *= 0.5;
      else fl *= 0.5;
    }
    side = s_now;
  }
  *lo = wlo;
  *hi = whi;
}

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
