// pm_flow.cu -- the scheduled in-place merge ("flow" engine, sm_100a).
//
// Same job as k_engine (pm_engine.cu): the stable merge (A wins ties) of the
// adjacent sorted runs A = [s, m) and B = [m, e) in place, bit-exact to the
// reference's stable core (seqmerge.py:55-75 / _kernels.py:227-313; the t >= 1
// drivers srecpar.py:33-84, soptmov.py:146-192 produce the same records).  The
// difference is WHEN the work is decided: k_engine discovers at run time, region
// by region, which units must be moved out of the way (a chain of dependent
// global round trips per region); here a plan computed on the device before the
// merge fixes the whole schedule, so the merge itself is a streaming pipeline
// whose only synchronisation is one counter per region.
//
// Output region q (M records) == slot q of the array.  Writing region q destroys
// slot q's input records; every other region that reads some of them ("reader")
// must have read them first, or they must have been saved ("salvaged") into the
// pool.  For a processing order (rank), reader c of slot j reads
//   * the original slot when rank(c) < rank(j)  (j's store waits for c's read:
//     pend[j] counts those readers, each decrements it once its loads landed),
//   * the slot's salvage entry otherwise (copied before the merge starts).
// So the salvage volume is the weight of the order's backward edges in the
// reader graph.  For two uniform runs that graph is the binary de Bruijn graph
// (slot j is read by regions 2j, 2j+1 mod K), whose cycles force some salvage.
// Two orders are evaluated per job and the cheaper one is taken:
//   * two fronts out of the A/B boundary (k_engine's order): 1/3 of N for uniform
//     runs, near zero for skewed/translated inputs;
//   * the itinerary angle: slot j's symbolic orbit (side of j, side of the region
//     reading j's middle record, side of the region reading that slot, ...) b_1..b_n
//     gives z_j = sum_i b_i exp(2 pi i k / n); a reader's z is z_j rotated by
//     -2 pi / n up to a +-1 perturbation, so processing in increasing arg(z) puts
//     readers first except across the cut and where the perturbation wins (the
//     circle-valued potential behind Mykkeltveit's de Bruijn feedback sets):
//     ~0.20 N salvaged for uniform runs (tools/sim_flow.py).
//
// Plan kernels (one pass each, all on the device, no host round trip):
//   k_plan_coarse/k_plan (pm_engine.cu) : merge-path split at every region boundary
//   k_flow_readers : identity regions; the reader of each slot's middle record
//   k_flow_angle   : itinerary angle key per slot, angle histogram
//   k_flow_choose  : salvage volume of both orders (per region, its <= 4 pieces)
//   k_flow_decide  : pick the order; scan the histogram / identity counts
//   k_flow_rank    : order[] / rank[] (counting sort / two-front compaction)
//   k_flow_hull    : per slot the hull of records later readers need; pend[] counts
//   k_flow_alloc   : pool entries (16-record aligned, phase-matched)
//   k_flow_tickets : the 80-byte per-ticket descriptor
// Merge:
//   k_flow_save    : copy every salvage entry into the pool
//   k_flow         : persistent streaming pipeline (k_buffered's shape): TMA
//                    gathers of the next region while the current one merges in
//                    shared memory, TMA bulk store in place once pend[r] == 0.
// If the salvage does not fit the pool the plan raises FC_FAIL; k_flow then
// exits at once and the bounded-pool engine (gated on that word) runs instead.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "pm_common.cuh"
#include "pm_engine.cuh"
#include "pm_launch.h"
#include "pm_tile.cuh"
#include "pm_search.cuh"

#include <cooperative_groups.h>
#include <nvtx3/nvToolsExt.h>
namespace cg = cooperative_groups;

namespace pm {

constexpr int kFlowChunk = 1024;
// -DPM_FLOW_CHECKED=1 (tools/checked.sh): device-side bounds and invariant checks
// on every access of the scheduled engine -- a failed check prints and traps (the
// substitute for compute-sanitizer, which this pool does not run)
#ifndef PM_FLOW_CHECKED
#define PM_FLOW_CHECKED 0
#endif
#define FLOW_CHECK(cond, ...)                                                      \
  do {                                                                             \
    if (PM_FLOW_CHECKED && !(cond)) {                                              \
      printf("FLOW_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#ifndef PM_FLOW_ABLATE
#define PM_FLOW_ABLATE 0  // k_flow timing ablations (tuning builds; results are wrong): 1 no pend wait, 2 no merge, 4 no store
#endif  // two-front tickets per compaction block

struct FlowGeo : Geo {
  __device__ explicit FlowGeo(const EngineParams& p) : Geo(p) {}
  // (plain load: the plan kernel writes split_a itself, so no read-only path)
  __device__ int64_t split(int64_t q) const { return P.split_a[q]; }
  __device__ int64_t diag(int64_t q) const { return Geo::diag(q); }
  __device__ int64_t bsplit(int64_t q) const { return diag(q) - split(q); }
  // smallest region q whose A range ends after A-local index v (0 <= v < LA)
  __device__ int64_t reader_a(int64_t v) const {
    int64_t lo = 0, hi = P.Q - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (split(mid + 1) > v) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  }
  __device__ int64_t reader_b(int64_t v) const {
    int64_t lo = 0, hi = P.Q - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (bsplit(mid + 1) > v) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  }
  __device__ bool identity(int64_t q, int64_t a0, int64_t a1) const {
    const int64_t la = LA();
    return (a0 == diag(q) && a1 == diag(q + 1)) || (a0 == la && a1 == la);
  }
};

// The pieces of region q: A records [s+a0, s+a1) and B records [m+b0, m+b1), each
// cut at slot boundaries (at most two pieces per run: a run of a region holds at
// most M == T records).  f(slot, lo, hi, k, is_b): absolute record range [lo, hi).
template <class F>
__device__ __forceinline__ void for_pieces(const EngineParams& P, int64_t xa0, int64_t xa1, int64_t xb0, int64_t xb1,
                                           F&& f) {
  for (int side = 0; side < 2; ++side) {
    int64_t x = side ? xb0 : xa0;
    const int64_t xe = side ? xb1 : xa1;
    for (int k = 0; x < xe && k < 2; ++k) {
      const int64_t y = min(xe, ((x >> P.lT) + 1) << P.lT);
      f((x >> P.lT) - P.k0, x, y, k, side);
      x = y;
    }
  }
}

__device__ __forceinline__ bool flow_off(const FlowParams& F) {
  return *(volatile int32_t*)F.P.noop || *(volatile long long*)&F.fc[FC_FAIL] ||
         *(volatile long long*)&F.fc[FC_ROTFAIL];
}
// The same test inside the cooperative plan, where FC_FAIL may be raised during a
// phase (k_flow_alloc / the forced fallback): one thread reads it for the whole
// CTA, so every thread of a CTA takes the same branch around the phase's CTA
// barriers.
__device__ __forceinline__ bool block_flow_off(const FlowParams& F) {
  __shared__ int32_t s_off;
  __syncthreads();
  if (threadIdx.x == 0) s_off = flow_off(F) ? 1 : 0;
  __syncthreads();
  return s_off != 0;
}

// ---- k_flow_sample / k_flow_split: the stable merge path at every region boundary
// Two levels instead of one long binary search per boundary (whose ~17 probes are
// mostly DRAM misses): the predicate A[i] <= B[d-1-i] at i = k S only touches
// A[k S] and B[d-1-k S] = B[k' S + phi] (every diagonal d = (R0+q) M - s is
// congruent mod S), so a search over the two sample arrays (L2-resident) brackets
// the split within S, and a last search of log2 S steps in the arrays finishes it.
template <typename KT>
__device__ __forceinline__ void ph_sample(const FlowParams& F) {
  const EngineParams& P = F.P;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const KT* A = reinterpret_cast<const KT*>(P.keys) + P.s;
  const KT* B = reinterpret_cast<const KT*>(P.keys) + P.m;
  KT* sa = reinterpret_cast<KT*>(F.samp_a);
  KT* sb = reinterpret_cast<KT*>(F.samp_b);
  if (tid < FC_WORDS && tid != FC_ROT && tid != FC_ROTFAIL) F.fc[tid] = 0;  // (FC_ROT, FC_ROTFAIL: thread 0 below)
  for (int64_t b = tid; b <= F.nb; b += nthr) F.hist[b] = 0;  // (before ph_readers counts identity regions)
  for (int64_t c = tid; c < P.Q / kFlowChunk + 2; c += nthr) F.chunk[c] = 0;
  if (tid == 0) {
    *P.ticket = 0;
    // (a prescribed layout has no such shortcut: identity regions are skipped instead)
    const bool nothing = P.m == P.s || P.m == P.e || (!F.nleaves && A[P.m - P.s - 1] <= B[0]);  // srecpar.py:56-57
    *P.noop = nothing ? 1 : 0;
    const bool rot = !nothing && !F.nleaves && A[0] > B[P.e - P.m - 1];
    F.fc[FC_ROT] = rot ? 1 : 0;
    // equal runs: the block swap (2 N w) always beats the engine (N/2 salvaged); the
    // plan stops here.  Unequal rotations only take the reversals (4 N w) when the
    // engine's salvage overflows the pool (ph_alloc).
    F.fc[FC_ROTFAIL] = rot && P.m - P.s == P.e - P.m ? 1 : 0;
    for (int i = 0; i < 16; ++i) P.stats[i] = 0;
    if (F.fc[FC_ROTFAIL]) P.stats[13] = 1;
  }
  // (four independent strided loads in flight per thread before their stores)
  for (int64_t k0 = tid; !F.nleaves && k0 < F.nsa + F.nsb; k0 += 4 * nthr) {
    KT v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u * nthr;
      v[u] = k < F.nsa ? __ldcs(A + (k << F.lS)) : k < F.nsa + F.nsb ? __ldcs(B + ((k - F.nsa) << F.lS) + F.phi) : (KT)0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u * nthr;
      if (k < F.nsa) sa[k] = v[u];
      else if (k < F.nsa + F.nsb) sb[k - F.nsa] = v[u];
    }
  }
}

// Largest k in [lo, hi] with pred(k) true, for pred monotone (true, then false) and
// pred(lo) true: an 8-ary search, seven independent probes per step, so a search
// over 2^20 candidates is 7 dependent round trips instead of 20.
template <class Pred>
__device__ __forceinline__ int64_t last_true8(int64_t lo, int64_t hi, Pred&& pred) {
  while (lo < hi) {
    const int64_t span = hi - lo;
    int64_t p[7];
    bool f[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) p[i] = lo + (span * (i + 1) + 7) / 8;  // in (lo, hi], non-decreasing
#pragma unroll
    for (int i = 0; i < 7; ++i) f[i] = pred(p[i]);
    int64_t nlo = lo, nhi = hi;
#pragma unroll
    for (int i = 6; i >= 0; --i) {
      if (f[i]) {
        nlo = max(nlo, p[i]);
      } else {
        nhi = min(nhi, p[i] - 1);
      }
    }
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// leaf of job-local output position d: the largest i with leaf_l[i] <= d
__device__ __forceinline__ int32_t leaf_of(const FlowParams& F, int64_t d) {
  int32_t lo = 0, hi = F.nleaves - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (F.leaf_l[mid] <= d) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// prescribed layout: A records among the first d outputs of A_0 B_0 A_1 B_1 ...
__device__ __forceinline__ void ph_split_leaves(const FlowParams& F) {
  const EngineParams& P = F.P;
  FlowGeo g(P);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = tid; q <= P.Q; q += nthr) {
    const int64_t d = g.diag(q);
    int64_t a;
    if (d >= g.N()) {
      a = g.LA();
    } else {
      const int32_t i = leaf_of(F, d);
      const int64_t na = F.leaf_a[i + 1] - F.leaf_a[i];
      a = F.leaf_a[i] + min(d - F.leaf_l[i], na);
    }
    P.split_a[q] = a;
  }
}

#ifndef PM_FLOW_SPLIT_ABLATE
#define PM_FLOW_SPLIT_ABLATE 0  // timing ablations of the split search (tuning builds; wrong splits): 1 no window search, 2 no sample search
#endif
#ifndef PM_FLOW_INTERP
#define PM_FLOW_INTERP 8  // tune: interpolation probes of the split search before binary search (2^30: split 66 -> 30 us)
#endif
template <typename KT>
__device__ __forceinline__ void ph_split(const FlowParams& F) {
  const EngineParams& P = F.P;
  FlowGeo g(P);
  if (*(volatile int32_t*)P.noop) return;
  if (F.nleaves) {
    ph_split_leaves(F);
    return;
  }
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const KT* A = reinterpret_cast<const KT*>(P.keys) + P.s;
  const KT* B = reinterpret_cast<const KT*>(P.keys) + P.m;
  const KT* sa = reinterpret_cast<const KT*>(F.samp_a);
  const KT* sb = reinterpret_cast<const KT*>(F.samp_b);
  const int64_t la = g.LA(), lb = g.LB(), S = (int64_t)1 << F.lS;
  for (int64_t q = tid; q <= P.Q; q += nthr) {
    const int64_t d = g.diag(q);
    const int64_t lo = max(d - lb, (int64_t)0), hi = min(d, la);
    int64_t a;
    if (q == 0 || q == P.Q || lo == hi) {
      a = q == 0 ? 0 : q == P.Q ? la : lo;
    } else {
      // largest k with k S in [lo, hi) and A[k S] <= B[d-1-k S]  (B index = (c - k) S + phi)
      const int64_t klo = (lo + S - 1) >> F.lS, khi = (hi - 1) >> F.lS;
      const int64_t c = (d - 1 - F.phi) >> F.lS;  // exact: d - 1 - phi is a multiple of S
      int64_t wlo = lo, whi = min(hi, klo << F.lS);  // window if no sample point passes
      // f(x) = A[x] - B[d-1-x] rises with x; the split is the first x with f(x) > 0.
      // Known: f <= 0 at xl = wlo - 1 (fl), f > 0 at xh = whi (fh) when `ends`.
      double fl = 0.0, fh = 0.0;
      bool ends = false;
      if (!(PM_FLOW_SPLIT_ABLATE & 2) && klo <= khi && sa[klo] <= sb[c - klo]) {
        const int64_t k = last_true8(klo, khi, [&](int64_t x) { return sa[x] <= sb[c - x]; });
        wlo = (k << F.lS) + 1;
        whi = min(hi, wlo - 1 + S);
        if (k < khi) {  // (k + 1) S <= hi - 1: both bracket values are samples
          fl = (double)sa[k] - (double)sb[c - k];
          fh = (double)sa[k + 1] - (double)sb[c - k - 1];
          ends = true;
        }
      }
      // a window at an end of the feasible range: one probe of the predicate there --
      // all of A's part (pred(hi - 1)) or none of it (!pred(lo)) settles the boundary
      // without the window search (the identity stretches of skewed jobs: half of
      // config 3's boundaries); interior windows (uniform runs) never pay for it
      if (wlo < whi && whi == hi && __ldg(A + hi - 1) <= __ldg(B + d - hi)) wlo = whi = hi;
      else if (wlo < whi && wlo == lo && !(__ldg(A + lo) <= __ldg(B + d - 1 - lo))) wlo = whi = lo;
      // the split is in [wlo, whi]: interpolation between the bracketing samples
      // (pm_search.cuh), then binary search.  The probes are the random DRAM reads
      // the split phase is bound by: ~2-3 instead of ~6 distinct lines per run.
      if (ends && wlo < whi) interp_bracket<KT>(A, B, d, &wlo, &whi, fl, fh, PM_FLOW_INTERP);
      if (PM_FLOW_SPLIT_ABLATE & 1) whi = wlo;  // (timing ablation: wrong splits)
      while (wlo < whi) {  // binary (its late probes share DRAM lines)
        const int64_t mid = (wlo + whi) >> 1;
        if (__ldg(A + mid) <= __ldg(B + d - 1 - mid)) wlo = mid + 1;
        else whi = mid;
      }
      a = wlo;
    }
    P.split_a[q] = a;
  }
}

// ---- k_flow_readers: pieces, identity flags, middle-record reader, resets -------
// Region q's pieces (FlowPiece[4 q .. 4 q + 3]): slot j, the record offsets
// [lo, hi) it reads in that slot, and 2 * side + k (side 0: A, 1: B; k: piece of
// the side).  j == -1: no piece.
__device__ __forceinline__ void ph_readers(const FlowParams& F) {
  const EngineParams& P = F.P;
  FlowGeo g(P);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  if (*(volatile int32_t*)P.noop) return;
  TwoFront tf{P.Q, P.qc};
  unsigned long long sal_tf = 0, nid = 0;
  const int lane = threadIdx.x & 31;
  // (warp-uniform trip count: the identity counts below are warp-aggregated --
  //  one atomic per warp and chunk instead of one per region; skewed jobs such as
  //  config 3 have tens of thousands of identity regions)
  for (int64_t jb = tid - lane; jb < P.K; jb += nthr) {  // (Q == K: region j writes slot j)
    const int64_t j = jb + lane;
    bool idn = false;
    if (j < P.K) {
      const int64_t a0 = g.split(j), a1 = g.split(j + 1), d0 = g.diag(j), d1 = g.diag(j + 1);
      idn = g.identity(j, a0, a1);
      F.idn[j] = idn ? 1 : 0;
      int4 pc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pc[i] = make_int4(-1, 0, 0, 0);
      int i = 0;
      // every slot's middle record lies in exactly one region's A or B range: that
      // region is the slot's reader D[] (the itinerary's next step); the two-front
      // order's salvage is counted here (it decides whether the itinerary phases run)
      const int64_t oj = tf.order(j);
      for_pieces(P, P.s + a0, P.s + a1, P.m + d0 - a0, P.m + d1 - a1, [&](int64_t jj, int64_t lo, int64_t hi, int k, int sd) {
        const int64_t ymid = (g.slot_lo(jj) + g.slot_hi(jj) - 1) >> 1;
        if (lo <= ymid && ymid < hi) F.D[jj] = (int32_t)j | (sd ? (int32_t)0x80000000 : 0);
        if (!idn) {
          const int64_t base = g.slot_base(jj);
          pc[i++] = make_int4((int32_t)jj, (int32_t)(lo - base), (int32_t)(hi - base), 2 * sd + k);
          if (jj != j && oj > tf.order(jj)) sal_tf += (unsigned long long)(hi - lo);
        }
      });
#pragma unroll
      for (int k = 0; k < 4; ++k) F.pieces[4 * j + k] = pc[k];
      F.rank[j] = INT32_MAX;
      F.slo[j] = (int32_t)P.T;
      F.shi[j] = 0;
      F.pend[j] = 0;
    }
    // identity regions per two-front chunk (ph_rank's compaction), and in total
    if (__ballot_sync(0xffffffffu, idn)) {
      const int64_t c = idn ? tf.order(j) / kFlowChunk : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      if (idn && lane == __ffs(peers) - 1) atomicAdd(&F.chunk[c], __popc(peers));
      nid += idn ? 1 : 0;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sal_tf += __shfl_xor_sync(0xffffffffu, sal_tf, o);
    nid += __shfl_xor_sync(0xffffffffu, nid, o);
  }
  if (lane == 0 && sal_tf) atomicAdd((unsigned long long*)&F.fc[FC_SAL_TF], sal_tf);
  if (lane == 0 && nid) atomicAdd((unsigned long long*)&F.fc[FC_NIDENT], nid);
}

// ---- k_flow_angle: itinerary vector per slot --------------------------------------
__device__ __forceinline__ void ph_angle(const FlowParams& F) {
  const EngineParams& P = F.P;
  if (block_flow_off(F)) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const int n = F.nbits;
  const float step = 6.283185307179586f / (float)n;
  for (int64_t j = tid; j < P.K; j += nthr) {
    float zr = 0.f, zi = 0.f;
    if (!F.idn[j]) {
      int32_t x = (int32_t)j;
      for (int i = 1; i <= n; ++i) {
        const int32_t v = F.D[x];
        if (v < 0) {
          float sn, cs;
          __sincosf(step * (float)i, &sn, &cs);
          zr += cs;
          zi += sn;
        }
        x = v & 0x7fffffff;
      }
    }
    F.z[j] = make_float2(zr, zi);
    F.z[P.K + j] = make_float2(0.f, 0.f);
    F.z[2 * P.K + j] = make_float2(0.f, 0.f);
  }
}

// ---- k_flow_sync: one step of angular synchronisation on the reader graph ------
// The angle order wants arg z(reader) = arg z(slot) - delta on every edge; one
// power-iteration step of the edge-weighted phase-synchronisation matrix moves
// each slot's phase to the weighted circular mean of what its readers and the
// slots it reads imply (tools/sim_flow.py: salvage 0.20 N -> 0.15 N in 4 steps).
// z[(it % 3) K ..] is read (normalised on the fly), z[((it + 1) % 3) K ..]
// accumulated, z[((it + 2) % 3) K ..] zeroed for the next step.
__device__ __forceinline__ void ph_sync(const FlowParams& F, int it) {
  const EngineParams& P = F.P;
  if (block_flow_off(F) || F.force >= 0 && F.force != 1) return;
  const int64_t K = P.K;
  const float2* zin = F.z + (it % 3) * K;
  float2* zout = F.z + ((it + 1) % 3) * K;
  float2* zclr = F.z + ((it + 2) % 3) * K;
  float cd, sd;
  __sincosf(6.283185307179586f / (float)F.nsync_div, &sd, &cd);
  auto unit = [](float2 v) {
    const float r = rsqrtf(fmaxf(v.x * v.x + v.y * v.y, 1e-30f));
    return make_float2(v.x * r, v.y * r);
  };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = tid; q < P.Q; q += nthr) {
    zclr[q] = make_float2(0.f, 0.f);
    if (F.idn[q]) continue;
    const float2 zq = unit(zin[q]);
    float ar = 0.f, ai = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int4 pc = F.pieces[4 * q + i];
      if (pc.x < 0 || pc.x == q) continue;
      const float wgt = (float)(pc.z - pc.y);
      const float2 zj = unit(zin[pc.x]);
      // slot j (writer) wants zq * e^{+i delta}; region q (reader) wants zj * e^{-i delta}
      atomicAdd(&zout[pc.x].x, wgt * (zq.x * cd - zq.y * sd));
      atomicAdd(&zout[pc.x].y, wgt * (zq.x * sd + zq.y * cd));
      ar += wgt * (zj.x * cd + zj.y * sd);
      ai += wgt * (zj.y * cd - zj.x * sd);
    }
    if (ar != 0.f || ai != 0.f) {
      atomicAdd(&zout[q].x, ar);
      atomicAdd(&zout[q].y, ai);
    }
  }
}

// ---- k_flow_key: angle bin per slot, histogram ----------------------------------
__device__ __forceinline__ void ph_key(const FlowParams& F, int zbuf) {
  const EngineParams& P = F.P;
  if (block_flow_off(F)) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const float2* z = F.z + zbuf * P.K;
  for (int64_t j = tid; j < P.K; j += nthr) {
    uint32_t key = (uint32_t)F.nb;  // identity: the last bin (never ranked)
    if (!F.idn[j]) {
      const float2 v = z[j];
      float ang = atan2f(v.y, v.x);
      if (ang < 0.f) ang += 6.283185307179586f;
      key = min((uint32_t)(ang * (float)F.nb * 0.15915494309189535f), (uint32_t)F.nb - 1);
      atomicAdd(&F.hist[key], 1);
    }
    F.key[j] = key;
  }
}

// ---- k_flow_choose: salvage volume of the angle order (two fronts: ph_readers) ---
// Region q reads piece (slot j, n records); it reads the salvage entry iff it
// comes after j.  Angle order ties (same bin) are broken by region index here
// (the counting sort breaks them arbitrarily -- an estimate suffices).
__device__ __forceinline__ void ph_choose(const FlowParams& F) {
  const EngineParams& P = F.P;
  if (block_flow_off(F) || F.force >= 0) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  unsigned long long sa = 0;
  for (int64_t q = tid; q < P.Q; q += nthr) {
    if (F.idn[q]) continue;
    const uint32_t kq = F.key[q];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int4 pc = F.pieces[4 * q + i];
      if (pc.x < 0 || pc.x == q) continue;
      const uint32_t kj = F.key[pc.x];
      if (kq > kj || (kq == kj && q > pc.x)) sa += (unsigned long long)(pc.z - pc.y);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sa += __shfl_xor_sync(0xffffffffu, sa, o);
  if ((threadIdx.x & 31) == 0 && sa) atomicAdd((unsigned long long*)&F.fc[FC_SAL_ANGLE], sa);
}

// block-wide exclusive scan of one int32 per thread (blockDim.x <= 1024); returns
// the exclusive prefix, *total the block sum
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* total) {
  __shared__ int32_t ws[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // (ws reuse across calls)
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t s = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) ws[lane] = s;
  }
  __syncthreads();
  *total = ws[nw - 1];
  return (wid ? ws[wid - 1] : 0) + x - v;
}

// one CTA: exclusive scan of v[0, n) in place; each thread scans a contiguous
// segment serially around a single block scan of the segment sums
__device__ __forceinline__ void cta_scan_inplace(int32_t* v, int64_t n) {
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t i0 = min(n, (int64_t)threadIdx.x * per), i1 = min(n, i0 + per);
  int32_t sum = 0;
  for (int64_t i = i0; i < i1; ++i) sum += v[i];
  int32_t tot;
  int32_t run = block_excl_scan(sum, &tot);
  for (int64_t i = i0; i < i1; ++i) {
    const int32_t x = v[i];
    v[i] = run;
    run += x;
  }
}

// ---- k_flow_decide (one CTA): the order, then its scan ------------------------
__device__ __forceinline__ void ph_decide(const FlowParams& F, bool skipped) {
  const EngineParams& P = F.P;
  if (block_flow_off(F)) return;
  __shared__ int32_t s_mode;
  if (threadIdx.x == 0) {
    int32_t mode = F.force;
    if (mode < 0) mode = !skipped && F.fc[FC_SAL_ANGLE] < F.fc[FC_SAL_TF] ? 1 : 0;
    if (skipped) F.fc[FC_SAL_ANGLE] = -1;  // (not evaluated)
    if (mode == 2) {  // debug: exercise the device-side fallback
      F.fc[FC_FAIL] = 1;
      mode = 0;
    }
    s_mode = mode;
    F.fc[FC_MODE] = mode;
    F.fc[FC_NTICK] = (long long)P.Q - F.fc[FC_NIDENT];
  }
  __syncthreads();
  if (s_mode == 1 && F.nb == 16 * (int)blockDim.x) {  // angle bins -> cursors: 16 per thread, vector loads
    int4* h4 = reinterpret_cast<int4*>(F.hist) + 4 * threadIdx.x;
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = h4[u];
    int32_t sum = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) sum += v[u].x + v[u].y + v[u].z + v[u].w;
    int32_t tot;
    int32_t run = block_excl_scan(sum, &tot);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int4 o;
      o.x = run; run += v[u].x;
      o.y = run; run += v[u].y;
      o.z = run; run += v[u].z;
      o.w = run; run += v[u].w;
      h4[u] = o;
    }
  } else if (s_mode == 1) cta_scan_inplace(F.hist, F.nb);
  else cta_scan_inplace(F.chunk, P.Q / kFlowChunk + 1);  // identity regions before each chunk
}

// ---- k_flow_rank: order[] / rank[] -------------------------------------------
// angle order: counting-sort scatter (ties in arrival order); two-front: block b
// compacts tickets [1024 b, 1024 b + 1024) minus identity regions.
__device__ __forceinline__ void ph_rank(const FlowParams& F) {
  const EngineParams& P = F.P;
  if (block_flow_off(F)) return;
  const int32_t mode = (int32_t)F.fc[FC_MODE];
  if (mode == 1) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = tid; j < P.Q; j += nthr) {
      if (F.idn[j]) continue;
      const int32_t t = atomicAdd(&F.hist[F.key[j]], 1);
      F.order[t] = (int32_t)j;
      F.rank[j] = t;
    }
  } else {
    TwoFront tf{P.Q, P.qc};
    for (int64_t b = blockIdx.x; b * kFlowChunk < P.Q; b += gridDim.x) {
      const int64_t t = b * kFlowChunk + threadIdx.x;
      int32_t q = -1, f = 0;
      if (t < P.Q) {
        q = (int32_t)tf.region_of_ticket(t);
        f = F.idn[q] ? 0 : 1;
      }
      int32_t tot;
      const int32_t ex = block_excl_scan(f, &tot);
      if (f) {
        const int32_t pos = (int32_t)(b * kFlowChunk - F.chunk[b]) + ex;
        F.order[pos] = q;
        F.rank[q] = pos;
      }
    }
  }
}

// ---- k_flow_hull: salvage hulls and pending-reader counts ----------------------
__device__ __forceinline__ void ph_hull(const FlowParams& F) {
  const EngineParams& P = F.P;
  if (block_flow_off(F)) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = tid; q < P.Q; q += nthr) {
    if (F.idn[q]) continue;
    const int32_t rq = F.rank[q];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int4 pc = F.pieces[4 * q + i];
      if (pc.x < 0 || pc.x == q) continue;
      if (rq > F.rank[pc.x]) {  // j is written first: q reads its salvage entry
        atomicMin(&F.slo[pc.x], pc.y);
        atomicMax(&F.shi[pc.x], pc.z);
      } else {
        atomicAdd(&F.pend[pc.x], 1);  // j's store waits for this read
      }
    }
  }
}

// ---- k_flow_alloc: pool entries ------------------------------------------------
// Entry of slot j: records [L, H) of the slot, L/H its salvage hull rounded to
// multiples of 16 records (so an entry keeps the caller's 16-byte phase and every
// superset TMA load of a piece stays inside it).  One atomic per block.
__device__ __forceinline__ void ph_alloc(const FlowParams& F) {
  const EngineParams& P = F.P;
  FlowGeo g(P);
  if (block_flow_off(F)) return;
  __shared__ long long s_base;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x; j0 < P.K; j0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    int32_t sz = 0, L = 0;
    if (j < P.K) {
      const int32_t lo = F.slo[j], hi = F.shi[j];
      if (hi > lo) {
        L = lo & ~15;
        sz = ((hi + 15) & ~15) - L;
      }
    }
    int32_t tot;
    const int32_t ex = block_excl_scan(sz, &tot);
    if (threadIdx.x == 0)
      s_base = tot ? (long long)atomicAdd((unsigned long long*)&F.fc[FC_POOL], (unsigned long long)tot) : 0ll;
    __syncthreads();
    const long long base = s_base;
    __syncthreads();
    if (sz) {
      const long long off = base + ex;  // multiple of 16 records
      if (off + sz > F.pool_cap) {  // (a pure rotation takes the block exchange instead)
        atomicExch((unsigned long long*)&F.fc[F.fc[FC_ROT] ? FC_ROTFAIL : FC_FAIL], 1ull);
        if (F.fc[FC_ROT]) P.stats[13] = 1;  // pm_status: the block-exchange route ran
      } else {
        F.pdelta[j] = off - (g.slot_base(j) + L);
        atomicAdd((unsigned long long*)&F.fc[FC_NSALV], 1ull);
      }
    }
  }
}

// ---- k_flow_tickets: per-ticket descriptors ------------------------------------
__device__ __forceinline__ void ph_tickets(const FlowParams& F) {
  const EngineParams& P = F.P;
  FlowGeo g(P);
  if (block_flow_off(F)) return;
  const int64_t nt = F.fc[FC_NTICK];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {  // pm_status: salvaged slots / records, identity regions, order, both salvage estimates
    P.stats[0] = (unsigned long long)F.fc[FC_NSALV];
    P.stats[1] = (unsigned long long)F.fc[FC_POOL];
    P.stats[3] = (unsigned long long)F.fc[FC_NIDENT];
    P.stats[4] = (unsigned long long)(F.fc[FC_MODE] + 1);
    P.stats[5] = (unsigned long long)F.fc[FC_SAL_ANGLE];
    P.stats[6] = (unsigned long long)F.fc[FC_SAL_TF];
  }
  for (int64_t t = tid; t < nt; t += nthr) {
    const int32_t q = F.order[t];
    FLOW_CHECK(q >= 0 && q < P.Q && F.rank[q] == (int32_t)t && !F.idn[q]);
    FlowTicket T;
    T.r = q;
    T.flags = 0;
    T.ja[0] = T.ja[1] = T.jb[0] = T.jb[1] = -1;
    T.pad_[0] = T.pad_[1] = 0;
    T.a0 = g.split(q);
    T.a1 = g.split(q + 1);
    T.dA[0] = T.dA[1] = T.dB[0] = T.dB[1] = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int4 pc = F.pieces[4 * q + i];
      if (pc.x < 0) continue;
      const int k = pc.w & 1;
      const bool pool = pc.x != q && F.rank[pc.x] < (int32_t)t;
      if (pc.w < 2) {
        T.ja[k] = pc.x;
        if (pool) {
          T.flags |= 1 << (1 + k);
          T.dA[k] = F.pdelta[pc.x];
        }
      } else {
        T.jb[k] = pc.x;
        if (pool) {
          T.flags |= 1 << (3 + k);
          T.dB[k] = F.pdelta[pc.x];
        }
      }
    }
    F.tk[t] = T;
  }
}

// ---- k_flow_save: copy the salvage entries into the pool ------------------------
// Work items are (slot, chunk of the slot): a skewed job's salvage sits in a few
// slots, and one warp copying a whole 32 KB entry is a chain of dependent round
// trips; chunks spread an entry over several warps.  As many chunks per slot as
// keep the scan to one pass (lanes of all warps >= items), at least 8 KB of keys
// each (2 KB items: 0.24 -> 0.35 ms at 2^30 int32, 0.07 -> 0.11 ms at config 4).
// Each warp scans 32 items at a time (one per lane, lane-strided so every warp
// gets items), then copies the items that hold salvage one after another with
// the whole warp (16-byte vectors, identical phase on both sides).
__device__ __forceinline__ void ph_save(const FlowParams& F) {
  const EngineParams& P = F.P;
  FlowGeo g(P);
  const int lane = threadIdx.x & 31;
  const int64_t ks = P.ks, w = P.w;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nc = max((int64_t)1, min(32 * nw / P.K, P.T * ks / 8192)), items = P.K * nc;
  const int32_t csz = (int32_t)((P.T + nc - 1) / nc);
  for (int64_t i0 = w0; i0 < items; i0 += nw * 32) {
    const int64_t it = i0 + lane * nw;  // (lane-strided: every warp gets items while items >= warps)
    int64_t x0 = 0, x1 = 0, dl = 0;
    if (it < items) {
      const int64_t j = it / nc, c = it - j * nc;
      const int32_t lo = max(F.slo[j], (int32_t)c * csz), hi = min(F.shi[j], (int32_t)(c + 1) * csz);
      if (hi > lo) {
        const int64_t base = g.slot_base(j);
        // the records of the hull that belong to the job
        x0 = max(base + lo, g.slot_lo(j));
        x1 = min(base + hi, g.slot_hi(j));
        dl = F.pdelta[j];
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, x1 > x0);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t y0 = __shfl_sync(0xffffffffu, x0, src), y1 = __shfl_sync(0xffffffffu, x1, src);
      const int64_t d = __shfl_sync(0xffffffffu, dl, src);
      FLOW_CHECK(y0 + d >= 0 && y1 + d <= F.pool_cap && y0 >= P.s && y1 <= P.e);
      copy_g2g_warp(reinterpret_cast<uint8_t*>(F.pool_keys + (y0 + d) * ks),
                    reinterpret_cast<const uint8_t*>(P.keys + y0 * ks), (y1 - y0) * ks, lane);
      if (w) copy_g2g_warp(F.pool_pay + (y0 + d) * w, P.pay + y0 * w, (y1 - y0) * w, lane);
    }
  }
}

// ---- k_flow_plan: every plan phase in one cooperative launch --------------------
// One CTA of 1024 threads per SM; a grid-wide barrier between phases replaces a
// kernel boundary (the phases are short and latency-bound: launch gaps and tails
// dominated when they were separate kernels).  Every early exit (noop, FC_FAIL)
// is taken by the whole grid, after a barrier, so no CTA is left waiting.
#ifndef PM_FLOW_DEBUG
#define PM_FLOW_DEBUG 0
#endif
#ifndef PM_FLOW_SAVE_IN_PLAN
#define PM_FLOW_SAVE_IN_PLAN 0  // 1: salvage copy inside the plan kernel, beside the tickets (2^30: plan + copy 0.401 vs 0.129 + 0.225 ms separate -- the plan grid copies slower)
#endif
#ifndef PM_FLOW_TF_EARLY
#define PM_FLOW_TF_EARLY 32
#endif
// tuning builds (-DPM_FLOW_DEBUG=1): %globaltimer after each phase -> stats[32 + k]
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PM_FLOW_DBG(k) \
  if (PM_FLOW_DEBUG && threadIdx.x == 0 && blockIdx.x == 0) F.P.stats[32 + (k)] = gtimer()
template <typename KT>
__global__ void __launch_bounds__(kFlowChunk, 1) k_flow_plan(FlowParams F) {
  cg::grid_group grid = cg::this_grid();
  PM_FLOW_DBG(0);
  ph_sample<KT>(F);
  grid.sync();
  PM_FLOW_DBG(1);
  if (*(volatile int32_t*)F.P.noop || *(volatile long long*)&F.fc[FC_ROTFAIL]) return;
  ph_split<KT>(F);
  grid.sync();
  PM_FLOW_DBG(2);
  ph_readers(F);
  grid.sync();
  PM_FLOW_DBG(3);
  // the two-front order needs no itinerary (lean plan): forced, or in auto mode
  // when its salvage is already below 1/PM_FLOW_TF_EARLY of the job (skewed or
  // translated inputs: the angle order could save at most that copy, its phases
  // cost more); the word is final after the barrier, so every CTA agrees
  const bool skip = F.force == 0 || (F.force < 0 && *(volatile long long*)&F.fc[FC_SAL_TF] * PM_FLOW_TF_EARLY <=
                                                        (long long)(F.P.e - F.P.s));
  if (!skip) {
    ph_angle(F);
    grid.sync();
    PM_FLOW_DBG(4);
    const bool angle = F.force < 0 || F.force == 1;
    for (int it = 0; angle && it < F.nsync; ++it) {
      ph_sync(F, it);
      grid.sync();
      PM_FLOW_DBG(5);
    }
    ph_key(F, angle ? F.nsync % 3 : 0);
    grid.sync();
    PM_FLOW_DBG(6);
    ph_choose(F);
    grid.sync();
    PM_FLOW_DBG(7);
  }
  if (blockIdx.x == 0) ph_decide(F, skip && F.force < 0);
  grid.sync();
  PM_FLOW_DBG(8);
  ph_rank(F);
  grid.sync();
  PM_FLOW_DBG(9);
  ph_hull(F);
  grid.sync();
  PM_FLOW_DBG(10);
  ph_alloc(F);
  grid.sync();
  PM_FLOW_DBG(11);
  ph_tickets(F);
  PM_FLOW_DBG(12);
#if PM_FLOW_SAVE_IN_PLAN
  // the salvage copy in the same phase as the tickets (both need only the pool
  // offsets): no kernel boundary, and the tickets overlap the copy
  if (!block_flow_off(F)) ph_save(F);
#endif
}

__global__ void __launch_bounds__(256) k_flow_save(FlowParams F) {
  if (flow_off(F)) return;
  ph_save(F);
}

// Prescribed layout (pm_reorder): output o of the region at job-local diagonal d0
// is A[a] or B[b] of its leaf; thread gt writes outputs [o0, o1) (consecutive,
// one leaf search per thread, then a linear walk across leaf boundaries).
template <typename KT, int GT>
__device__ __forceinline__ void concat_tile(const FlowParams& F, int64_t d0, int64_t a0, int64_t b0, const KT* As,
                                            const KT* Bs, int32_t nout, KT* ko, uint8_t* po, const uint8_t* PA,
                                            const uint8_t* PB, int64_t w, int gt) {
  const int32_t E = (nout + GT - 1) / GT;
  const int32_t o0 = min(gt * E, nout), o1 = min(o0 + E, nout);
  if (o0 >= o1) return;
  int32_t i = leaf_of(F, d0 + o0);
  int64_t lend = F.leaf_l[i + 1], lstart = F.leaf_l[i], na = F.leaf_a[i + 1] - F.leaf_a[i], apre = F.leaf_a[i];
  for (int32_t o = o0; o < o1; ++o) {
    const int64_t d = d0 + o;
    while (d >= lend) {
      ++i;
      lstart = lend;
      lend = F.leaf_l[i + 1];
      apre = F.leaf_a[i];
      na = F.leaf_a[i + 1] - apre;
    }
    const int64_t off = d - lstart;
    if (off < na) {
      const int64_t x = apre + off - a0;  // staged A position
      ko[o] = As[x];
      if (w) for (int64_t c = 0; c < w; ++c) po[(int64_t)o * w + c] = PA[x * w + c];
    } else {
      const int64_t x = d - (apre + na) - b0;  // B index d - leaf_a[i+1], staged
      ko[o] = Bs[x];
      if (w) for (int64_t c = 0; c < w; ++c) po[(int64_t)o * w + c] = PB[x * w + c];
    }
  }
}

// ---- k_flow: the streaming in-place merge ---------------------------------------
struct FlowDesc {
  int64_t d0;
  int32_t r, alpha, beta, nout, offA, offB, poffA, poffB;
  int32_t rd[4];  // slots read from their original place (pend[] to release), -1: none
};

__device__ __forceinline__ FlowTicket load_ticket(const FlowTicket* p) {
  FlowTicket T;
  const uint4* s = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(&T);
#pragma unroll
  for (int i = 0; i < 5; ++i) d[i] = __ldg(s + i);
  return T;
}

// leader: the region's geometry, then TMA loads of its pieces into the stage
template <typename KT>
__device__ __forceinline__ void flow_issue(const FlowParams& F, const FlowGeo& g, const FlowTicket& T,
                                           FlowDesc& D, uint8_t* kin, uint8_t* pin, uint64_t* bar) {
  const EngineParams& P = F.P;
  const int64_t ks = sizeof(KT), w = P.w;
  const int64_t q = T.r;
  const int64_t d0 = g.diag(q), d1 = g.diag(q + 1);
  const int64_t a0 = T.a0, a1 = T.a1, b0 = d0 - a0, b1 = d1 - a1;
  const int64_t alpha = a1 - a0, beta = b1 - b0;
  const int64_t xa = P.s + a0, xb = P.m + b0;
  D.d0 = d0;
  D.r = (int32_t)q;
  D.alpha = (int32_t)alpha;
  D.beta = (int32_t)beta;
  D.nout = (int32_t)(d1 - d0);
  const int64_t offA = ((uintptr_t)(P.keys + xa * ks)) & 15;
  const int64_t offB = ((offA + (alpha + kSent) * ks + 15) & ~(int64_t)15) + (((uintptr_t)(P.keys + xb * ks)) & 15);
  int64_t poffA = 0, poffB = 0;
  if (w) {
    poffA = ((uintptr_t)(P.pay + xa * w)) & 15;
    poffB = ((poffA + alpha * w + 15) & ~(int64_t)15) + (((uintptr_t)(P.pay + xb * w)) & 15);
  }
  D.offA = (int32_t)offA;
  D.offB = (int32_t)offB;
  D.poffA = (int32_t)poffA;
  D.poffB = (int32_t)poffB;
  int nrd = 0;
  D.rd[0] = D.rd[1] = D.rd[2] = D.rd[3] = -1;
  // slot boundaries are 16-byte aligned only when both bases are (see copy_g2s_piece)
  const bool exact = (((uintptr_t)P.keys) & 15) || (w && (((uintptr_t)P.pay) & 15));
  for_pieces(P, xa, xa + alpha, xb, xb + beta, [&](int64_t j, int64_t x, int64_t y, int k, int side) {
    const bool pool = (T.flags >> (side ? 3 + k : 1 + k)) & 1;
    const int64_t dl = pool ? (side ? T.dB[k] : T.dA[k]) : 0;
    FLOW_CHECK(x < y && (side ? (x >= P.m && y <= P.e) : (x >= P.s && y <= P.m)));
    FLOW_CHECK(j == (x >> P.lT) - P.k0 && j == ((y - 1) >> P.lT) - P.k0 && j >= 0 && j < P.K);
    FLOW_CHECK(!pool || (x + dl >= 0 && y + dl <= F.pool_cap));
    FLOW_CHECK(!pool || (j != q && F.rank[j] < F.rank[q] && x - g.slot_base(j) >= F.slo[j] &&
                         y - g.slot_base(j) <= F.shi[j]));
    FLOW_CHECK(pool || j == q || F.rank[j] > F.rank[q]);
    const int64_t o = side ? x - xb : x - xa;  // records already staged on this side
    const char* ksrc = (pool ? F.pool_keys : P.keys) + (x + dl) * ks;
    copy_g2s_piece(kin + (side ? offB : offA) + o * ks, reinterpret_cast<const uint8_t*>(ksrc), (y - x) * ks, bar,
                   exact);
    if (w) {
      const uint8_t* psrc = (pool ? F.pool_pay : P.pay) + (x + dl) * w;
      copy_g2s_piece(pin + (side ? poffB : poffA) + o * w, psrc, (y - x) * w, bar, exact);
    }
    if (!pool && j != q) D.rd[nrd++] = (int32_t)j;
  });
  mbar_arrive(bar);
}

// the region's reads have landed: release the original slots it read
__device__ __forceinline__ void flow_release(const FlowParams& F, const FlowDesc& D) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (D.rd[i] >= 0) {
      const int32_t old = atomicSub(&F.pend[D.rd[i]], 1);
      FLOW_CHECK(old > 0);  // every release was counted by the plan
      (void)old;
    }
}

// Persistent, software-pipelined (k_buffered's shape).  The control warp's lane 0
// ("leader") claims tickets two ahead and loads each ticket's descriptor one
// iteration before it issues the region's TMA loads, so the only round trips left
// on its path are the pend[] polls, which are issued before the stage wait.
template <typename KT>
__global__ void __launch_bounds__(kFlowThreads) k_flow(FlowParams F) {
  constexpr int NS = kFlowStages;
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ uint64_t bar[NS];
  __shared__ int64_t s_t[NS];
  __shared__ FlowDesc s_d[NS];
  __shared__ int32_t s_early[NS];
  __shared__ FlowTicket s_next;  // the leader's prefetched ticket (in shared memory: no registers for all threads)
  const EngineParams& P = F.P;
  FlowGeo g(P);
  constexpr int NT = kFlowThreads;
  const int tid = threadIdx.x, lane = tid & 31;
  const int NW = NT >> 5;
  const bool ctrl = (tid >> 5) == NW - 1;
  const bool leader = ctrl && lane == 0;
  const int MT = NT - 32;
  const int64_t ks = sizeof(KT), w = P.w;
  if (flow_off(F)) return;
  const int64_t ntick = F.fc[FC_NTICK];
  const size_t tile = P.smem_keys + P.smem_pay;
#define STAGE(b) (dyn + (size_t)(b) * tile)
#define OUTB(b) (dyn + (size_t)(NS + (b)) * tile)
  int64_t t_next = ntick;  // leader: the next ticket to issue, its descriptor loaded ahead
  if (leader) {
    for (int k = 0; k < NS; ++k) {
      mbar_init(&bar[k], 1);
      s_early[k] = 0;
      s_t[k] = ntick;
    }
    for (int k = 0; k < NS - 1; ++k) {
      const int64_t t0 = (*(volatile int32_t*)P.err) ? ntick : atomicAdd(P.ticket, 1);
      s_t[k] = t0 < ntick ? t0 : ntick;
      if (t0 >= ntick) break;
      flow_issue<KT>(F, g, load_ticket(F.tk + t0), s_d[k], STAGE(k), STAGE(k) + P.smem_keys, &bar[k]);
    }
    t_next = atomicAdd(P.ticket, 1);
    if (t_next < ntick) s_next = load_ticket(F.tk + t_next);
    else t_next = ntick;
  }
  __syncthreads();
  uint32_t phmask = 0;
  unsigned long long n_reg = 0;
  for (int it = 0;; ++it) {
    const int cur = it % NS, ob = kFlowOut == 2 ? (it & 1) : 0;
    const int64_t t = s_t[cur];
    if (t >= ntick) break;
    const FlowDesc& R = s_d[cur];  // (read in place: the leader rewrites it only after the next barrier)
    int32_t pv = 0;
    if (leader) {
      pv = ld_relaxed(&F.pend[R.r]);  // first poll of this region's store condition, in flight now
      // keep NS-1 regions in flight: the previous iteration's stage is free
      const int nx = (it + NS - 1) % NS;
      const int64_t tn = (*(volatile int32_t*)P.err) ? ntick : t_next;
      s_t[nx] = tn;
      s_early[nx] = 0;
      if (tn < ntick) {
        flow_issue<KT>(F, g, s_next, s_d[nx], STAGE(nx), STAGE(nx) + P.smem_keys, &bar[nx]);
        t_next = atomicAdd(P.ticket, 1);
        if (t_next < ntick) s_next = load_ticket(F.tk + t_next);  // used next iteration
        else t_next = ntick;
      }
    }
    while (!mbar_try_wait(&bar[cur], (phmask >> cur) & 1)) {
    }
    phmask ^= 1u << cur;
    const int64_t phk = ((uintptr_t)(P.keys + (P.s + R.d0) * ks)) & 15;
    const int64_t php = w ? (((uintptr_t)(P.pay + (P.s + R.d0) * w)) & 15) : 0;
    uint8_t* kout_s = OUTB(ob);
    uint8_t* pout_s = OUTB(ob) + P.smem_keys;
    if (ctrl) {
      if (leader) {
        // (relaxed: the loads have completed -- the barrier said so -- so a writer that
        // sees the count drop cannot change what this region read)
        if (!s_early[cur]) flow_release(F, R);
        // regions in flight whose loads have landed: release their reads now -- other
        // CTAs' stores may be waiting for them (checked again while this one waits)
        auto release_landed = [&]() {
          for (int k = 1; k < NS; ++k) {
            const int sk = (it + k) % NS;
            if (s_t[sk] < ntick && !s_early[sk] && mbar_try_wait(&bar[sk], (phmask >> sk) & 1)) {
              flow_release(F, s_d[sk]);
              s_early[sk] = 1;
            }
          }
        };
        release_landed();
        // every lower-ranked reader of this slot has read it
        if (PM_FLOW_ABLATE & 1) pv = 0;  // (timing ablation: results are wrong)
        for (uint32_t it2 = 0; pv != 0; ++it2) {
          if ((it2 & 255) == 255 && ld_relaxed(P.err)) break;
          if (it2 > kSpinLimit) {
            raise_error(P.err, PM_ERR_TIMEOUT);
            break;
          }
          backoff(it2);
          release_landed();
          pv = ld_relaxed(&F.pend[R.r]);
        }
      }
      __syncwarp();
    } else {
      uint8_t* kin = STAGE(cur);
      uint8_t* pin = STAGE(cur) + P.smem_keys;
      if (F.nleaves) {  // prescribed layout: concatenate the leaf slices
        const int64_t a0 = F.P.split_a[R.r];
        concat_tile<KT, kFlowThreads - 32>(F, R.d0, a0, R.d0 - a0, reinterpret_cast<const KT*>(kin + R.offA),
                                           reinterpret_cast<const KT*>(kin + R.offB), R.nout,
                                           reinterpret_cast<KT*>(kout_s + phk), pout_s + php, pin + R.poffA,
                                           pin + R.poffB, w, tid);
      } else {
        if (!w) {
          write_sentinels<KT>(kin, R.offA, R.alpha, R.offB, R.beta, tid, MT);
          named_barrier_sync(1, MT);
        }
        const bool wq4 = w && (w & 3) == 0 && ((php | R.poffA | R.poffB) & 3) == 0;
        if (wq4 && w >= kWideRow)
          merge_tile_wide<KT, kFlowThreads - 32>(reinterpret_cast<const KT*>(kin + R.offA),
                                                 reinterpret_cast<const KT*>(kin + R.offB), R.alpha, R.beta, R.nout,
                                                 reinterpret_cast<KT*>(kout_s + phk), pout_s + php, pin + R.poffA,
                                                 pin + R.poffB, w, tid, 1);
        else if (!(PM_FLOW_ABLATE & 2))
          merge_tile<KT, kFlowThreads - 32>(MODE_MERGE, reinterpret_cast<const KT*>(kin + R.offA),
                                            reinterpret_cast<const KT*>(kin + R.offB), R.alpha, R.beta, R.nout,
                                            reinterpret_cast<KT*>(kout_s + phk), pout_s + php, pin + R.poffA,
                                            pin + R.poffB, w, wq4, tid);
      }
      fence_proxy_async_smem();
    }
    __syncthreads();  // tile complete, slot clear
    const int gt = (tid + 32) % NT;
    FLOW_CHECK(R.d0 >= 0 && R.d0 + R.nout <= P.e - P.s && R.nout == g.slot_hi(R.r) - g.slot_lo(R.r) &&
               P.s + R.d0 == g.slot_lo(R.r));
    FLOW_CHECK(F.pend[R.r] == 0 || *(volatile int32_t*)P.err);
    if (!(PM_FLOW_ABLATE & 4)) {
      stream_out(kout_s + phk, reinterpret_cast<uint8_t*>(P.keys + (P.s + R.d0) * ks), (int64_t)R.nout * ks, gt, NT);
      if (w) stream_out(pout_s + php, P.pay + (P.s + R.d0) * w, (int64_t)R.nout * w, gt, NT);
    }
    ++n_reg;
    if (leader) {
      if (kFlowOut == 2) bulk_wait_read<1>();  // the store that used the other output buffer has read it
      else bulk_wait_read<0>();                // one output tile: this store has read it
    }
    __syncthreads();
  }
  if (leader) {
    bulk_wait_all();
    atomicAdd(&P.stats[2], n_reg);
  }
#undef STAGE
#undef OUTB
}

// ---- host launcher ---------------------------------------------------------------
// (the caller caches both answers per device and geometry: these queries and the
// attribute call cost more host time than the launches they configure)
// attr_smem: the k_flow dynamic shared memory limit to set (>= smem; the largest any
// call on this device has needed, so a cached geometry never sees a lowered limit)
template <typename KT>
cudaError_t flow_occupancy(size_t smem, size_t attr_smem, int* blocks_per_sm, int* plan_blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_flow<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attr_smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_flow<KT>, kFlowThreads, smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(plan_blocks_per_sm, k_flow_plan<KT>, kFlowChunk, 0);
}

// plan kernels (after launch_plan's splits); ev (may be null) is recorded between
// the plan and the merge
struct NvtxRange {
  explicit NvtxRange(const char* what) { nvtxRangePushA(what); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <typename KT>
cudaError_t launch_flow(const FlowParams& F, int grid, size_t smem, int num_sms, int bps, cudaStream_t st,
                        cudaEvent_t ev, cudaEvent_t ev_merge, cudaEvent_t ev_fork) {
  cudaError_t e;
  if (bps < 1) return cudaErrorInvalidConfiguration;
  FlowParams Fa = F;
  void* args[] = {&Fa};
  // NVTX phase ranges (host-side enqueue spans; nsys correlates them with the kernels)
  NvtxRange r_all("pm_merge: scheduled engine");
  // plan grid sized to the job (grid barriers over fewer CTAs are cheaper; every phase
  // strides over its items): ~PM_FLOW_PLAN_PER regions per CTA, at most every SM
#ifndef PM_FLOW_PLAN_PER
#define PM_FLOW_PLAN_PER 256
#endif
  const int pgrid = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)num_sms * std::min(bps, 2), (F.P.Q + PM_FLOW_PLAN_PER - 1) / PM_FLOW_PLAN_PER));
  e = cudaLaunchCooperativeKernel((const void*)k_flow_plan<KT>, dim3(pgrid), dim3(kFlowChunk), args,
                                  0, st);
  if (e != cudaSuccess) return e;
  count_launches(1);
  if (ev) {
    e = cudaEventRecord(ev, st);
    if (e != cudaSuccess) return e;
  }
  if (ev_fork) {  // the gated fallback engine may start on a side stream from here
    e = cudaEventRecord(ev_fork, st);
    if (e != cudaSuccess) return e;
  }
  if (!PM_FLOW_SAVE_IN_PLAN) {
    NvtxRange r("pm_flow: salvage copy");
    k_flow_save<<<num_sms * 8, 256, 0, st>>>(F);
    count_launches(1);
  }
  if (ev_merge) {
    e = cudaEventRecord(ev_merge, st);
    if (e != cudaSuccess) return e;
  }
  {
    NvtxRange r("pm_flow: merge");
    k_flow<KT><<<grid, kFlowThreads, smem, st>>>(F);
  }
  count_launches(1);

  return cudaGetLastError();
}

template cudaError_t flow_occupancy<int32_t>(size_t, size_t, int*, int*);
template cudaError_t flow_occupancy<int64_t>(size_t, size_t, int*, int*);
template cudaError_t launch_flow<int32_t>(const FlowParams&, int, size_t, int, int, cudaStream_t, cudaEvent_t,
                                          cudaEvent_t, cudaEvent_t);
template cudaError_t launch_flow<int64_t>(const FlowParams&, int, size_t, int, int, cudaStream_t, cudaEvent_t,
                                          cudaEvent_t, cudaEvent_t);

}  // namespace pm
