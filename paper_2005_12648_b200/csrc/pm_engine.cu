// pm_engine.cu -- plan + in-place merge engine + streaming pipeline kernels (sm_100a).
//
// k_plan_coarse / k_plan : stable merge-path splits at every region diagonal
//            (a warp per coarse boundary, bracketed per-thread searches between)
//            + workspace reset; k_flags / k_compact: the engine's ticket list.
// k_engine : persistent kernel; salvage workers close each
//            region's slot and move still-needed units out, the data team
//            gathers the region's A/B pieces into shared memory with TMA bulk
//            copies, merges there and streams the region back in place.
// k_buffered : streaming TMA pipeline -- the out-of-place merge (pm_merge_copy)
//            and the min-side-buffered in-place mode (seq_merge_buffered budget).
//
// Reference behaviour being reproduced (bit-exact): the stable merge of
// seq_merge_buffered (seqmerge.py:55-75 / _kernels.py:227-313, A wins ties)
// and the block exchange of linear_shift / circular_shift (_kernels.py:92-197).
#include <cuda_runtime.h>

#include <algorithm>

#include "pm_common.cuh"
#include "pm_launch.h"
#include "pm_engine.cuh"
#include "pm_search.cuh"
#include "pm_tile.cuh"
#include "pm_hostcache.h"

namespace pm {

// -DPM_STATS=1 (tuning builds): cycle counters and path counters in pm_debug_stats
#ifndef PM_STATS
#define PM_STATS 0
#endif
#ifndef PM_ITEM_RESAMPLE
#define PM_ITEM_RESAMPLE 0
#endif
#ifndef PM_PREFETCH_ITEM
#define PM_PREFETCH_ITEM 1
#endif
#ifndef PM_PREFETCH_MOVE
#define PM_PREFETCH_MOVE 0
#endif
#ifndef PM_TLIST
#define PM_TLIST 1  // tune: engine tickets skip identity regions
#endif
// timing ablations (tuning builds only; results are wrong)
#ifndef PM_ABLATE
#define PM_ABLATE 0  // bit 0: tile merge, 1: salvage copies, 2: gather loads, 3: output stores
#endif


// ============================================================================
// lock-free stacks of free slots / scratch units (Treiber stack, ABA tag)
// ============================================================================
__device__ __forceinline__ void stack_push(unsigned long long* top, int32_t* next, int32_t idx) {
  unsigned long long old = *(volatile unsigned long long*)top, nw;
  do {
    next[idx] = (int32_t)(uint32_t)(old & 0xFFFFFFFFull);
    fence_acq_rel_gpu();
    nw = (((old >> 32) + 1ull) << 32) | (uint32_t)idx;
    unsigned long long seen = atomicCAS(top, old, nw);
    if (seen == old) break;
    old = seen;
  } while (true);
}
__device__ __forceinline__ int32_t stack_pop(unsigned long long* top, int32_t* next) {
  unsigned long long old = *(volatile unsigned long long*)top;
  while (true) {
    uint32_t idx = (uint32_t)(old & 0xFFFFFFFFull);
    if (idx == kEmpty32) return -1;
    int32_t nxt = *(volatile int32_t*)&next[idx];
    unsigned long long nw = (((old >> 32) + 1ull) << 32) | (uint32_t)nxt;
    unsigned long long seen = atomicCAS(top, old, nw);
    if (seen == old) {
      fence_acq_rel_gpu();
      return (int32_t)idx;
    }
    old = seen;
  }
}

// ============================================================================
// k_plan: merge-path splits + workspace reset
// ============================================================================
#ifndef PM_PLAN_INTERP
#define PM_PLAN_INTERP 8  // tune: interpolation probes of k_plan's split search (0: binary only)
#endif
constexpr int kCoarse = 64;  // k_plan_coarse searches every kCoarse-th region boundary
// Up to kWarpPlan boundaries (jobs of up to ~2^24 records) k_plan alone runs one
// warp per boundary over the full range (33-ary ballot search: ~5 dependent
// probes), without k_plan_coarse: the two-level plan's thread-per-boundary
// binary searches were a chain of ~18 dependent DRAM probes on 3 CTAs (2^21
// records: 6 + 15 us of plan for an 11 us merge).  Larger jobs keep the two
// levels (a warp per boundary would multiply the probe traffic by 32).
#ifndef PM_WARP_PLAN
#define PM_WARP_PLAN 8192
#endif
constexpr int64_t kWarpPlan = PM_WARP_PLAN;
// Full-range merge-path searches at every kCoarse-th boundary (and the last);
// k_plan then searches the boundaries in between inside these brackets.
template <typename KT>
__global__ void __launch_bounds__(256) k_plan_coarse(EngineParams P) {
  if (!P.gate_out && P.gate && !*(volatile const int32_t*)P.gate) return;  // (gate_out: k_plan computes it next)
  Geo g(P);
  const KT* keys = reinterpret_cast<const KT*>(P.keys);
  const int64_t la = g.LA(), lb = g.LB();
  const KT* B = P.keys_b ? reinterpret_cast<const KT*>(P.keys_b) : keys + P.m;
  // one warp per coarse boundary: 33-ary ballot search, ~6 dependent probes at 2^29
  const int lane = threadIdx.x & 31;
  const int64_t nc = P.Q / kCoarse + 1;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w0; c <= nc; c += nw) {
    const int64_t q = min(c * kCoarse, P.Q);
    const int64_t d = g.diag(q);
    int64_t a;
    if (P.mode == MODE_MERGE) {
      a = merge_path_warp<KT>(keys + P.s, la, B, lb, d, lane);
    } else {
      a = d - lb;
      a = a < 0 ? 0 : (a > la ? la : a);
    }
    if (lane == 0) P.split_a[q] = a;
  }
}

template <typename KT>
__global__ void k_plan(EngineParams P) {
  Geo g(P);
  const KT* keys = reinterpret_cast<const KT*>(P.keys);
  const int64_t la = g.LA(), lb = g.LB();
  if (P.gate_out) {  // staged path: the gate the later kernels read (srecpar.py:56-57)
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.gate_out = keys[P.m - 1] > keys[P.m] ? 1 : 0;
  } else if (P.gate && !*(volatile const int32_t*)P.gate) {
    return;
  }
  if (P.Q + 1 <= kWarpPlan) {  // one warp per boundary, full range
    const KT* B = P.keys_b ? reinterpret_cast<const KT*>(P.keys_b) : keys + P.m;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = w0; q <= P.Q; q += nw) {
      const int64_t d = g.diag(q);
      int64_t a;
      if (P.mode == MODE_MERGE) {
        a = merge_path_warp<KT>(keys + P.s, la, B, lb, d, lane);
      } else {
        a = d - lb;
        a = a < 0 ? 0 : (a > la ? la : a);
      }
      if (lane == 0) P.split_a[q] = a;
    }
  } else {
  // one thread per region boundary: binary search of the stable merge path
  // (2 independent loads per step, every search in flight at once), bounded by
  // the coarse splits k_plan_coarse found every kCoarse boundaries
    const int64_t tid0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthr0 = (int64_t)gridDim.x * blockDim.x;
    const KT* B = P.keys_b ? reinterpret_cast<const KT*>(P.keys_b) : keys + P.m;
    for (int64_t q = tid0; q <= P.Q; q += nthr0) {
      if ((q & (kCoarse - 1)) == 0 || q == P.Q) continue;  // (coarse boundary: done)
      const int64_t d = g.diag(q);
      int64_t a;
      if (P.mode == MODE_MERGE) {
        const int64_t q0 = q & ~(int64_t)(kCoarse - 1), q1 = min(q0 + kCoarse, P.Q);
        const int64_t a0 = P.split_a[q0], a1 = P.split_a[q1];
        const int64_t b0 = g.diag(q0) - a0, b1 = g.diag(q1) - a1;
        // a is monotone in d and so is b = d - a: both stay between the coarse splits
        int64_t lo = max(max(a0, d - b1), max(d - lb, (int64_t)0));
        int64_t hi = min(min(a1, d - b0), min(d, la));
        // both bracket ends inside the runs: their values (one round trip), then
        // interpolation (pm_search.cuh) before the binary search
        if (hi - lo > 64 && lo - 1 >= max(d - lb, (int64_t)0) && hi < la && d - 1 - hi >= 0) {
          const KT* A = keys + P.s;
          const double fl = (double)__ldg(A + lo - 1) - (double)__ldg(B + d - lo);
          const double fh = (double)__ldg(A + hi) - (double)__ldg(B + d - 1 - hi);
          if (fl <= 0.0 && fh > 0.0) interp_bracket<KT>(A, B, d, &lo, &hi, fl, fh, PM_PLAN_INTERP);
        }
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (__ldg(keys + P.s + mid) <= __ldg(B + d - 1 - mid)) lo = mid + 1;
          else hi = mid;
        }
        a = lo;
      } else {  // rotation: outputs are B then A
        a = d - lb;
        a = a < 0 ? 0 : (a > la ? la : a);
      }
      P.split_a[q] = a;
    }
  }
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (P.state) {  // (the scheduled engine keeps none of the engine's unit bookkeeping)
    for (int64_t j = tid; j < P.K; j += nthr) {
      P.state[j] = (int32_t)j;
      P.loc[j] = (int32_t)j;
      P.reads[j] = 0;
    }
    // scratch units [0, G) start in the engine CTAs' caches (s_per each, k_engine);
    // unit i >= G starts on shard (i - G) % kShards
    const int64_t G = (int64_t)P.grid * P.s_per;
    for (int64_t i = G + tid; i < P.S; i += nthr)
      P.next_scr[i] = (i + kShards < P.S) ? (int32_t)(i + kShards) : (int32_t)kEmpty32;
    for (int64_t sh = tid; sh < kShards; sh += nthr) {
      P.free_top[sh * kTopStride] = (unsigned long long)kEmpty32;
      P.scr_top[sh * kTopStride] = G + sh < P.S ? (unsigned long long)(G + sh) : (unsigned long long)kEmpty32;
    }
  }
  if (tid == 0) {
    *P.ticket = 0;
    bool nothing = (la == 0 || lb == 0);
    if (P.out_keys) nothing = false;  // out of place: every record still moves
    else if (!nothing && P.mode == MODE_MERGE) nothing = keys[P.m - 1] <= keys[P.m];  // srecpar.py:56-57
    *P.noop = nothing ? 1 : 0;
    *P.need_space = 0;
    if (P.ntick) P.ntick[1] = 0;  // identity regions (k_flags)
    for (int i = 0; i < 64; ++i) P.stats[i] = 0;
  }
}

// ============================================================================
// k_engine
// ============================================================================

#ifndef PM_CACHE
#define PM_CACHE 64
#endif
constexpr int kCache = PM_CACHE;  // CTA-local caches of free slots / free scratch units

// Splits a ticket's salvage and data phases need, loaded once (one round trip of
// independent loads) an iteration ahead: region q = region_of_ticket(t) has
// splits a0 = split(q), a1 = split(q+1); the windows of tickets t-1 and t have
// boundary splits (plo, phi) and (clo, chi).
struct TInfo {
  int64_t t, a0, a1, plo, phi, clo, chi;
};
__device__ __forceinline__ void load_tinfo(const Geo& g, int64_t t, TInfo& o) {
  const int64_t q = g.region_of_ticket(t);
  int64_t pl = 0, pr = -1, cl, cr;
  if (t > 0) g.window(t - 1, pl, pr);
  g.window(t, cl, cr);
  const int64_t a0 = g.split(q), a1 = g.split(q + 1);
  const int64_t plo = t > 0 ? g.split(pl) : 0, phi = t > 0 ? g.split(pr + 1) : 0;
  const int64_t clo = g.split(cl), chi = g.split(cr + 1);
  o.a0 = a0;
  o.a1 = a1;
  o.plo = plo;
  o.phi = phi;
  o.clo = clo;
  o.chi = chi;
  o.t = t;
}


// ---- sharded global free lists (one CAS word per shard) --------------------
// warp-cooperative pop: lanes read all shard tops at once, then lane 0 pops the
// nearest non-empty shard (home first), reusing the scanned top as the CAS
// expectation.  Returns -1 if every shard looked empty.
__device__ __forceinline__ int32_t warp_pop(unsigned long long* tops, int32_t* next, int home, int lane) {
  const unsigned long long a = *(volatile unsigned long long*)&tops[((home + lane) & (kShards - 1)) * kTopStride];
  const unsigned long long b = *(volatile unsigned long long*)&tops[((home + 32 + lane) & (kShards - 1)) * kTopStride];
  unsigned ma = __ballot_sync(0xffffffffu, (uint32_t)a != kEmpty32);
  unsigned mb = __ballot_sync(0xffffffffu, (uint32_t)b != kEmpty32);
  int32_t v = -1;
  while ((ma | mb) && v < 0) {
    int src_lane, sh;
    unsigned long long old;
    if (ma) {
      src_lane = __ffs(ma) - 1;
      ma &= ma - 1;
      old = __shfl_sync(0xffffffffu, a, src_lane);
      sh = (home + src_lane) & (kShards - 1);
    } else {
      src_lane = __ffs(mb) - 1;
      mb &= mb - 1;
      old = __shfl_sync(0xffffffffu, b, src_lane);
      sh = (home + 32 + src_lane) & (kShards - 1);
    }
    if (lane == 0) {
      while ((uint32_t)old != kEmpty32) {
        const uint32_t idx = (uint32_t)old;
        const int32_t nxt = *(volatile int32_t*)&next[idx];
        const unsigned long long nw = (((old >> 32) + 1ull) << 32) | (uint32_t)nxt;
        const unsigned long long seen = atomicCAS(&tops[sh * kTopStride], old, nw);
        if (seen == old) {
          fence_acq_rel_gpu();
          v = (int32_t)idx;
          break;
        }
        old = seen;
      }
    }
    v = __shfl_sync(0xffffffffu, v, 0);
  }
  return v;
}

// ---- CTA-local caches (shared memory, short spinlock) -----------------------
template <class Ctl>
__device__ __forceinline__ void cta_lock(Ctl& c) {
  while (atomicCAS(&c.lock, 0, 1) != 0) {
  }
  __threadfence_block();
}
template <class Ctl>
__device__ __forceinline__ void cta_unlock(Ctl& c) {
  __threadfence_block();
  atomicExch(&c.lock, 0);
}
// Make slot v FREE on the global lists: a cached slot may still record its last
// occupant `expect` (released without a round trip); it is handed over only if
// it still holds that occupant (its region may have closed it meanwhile).
__device__ __forceinline__ void release_slot_global(const EngineParams& P, int32_t v, int32_t expect, int home) {
  if (expect != ST_FREE && atomicCAS(&P.state[v], expect, ST_FREE) != expect) return;
  stack_push(&P.free_top[home * kTopStride], P.next_free, v);
}
// push a freed slot (v >= 0; state still `expect`) or scratch unit (v = -(i+1));
// overflow goes global
template <class Ctl>
__device__ __forceinline__ void cache_push(Ctl& c, const EngineParams& P, int32_t v, int home,
                                           int32_t expect = ST_FREE) {
  cta_lock(c);
  bool done = false;
  if (v >= 0 && c.n_fs < kCache) {
    c.fx[c.n_fs] = expect;
    c.fs[c.n_fs++] = v;
    done = true;
  } else if (v < 0 && c.n_sc < kCache) {
    c.sc[c.n_sc++] = -v - 1;
    done = true;
  }
  cta_unlock(c);
  if (!done) {
    if (v >= 0) release_slot_global(P, v, expect, home);
    else stack_push(&P.scr_top[home * kTopStride], P.next_scr, -v - 1);
  }
}
// give every cached unit back to the global lists (another CTA is starving)
template <class Ctl>
__device__ __forceinline__ void cache_flush(Ctl& c, const EngineParams& P, int home) {
  cta_lock(c);
  const int nf = c.n_fs, ns = c.n_sc;
  c.n_fs = 0;
  c.n_sc = 0;
  int32_t fs[kCache], fx[kCache], sc[kCache];
  for (int i = 0; i < nf; ++i) {
    fs[i] = c.fs[i];
    fx[i] = c.fx[i];
  }
  for (int i = 0; i < ns; ++i) sc[i] = c.sc[i];
  cta_unlock(c);
  for (int i = 0; i < nf; ++i) release_slot_global(P, fs[i], fx[i], home);
  for (int i = 0; i < ns; ++i) stack_push(&P.scr_top[home * kTopStride], P.next_scr, sc[i]);
}

// Warp-wide: a salvage destination for unit u, moved by ticket t.  Scratch first
// (a parked unit is never moved again), then free slots; CTA cache first, then
// the global lists.  A free slot qualifies only if its region's order exceeds t:
// units only ever move to higher order (or scratch), so while u sits in region
// r's slot, reads[u] counts exactly its consumers of order <= r -- the count
// the region's store waits on.  (A free slot of a lower-order region belongs to a
// ticket already in flight that is about to close it: it is dropped.)
// Blocking callers have published their own region's reads first, so a blocked
// caller never holds space other regions wait for; after a while they raise
// need_space so CTAs flush their caches.
template <class Ctl>
__device__ __forceinline__ int32_t acquire_dest(Ctl& c, const EngineParams& P, int32_t u, int64_t t, int home,
                                                int lane, bool block) {
  bool flagged = false;
  int32_t dest = INT32_MIN;
  const Geo g(P);
  auto usable = [&](int32_t f, int32_t x) {
    return g.order(g.region_of_slot(f)) > t && atomicCAS(&P.state[f], x, u) == x;
  };
  for (uint32_t it = 0;; ++it) {
    // scratch first (cache, then the global lists): a unit parked in scratch is
    // final, one parked in a free slot moves again when that slot's region starts
    int32_t d = INT32_MIN;
    if (lane == 0) {
      cta_lock(c);
      if (c.n_sc > 0) d = -c.sc[--c.n_sc] - 1;
      cta_unlock(c);
    }
    d = __shfl_sync(0xffffffffu, d, 0);
    if (d != INT32_MIN) {
      dest = d;
#if PM_STATS
      if (lane == 0) atomicAdd(&P.stats[16], 1ull);
#endif
      break;
    }
    const int32_t si = warp_pop(P.scr_top, P.next_scr, home, lane);
    if (si >= 0) {
      dest = -si - 1;
#if PM_STATS
      if (lane == 0) atomicAdd(&P.stats[18], 1ull);
#endif
      break;
    }
    if (lane == 0) {
      cta_lock(c);
      int32_t f = -1;
      while (c.n_fs > 0) {
        --c.n_fs;
        f = c.fs[c.n_fs];
        if (usable(f, c.fx[c.n_fs])) break;
        f = -1;  // its region started meanwhile (or precedes t)
      }
      cta_unlock(c);
      if (f >= 0) d = f;
    }
    d = __shfl_sync(0xffffffffu, d, 0);
    if (d != INT32_MIN) {
      dest = d;
#if PM_STATS
      if (lane == 0) atomicAdd(&P.stats[17], 1ull);
#endif
      break;
    }
    int32_t f;
    bool got = false;
    while ((f = warp_pop(P.free_top, P.next_free, home, lane)) >= 0) {
      int ok = 0;
      if (lane == 0) ok = usable(f, ST_FREE);
      if (__shfl_sync(0xffffffffu, ok, 0)) {
        got = true;
        break;
      }
    }
    if (got) {
      dest = f;
#if PM_STATS
      if (lane == 0) atomicAdd(&P.stats[19], 1ull);
#endif
      break;
    }
    if (!block || ((it & 15) == 15 && ld_relaxed(P.err))) break;
    if (!flagged && it > 32) {
      if (lane == 0) atomicAdd(P.need_space, 1);
      flagged = true;
    }
    if (it > kSpinLimit) {
      if (lane == 0) raise_error(P.err, PM_ERR_NOSPACE);
      break;
    }
    backoff(it);
  }
  if (flagged && lane == 0) atomicSub(P.need_space, 1);
  return dest;
}

// Close slot j (the region has started) and sample its occupant's reads / loc.
// The home unit's state is read together with the exchange (it is usually the
// occupant); the sample precedes any read this region publishes.
__device__ __forceinline__ void close_and_sample(const Geo& g, const EngineParams& P, int64_t j, bool identity,
                                                 int32_t& u, int32_t& r, int32_t& l) {
  const int32_t home_u = (int32_t)j;
  int32_t r_h = 0, l_h = -1;
  if (!identity) {
    r_h = ld_acquire(&P.reads[home_u]);
    l_h = ld_acquire(&P.loc[home_u]);
  }
  u = atomicExch(&P.state[j], ST_CLOSED);
  r = 0;
  l = -1;
  if (u == home_u) {
    r = r_h;
    l = l_h;
  } else if (u >= 0 && !identity) {
    r = ld_acquire(&P.reads[u]);
  }
}

// Move unit u out of slot `slot` into `dest` (warp-wide) and publish its new home.
template <typename KT>
__device__ __forceinline__ void move_unit(const Geo& g, const EngineParams& P, int32_t u, int64_t slot, int32_t dest,
                                          int lane, Prof& prof, bool publish = true) {
  const int64_t ks = sizeof(KT), w = P.w;
  const int64_t x0 = g.slot_lo(u), x1 = g.slot_hi(u), hb = g.slot_base(u);
  const int64_t sbase = g.slot_base(slot);
  const int64_t dbase = dest >= 0 ? g.slot_base(dest) : 0;
  char* kd = dest >= 0 ? P.keys + (dbase + (x0 - hb)) * ks : P.scr_keys + ((-(int64_t)dest - 1) * P.T + (x0 - hb)) * ks;
#if PM_PREFETCH_MOVE
  // pull the whole unit toward L2 at once: the warp's batched loads then mostly hit L2
  if (lane == 0) {
    prefetch_l2(P.keys + (sbase + (x0 - hb)) * ks, (x1 - x0) * ks);
    if (w) prefetch_l2(P.pay + (sbase + (x0 - hb)) * w, (x1 - x0) * w);
  }
#endif
  if (!(PM_ABLATE & 2))
    copy_g2g_warp(reinterpret_cast<uint8_t*>(kd), reinterpret_cast<const uint8_t*>(P.keys + (sbase + (x0 - hb)) * ks),
                  (x1 - x0) * ks, lane);
  if (w) {
    uint8_t* pd = dest >= 0 ? P.pay + (dbase + (x0 - hb)) * w : P.scr_pay + ((-(int64_t)dest - 1) * P.T + (x0 - hb)) * w;
    copy_g2g_warp(pd, P.pay + (sbase + (x0 - hb)) * w, (x1 - x0) * w, lane);
  }
  if (!publish) return;  // the caller fences and publishes later (publish_pending)
  fence_acq_rel_gpu();  // every lane's part is visible before the new home is published
  __syncwarp();
  if (lane == 0) st_release(&P.loc[u], dest);
}

// Decoupled persistent engine.  A CTA holds a ring of up to kRing tickets:
//   salvage workers (warps 0..kTeam-1) each take the next (ticket, slot) item in
//     ticket order and run its chain on their own: close the slot and sample its
//     occupant, wait for the occupant to land, then move it (scratch first, else
//     a free slot of a higher-order region) if a later region still needs it.
//     No space -> wait for the ticket's reads to be published, then block for
//     space (the region's own reads free space first).
//   data team (the other kDataWarps warps) takes the ring's tickets in order:
//     gathers the A/B pieces into shared memory (TMA bulk), publishes the reads,
//     merges in shared memory, issues the next ticket's gather, waits until every
//     slot item of the ticket is done and every consumer of order <= t has read
//     each occupant, and streams the output tile back in place (TMA bulk store).
// The teams meet only on shared-memory counters, so a worker's long chain
// (waits on other CTAs, round trips of the copy) overlaps the other workers'
// chains and the data team's work on earlier tickets.

constexpr int kMaxMu = 8;  // slots per region (pm_capi.cu enforces mu <= kMaxMu)
struct RingEntry {
  TInfo ti;             // ti.t = ticket (>= Q: the end)
  int32_t nslot;        // slot items of the ticket
  int32_t items_done;   // finished slot items
  int32_t published;    // the data team has published the ticket's reads
  int32_t pad_;
  int32_t occ[kMaxMu];    // occupant sampled by each slot item (-1: none)
  int32_t occ_r[kMaxMu];  // its reads[] as sampled by the item
};
struct EngCtl {
  uint64_t bar;
  RingEntry ring[kRing];
  int32_t filled;       // entries filled so far (monotone)
  int32_t d_done;       // entries the data team has finished (monotone)
  int32_t cur_e, cur_i; // next salvage item: entry, slot
  int32_t claim_lock;
  int32_t next_t;       // prefetched ticket
  int32_t lock;         // protects the caches below (cache_push / acquire_dest)
  int32_t n_fs, n_sc;
  int32_t abort;
  int32_t fs[kCache];
  int32_t fx[kCache];   // the occupant fs[i] still records (ST_FREE once released)
  int32_t sc[kCache];
  int32_t ntick;        // tickets with work (k_compact; kept last: the layout above is register-sensitive)
};

// The data team's view of one region: its input pieces and staging offsets.
struct DataRegion {
  int64_t t, d0, nout, alpha, beta, xa, xb, offA, offB, poffA, poffB, ua0, ub0;
  int32_t npa, np;
  bool identity;
  __device__ __forceinline__ void init(const Geo& g, const EngineParams& P, const TInfo& ti, int64_t la) {
    t = ti.t;
    if (t >= P.Q) return;
    const int64_t ks = P.ks, w = P.w;
    const int64_t q = g.region_of_ticket(t);
    d0 = g.diag(q);
    const int64_t d1 = g.diag(q + 1);
    const int64_t a0 = ti.a0, a1 = ti.a1, b0 = d0 - a0, b1 = d1 - a1;
    alpha = a1 - a0;
    beta = b1 - b0;
    nout = d1 - d0;
    identity = P.mode == MODE_MERGE && ((a0 == d0 && a1 == d1) || (a0 == la && a1 == la));
    xa = P.s + a0;
    xb = P.m + b0;
    offA = ((uintptr_t)(P.keys + xa * ks)) & 15;
    offB = ((offA + (alpha + kSent) * ks + 15) & ~(int64_t)15) + (((uintptr_t)(P.keys + xb * ks)) & 15);
    poffA = poffB = 0;
    if (w) {
      poffA = ((uintptr_t)(P.pay + xa * w)) & 15;
      poffB = ((poffA + alpha * w + 15) & ~(int64_t)15) + (((uintptr_t)(P.pay + xb * w)) & 15);
    }
    ua0 = alpha ? ((xa >> P.lT) - P.k0) : 0;
    const int64_t ua1 = alpha ? (((xa + alpha - 1) >> P.lT) - P.k0 + 1) : 0;
    ub0 = beta ? ((xb >> P.lT) - P.k0) : 0;
    const int64_t ub1 = beta ? (((xb + beta - 1) >> P.lT) - P.k0 + 1) : 0;
    npa = (int32_t)(ua1 - ua0);
    np = npa + (int32_t)(ub1 - ub0);
  }
};

// Tickets with work are tlist[k] for k = 0, 1, ... (identity regions -- inputs
// already on their outputs -- never get one); Q marks the end.
__device__ __forceinline__ int32_t resolve_ticket(const EngineParams& P, int32_t k, int32_t ntick) {
  if (ntick == P.Q) return k < ntick ? k : (int32_t)P.Q;  // nothing left out: the identity map
  return k < ntick ? __ldg(&P.tlist[k]) : (int32_t)P.Q;
}

// Fill ring entry e with the prefetched ticket (caller holds the claim lock and
// has checked that the entry is free: e - d_done < kRing).
__device__ __forceinline__ void open_entry(EngCtl& c, const Geo& g, const EngineParams& P, int32_t e) {
  volatile EngCtl& vc = c;
  RingEntry& re = c.ring[e % kRing];
  const int64_t t = vc.next_t;
  if (t < P.Q) {
    // the next ticket's fetch and this ticket's split loads share one round trip
    const int32_t k_next = atomicAdd(P.ticket, 1);
    load_tinfo(g, t, re.ti);
    const int64_t q = g.region_of_ticket(t);
    re.nslot = (int32_t)(g.region_end_slot(q) - g.region_first_slot(q));
    vc.next_t = resolve_ticket(P, k_next, vc.ntick);  // (a load only if tickets were left out)

  } else {
    re.ti.t = P.Q;
    re.nslot = 0;
  }
  re.items_done = 0;
  re.published = 0;
  __threadfence_block();
  vc.filled = e + 1;
}
__device__ __forceinline__ void claim_lock(EngCtl& c) {
  while (atomicCAS(&c.claim_lock, 0, 1) != 0) {
  }
  __threadfence_block();
}
__device__ __forceinline__ void claim_unlock(EngCtl& c) {
  __threadfence_block();
  atomicExch(&c.claim_lock, 0);
}

template <typename KT>
__global__ void __launch_bounds__(kEngineThreads, kEngineMinBlocks) k_engine(EngineParams P) {
  if (P.gate && !*(volatile const int32_t*)P.gate) return;
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ EngCtl ctl;
  Geo g(P);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NT = kEngineThreads;  // (launched with exactly this many)
  const int64_t ks = sizeof(KT);
  const int64_t w = P.w;
  if (*(volatile int32_t*)P.noop) return;

  uint8_t* kin = dyn;                                 // staged keys (A then B, phase-shifted)
  uint8_t* pin = dyn + P.smem_keys;                   // staged payload
  uint8_t* kout_s = dyn + P.smem_keys + P.smem_pay;   // merged output tile (keys), phase-aligned
  uint8_t* pout_s = kout_s + P.smem_keys;             // merged output tile (payload)
  constexpr int kTeam = kEngineTeam;                  // warps per team
  const int home = blockIdx.x & (kShards - 1);
  const int64_t la = g.LA();
  Prof prof;
  uint32_t n_salv = 0, r_salv = 0, n_reg = 0, n_ident = 0;
  if (tid == 0) {
    mbar_init(&ctl.bar, 1);
    ctl.lock = 0;
    ctl.claim_lock = 0;
    ctl.n_fs = 0;
    ctl.n_sc = 0;
    ctl.abort = 0;
    ctl.filled = 0;
    ctl.d_done = 0;
    ctl.cur_e = 0;
    ctl.cur_i = 0;
    ctl.ntick = PM_TLIST ? *P.ntick : (int32_t)P.Q;
    ctl.next_t = resolve_ticket(P, atomicAdd(P.ticket, 1), ctl.ntick);
    // this CTA's share of the scratch pool starts in its cache (k_plan)
    ctl.n_sc = (int32_t)P.s_per;
    for (int32_t k = 0; k < (int32_t)P.s_per; ++k) ctl.sc[k] = (int32_t)(blockIdx.x * P.s_per + k);
  }
  __syncthreads();
  volatile EngCtl& vc = ctl;

  if (wid < kTeam) {
    // ===================== salvage workers ====================================
    long long cw = prof.now();
    for (uint32_t spin = 0;;) {
      // ---- claim the next item (lane 0, under the claim lock) ----
      int32_t e = -1, i = 0;
      int status = 0;  // 0 = got an item, 1 = retry (ring full), 2 = finished
      if (lane == 0) {
        claim_lock(ctl);
        e = vc.cur_e;
        if (vc.abort) {
          status = 2;
        } else if (e == vc.filled) {
          if (e - vc.d_done >= kRing) status = 1;  // ring full: the data team is behind
          else open_entry(ctl, g, P, e);
        }
        if (status == 0) {
          const RingEntry& re = ctl.ring[e % kRing];
          if (re.ti.t >= P.Q) {
            status = 2;
          } else {
            i = vc.cur_i;
            if (i + 1 >= re.nslot) {
              vc.cur_e = e + 1;
              vc.cur_i = 0;
            } else {
              vc.cur_i = i + 1;
            }
          }
        }
        claim_unlock(ctl);
      }
      status = __shfl_sync(0xffffffffu, status, 0);
      if (status == 2) break;
      if (status == 1) {
        if (lane == 0 && (++spin & 63) == 0 && *(volatile int32_t*)P.need_space) cache_flush(ctl, P, home);
        __nanosleep(64);
        continue;
      }
      e = __shfl_sync(0xffffffffu, e, 0);
      i = __shfl_sync(0xffffffffu, i, 0);
      const long long c0 = prof.now();
      prof.add(PS_STEP1, c0 - cw);  // claiming, incl. waiting for ring space
      // ---- run the item: slot j0 + i of ticket t ----
      RingEntry& re = ctl.ring[e % kRing];
      const int64_t t = re.ti.t;
      const int64_t q = g.region_of_ticket(t);
      const int64_t j0 = g.region_first_slot(q);
      const int32_t slot = (int32_t)(j0 + i);
      const int64_t d0 = g.diag(q), d1 = g.diag(q + 1);
      const int64_t a0 = re.ti.a0, a1 = re.ti.a1;
      const bool identity = P.mode == MODE_MERGE && ((a0 == d0 && a1 == d1) || (a0 == la && a1 == la));
      int32_t u = -1, early_r = 0, early_l = -1;
      if (lane == 0) {
        close_and_sample(g, P, slot, identity, u, early_r, early_l);
        re.occ[i] = identity ? -1 : u;
        re.occ_r[i] = early_r;
      }
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u >= 0 && !identity) {
        int alive = 0;
        if (lane == 0) {
          for (uint32_t it = 0; early_l != slot && ld_acquire(&P.loc[u]) != slot; ++it) {  // landing
            if ((it & 255) == 255 && ld_relaxed(P.err)) {
              ctl.abort = 1;
              break;
            }
            if (it > kSpinLimit) {
              raise_error(P.err, PM_ERR_TIMEOUT);
              ctl.abort = 1;
              break;
            }
            backoff(it);
          }
          prof.add(PS_SLAND, prof.now() - c0);
          // move u now if a region after t still needs it: earlier consumers that
          // have not read it yet read either copy -- t's store waits for them
          int64_t cwl, cwr;
          g.window(t, cwl, cwr);
          alive = g.consumed_in(u, cwl, cwr, re.ti.clo, re.ti.chi) < g.slot_hi(u) - g.slot_lo(u) && !vc.abort;
#if PM_PREFETCH_ITEM
          if (alive) {  // the copy comes after the destination search: warm L2 now
            const int64_t ux0 = g.slot_lo(u), src = g.slot_base(slot) + (ux0 - g.slot_base(u));
            prefetch_l2(P.keys + src * (int64_t)sizeof(KT), (g.slot_hi(u) - ux0) * (int64_t)sizeof(KT));
            if (w) prefetch_l2(P.pay + src * w, (g.slot_hi(u) - ux0) * w);
          }
#endif
        }
        alive = __shfl_sync(0xffffffffu, alive, 0);
        const long long c2 = prof.now();
        prof.add(PS_THR, c2 - c0);
        if (alive) {
          int32_t dest = acquire_dest(ctl, P, u, t, home, lane, false);
          if (dest == INT32_MIN) {
            // no space: the region's own reads free space first, then block
            const long long cb = prof.now();
            if (lane == 0)
              while (!vc.ring[e % kRing].published && !vc.abort) __nanosleep(128);
            __syncwarp();
            if (!vc.abort) dest = acquire_dest(ctl, P, u, t, home, lane, true);
            if (lane == 0) {
              prof.hist(P.stats, 20, 0, 1, 1);
              prof.hist(P.stats, 21, 0, 1, prof.now() - cb);
            }
          }
          prof.add(PS_DEST, prof.now() - c2);
          if (dest == INT32_MIN) {
            if (lane == 0) ctl.abort = 1;
          } else {
            const long long c3 = prof.now();
            move_unit<KT>(g, P, u, slot, dest, lane, prof);
            prof.add(PS_COPY, prof.now() - c3);
            if (lane == 0) {
              ++n_salv;
              r_salv += (uint32_t)(g.slot_hi(u) - g.slot_lo(u));
            }
          }
        }
      }
#if PM_ITEM_RESAMPLE
      // refresh the occupant's reads sample for the store-time check
      if (lane == 0 && u >= 0 && !identity) {
        int64_t cwl, cwr;
        g.window(t, cwl, cwr);
        if (early_r < g.consumed_in(u, cwl, cwr, re.ti.clo, re.ti.chi)) re.occ_r[i] = ld_acquire(&P.reads[u]);
      }
#endif
      __syncwarp();
      if (lane == 0) atomicAdd(&re.items_done, 1);
      cw = prof.now();
      prof.add(PS_STEP2, cw - c0);
    }
  } else {
    // ===================== data team ==========================================
    // Per entry: land the gathered pieces, publish the reads, merge into the output
    // tile, issue the NEXT entry's gather into the freed input tile, then wait for
    // the slot items and earlier consumers and stream the tile back.
    const int gt = tid - kTeam * 32, GT = NT - kTeam * 32;
    uint32_t phase = 0;
    long long td = prof.now();
#define PM_TICK(k)                      \
  if (gt == 0) {                        \
    const long long n_ = prof.now();    \
    prof.add(PS_GATHER + (k), n_ - td); \
    td = n_;                            \
  }
    // open entry e (if the workers have not) and describe its region
    auto open_and_describe = [&](int32_t e, DataRegion& R) {
      if (gt == 0 && vc.filled <= e && !vc.abort) {
        claim_lock(ctl);
        if (vc.filled <= e) open_entry(ctl, g, P, e);
        claim_unlock(ctl);
      }
      named_barrier_sync(1, GT);
      R.init(g, P, ctl.ring[e % kRing].ti, la);
    };
    // open entries up to e ahead of need (thread gt == 0, while the team waits anyway)
    auto open_ahead = [&](int32_t e) {
      if (gt == 0 && vc.filled <= e && e - vc.d_done < kRing && !vc.abort) {
        claim_lock(ctl);
        while (vc.filled <= e && vc.filled - vc.d_done < kRing) {
          const int32_t f = vc.filled;
          if (f > 0 && ctl.ring[(f - 1) % kRing].ti.t >= P.Q) break;  // the end is open already
          open_entry(ctl, g, P, f);
        }
        claim_unlock(ctl);
      }
    };
    // wait until every piece sits where nobody moves it before it is read, then
    // issue its TMA bulk load (thread per piece) and arm the barrier
    // returns the location this thread read its first piece from (INT32_MIN: none):
    // if this region turns out to be the unit's last reader, the unit is still
    // there (nobody moves a unit without a later consumer), so it is released
    // without another round trip
    // pl: this thread's piece location loaded (relaxed) one merge earlier, or
    // INT32_MIN.  A location of order >= t (or scratch) seen then is still safe to
    // read: the unit only moves up, and its old slot is not overwritten before
    // this region's read is counted.
    auto gather_issue = [&](const DataRegion& R, int32_t pl) -> int32_t {
      int32_t mine = INT32_MIN;
      for (int p = gt; p < R.np; p += GT) {
        const bool isA = p < R.npa;
        const int64_t j = isA ? R.ua0 + p : R.ub0 + (p - R.npa);
        const int64_t run0 = isA ? R.xa : R.xb, run1 = isA ? R.xa + R.alpha : R.xb + R.beta;
        const int64_t x0 = max(run0, g.slot_lo(j)), x1 = min(run1, g.slot_hi(j));
        int32_t l = p == gt ? pl : INT32_MIN;
        for (uint32_t it = 0;; ++it) {
          if (l != INT32_MIN && (l < 0 || g.order(g.region_of_slot(l)) >= R.t)) {
            // the prefetch was relaxed: acquire a moved unit's data (a unit still
            // in its home slot holds the caller's original records)
            if (l != (int32_t)j) fence_acq_rel_gpu();
            break;
          }
          l = ld_acquire(&P.loc[j]);
          if (l < 0 || g.order(g.region_of_slot(l)) >= R.t) break;
          if ((it & 255) == 255 && ld_relaxed(P.err)) {
            ctl.abort = 1;
            break;
          }
          if (it > kSpinLimit) {
            raise_error(P.err, PM_ERR_TIMEOUT);
            ctl.abort = 1;
            break;
          }
          if ((it & 63) == 63 && *(volatile int32_t*)P.need_space) cache_flush(ctl, P, home);
          backoff(it);
        }
        const int64_t hb = g.slot_base(j);
        const char* ksrc;
        const uint8_t* psrc;
        if (l >= 0) {
          const int64_t base = g.slot_base(l);
          ksrc = P.keys + (base + (x0 - hb)) * ks;
          psrc = P.pay + (base + (x0 - hb)) * w;
        } else {
          const int64_t si = -(int64_t)l - 1;
          ksrc = P.scr_keys + (si * P.T + (x0 - hb)) * ks;
          psrc = P.scr_pay + (si * P.T + (x0 - hb)) * w;
        }
        uint8_t* kdst = kin + (isA ? R.offA + (x0 - R.xa) * ks : R.offB + (x0 - R.xb) * ks);
        // (unit boundaries are 16-byte aligned only when both bases are)
        const bool exact = (((uintptr_t)P.keys) & 15) || (w && (((uintptr_t)P.pay) & 15));
        if (!(PM_ABLATE & 4))
          copy_g2s_piece(kdst, reinterpret_cast<const uint8_t*>(ksrc), (x1 - x0) * ks, &ctl.bar, exact);
        if (w) {
          uint8_t* pdst = pin + (isA ? R.poffA + (x0 - R.xa) * w : R.poffB + (x0 - R.xb) * w);
          copy_g2s_piece(pdst, psrc, (x1 - x0) * w, &ctl.bar, exact);
        }
        if (p == gt) mine = l;
      }
      named_barrier_sync(1, GT);  // every expect_tx registered before the single arrive
      if (gt == 0) mbar_arrive(&ctl.bar);
      return mine;
    };

    DataRegion R;
    int32_t e = 0;
    open_and_describe(0, R);
    bool pending = false;  // a gather is in flight on ctl.bar
    int32_t gl = INT32_MIN;  // where this thread read its piece of the current region
    if (R.t < P.Q && !R.identity && !vc.abort) {
      gl = gather_issue(R, INT32_MIN);
      pending = true;
    }
    while (true) {
      RingEntry& re = ctl.ring[e % kRing];
      if (R.t >= P.Q || vc.abort) break;
      td = prof.now();
      DataRegion Rn;
      if (R.identity) {
        if (gt == 0) {
          ++n_ident;
          atomicExch(&re.published, 1);
          // the slot items still close the region's slots; wait for them so the
          // ring entry is not reused under a worker
          while (vc.ring[e % kRing].items_done < re.nslot && !vc.abort) {
          }
          __threadfence_block();
          vc.d_done = e + 1;
        }
        open_and_describe(e + 1, Rn);
        gl = INT32_MIN;
        if (Rn.t < P.Q && !Rn.identity && !vc.abort) {
          gl = gather_issue(Rn, INT32_MIN);
          pending = true;
        }
        R = Rn;
        ++e;
        continue;
      }
      // ---- land entry e ----
      while (!mbar_try_wait(&ctl.bar, phase)) {
      }
      phase ^= 1;
      pending = false;
      PM_TICK(1);
      // prefetch (relaxed) the locations of the next entry's pieces for its gather
      int32_t pl = INT32_MIN;
      if (vc.filled > e + 1) {
        __threadfence_block();
        const TInfo& tn = ctl.ring[(e + 1) % kRing].ti;
        if (tn.t < P.Q) {
          DataRegion Rp;
          Rp.init(g, P, tn, la);
          if (!Rp.identity && gt < Rp.np) pl = ld_relaxed(&P.loc[gt < Rp.npa ? Rp.ua0 + gt : Rp.ub0 + (gt - Rp.npa)]);
        }
      }
      // publish the reads (one piece per thread; np <= GT): the atomics stay in
      // flight during the merge, deaths are handled after it
      int64_t pj = -1;
      int32_t pn = 0, pold = 0;
      if (gt < R.np) {
        const bool isA = gt < R.npa;
        pj = isA ? R.ua0 + gt : R.ub0 + (gt - R.npa);
        const int64_t run0 = isA ? R.xa : R.xb, run1 = isA ? R.xa + R.alpha : R.xb + R.beta;
        pn = (int32_t)(min(run1, g.slot_hi(pj)) - max(run0, g.slot_lo(pj)));
        // (no fence: the bulk loads have completed -- the mbarrier said so -- so a
        // writer that sees this count cannot change what this region read)
        pold = atomicAdd(&P.reads[pj], pn);
      }
      if (P.mode == MODE_MERGE && !w) write_sentinels<KT>(kin, R.offA, R.alpha, R.offB, R.beta, gt, GT);
      if (gt == 0) bulk_wait_read_all();  // the previous tile's TMA store has read the output tile
      named_barrier_sync(1, GT);
      if (gt == 0) atomicExch(&re.published, 1);
      PM_TICK(2);
      // merge path (A wins ties): every thread merges an odd-length run of outputs
      // (odd stride -> conflict-free smem) straight into the phase-aligned output tile
      const KT* As = reinterpret_cast<const KT*>(kin + R.offA);
      const KT* Bs = reinterpret_cast<const KT*>(kin + R.offB);
      const int64_t phk = ((uintptr_t)(P.keys + (P.s + R.d0) * ks)) & 15;
      KT* ko = reinterpret_cast<KT*>(kout_s + phk);
      const int64_t php = w ? (((uintptr_t)(P.pay + (P.s + R.d0) * w)) & 15) : 0;
      uint8_t* po = pout_s + php;
      const uint8_t* PA = pin + R.poffA;
      const uint8_t* PB = pin + R.poffB;
      const bool wq4 = w && (w & 3) == 0 && ((php | R.poffA | R.poffB) & 3) == 0;
      if (!(PM_ABLATE & 1))
        merge_tile<KT, kEngineThreads - kTeam * 32>(P.mode, As, Bs, R.alpha, R.beta, R.nout, ko, po, PA, PB, w, wq4, gt);
      fence_proxy_async_smem();  // our smem writes -> visible to the TMA (async proxy)
      PM_TICK(3);
      // ---- the input tile is free: start the next entry's gather now ----
      open_and_describe(e + 1, Rn);  // (its barrier also ends every thread's merge)
      PM_TICK(1);
      int32_t gl_next = INT32_MIN;
      if (Rn.t < P.Q && !Rn.identity && !vc.abort) {
        gl_next = gather_issue(Rn, pl);
        pending = true;
      }
      PM_TICK(0);
      const long long q0 = prof.now();
      if (pj >= 0 && pold + pn == (int32_t)(g.slot_hi(pj) - g.slot_lo(pj))) {
        // last reader: release the unit's location into the CTA cache (a slot keeps
        // recording pj until a salvage worker claims it: no round trip here)
        const int32_t l = gl;
        if (l < 0) {
          cache_push(ctl, P, l, home);
        } else if (g.slot_full(l)) {
          cache_push(ctl, P, l, home, (int32_t)pj);
        }
      }
      const long long q1 = prof.now();
      open_ahead(e + 2);
      const long long q2 = prof.now();
      // ---- every slot of the region must be cleared before the tile lands there:
      //      all slot items are done, and every consumer of order <= t has read
      //      each occupant (t's own reads are published by now) ----
      if (gt == 0)
        while (vc.ring[e % kRing].items_done < re.nslot && !vc.abort) {
        }
      named_barrier_sync(1, GT);
      const long long q3 = prof.now();
      if (gt < re.nslot) {
        const int32_t u = re.occ[gt];
        if (u >= 0) {
          int64_t cwl, cwr;
          g.window(R.t, cwl, cwr);
          const int64_t before = g.consumed_in(u, cwl, cwr, re.ti.clo, re.ti.chi);
          // (reads[] only counts consumers of order <= t while u sits in t's slot, so
          // the item's sample settles it without a round trip when it suffices)
          for (uint32_t it = 0; re.occ_r[gt] < before && ld_acquire(&P.reads[u]) < before; ++it) {
            if ((it & 255) == 255 && ld_relaxed(P.err)) {
              ctl.abort = 1;
              break;
            }
            if (it > kSpinLimit) {
              raise_error(P.err, PM_ERR_TIMEOUT);
              ctl.abort = 1;
              break;
            }
            backoff(it);
          }
        }
      }
      named_barrier_sync(1, GT);
#if PM_STATS
      if (gt == 0) {  // stats[24..27]: free, open-ahead, items wait, consumer wait
        const long long q4 = prof.now();
        atomicAdd(&P.stats[24], (unsigned long long)(q1 - q0));
        atomicAdd(&P.stats[25], (unsigned long long)(q2 - q1));
        atomicAdd(&P.stats[26], (unsigned long long)(q3 - q2));
        atomicAdd(&P.stats[27], (unsigned long long)(q4 - q3));
      }
#endif
      PM_TICK(4);
      if (!vc.abort) {
        // stream the tile back in place: TMA bulk store for the 16-byte-aligned body,
        // generic stores for the unaligned head and tail bytes
        if (!(PM_ABLATE & 8))
          stream_out(kout_s + phk, reinterpret_cast<uint8_t*>(P.keys + (P.s + R.d0) * ks), R.nout * ks, gt, GT);
        if (w) stream_out(pout_s + php, P.pay + (P.s + R.d0) * w, R.nout * w, gt, GT);
      }
      if (gt == 0) {
        ++n_reg;
        __threadfence_block();
        vc.d_done = e + 1;  // the ring entry may be reused
      }
      PM_TICK(5);
      R = Rn;
      gl = gl_next;
      ++e;
    }
    if (gt == 0) {
      // an aborted job may leave a gather in flight: let it land before the CTA exits
      if (pending)
        for (uint32_t it = 0; !mbar_try_wait(&ctl.bar, phase) && it < (1u << 20); ++it) {
        }
      bulk_wait_all();  // the last output tile has landed
    }
#undef PM_TICK
  }
  __syncthreads();
  // leave nothing behind in the CTA cache (another job reuses the lists)
  if (tid == 0) cache_flush(ctl, P, home);
  if (lane == 0 && n_salv) {
    atomicAdd(&P.stats[0], (unsigned long long)n_salv);
    atomicAdd(&P.stats[1], (unsigned long long)r_salv);
  }
  if (tid == kTeam * 32) {
    atomicAdd(&P.stats[2], (unsigned long long)n_reg);
    atomicAdd(&P.stats[3], (unsigned long long)n_ident);
  }
  if (lane == 0) prof.flush(P.stats);
}


// ============================================================================
// Buffered mode: the reference's min-side-buffered core (seq_merge_buffered,
// seqmerge.py:55-75 / _kernels.py:227-313) as a streaming GPU pipeline.  The
// shorter run is copied to the caller-sized buffer; regions are then merged in
// the direction that only ever overwrites already-consumed records of the
// other run (ascending when A is buffered, descending when B is), each region
// waiting only for the few earlier regions that read the records it overwrites.
// 1.5 passes over the data for equal runs, no unit bookkeeping.
// ============================================================================
// For every region r of the buffered pipeline: the regions that read the
// unbuffered-run records r overwrites (c_lo..c_hi, stored in state[] / loc[],
// which the buffered mode does not otherwise use).  One thread per region.
__global__ void __launch_bounds__(256) k_consumers(EngineParams P, int32_t buf_a) {
  Geo g(P);
  const int64_t la = g.LA();
  auto last_le = [&](int64_t v, int64_t lo, int64_t hi, bool on_b) {  // largest c in [lo,hi], run_c <= v
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      const int64_t rc = on_b ? g.diag(mid) - g.split(mid) : g.split(mid);
      if (rc <= v) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < P.Q; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d0 = g.diag(r), d1 = g.diag(r + 1);
    int64_t c_lo = 0, c_hi = -1;
    if (buf_a) {  // r writes into B's area [m, e): B indices [jlo, jhi); consumers are <= r
      const int64_t jlo = max(P.s + d0, P.m) - P.m, jhi = P.s + d1 - P.m;
      if (jhi > jlo) {
        c_lo = last_le(jlo, 0, r, true);
        c_hi = last_le(jhi - 1, c_lo, r, true);
      }
    } else {  // r writes into A's area [s, m): A indices [ilo, ihi); consumers are >= r
      const int64_t ilo = d0, ihi = min(d1, la);
      if (ihi > ilo) {
        c_lo = last_le(ilo, r, P.Q - 1, false);
        c_hi = last_le(ihi - 1, c_lo, P.Q - 1, false);
      }
    }
    P.state[r] = (int32_t)c_lo;
    P.loc[r] = (int32_t)c_hi;
  }
}

template <typename KT>
__global__ void __launch_bounds__(256) k_copy_run(EngineParams P, int64_t x0, int64_t x1) {
  const int64_t ks = sizeof(KT);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  for (int part = 0; part < (P.w ? 2 : 1); ++part) {
    const int64_t rb = part ? P.w : ks;
    const uint8_t* src = part ? P.pay + x0 * rb : reinterpret_cast<const uint8_t*>(P.keys) + x0 * rb;
    uint8_t* dst = part ? P.scr_pay : reinterpret_cast<uint8_t*>(P.scr_keys);  // same 16-byte phase as src
    const int64_t n = (x1 - x0) * rb;
    int64_t head = (16 - ((uintptr_t)src & 15)) & 15;
    if (head > n) head = n;
    const int64_t nv = (n - head) >> 4;
    for (int64_t b = tid; b < head; b += nthr) dst[b] = src[b];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    for (int64_t i = tid; i < nv; i += nthr) d4[i] = PM_COPY_LD(s4 + i);
    for (int64_t b = head + (nv << 4) + tid; b < n; b += nthr) dst[b] = src[b];
  }
}

// Per-region geometry of the buffered pipeline (staged tile layout in smem).
struct BufRegion {
  int64_t r, d0, d1, a0, a1, b0, b1, alpha, beta, nout;
  int64_t offA, offB, poffA, poffB;
  bool identity;
};
// What the merging warps need of a staged region: the leader derives it once
// when it issues the region's loads and leaves it in shared memory (the
// region-local quantities fit in 32 bits: nout <= M).
struct BufDesc {
  int64_t d0, r;
  int32_t alpha, beta, nout, offA, offB, poffA, poffB, identity;
  __device__ void set(const BufRegion& R) {
    d0 = R.d0;
    r = R.r;
    alpha = (int32_t)R.alpha;
    beta = (int32_t)R.beta;
    nout = (int32_t)R.nout;
    offA = (int32_t)R.offA;
    offB = (int32_t)R.offB;
    poffA = (int32_t)R.poffA;
    poffB = (int32_t)R.poffB;
    identity = R.identity;
  }
};

// region of ticket t; its boundary splits a0/a1 are passed in when already at hand
// (a0 < 0: load them)
template <typename KT>
__device__ __forceinline__ BufRegion buf_region(const Geo& g, const EngineParams& P, int64_t t, int32_t buf_a,
                                                int64_t a0 = -1, int64_t a1 = -1) {
  BufRegion R;
  const int64_t ks = sizeof(KT), w = P.w, la = g.LA();
  R.r = buf_a ? t : P.Q - 1 - t;
  R.d0 = g.diag(R.r);
  R.d1 = g.diag(R.r + 1);
  R.a0 = a0 >= 0 ? a0 : g.split(R.r);
  R.a1 = a0 >= 0 ? a1 : g.split(R.r + 1);
  R.b0 = R.d0 - R.a0;
  R.b1 = R.d1 - R.a1;
  R.alpha = R.a1 - R.a0;
  R.beta = R.b1 - R.b0;
  R.nout = R.d1 - R.d0;
  R.identity = !P.out_keys && ((R.a0 == R.d0 && R.a1 == R.d1) || (R.a0 == la && R.a1 == la));
  const int64_t xa = P.s + R.a0, xb = P.m + R.b0;
  const char* kbsrc = P.keys_b ? P.keys_b + R.b0 * ks : P.keys + xb * ks;
  R.offA = ((uintptr_t)(P.keys + xa * ks)) & 15;
  R.offB = ((R.offA + (R.alpha + kSent) * ks + 15) & ~(int64_t)15) + (((uintptr_t)kbsrc) & 15);
  R.poffA = R.poffB = 0;
  if (w) {
    const uint8_t* pbsrc = P.pay_b ? P.pay_b + R.b0 * w : P.pay + xb * w;
    R.poffA = ((uintptr_t)(P.pay + xa * w)) & 15;
    R.poffB = ((R.poffA + R.alpha * w + 15) & ~(int64_t)15) + (((uintptr_t)pbsrc) & 15);
  }
  return R;
}

// thread 0: TMA-load region R's runs into staging buffer (kin, pin); the
// buffered run comes from the phase-matched scratch copy
template <typename KT>
__device__ __forceinline__ void buf_issue(const EngineParams& P, const BufRegion& R, int32_t buf_a, uint8_t* kin,
                                          uint8_t* pin, uint64_t* bar) {
  const int64_t ks = sizeof(KT), w = P.w;
  const int64_t xa = P.s + R.a0, xb = P.m + R.b0;
  // (copy mode: both runs come from the source array)
  const bool oop = P.out_keys != nullptr;
  const char* ka = buf_a && !oop ? P.scr_keys + R.a0 * ks : P.keys + xa * ks;
  const char* kb = P.keys_b ? P.keys_b + R.b0 * ks : buf_a || oop ? P.keys + xb * ks : P.scr_keys + R.b0 * ks;
  copy_g2s_superset(kin + R.offA, reinterpret_cast<const uint8_t*>(ka), R.alpha * ks, bar);
  copy_g2s_superset(kin + R.offB, reinterpret_cast<const uint8_t*>(kb), R.beta * ks, bar);
  if (w) {
    const uint8_t* pa = buf_a && !oop ? P.scr_pay + R.a0 * w : P.pay + xa * w;
    const uint8_t* pb = P.pay_b ? P.pay_b + R.b0 * w : buf_a || oop ? P.pay + xb * w : P.scr_pay + R.b0 * w;
    copy_g2s_superset(pin + R.poffA, pa, R.alpha * w, bar);
    copy_g2s_superset(pin + R.poffB, pb, R.beta * w, bar);
  }
  mbar_arrive(bar);
}

// Persistent, software-pipelined: while the CTA merges one region out of its
// staging buffer, the TMA loads of the next kBufStages-1 regions are already in
// flight in the other staging buffers; the merged tile leaves through a TMA bulk
// store from one of two output buffers.  The last warp is the control warp
// (tickets, TMA issue, read flags, consumer checks, bulk stores); the other warps
// only merge, so no round trip sits on the merge's critical path.
template <typename KT>
__global__ void __launch_bounds__(kBufferedThreads) k_buffered(EngineParams P, int32_t buf_a) {
  if (P.gate && !*(volatile const int32_t*)P.gate) return;  // (staged path: the runs are already in order)
  constexpr int NS = kBufStages;
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ uint64_t bar[NS];
  __shared__ int64_t s_t[NS];
  __shared__ BufDesc s_d[NS];      // the staged region's geometry (set by the leader)
  __shared__ int32_t s_early[NS];  // the region's read flag was already raised
  Geo g(P);
  constexpr int NT = kBufferedThreads;  // (launched with exactly this many)
  const int tid = threadIdx.x, lane = tid & 31;
  const int NW = NT >> 5;
  const bool ctrl = (tid >> 5) == NW - 1;
  const bool leader = ctrl && lane == 0;  // issues every TMA op of the CTA
  const int MT = NT - 32;                 // merge threads
  const int64_t ks = sizeof(KT), w = P.w;
  if (*(volatile int32_t*)P.noop) return;
  int32_t t_pref = 0;
  const size_t tile = P.smem_keys + P.smem_pay;
  // tiles are addressed as dyn + offset so the compiler keeps them in the shared
  // space (a local pointer array would turn every access into a generic LD/ST)
#define STAGE(b) (dyn + (size_t)(b) * tile)
#define OUTB(b) (dyn + (size_t)(NS + (b)) * tile)
  int32_t* flags = P.reads;  // flags[r] = 1 once region r has read its inputs
  const bool oop = P.out_keys != nullptr;  // copy mode: no overlap, no flags
  char* const okeys = oop ? P.out_keys : P.keys;
  uint8_t* const opay = oop ? P.out_pay : P.pay;
  if (leader) {
    // fill the pipeline: tickets of the first NS-1 iterations, their loads in flight
    for (int k = 0; k < NS; ++k) {
      mbar_init(&bar[k], 1);
      s_early[k] = 0;
      s_t[k] = P.Q;
    }
    for (int k = 0; k < NS - 1; ++k) {
      const int64_t t0 = (*(volatile int32_t*)P.err) ? P.Q : atomicAdd(P.ticket, 1);
      s_t[k] = t0 < P.Q ? t0 : P.Q;
      if (t0 < P.Q) {
        const BufRegion R = buf_region<KT>(g, P, t0, buf_a);
        s_d[k].set(R);
        if (!R.identity) buf_issue<KT>(P, R, buf_a, STAGE(k), STAGE(k) + P.smem_keys, &bar[k]);
      } else {
        break;
      }
    }
    t_pref = atomicAdd(P.ticket, 1);  // the ticket after those, in flight
  }
  __syncthreads();
  uint32_t phmask = 0;  // bit k: parity of stage k's barrier
  // control warp: consumer range of the region one iteration ahead (in-place mode)
  int64_t cn_lo = 1, cn_hi = 0;
  if (ctrl && !oop && s_t[0] < P.Q && !s_d[0].identity) {
    cn_lo = __ldg(&P.state[s_d[0].r]);
    cn_hi = __ldg(&P.loc[s_d[0].r]);
  }
  unsigned long long n_reg = 0;
  Prof prof;
  long long tb = prof.now();
#define PB_TICK(k)                       \
  if (tid == 0) {                        \
    const long long n_ = prof.now();     \
    prof.add(PS_GATHER + (k), n_ - tb);  \
    tb = n_;                             \
  }
  for (int it = 0;; ++it) {
    const int cur = it % NS, ob = it & 1;
    const int64_t t = s_t[cur];
    if (t >= P.Q) break;
    const BufDesc R = s_d[cur];
    if (leader) {  // (writes only the previous iteration's stage slot: no race with R above)
      // keep NS-1 regions in flight: the stage of the previous iteration is free
      const int nx = (it + NS - 1) % NS;
      const int64_t tn = (*(volatile int32_t*)P.err) ? P.Q : (t_pref < P.Q ? t_pref : P.Q);
      if (t_pref < P.Q) t_pref = atomicAdd(P.ticket, 1);
      s_t[nx] = tn;
      s_early[nx] = 0;
      if (tn < P.Q) {
        const BufRegion Rn = buf_region<KT>(g, P, tn, buf_a);
        s_d[nx].set(Rn);
        if (!Rn.identity) buf_issue<KT>(P, Rn, buf_a, STAGE(nx), STAGE(nx) + P.smem_keys, &bar[nx]);
      }
    }
    PB_TICK(0);
    // in-place mode, control warp: this region's consumer range (loaded one iteration
    // ago), and the next region's, loaded now -- only the flag round trip is left
    // to overlap the merge
    const int64_t c_lo = cn_lo, c_hi = cn_hi;
    if (ctrl && !oop) {
      __syncwarp();  // (the leader's stage writes above)
      const int sn = (it + 1) % NS;
      cn_lo = 1;
      cn_hi = 0;
      if (s_t[sn] < P.Q && !s_d[sn].identity) {
        cn_lo = __ldg(&P.state[s_d[sn].r]);
        cn_hi = __ldg(&P.loc[s_d[sn].r]);
      }
    }
    if (R.identity) {  // records already on their outputs and read by r only
      if (leader) st_relaxed(&flags[R.r], 1);
    } else {
      while (!mbar_try_wait(&bar[cur], (phmask >> cur) & 1)) {
      }
      phmask ^= 1u << cur;
      PB_TICK(1);
      const int64_t phk = ((uintptr_t)(okeys + (P.s + R.d0) * ks)) & 15;
      const int64_t php = w ? (((uintptr_t)(opay + (P.s + R.d0) * w)) & 15) : 0;
      uint8_t* kout_s = OUTB(ob);
      uint8_t* pout_s = OUTB(ob) + P.smem_keys;
      if (ctrl && oop) {
        // copy mode: nothing to announce or wait for
      } else if (ctrl) {
        // (a relaxed flag: the region's loads have completed -- its barrier said so --
        // so a writer that sees the flag cannot change what the region read; a
        // release here would be a full GPU membar behind this CTA's bulk stores)
        if (leader && !s_early[cur]) st_relaxed(&flags[R.r], 1);
        // the records this region overwrites in the unbuffered run must have been read
        // by their consumers (regions c_lo..c_hi, precomputed by k_consumers)
        for (int64_t c = c_lo + lane; c <= c_hi; c += 32) {
          if (c == R.r) continue;
          for (uint32_t it2 = 0; ld_acquire(&flags[c]) == 0; ++it2) {
            if ((it2 & 255) == 255 && ld_relaxed(P.err)) break;
            if (it2 > kSpinLimit) {
              raise_error(P.err, PM_ERR_TIMEOUT);
              break;
            }
            backoff(it2);
          }
        }
        // regions in flight whose loads have landed: announce their reads early
        if (leader) {
          for (int k = 1; k < NS; ++k) {
            const int sk = (it + k) % NS;
            const int64_t tk = s_t[sk];
            if (tk < P.Q && !s_early[sk] && mbar_try_wait(&bar[sk], (phmask >> sk) & 1)) {
              if (!s_d[sk].identity) {
                st_relaxed(&flags[s_d[sk].r], 1);
                s_early[sk] = 1;
              }
            }
          }
        }
      } else {
        uint8_t* kin = STAGE(cur);
        uint8_t* pin = STAGE(cur) + P.smem_keys;
        if (!w) {
          write_sentinels<KT>(kin, R.offA, R.alpha, R.offB, R.beta, tid, MT);
          named_barrier_sync(1, MT);
        }
        const bool wq4 = w && (w & 3) == 0 && ((php | R.poffA | R.poffB) & 3) == 0;
        merge_tile<KT, kBufferedThreads - 32>(MODE_MERGE, reinterpret_cast<const KT*>(kin + R.offA),
                                              reinterpret_cast<const KT*>(kin + R.offB), R.alpha, R.beta, R.nout,
                                              reinterpret_cast<KT*>(kout_s + phk), pout_s + php, pin + R.poffA,
                                              pin + R.poffB, w, wq4, tid);
        PB_TICK(2);
        fence_proxy_async_smem();
      }
      PB_TICK(5);
      __syncthreads();  // tile complete, consumers done
      PB_TICK(3);
      // the leader (gt == 0) issues the bulk stores; everyone writes unaligned edges
      const int gt = (tid + 32) % NT;
      stream_out(kout_s + phk, reinterpret_cast<uint8_t*>(okeys + (P.s + R.d0) * ks), R.nout * ks, gt, NT);
      if (w) stream_out(pout_s + php, opay + (P.s + R.d0) * w, R.nout * w, gt, NT);
      ++n_reg;
    }
    if (leader) bulk_wait_read<1>();  // the store that used the other output buffer has read it
    __syncthreads();
    PB_TICK(4);
  }
  if (leader) {
    bulk_wait_all();
    atomicAdd(&P.stats[2], n_reg);
  }
  if (tid == 0) prof.flush(P.stats);
#undef STAGE
#undef OUTB
}

// The engine's ticket list: every ticket (two-front order) whose region is not an
// identity region, in order.  k_flags marks them (grid-wide, into tlist), then
// one CTA compacts: per-thread chunk counts, a block scan, chunk writes.
__global__ void __launch_bounds__(256) k_flags(EngineParams P) {
  if (P.gate && !*(volatile const int32_t*)P.gate) return;
  Geo g(P);
  const int64_t la = g.LA();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < P.Q; t += (int64_t)gridDim.x * blockDim.x) {
    bool work = true;
    if (P.mode == MODE_MERGE) {
      const int64_t q = g.region_of_ticket(t);
      const int64_t d0 = g.diag(q), d1 = g.diag(q + 1), a0 = g.split(q), a1 = g.split(q + 1);
      work = !((a0 == d0 && a1 == d1) || (a0 == la && a1 == la));
    }
    P.tlist[P.Q + 8 + t] = work ? 1 : 0;  // flags live after the list
    const unsigned idle = __ballot_sync(__activemask(), !work);
    if (idle && (threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(&P.ntick[1], __popc(idle));
  }
}
__global__ void __launch_bounds__(1024) k_compact(EngineParams P) {
  if (P.gate && !*(volatile const int32_t*)P.gate) return;
  __shared__ int32_t wsum[32];
  __shared__ int32_t base;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int32_t* flag = P.tlist + P.Q + 8;
  if (*(volatile int32_t*)&P.ntick[1] == 0) {  // no identity region: tickets map to themselves
    if (tid == 0) P.ntick[0] = (int32_t)P.Q;
    return;
  }
  if (tid == 0) base = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < P.Q; t0 += blockDim.x) {  // coalesced tiles, running offset
    const int64_t t = t0 + tid;
    const int32_t f = t < P.Q ? flag[t] : 0;
    int32_t x = f;  // warp inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int32_t s = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      if (lane < nw) wsum[lane] = s;  // inclusive warp prefix sums
    }
    __syncthreads();
    const int32_t pos = base + (wid ? wsum[wid - 1] : 0) + x - f;
    if (f) P.tlist[pos] = (int32_t)t;
    __syncthreads();
    if (tid == 0) base += wsum[nw - 1];
    __syncthreads();
  }
  if (tid == 0) *P.ntick = base;
}

// ---- staged path helpers: skip the whole pass when the runs are already in order ----
// dst <- src (n bytes, identical 16-byte phase), only if *gate
__global__ void __launch_bounds__(256) k_copy_gated(uint8_t* dst, const uint8_t* src, int64_t n, const int32_t* gate) {
  if (!*(volatile const int32_t*)gate) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  int64_t head = (16 - ((uintptr_t)src & 15)) & 15;
  if (head > n) head = n;
  const int64_t nv = (n - head) >> 4;
  for (int64_t b = tid; b < head; b += nthr) dst[b] = src[b];
  const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (int64_t i = tid; i < nv; i += nthr) d4[i] = PM_COPY_LD(s4 + i);
  for (int64_t b = head + (nv << 4) + tid; b < n; b += nthr) dst[b] = src[b];
}

cudaError_t launch_copy_gated(void* dst, const void* src, int64_t n, const int32_t* gate, int num_sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((n / 16 + 255) / 256 + 1, (int64_t)num_sms * 8);
  k_copy_gated<<<grid, 256, 0, st>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), n, gate);
  count_launches(1);
  return cudaGetLastError();
}

// ---- host launchers (called from pm_capi.cu) --------------------------------
template <typename KT>
cudaError_t launch_plan(const EngineParams& P, int grid, cudaStream_t st) {
  if (P.Q + 1 <= kWarpPlan) {  // one level: a warp per boundary (k_plan)
    grid = (int)std::max<int64_t>(grid, std::min<int64_t>((P.Q + 1 + 7) / 8, 2048));
    k_plan<KT><<<grid, 256, 0, st>>>(P);
    count_launches(1);
  } else {
    k_plan_coarse<KT><<<(int)std::min<int64_t>((P.Q / kCoarse + 8) / 8, 2048), 256, 0, st>>>(P);
    k_plan<KT><<<grid, 256, 0, st>>>(P);
    count_launches(2);
  }
  if (P.tlist && PM_TLIST) {
    k_flags<<<(int)std::min<int64_t>((P.Q + 255) / 256, 1184), 256, 0, st>>>(P);
    k_compact<<<1, 1024, 0, st>>>(P);
    count_launches(2);
  }
  return cudaGetLastError();
}
template <typename KT>
cudaError_t launch_engine(const EngineParams& P, int grid, int block, size_t smem, cudaStream_t st) {
  if (block != kEngineThreads) return cudaErrorInvalidValue;  // the kernel's team split is compile-time
  k_engine<KT><<<grid, block, smem, st>>>(P);
  count_launches(1);
  return cudaGetLastError();
}
template <typename KT>
cudaError_t engine_occupancy(int block, size_t smem, int* blocks_per_sm) {
  cudaError_t e = ensure_smem_attr((const void*)k_engine<KT>, smem);
  if (e != cudaSuccess) return e;
  return cached_occupancy(blocks_per_sm, (const void*)k_engine<KT>, block, smem);
}
template <typename KT>
cudaError_t buffered_occupancy(size_t smem, int* blocks_per_sm) {
  cudaError_t e = ensure_smem_attr((const void*)k_buffered<KT>, smem);
  if (e != cudaSuccess) return e;
  return cached_occupancy(blocks_per_sm, (const void*)k_buffered<KT>, kBufferedThreads, smem);
}
template <typename KT>
cudaError_t launch_buffered(const EngineParams& P, int32_t buf_a, int grid, size_t smem, cudaStream_t st) {
  const int64_t x0 = buf_a ? P.s : P.m, x1 = buf_a ? P.m : P.e;
  const int cgrid = (int)std::min<int64_t>(std::max<int64_t>(((x1 - x0) * (int64_t)sizeof(KT) / 16 + 255) / 256, 1),
                                           (int64_t)grid * 4);
  k_copy_run<KT><<<cgrid, 256, 0, st>>>(P, x0, x1);
  k_consumers<<<(int)std::min<int64_t>((P.Q + 255) / 256, 4096), 256, 0, st>>>(P, buf_a);
  count_launches(2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = ensure_smem_attr((const void*)k_buffered<KT>, smem);
  if (e != cudaSuccess) return e;
  k_buffered<KT><<<grid, kBufferedThreads, smem, st>>>(P, buf_a);
  count_launches(1);
  return cudaGetLastError();
}
template <typename KT>
cudaError_t launch_merge_copy(const EngineParams& P, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = ensure_smem_attr((const void*)k_buffered<KT>, smem);
  if (e != cudaSuccess) return e;
  k_buffered<KT><<<grid, kBufferedThreads, smem, st>>>(P, 1);
  count_launches(1);
  return cudaGetLastError();
}
template cudaError_t launch_merge_copy<int32_t>(const EngineParams&, int, size_t, cudaStream_t);
template cudaError_t launch_merge_copy<int64_t>(const EngineParams&, int, size_t, cudaStream_t);
template cudaError_t launch_buffered<int32_t>(const EngineParams&, int32_t, int, size_t, cudaStream_t);
template cudaError_t launch_buffered<int64_t>(const EngineParams&, int32_t, int, size_t, cudaStream_t);
template cudaError_t launch_plan<int32_t>(const EngineParams&, int, cudaStream_t);
template cudaError_t launch_plan<int64_t>(const EngineParams&, int, cudaStream_t);
template cudaError_t launch_engine<int32_t>(const EngineParams&, int, int, size_t, cudaStream_t);
template cudaError_t launch_engine<int64_t>(const EngineParams&, int, int, size_t, cudaStream_t);
template cudaError_t engine_occupancy<int32_t>(int, size_t, int*);
template cudaError_t buffered_occupancy<int32_t>(size_t, int*);
template cudaError_t buffered_occupancy<int64_t>(size_t, int*);
template cudaError_t engine_occupancy<int64_t>(int, size_t, int*);

}  // namespace pm
