// pm_tile.cuh -- device pieces shared by the in-place engines (k_engine, k_buffered
// in pm_engine.cu; k_flow in pm_flow.cu): job/slot/region geometry, the staged
// tile copies (TMA bulk global->shared superset copies, warp vector copies), the
// stable shared-memory tile merge and the bulk-store stream-out.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pm_common.cuh"
#include "pm_engine.cuh"

namespace pm {

#ifndef PM_ABLATE
#define PM_ABLATE 0  // bit 0: tile merge, 1: salvage copies, 2: gather loads, 3: output stores (tuning builds)
#endif
#ifndef PM_STATS
#define PM_STATS 0
#endif

// ============================================================================
// geometry helpers (all indices int64; "local" = relative to the job)
// ============================================================================
struct Geo {
  const EngineParams& P;
  __device__ explicit Geo(const EngineParams& p) : P(p) {}
  __device__ int64_t LA() const { return P.m - P.s; }
  __device__ int64_t LB() const { return P.e - P.m; }
  __device__ int64_t N() const { return P.e - P.s; }
  // slot j (local) -> absolute element range (clipped to the job)
  __device__ int64_t slot_lo(int64_t j) const { return max(P.s, (P.k0 + j) * P.T); }
  __device__ int64_t slot_hi(int64_t j) const { return min(P.e, (P.k0 + j + 1) * P.T); }
  __device__ int64_t slot_base(int64_t j) const { return (P.k0 + j) * P.T; }  // unclipped
  __device__ bool slot_full(int64_t j) const { return slot_hi(j) - slot_lo(j) == P.T; }
  __device__ int64_t region_of_slot(int64_t j) const { return ((P.k0 + j) >> P.lmu) - P.R0; }
  __device__ int64_t region_first_slot(int64_t q) const { return max((int64_t)0, (P.R0 + q) * P.mu - P.k0); }
  __device__ int64_t region_end_slot(int64_t q) const { return min(P.K, (P.R0 + q + 1) * P.mu - P.k0); }
  // local output diagonal at the start of region q (q in [0, Q])
  __device__ int64_t diag(int64_t q) const {
    if (q <= 0) return 0;
    if (q >= P.Q) return N();
    return (P.R0 + q) * P.M - P.s;
  }
  // ---- two-front ticket order (pm_engine.cuh) ----
  __device__ TwoFront tf() const { return TwoFront{P.Q, P.qc}; }
  __device__ int64_t region_of_ticket(int64_t t) const { return tf().region_of_ticket(t); }
  __device__ int64_t order(int64_t q) const { return tf().order(q); }
  __device__ void window(int64_t t, int64_t& lo, int64_t& hi) const { tf().window(t, lo, hi); }
  // split of boundary q (computed by k_plan before the engine starts; read-only here)
  __device__ int64_t split(int64_t q) const { return __ldg(&P.split_a[q]); }
  // records of unit j consumed by the regions of the ticket window <= t
  __device__ int64_t consumed_by_window(int64_t j, int64_t t) const {
    int64_t wl, wr;
    window(t, wl, wr);
    return consumed_in(j, wl, wr, split(wl), split(wr + 1));
  }
  // same, with the window [wl, wr] and its boundary splits already at hand
  __device__ int64_t consumed_in(int64_t j, int64_t wl, int64_t wr, int64_t a_lo, int64_t a_hi) const {
    int64_t b_lo = diag(wl) - a_lo, b_hi = diag(wr + 1) - a_hi;
    int64_t x0 = slot_lo(j), x1 = slot_hi(j), c = 0;
    // A part of the unit, A-local indices
    int64_t ua0 = x0 - P.s, ua1 = min(x1, P.m) - P.s;
    if (ua1 > ua0) c += max((int64_t)0, min(ua1, a_hi) - max(ua0, a_lo));
    int64_t ub0 = max(x0, P.m) - P.m, ub1 = x1 - P.m;
    if (ub1 > ub0) c += max((int64_t)0, min(ub1, b_hi) - max(ub0, b_lo));
    return c;
  }
};

// copy n (< 16) bytes that lie inside one aligned 16-byte chunk, from a vector
// already loaded by the caller
__device__ __forceinline__ void put_small(uint8_t* dst, const uint4& v, const uint8_t* src, int n) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  const int o = (int)((uintptr_t)src & 15);
  for (int i = 0; i < n; ++i) dst[i] = b[o + i];
}
__device__ __forceinline__ uint4 load_chunk(const uint8_t* src, int n) {
  if (n <= 0) return make_uint4(0, 0, 0, 0);
  return __ldcg(reinterpret_cast<const uint4*>((uintptr_t)src & ~(uintptr_t)15));
}

// global -> shared, identical 16-byte phase on both sides: TMA bulk copy for the
// aligned body, one vector load each for the unaligned head and tail (both
// issued before either is used)
__device__ __forceinline__ void copy_g2s_phased(uint8_t* dst, const uint8_t* src, int64_t nbytes, uint64_t* bar) {
  if (nbytes <= 0) return;
  int64_t head = (16 - ((uintptr_t)src & 15)) & 15;
  if (head > nbytes) head = nbytes;
  const int64_t body = ((nbytes - head) >> 4) << 4;
  const int tail = (int)(nbytes - head - body);
  const uint4 vh = load_chunk(src, (int)head);
  const uint4 vt = load_chunk(src + head + body, tail);
  if (body > 0) {
    mbar_expect_tx(bar, (uint32_t)body);
    bulk_g2s(dst + head, src + head, (uint32_t)body, bar);
  }
  if (head) put_small(dst, vh, src, (int)head);
  if (tail) put_small(dst + head + body, vt, src + head + body, tail);
}

// global -> shared by TMA over the 16-byte-aligned superset of the piece: bytes
// just outside it are copied too and ignored (they land in the tile's phase/pad
// bytes; interior piece boundaries are unit boundaries, which are aligned)
__device__ __forceinline__ void copy_g2s_superset(uint8_t* dst, const uint8_t* src, int64_t nbytes, uint64_t* bar) {
  if (nbytes <= 0) return;
  const uintptr_t a = (uintptr_t)src & ~(uintptr_t)15;
  const uintptr_t b = ((uintptr_t)src + nbytes + 15) & ~(uintptr_t)15;
  const uint32_t n = (uint32_t)(b - a);
  mbar_expect_tx(bar, n);
  bulk_g2s(dst - ((uintptr_t)src - a), reinterpret_cast<const void*>(a), n, bar);
}

// One staged piece: the superset copy when the caller's slot boundaries are 16-byte
// aligned (consecutive pieces then meet on aligned bytes), else the exact copy --
// with an unaligned base two adjacent pieces from different sources would both
// write the bytes around their common boundary.
__device__ __forceinline__ void copy_g2s_piece(uint8_t* dst, const uint8_t* src, int64_t nbytes, uint64_t* bar,
                                               bool exact) {
  if (exact) copy_g2s_phased(dst, src, nbytes, bar);
  else copy_g2s_superset(dst, src, nbytes, bar);
}

// warp copy global -> global, identical 16-byte phase on both sides; all loads of
// a lane are issued before its stores (8 x 16 B in flight per lane)
#ifndef PM_COPY_LDCS
#define PM_COPY_LDCS 0  // 1: streaming (evict-first) loads in the warp copies (salvage copy at 2^30: 0.238 ms vs 0.234 without)
#endif
#if PM_COPY_LDCS
#define PM_COPY_LD(p) __ldcs(p)
#else
#define PM_COPY_LD(p) (*(p))
#endif
__device__ __forceinline__ void copy_g2g_warp(uint8_t* dst, const uint8_t* src, int64_t nbytes, int lane) {
  if (nbytes <= 0) return;
  int64_t head = (16 - ((uintptr_t)src & 15)) & 15;
  if (head > nbytes) head = nbytes;
  if (lane < head) dst[lane] = src[lane];
  const int64_t nvec = (nbytes - head) >> 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  int64_t i = lane;
#ifndef PM_COPY_UNROLL
#define PM_COPY_UNROLL 8
#endif
  constexpr int CU = PM_COPY_UNROLL;
  for (; i + 32 * (CU - 1) < nvec; i += 32 * CU) {
    uint4 v[CU];
#pragma unroll
    for (int k = 0; k < CU; ++k) v[k] = PM_COPY_LD(s4 + i + 32 * k);
#pragma unroll
    for (int k = 0; k < CU; ++k) d4[i + 32 * k] = v[k];
  }
  for (; i < nvec; i += 32) d4[i] = PM_COPY_LD(s4 + i);
  const int64_t tail0 = head + (nvec << 4);
  if (tail0 + lane < nbytes) dst[tail0 + lane] = src[tail0 + lane];
}

// Merge (A wins ties) or concatenate (rotation: B then A) the staged runs As[0,alpha),
// Bs[0,beta) into the output tile ko[0,nout) (+ payload rows), thread gt of GT.
// Every thread takes an odd-length run of outputs: odd strides keep the shared
// memory accesses of a warp on distinct banks.
// +max sentinels after both staged runs (keys-only merges; threads gt of GT).
template <typename KT>
__device__ __forceinline__ void write_sentinels(uint8_t* kin, int64_t offA, int64_t alpha, int64_t offB, int64_t beta,
                                                int gt, int GT) {
  KT* a = reinterpret_cast<KT*>(kin + offA) + alpha;
  KT* b = reinterpret_cast<KT*>(kin + offB) + beta;
  const KT mx = sizeof(KT) == 4 ? (KT)INT32_MAX : (KT)INT64_MAX;
  for (int k = gt; k < 2 * kSent; k += GT) (k < kSent ? a[k] : b[k - kSent]) = mx;
}

// GT (the merging threads) is a compile-time constant: the per-thread span E is
// then a multiply-shift, not a division, on every region
template <typename KT, int GT>
__device__ __forceinline__ void merge_tile(int32_t mode, const KT* As, const KT* Bs, int64_t alpha, int64_t beta,
                                           int64_t nout, KT* ko, uint8_t* po, const uint8_t* PA, const uint8_t* PB,
                                           int64_t w, bool wq4, int gt) {
  int32_t E = (int32_t)(((uint32_t)nout + GT - 1) / (uint32_t)GT);  // 32-bit: nout <= M
  E |= 1;
  {
    // region-local indices fit in 32 bits (nout <= M)
    const int32_t al = (int32_t)alpha, bl = (int32_t)beta, no = (int32_t)nout, e32 = (int32_t)E;
    int32_t o = min(gt * e32, no);
    const int32_t oe = min(o + e32, no);
    if (mode == MODE_MERGE && !w) {
      // keys only.  Shared-memory bandwidth bounds this loop (lanes sit at random
      // offsets, ~3.5-way bank conflicts per load), so each step loads exactly one
      // candidate -- the replacement for the side just taken -- via an address select
      // Both runs are followed by kSent +max sentinels (write_sentinels): an
      // exhausted run offers +max, which loses to every real key except +max
      // itself -- and then either choice emits the same value.  No bound checks.
      int32_t lo = o > bl ? o - bl : 0, hi = o < al ? o : al;
      const KT* Bq = Bs + (o - 1);  // Bs[o - 1 - mid] == Bq[-mid]
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (As[mid] <= *(Bq - mid)) lo = mid + 1;
        else hi = mid;
      }
      // run cursors as pointers: a step is compare, min, store, one predicated
      // advance per side, the candidate address select, load, and the refill
      const KT* pa = As + lo;
      const KT* pb = Bs + (o - lo);
      KT va = *pa, vb = *pb;
#pragma unroll 4
      for (; o < oe; ++o) {
        const bool takeA = va <= vb;
        ko[o] = takeA ? va : vb;
        if (takeA) ++pa; else ++pb;
        const KT v = *(takeA ? pa : pb);
        if (takeA) va = v; else vb = v;
      }
    } else if (mode == MODE_MERGE) {
      int32_t lo = o > bl ? o - bl : 0, hi = o < al ? o : al;
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (As[mid] <= Bs[o - 1 - mid]) lo = mid + 1;
        else hi = mid;
      }
      int32_t i = lo, jb = o - lo;
      const int32_t amax = al > 0 ? al - 1 : 0, bmax = bl > 0 ? bl - 1 : 0;
      KT va = As[min(i, amax)], vb = Bs[min(jb, bmax)];
      // with payload (stability visible): bound-checked, branch-free steps -- the
      // taken record's payload row is copied, then only the taken side reloads
      if (wq4 && w == 4) {
        const uint32_t* pa = reinterpret_cast<const uint32_t*>(PA);
        const uint32_t* pb = reinterpret_cast<const uint32_t*>(PB);
        uint32_t* pd = reinterpret_cast<uint32_t*>(po);
#pragma unroll 4
        for (; o < oe; ++o) {
          const bool takeA = (jb >= bl) | ((i < al) & (va <= vb));
          ko[o] = takeA ? va : vb;
          pd[o] = *(takeA ? pa + i : pb + jb);
          i += takeA;
          jb += !takeA;
          const KT v = *(takeA ? As + min(i, amax) : Bs + min(jb, bmax));
          va = takeA ? v : va;
          vb = takeA ? vb : v;
        }
      } else {
        for (; o < oe; ++o) {
          const bool takeA = (jb >= bl) | ((i < al) & (va <= vb));
          ko[o] = takeA ? va : vb;
          const uint8_t* rs = takeA ? PA + (int64_t)i * w : PB + (int64_t)jb * w;
          uint8_t* rd = po + (int64_t)o * w;
          if (wq4) {
            for (int64_t c = 0; c < w; c += 4)
              *reinterpret_cast<uint32_t*>(rd + c) = *reinterpret_cast<const uint32_t*>(rs + c);
          } else {
            for (int64_t c = 0; c < w; ++c) rd[c] = rs[c];
          }
          i += takeA;
          jb += !takeA;
          const KT v = *(takeA ? As + min(i, amax) : Bs + min(jb, bmax));
          va = takeA ? v : va;
          vb = takeA ? vb : v;
        }
      }
    } else {  // rotation: B piece then A piece
      for (; o < oe; ++o) {
        const bool fromB = o < bl;
        const int32_t si = fromB ? o : o - bl;
        ko[o] = fromB ? Bs[si] : As[si];
        if (w) {
          const uint8_t* rs = fromB ? PB + (int64_t)si * w : PA + (int64_t)si * w;
          uint8_t* rd = po + (int64_t)o * w;
          for (int64_t c = 0; c < w; ++c) rd[c] = rs[c];
        }
      }
    }
  }
}

// merge_tile for wide payload rows (w >= kWideRow, rows 4-byte aligned): the
// per-thread spans of merge_tile would leave most threads idle (a 32 KB tile holds
// only 32 KB / w records) and copy each row with one thread.  Phase 1: one thread
// per output finds its source by the merge-path search (A first on ties: stable),
// writes the key and parks the source row's offset in the first word of its output
// row.  Phase 2, after a barrier over the GT merging threads: one warp per output
// row reads the offset and copies the row with 16-byte (or 4-byte) words.
#ifndef PM_WIDE_ROW
#define PM_WIDE_ROW 384  // tune: payload bytes from which the tile merge copies rows warp-cooperatively (124 B: 1.18 vs 1.37 ms per-thread)
#endif
constexpr int64_t kWideRow = PM_WIDE_ROW;
template <typename KT, int GT>
__device__ __forceinline__ void merge_tile_wide(const KT* As, const KT* Bs, int64_t alpha, int64_t beta, int64_t nout,
                                                KT* ko, uint8_t* po, const uint8_t* PA, const uint8_t* PB, int64_t w,
                                                int gt, int bar_id) {
  const int32_t al = (int32_t)alpha, bl = (int32_t)beta, no = (int32_t)nout, w32 = (int32_t)w;
  for (int32_t o = gt; o < no; o += GT) {
    int32_t lo = o > bl ? o - bl : 0, hi = o < al ? o : al;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (As[mid] <= Bs[o - 1 - mid]) lo = mid + 1;
      else hi = mid;
    }
    const int32_t i = lo, j = o - lo;
    const bool takeA = j >= bl || (i < al && As[i] <= Bs[j]);
    ko[o] = takeA ? As[i] : Bs[j];
    const uint8_t* src = takeA ? PA + (int64_t)i * w32 : PB + (int64_t)j * w32;
    *reinterpret_cast<int32_t*>(po + (int64_t)o * w32) = (int32_t)(src - PA);
  }
  named_barrier_sync(bar_id, GT);
  // lane groups of L = 2^lg lanes per row (>= ~4 vector words per lane), 32 / L rows
  // per warp step; a group reads its row's parked offset before anyone overwrites it
  const int lane = gt & 31;
  const bool v16 = (w32 & 15) == 0 && ((((uintptr_t)po) | ((uintptr_t)PA) | ((uintptr_t)PB)) & 15) == 0;
  const int vb = v16 ? 16 : 4;
  int lg = 5;
  while (lg > 0 && (w32 / vb) < (4 << lg)) --lg;
  const int L = 1 << lg, grp = lane >> lg, sub = lane & (L - 1), rpw = 32 >> lg;
  for (int32_t o0 = (gt >> 5) * rpw; o0 < no; o0 += (GT / 32) * rpw) {
    const int32_t o = o0 + grp;
    uint8_t* dst = po + (int64_t)o * w32;
    const int32_t off = o < no ? *reinterpret_cast<const int32_t*>(dst) : 0;
    __syncwarp();
    if (o < no) {
      const uint8_t* src = PA + off;
      if (v16) {
        for (int32_t c = sub * 16; c < w32; c += L * 16)
          *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
      } else {
        for (int32_t c = sub * 4; c < w32; c += L * 4)
          *reinterpret_cast<uint32_t*>(dst + c) = *reinterpret_cast<const uint32_t*>(src + c);
      }
    }
  }
}

// Stream n bytes from a shared-memory tile to global memory with the same 16-byte
// phase: thread `gt` == 0 issues one TMA bulk store for the aligned body; the
// first threads write the unaligned head / tail bytes.
__device__ __forceinline__ void stream_out(const uint8_t* src_s, uint8_t* dst_g, int64_t n, int gt, int GT) {
  if (n <= 0) return;
  int64_t head = (16 - ((uintptr_t)dst_g & 15)) & 15;
  if (head > n) head = n;
  const int64_t body = ((n - head) >> 4) << 4;
  const int64_t tail0 = head + body;
  if (gt == 0 && body > 0) {
    bulk_s2g(dst_g + head, src_s + head, (uint32_t)body);
    bulk_commit();
  }
  for (int64_t b = gt; b < head; b += GT) dst_g[b] = src_s[b];
  for (int64_t b = tail0 + gt; b < n; b += GT) dst_g[b] = src_s[b];
}

// Cycle counters of the engine phases (pm_status stats[4..15]); compiled in only
// with -DPM_STATS=1 (tuning builds) -- the counters cost registers.
enum : int { PS_GATHER = 4, PS_LAND = 5, PS_PUBLISH = 6, PS_MERGE = 7, PS_WAITDEF = 8, PS_STORE = 9,
             PS_STEP1 = 10, PS_STEP2 = 11, PS_SLAND = 12, PS_THR = 13, PS_DEST = 14, PS_COPY = 15 };
struct Prof {
#if PM_STATS
  unsigned long long v[16] = {};
  __device__ __forceinline__ long long now() const { return clock64(); }
  __device__ __forceinline__ void add(int k, long long d) { v[k] += (unsigned long long)d; }
  __device__ __forceinline__ void flush(unsigned long long* stats) const {
    for (int k = 4; k < 16; ++k)
      if (v[k]) atomicAdd(&stats[k], v[k]);
  }
  // per-ticket-range histogram: stats[base + 16*t/Q] += d
  __device__ __forceinline__ void hist(unsigned long long* stats, int base, int64_t t, int64_t Q, long long d) const {
    atomicAdd(&stats[base + (int)(t * 16 / Q)], (unsigned long long)d);
  }
#else
  __device__ __forceinline__ long long now() const { return 0; }
  __device__ __forceinline__ void add(int, long long) {}
  __device__ __forceinline__ void flush(unsigned long long*) const {}
  __device__ __forceinline__ void hist(unsigned long long*, int, int64_t, int64_t, long long) const {}
#endif
};

}  // namespace pm
