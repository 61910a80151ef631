// pm_rotate.cu -- in-place block exchange A|B -> B|A by three reversals
// (reverse A, reverse B, reverse A|B): two streaming passes over the records,
// every pass a perfectly parallel swap of mirrored records (coalesced on both
// sides), no bookkeeping.  Replaces _kernels.linear_shift / circular_shift
// (_kernels.py:92-197) behind pm_shift; the result is the same array (the
// reference's instrumented move counts are computed on the host, shift.py).
#include <cuda_runtime.h>
#include <type_traits>

#include <algorithm>
#include <cstdint>

#include "pm_common.cuh"
#include "pm_launch.h"
#include "pm_tile.cuh"
#include "pm_hostcache.h"

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
__global__ void __launch_bounds__(256) k_reverse(const int32_t* gate, KT* keys, uint8_t* pay, int64_t w, int64_t lo0,
                                                 int64_t len0, int64_t lo1, int64_t len1) {
  if (gate && !*(volatile const int32_t*)gate) return;
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

// Keys only, 16-byte vectors: block job b of a segment swaps the aligned left
// chunk [x0, x0+C) with its mirror [S-x0-C+1, S-x0] (S = 2 lo + len - 1).  Both
// ranges are read into shared memory with aligned vector loads (the right one
// as an aligned superset), then written back reversed -- aligned vector stores,
// element stores only for the right range's partial edge vectors.  The pairs
// before the first aligned chunk and after the last full one are swapped by one
// extra job per segment, element by element.  Jobs never share a record.
template <typename KT, int C>
__global__ void __launch_bounds__(256) k_reverse_vec(const int32_t* gate, KT* keys, int64_t lo0, int64_t len0, int64_t lo1,
                                                     int64_t len1) {
  if (gate && !*(volatile const int32_t*)gate) return;
  constexpr int V = 16 / sizeof(KT);
  __shared__ __align__(16) KT Lb[C];
  __shared__ __align__(16) KT Rb[C + 2 * V];
  auto plan = [&](int64_t lo, int64_t len, int64_t& L0, int64_t& nfull) {
    const int64_t half = len >> 1;
    L0 = (lo + V - 1) / V * V;
    nfull = L0 < lo + half ? (lo + half - L0) / C : 0;
  };
  int64_t L00, nf0, L01, nf1;
  plan(lo0, len0, L00, nf0);
  plan(lo1, len1, L01, nf1);
  const int64_t njobs = nf0 + nf1 + 2;
  for (int64_t job = blockIdx.x; job < njobs; job += gridDim.x) {
    // job order: full chunks of segment 0, of segment 1, then the two scalar jobs
    const bool s1 = job >= nf0 && job != nf0 + nf1;
    const int64_t lo = s1 ? lo1 : lo0, len = s1 ? len1 : len0, L0 = s1 ? L01 : L00, nf = s1 ? nf1 : nf0;
    const int64_t S = 2 * lo + len - 1, half = len >> 1;
    if (job >= nf0 + nf1) {  // scalar pairs of segment 0 (job nf0+nf1) or 1 (last job)
      const int64_t head_end = min(L0, lo + half), tail0 = max(L0 + nf * C, head_end);
      for (int64_t x = lo + threadIdx.x; x < head_end; x += blockDim.x) {
        const KT a = keys[x], b = keys[S - x];
        keys[x] = b;
        keys[S - x] = a;
      }
      for (int64_t x = tail0 + threadIdx.x; x < lo + half; x += blockDim.x) {
        const KT a = keys[x], b = keys[S - x];
        keys[x] = b;
        keys[S - x] = a;
      }
      continue;
    }
    const int64_t b = s1 ? job - nf0 : job;
    const int64_t x0 = L0 + b * C;
    const int64_t ylo = S - x0 - C + 1, yhi = S - x0;  // inclusive
    const int64_t r0 = ylo / V * V, r1 = (yhi + V) / V * V;  // aligned superset [r0, r1)
    const uint4* L4 = reinterpret_cast<const uint4*>(keys + x0);
    const uint4* R4 = reinterpret_cast<const uint4*>(keys + r0);
    for (int i = threadIdx.x; i < C / V; i += blockDim.x) reinterpret_cast<uint4*>(Lb)[i] = L4[i];
    for (int i = threadIdx.x; i < (int)((r1 - r0) / V); i += blockDim.x) {
      const int64_t yb = r0 + (int64_t)i * V;
      if (yb + V <= lo + len) {
        reinterpret_cast<uint4*>(Rb)[i] = R4[i];
      } else {  // (the segment's last partial vector: stay inside the caller's array)
        for (int c = 0; c < V && yb + c < lo + len; ++c) Rb[i * V + c] = keys[yb + c];
      }
    }
    __syncthreads();
    // left chunk <- mirror (reversed)
    uint4* Lo4 = reinterpret_cast<uint4*>(keys + x0);
    for (int i = threadIdx.x; i < C / V; i += blockDim.x) {
      KT v[V];
#pragma unroll
      for (int c = 0; c < V; ++c) v[c] = Rb[(S - (x0 + i * V + c)) - r0];
      Lo4[i] = *reinterpret_cast<const uint4*>(v);
    }
    // right range <- left chunk (reversed); partial edge vectors element by element
    for (int64_t i = threadIdx.x; i < (r1 - r0) / V; i += blockDim.x) {
      const int64_t yb = r0 + i * V;
      if (yb >= ylo && yb + V - 1 <= yhi) {
        KT v[V];
#pragma unroll
        for (int c = 0; c < V; ++c) v[c] = Lb[(S - (yb + c)) - x0];
        *reinterpret_cast<uint4*>(keys + yb) = *reinterpret_cast<const uint4*>(v);
      } else {
        for (int c = 0; c < V; ++c) {
          const int64_t y = yb + c;
          if (y >= ylo && y <= yhi) keys[y] = Lb[(S - y) - x0];
        }
      }
    }
    __syncthreads();
  }
}

// Wide payload rows: one warp per (mirrored pair, column chunk) swaps the two
// rows with V-byte vector words (lane 0 of chunk 0 also swaps the keys), so a
// row pair moves coalesced instead of one thread walking a whole row.
template <int V> struct RowWord;
template <> struct RowWord<16> { using T = uint4; };
template <> struct RowWord<8> { using T = uint2; };
template <> struct RowWord<4> { using T = uint32_t; };
template <> struct RowWord<2> { using T = uint16_t; };
template <> struct RowWord<1> { using T = uint8_t; };

template <typename KT, int V>
__global__ void __launch_bounds__(256) k_reverse_wide(const int32_t* gate, KT* keys, uint8_t* pay, int64_t w, int64_t lo0,
                                                      int64_t len0, int64_t lo1, int64_t len1) {
  if (gate && !*(volatile const int32_t*)gate) return;
  using T = typename RowWord<V>::T;
  constexpr int CW = 4;
  const int lane = threadIdx.x & 31;
  const int64_t W = w / V, span = 32 * CW, nch = (W + span - 1) / span;
  const int64_t p0 = len0 >> 1, np = p0 + (len1 >> 1), items = np * nch;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += nw) {
    const int64_t p = it / nch, c0 = (it - p * nch) * span;
    const bool s0 = p < p0;
    const int64_t i = s0 ? p : p - p0, lo = s0 ? lo0 : lo1, len = s0 ? len0 : len1;
    const int64_t xl = lo + i, xr = lo + len - 1 - i;
    if (c0 == 0 && lane == 0) {
      const KT a = keys[xl];
      keys[xl] = keys[xr];
      keys[xr] = a;
    }
    T* L = reinterpret_cast<T*>(pay + xl * w);
    T* R = reinterpret_cast<T*>(pay + xr * w);
    T a[CW], b[CW];
#pragma unroll
    for (int u = 0; u < CW; ++u) {
      const int64_t x = c0 + u * 32 + lane;
      if (x < W) {
        a[u] = L[x];
        b[u] = R[x];
      }
    }
#pragma unroll
    for (int u = 0; u < CW; ++u) {
      const int64_t x = c0 + u * 32 + lane;
      if (x < W) {
        L[x] = b[u];
        R[x] = a[u];
      }
    }
  }
}

template <typename KT, int V>
static void reverse_wide_pair(KT* k, uint8_t* p, int64_t w, int64_t lo, int64_t la, int64_t lb, int num_sms,
                              cudaStream_t st, const int32_t* gate) {
  const int64_t nch = (w / V + 127) / 128;
  const int64_t pairs = (la >> 1) + (lb >> 1), all = (la + lb) >> 1;
  auto grid_for = [&](int64_t items) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, (int64_t)num_sms * 8));
  };
  if (pairs > 0) k_reverse_wide<KT, V><<<grid_for(pairs * nch), 256, 0, st>>>(gate, k, p, w, lo, la, lo + la, lb);
  if (all > 0) k_reverse_wide<KT, V><<<grid_for(all * nch), 256, 0, st>>>(gate, k, p, w, lo, la + lb, 0, 0);
  count_launches((pairs > 0) + (all > 0));
}

#ifndef PM_ROTATE_WIDE_MIN
#define PM_ROTATE_WIDE_MIN 32  // payload bytes per row from which rows move warp-wide
#endif

// ---- one-pass block exchange when one block is small (the reference's staged
// exchange, _kernels.py:46-90, for blocks of up to PM_SLIDE_STASH bytes) ----
constexpr int kSlideTile = 32768;
constexpr int kSlideThreads = 256;
constexpr int kSlideStages = 2;

// Aligned 16-byte destination chunks [c0, c0 + 16 nc) from the staged source image:
// destination byte x reads stage byte x + dlt, and dlt's 16-byte phase is the same
// for every chunk (Q words + S bits).  Two conflict-free 16-byte shared loads per
// chunk and a funnel shift realign it.
template <int Q>
__device__ __forceinline__ void slide_chunks(uint8_t* dst, const uint8_t* src, int64_t nc, int sh) {
  for (int64_t c = threadIdx.x; c < nc; c += blockDim.x) {
    const uint4* q = reinterpret_cast<const uint4*>(src + c * 16);
    uint4 v;
    if (Q == 0 && sh == 0) {
      v = q[0];
    } else {
      const uint4 a = q[0], b = q[1];
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      v = make_uint4(__funnelshift_r(w[Q], w[Q + 1], sh), __funnelshift_r(w[Q + 1], w[Q + 2], sh),
                     __funnelshift_r(w[Q + 2], w[Q + 3], sh), __funnelshift_r(w[Q + 3], w[Q + 4], sh));
    }
    __stcs(reinterpret_cast<uint4*>(dst + c * 16), v);
  }
}

// One tile's destination bytes [d0, d1) from its staged source: stage byte of
// destination x is x + dlt.  Aligned 16-byte chunks, bytewise at the range edges.
__device__ __forceinline__ void slide_store(uint8_t* plane, const uint8_t* tile, int64_t d0, int64_t d1, int64_t dlt) {
  const uintptr_t c0 = ((uintptr_t)(plane + d0) + 15) & ~(uintptr_t)15;
  const uintptr_t c1 = (uintptr_t)(plane + d1) & ~(uintptr_t)15;
  if (c1 > c0) {
    const int64_t x0 = (int64_t)(c0 - (uintptr_t)plane), nc = (int64_t)((c1 - c0) >> 4);
    const int64_t so = x0 + dlt;  // stage offset of the first chunk's source
    const int r = (int)(so & 15), sh = (r & 3) * 8;
    const uint8_t* src = tile + (so - r);
    switch (r >> 2) {
      case 0: slide_chunks<0>(plane + x0, src, nc, sh); break;
      case 1: slide_chunks<1>(plane + x0, src, nc, sh); break;
      case 2: slide_chunks<2>(plane + x0, src, nc, sh); break;
      default: slide_chunks<3>(plane + x0, src, nc, sh); break;
    }
    const int64_t h = (int64_t)(c0 - (uintptr_t)(plane + d0)), tl = (int64_t)((uintptr_t)(plane + d1) - c1);
    for (int64_t bt = threadIdx.x; bt < h + tl; bt += blockDim.x) {
      const int64_t x = bt < h ? d0 + bt : (int64_t)(c1 - (uintptr_t)plane) + (bt - h);
      plane[x] = tile[x + dlt];
    }
  } else {
    for (int64_t x = d0 + threadIdx.x; x < d1; x += blockDim.x) plane[x] = tile[x + dlt];
  }
}

// The small block is stashed (stream-ordered copies on the host side), the big
// block slides over it in one pass, the stash lands at the far end.  The slide
// is an overlapping move: plane bytes [S0, S0+L) move by -D (left) or +D
// (right).  A persistent grid claims kSlideTile-byte source tiles in the
// direction of the move (ascending for left); each CTA keeps kSlideStages tiles in
// flight: the TMA bulk load of its next tile lands while it stores the current one.
// A landed tile publishes "read"; before storing, a tile waits until every
// earlier-claimed tile whose source its destination overlaps has been read.  Waits
// only ever target tiles claimed earlier (whose loads were issued at claim time),
// so they always resolve.
__global__ void __launch_bounds__(kSlideThreads) k_slide(uint8_t* plane, int64_t S0, int64_t L, int64_t D, int right,
                                                         int32_t* flags, int32_t* ticket, int32_t* err) {
  extern __shared__ __align__(128) uint8_t sdyn[];
  __shared__ uint64_t bar[kSlideStages];
  __shared__ int64_t s_i[kSlideStages];
  const int64_t ntiles = (L + kSlideTile - 1) / kSlideTile;
  constexpr size_t kStage = kSlideTile + 64;
  auto issue = [&](int stg) {  // thread 0: claim the next tile, TMA-load its 16-byte-aligned superset
    const int64_t t = atomicAdd(ticket, 1);
    const int64_t i = t < ntiles ? (right ? ntiles - 1 - t : t) : -1;
    s_i[stg] = i;
    if (i >= 0) {
      const int64_t s0 = S0 + i * kSlideTile, s1 = min(S0 + L, s0 + kSlideTile);
      copy_g2s_superset(sdyn + stg * kStage + (((uintptr_t)(plane + s0)) & 15), plane + s0, s1 - s0, &bar[stg]);
    }
    mbar_arrive(&bar[stg]);
  };
  if (threadIdx.x == 0) {
    for (int k = 0; k < kSlideStages; ++k) mbar_init(&bar[k], 1);
    for (int k = 0; k < kSlideStages; ++k) issue(k);
  }
  __syncthreads();
  uint32_t ph = 0;
  for (int it = 0;; ++it) {
    const int cur = it % kSlideStages;
    while (!mbar_try_wait(&bar[cur], (ph >> cur) & 1)) {
    }
    ph ^= 1u << cur;
    const int64_t i = s_i[cur];
    if (i < 0) break;
    if (threadIdx.x == 0) st_release(&flags[i], 1);  // this tile's source is read (it landed)
    const int64_t s0 = S0 + i * kSlideTile, s1 = min(S0 + L, s0 + kSlideTile);
    const int64_t d0 = right ? s0 + D : s0 - D, d1 = right ? s1 + D : s1 - D;
    const int64_t lo = max(d0, S0), hi = min(d1, S0 + L);  // the part over the big block's source
    if (hi > lo) {
      const int64_t j0 = (lo - S0) / kSlideTile, j1 = (hi - 1 - S0) / kSlideTile;
      for (int64_t j = j0 + threadIdx.x; j <= j1; j += blockDim.x) {
        if (j == i) continue;
        for (uint32_t w = 0; ld_acquire(&flags[j]) == 0; ++w) {
          if (w > kSpinLimit) {
            raise_error(err, PM_ERR_TIMEOUT);
            break;
          }
          backoff(w);
        }
      }
    }
    __syncthreads();
    const uint8_t* tile = sdyn + cur * kStage;
    // the stage holds the source's 16-byte-aligned superset from stage byte 0: plane byte x
    // sits at stage byte x - sbase
    const int64_t sbase = (int64_t)(((uintptr_t)(plane + s0)) & ~(uintptr_t)15) - (int64_t)(uintptr_t)plane;
    slide_store(plane, tile, d0, d1, (right ? -D : D) - sbase);
    __syncthreads();  // the stage is free
    if (threadIdx.x == 0) issue(cur);
  }
}

cudaError_t launch_slide(void* plane, int64_t S0, int64_t L, int64_t D, bool right, int32_t* flags, int32_t* ticket,
                         int32_t* err, int num_sms, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  const int64_t ntiles = (L + kSlideTile - 1) / kSlideTile;
  cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)ntiles * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ticket, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const size_t smem = kSlideStages * (kSlideTile + 64);
  e = ensure_smem_attr((const void*)k_slide, smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)num_sms * 3);
  k_slide<<<grid, kSlideThreads, smem, st>>>(static_cast<uint8_t*>(plane), S0, L, D, right ? 1 : 0, flags, ticket, err);
  count_launches(1);
  return cudaGetLastError();
}

#ifndef PM_SWAP_HINTS
#define PM_SWAP_HINTS 0  // 1: streaming (evict-first) loads / stores in the block swap (2^30: 0.67 of the copy peak vs 0.90 without)
#endif
#if PM_SWAP_HINTS
#define SWAP_LD(p) __ldcs(p)
#define SWAP_ST(p, v) __stcs(p, v)
#else
#define SWAP_LD(p) (*(p))
#define SWAP_ST(p, v) (*(p) = (v))
#endif
// ---- block swap of two equal adjacent blocks: [X | Y] -> [Y | X] ----------------
// A rotation with |A| == |B| needs no reversal: every word of X trades places with
// the word len bytes ahead (one read and one write per record: 2 N w of traffic
// instead of the reversals' 4 N w).  Grid-stride, four words per thread in flight;
// 16-byte words when both blocks share the 16-byte grid, else 4- or 1-byte words.
template <typename WT>
__global__ void __launch_bounds__(256) k_swap_blocks(const int32_t* gate, uint8_t* x, uint8_t* y, int64_t nbytes) {
  if (gate && !*(volatile const int32_t*)gate) return;
  WT* a = reinterpret_cast<WT*>(x);
  WT* b = reinterpret_cast<WT*>(y);
  const int64_t n = nbytes / (int64_t)sizeof(WT), stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
    WT va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        va[u] = SWAP_LD(a + i);
        vb[u] = SWAP_LD(b + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        SWAP_ST(a + i, vb[u]);
        SWAP_ST(b + i, va[u]);
      }
    }
  }
}

// grid: every resident CTA once (a grid-stride kernel with a second partial wave
// leaves the late CTAs running alone: 0.66 of the copy peak at 2^30 with 1184 CTAs)
template <typename WT>
static cudaError_t swap_launch(uint8_t* x, uint8_t* y, int64_t nbytes, int num_sms, cudaStream_t st,
                               const int32_t* gate) {
  int bps = 0;
  cudaError_t e = cached_occupancy(&bps, (const void*)k_swap_blocks<WT>, 256, 0);
  if (e != cudaSuccess) return e;
  const int64_t words = nbytes / (int64_t)sizeof(WT);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((words + 1023) / 1024, (int64_t)num_sms * std::max(bps, 1)));
  k_swap_blocks<WT><<<grid, 256, 0, st>>>(gate, x, y, nbytes);
  return cudaGetLastError();
}
// swap the disjoint byte blocks [x, x + nbytes) and [y, y + nbytes)
static cudaError_t swap_plane(uint8_t* x, uint8_t* y, int64_t nbytes, int num_sms, cudaStream_t st,
                              const int32_t* gate) {
  if (nbytes <= 0) return cudaSuccess;
  const uintptr_t al = (uintptr_t)x | (uintptr_t)y | (uintptr_t)nbytes;
  count_launches(1);
  if ((al & 15) == 0) return swap_launch<uint4>(x, y, nbytes, num_sms, st, gate);
  if ((al & 3) == 0) return swap_launch<uint32_t>(x, y, nbytes, num_sms, st, gate);
  return swap_launch<uint8_t>(x, y, nbytes, num_sms, st, gate);
}
// records [x0, x0 + len) <-> [y0, y0 + len) (disjoint) in the keys and payload planes
static cudaError_t swap_records(void* keys, int ks, void* payload, int64_t w, int64_t x0, int64_t y0, int64_t len,
                                int num_sms, cudaStream_t st, const int32_t* gate) {
  uint8_t* K = static_cast<uint8_t*>(keys);
  cudaError_t e = swap_plane(K + x0 * ks, K + y0 * ks, len * ks, num_sms, st, gate);
  if (e == cudaSuccess && w) {
    uint8_t* P = static_cast<uint8_t*>(payload);
    e = swap_plane(P + x0 * w, P + y0 * w, len * w, num_sms, st, gate);
  }
  return e;
}

// [lo, lo + len) <-> [lo + len, lo + 2 len) in the keys and the payload planes
cudaError_t launch_swap_blocks(void* keys, int ks, void* payload, int64_t w, int64_t lo, int64_t len, int num_sms,
                               cudaStream_t st, const int32_t* gate) {
  return swap_records(keys, ks, payload, w, lo, lo + len, len, num_sms, st, gate);
}

// Linear shifting by block swaps (the reference's Gries-Mills exchange,
// _kernels.py:92-150): swap the smaller block with the far end of the larger one
// -- it lands in its final place -- and continue on the rest.  Each step is one
// streaming swap (4 s w bytes for a block of s records); the steps stop once the
// smaller block is under 1/16 of the exchange (or after 16 steps), and three
// reversals finish the remainder.  Equal blocks: one swap.  The sequence depends
// only on the lengths, so it is enqueued whole (gated like the reversals).
template <typename KT>
cudaError_t launch_block_exchange(void* keys, void* payload, int64_t w, int64_t lo, int64_t la, int64_t lb,
                                  int num_sms, cudaStream_t st, const int32_t* gate) {
  const int64_t n = la + lb;
  cudaError_t e = cudaSuccess;
  int64_t a = la, b = lb;
  for (int step = 0; e == cudaSuccess && a > 0 && b > 0 && step < 16; ++step) {
    if (a == b) return swap_records(keys, sizeof(KT), payload, w, lo, lo + a, a, num_sms, st, gate);
    if (std::min(a, b) * 16 < n) break;
    if (a < b) {  // [X | Y1 Y2], |Y2| = a: X <-> Y2 puts X last; rotate [Y2 | Y1] next
      e = swap_records(keys, sizeof(KT), payload, w, lo, lo + b, a, num_sms, st, gate);
      b -= a;
    } else {  // [X1 X2 | Y], |X1| = b: X1 <-> Y puts Y first; rotate [X2 | X1] next
      e = swap_records(keys, sizeof(KT), payload, w, lo, lo + a, b, num_sms, st, gate);
      lo += b;
      a -= b;
    }
  }
  if (e != cudaSuccess || a == 0 || b == 0) return e;
  return launch_rotate<KT>(keys, payload, w, lo, a, b, num_sms, st, gate);
}
template cudaError_t launch_block_exchange<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int,
                                                    cudaStream_t, const int32_t*);
template cudaError_t launch_block_exchange<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int,
                                                    cudaStream_t, const int32_t*);

template <typename KT>
cudaError_t launch_rotate(void* keys, void* payload, int64_t w, int64_t lo, int64_t la, int64_t lb, int num_sms,
                          cudaStream_t st, const int32_t* gate) {
  KT* k = static_cast<KT*>(keys);
  uint8_t* p = static_cast<uint8_t*>(payload);
  const int64_t pairs = (la >> 1) + (lb >> 1);
  const int64_t all = (la + lb) >> 1;
  auto grid_for = [&](int64_t np) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((np + 1023) / 1024, (int64_t)num_sms * 8));
  };
  // vectorised block jobs on one plane of 4- or 8-byte elements (its base 16-byte aligned)
  auto vec_plane = [&](auto* base) {
    using ET = std::remove_pointer_t<decltype(base)>;
    constexpr int C = 8192 / sizeof(ET);
    auto jobs = [&](int64_t a, int64_t b) { return (a / 2) / C + (b / 2) / C + 2; };
    const int g1 = (int)std::max<int64_t>(1, std::min<int64_t>(jobs(la, lb), (int64_t)num_sms * 8));
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(jobs(la + lb, 0), (int64_t)num_sms * 8));
    if (pairs > 0) k_reverse_vec<ET, C><<<g1, 256, 0, st>>>(gate, base, lo, la, lo + la, lb);
    if (all > 0) k_reverse_vec<ET, C><<<g2, 256, 0, st>>>(gate, base, lo, la + lb, 0, 0);
    count_launches((pairs > 0) + (all > 0));
  };
  const bool kal = (((uintptr_t)keys) & 15) == 0, pal = (((uintptr_t)payload) & 15) == 0;
  if (kal && (!w || ((w == 4 || w == 8) && pal))) {
    // keys, and 4- / 8-byte payload rows as a plane of int32 / int64 elements (SoA):
    // each plane reversed with 16-byte vectors (a row-wise swap is 3-4x slower)
    vec_plane(k);
    if (w == 4) vec_plane(reinterpret_cast<int32_t*>(p));
    if (w == 8) vec_plane(reinterpret_cast<int64_t*>(p));
    return cudaGetLastError();
  }
  if (w >= PM_ROTATE_WIDE_MIN) {
    const uintptr_t al = (uintptr_t)p | (uintptr_t)w;
    if ((al & 15) == 0) reverse_wide_pair<KT, 16>(k, p, w, lo, la, lb, num_sms, st, gate);
    else if ((al & 7) == 0) reverse_wide_pair<KT, 8>(k, p, w, lo, la, lb, num_sms, st, gate);
    else if ((al & 3) == 0) reverse_wide_pair<KT, 4>(k, p, w, lo, la, lb, num_sms, st, gate);
    else if ((al & 1) == 0) reverse_wide_pair<KT, 2>(k, p, w, lo, la, lb, num_sms, st, gate);
    else reverse_wide_pair<KT, 1>(k, p, w, lo, la, lb, num_sms, st, gate);
    return cudaGetLastError();
  }
  if (pairs > 0) k_reverse<KT><<<grid_for(pairs), 256, 0, st>>>(gate, k, p, w, lo, la, lo + la, lb);
  if (all > 0) k_reverse<KT><<<grid_for(all), 256, 0, st>>>(gate, k, p, w, lo, la + lb, 0, 0);
  count_launches((pairs > 0) + (all > 0));
  return cudaGetLastError();
}
template cudaError_t launch_rotate<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, cudaStream_t,
                                            const int32_t*);
template cudaError_t launch_rotate<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, cudaStream_t,
                                            const int32_t*);

}  // namespace pm
