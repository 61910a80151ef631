// pm_wide.cu -- merges of wide records (payload rows of hundreds of bytes up to
// the reference's 65 540-byte elements, bench.py:22 DEFAULT_ELEM_BYTES).
//
// Wide rows do not fit the engine's staging tiles, and moving them through a
// key-ordered tile wastes shared memory on bytes no comparison reads.  The
// merge of wide records is therefore split into
//   (1) the stable merge of (key, row index) pairs -- the streaming pipeline in
//       copy mode (k_buffered), 8 or 12 bytes per record;
//   (2) the row permutation it defines, new_row[p] = old_row[idx[p]]:
//       * out of place (pm_merge_copy, pm_merge_host): a gather (k_gather_rows);
//       * in place (pm_merge): the permutation's cycles are cut into segments
//         at every position p = kG (G from a bounded save budget); a cycle with
//         no such position is one segment headed by its minimum.  k_cyc_mark
//         walks every cut segment (one thread each) and marks its positions;
//         k_cyc_walk follows each unmarked position for at most kWalk steps
//         and, when it closes the (uncut) cycle, makes the minimum its head.
//         Uncut cycles longer than kWalk switch on k_cyc_fallback, one
//         persistent launch doing pointer doubling over (value, next) pairs
//         behind grid barriers (it exits at once otherwise).  k_cyc_save copies
//         the cut rows aside and k_cyc_move walks every segment per column
//         chunk, several chains per warp: the columns of a row move
//         independently, so even one long cycle spreads over row_bytes / chunk
//         chains.  Each record is read once and written once (plus the saved
//         cut rows, ~1/G of them).
// Keys, row indices and the doubling arrays are 4-16 bytes per record against
// rows of >= kWideMin bytes, so the extra space is a few percent of the data.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "pm_launch.h"

namespace pm {

namespace {

constexpr int kWideThreads = 256;
#ifndef PM_CYC_MINB
#define PM_CYC_MINB 3  // tune: resident CTAs per SM the cycle walk is compiled for (1: 1.94 ms, 3: 1.67, 4: 2.62 at 508-byte rows)
#endif
constexpr int kChunkWords = 4;  // vector words per lane per chunk step

template <int V> struct VecT;
template <> struct VecT<16> { using T = uint4; };
template <> struct VecT<8> { using T = uint2; };
template <> struct VecT<4> { using T = uint32_t; };
template <> struct VecT<2> { using T = uint16_t; };
template <> struct VecT<1> { using T = uint8_t; };

__global__ void k_iota(int32_t* idx, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    idx[p] = (int32_t)p;
}

// out[p] = (idx[p] < la ? a[idx[p]] : b[idx[p] - la]); one warp per (row, chunk).
template <int V>
__global__ void __launch_bounds__(kWideThreads) k_gather_rows(uint8_t* __restrict__ out, const uint8_t* __restrict__ a,
                                                              const uint8_t* __restrict__ b, const int32_t* idx,
                                                              int64_t n, int64_t la, int64_t w) {
  using T = typename VecT<V>::T;
  const int lane = threadIdx.x & 31;
  const int64_t W = w / V, span = 32 * kChunkWords, nch = (W + span - 1) / span;
  const int64_t items = n * nch, nw = (int64_t)gridDim.x * (kWideThreads / 32);
  for (int64_t it = blockIdx.x * (int64_t)(kWideThreads / 32) + (threadIdx.x >> 5); it < items; it += nw) {
    const int64_t p = it / nch, c0 = (it - p * nch) * span;
    const int64_t src = idx[p];
    const T* s = reinterpret_cast<const T*>(src < la ? a + src * w : b + (src - la) * w);
    T* d = reinterpret_cast<T*>(out + p * w);
    T v[kChunkWords];
#pragma unroll
    for (int u = 0; u < kChunkWords; ++u) {
      const int64_t x = c0 + u * 32 + lane;
      if (x < W) v[u] = s[x];
    }
#pragma unroll
    for (int u = 0; u < kChunkWords; ++u) {
      const int64_t x = c0 + u * 32 + lane;
      if (x < W) d[x] = v[u];
    }
  }
}

// mark[q] = 1 for every q on a cut segment: one thread per cut position walks
// its segment up to the next cut (the positions of cut cycles, all of them).
__global__ void k_cyc_mark(const int32_t* __restrict__ idx, int64_t n, int32_t G, uint8_t* mark) {
  const int64_t ncut = (n + G - 1) / G;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ncut; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = (int32_t)(k * G);
    int32_t q = __ldg(idx + c);
    if (q == c) continue;
    mark[c] = 1;
    while (q % G != 0) {
      mark[q] = 1;
      q = __ldg(idx + q);
    }
  }
}

// Uncut cycles (positions left unmarked, not fixed): walk at most kWalk steps;
// closing the cycle makes its minimum a head.  A longer uncut cycle leaves its
// positions unresolved (mark = 2) and switches on the fallback.
constexpr int kWalk = 256;
__global__ void k_cyc_walk(const int32_t* __restrict__ idx, int64_t n, int32_t* heads, int32_t* cnt, uint8_t* mark,
                           int32_t* any_unres) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t q = __ldg(idx + p);
    if (q == (int32_t)p || mark[p]) continue;
    int32_t mn = (int32_t)p;
    bool closed = false;
    for (int k = 0; k < kWalk; ++k) {
      if (q == (int32_t)p) {
        closed = true;
        break;
      }
      mn = min(mn, q);
      q = __ldg(idx + q);
    }
    if (!closed) {
      mark[p] = 2;
      *any_unres = 1;
    } else if (mn == (int32_t)p) {
      heads[atomicAdd(cnt, 1)] = (int32_t)p;
    }
  }
}

// Grid-wide barrier of a cooperative launch (all blocks co-resident).
__device__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// Fallback for uncut cycles longer than kWalk (runs only when k_cyc_walk left
// some position unresolved, mark = 2): pointer doubling, ceil(log2 n) rounds; .x becomes
// the minimum over the cycle of val[p] = (p % G == 0 ? -1 : p), so an
// unresolved p is a head iff it is its cycle's value minimum.
__global__ void k_cyc_fallback(const int32_t* idx, int64_t n, int32_t G, int2* d0, int2* d1, const uint8_t* unres,
                               const int32_t* any_unres, int32_t* heads, int32_t* cnt, unsigned* bar, int rounds) {
  if (*(volatile const int32_t*)any_unres == 0) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t p = t0; p < n; p += stride) d0[p] = make_int2(p % G == 0 ? -1 : (int32_t)p, idx[p]);
  for (int r = 0; r < rounds; ++r) {
    grid_barrier(bar, bar + 1, gridDim.x);
    for (int64_t p = t0; p < n; p += stride) {
      const int2 a = d0[p], b = d0[a.y];
      d1[p] = make_int2(min(a.x, b.x), b.y);
    }
    int2* t = d0;
    d0 = d1;
    d1 = t;
  }
  grid_barrier(bar, bar + 1, gridDim.x);
  for (int64_t p = t0; p < n; p += stride)
    if (unres[p] == 2 && d0[p].x == (int32_t)p) heads[atomicAdd(cnt, 1)] = (int32_t)p;
}
// save[k] = row kG for every cut position kG that is not a fixed point.
template <int V>
__global__ void __launch_bounds__(kWideThreads) k_cyc_save(uint8_t* __restrict__ save, const uint8_t* __restrict__ pay,
                                                           const int32_t* idx, int64_t n, int64_t w, int32_t G) {
  using T = typename VecT<V>::T;
  const int64_t W = w / V, ncut = (n + G - 1) / G;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncut * W; t += nt) {
    const int64_t k = t / W, x = t - k * W, p = k * G;
    if (idx[p] == (int32_t)p) continue;
    reinterpret_cast<T*>(save + k * w)[x] = reinterpret_cast<const T*>(pay + p * w)[x];
  }
}

// Vector words per lane per chunk step (1 KB per warp step for 8/16-byte words)
// and independent chains per warp (each step of a chain waits for its successor
// link, so a warp keeps several segments in flight).
template <int V> __host__ __device__ constexpr int chunk_words() { return V == 16 ? 2 : 4; }
template <int V> __host__ __device__ constexpr int chains() { return V >= 8 ? 2 : 4; }

// Segment items (x column chunks): [0, ncut) start at the cut positions kG
// (fixed points skip); [ncut, ncut + *cnt) are the uncut cycles' heads.  A cut
// segment ends where its walk reaches the next cut position, whose old row is
// read from save[]; an uncut cycle ends back at its head, whose old chunk the
// warp kept in registers.  A step writes row d from its source s = idx[d] and
// the next step writes row s: every row is read before it is written.  Each
// warp runs kC chains side by side, refilling a slot from its item sequence.
template <int V>
__global__ void __launch_bounds__(kWideThreads, PM_CYC_MINB) k_cyc_move(uint8_t* pay, const uint8_t* __restrict__ save,
                                                           const int32_t* __restrict__ idx,
                                                           const int32_t* __restrict__ heads, const int32_t* cnt,
                                                           int64_t n, int64_t w, int32_t G) {
  using T = typename VecT<V>::T;
  constexpr int CW = chunk_words<V>(), kC = chains<V>();
  // uncut heads' old chunks (read back at the cycle's last step)
  __shared__ T stash[kWideThreads / 32][kC][CW * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t W = w / V, span = 32 * CW, nch = (W + span - 1) / span;
  const int64_t ncut = (n + G - 1) / G, nseg = ncut + *cnt;
  const int64_t items = nseg * nch, nw = (int64_t)gridDim.x * (kWideThreads / 32);
  int64_t next = blockIdx.x * (int64_t)(kWideThreads / 32) + wid;
  int32_t hh[kC], dd[kC], ss[kC];
  int64_t cc[kC];
  bool cut[kC], act[kC];
  // (re)fill slot k with the next non-trivial item of this warp (an idle slot
  // keeps a harmless state: chunk 0, position 0)
  auto refill = [&](int k) {
    act[k] = false;
    cc[k] = 0;
    hh[k] = dd[k] = ss[k] = 0;
    cut[k] = true;
    while (next < items) {
      const int64_t it = next;
      next += nw;
      const int64_t sg = it / nch;
      cc[k] = (it - sg * nch) * span;
      cut[k] = sg < ncut;
      hh[k] = cut[k] ? (int32_t)(sg * G) : heads[sg - ncut];
      ss[k] = __ldg(idx + hh[k]);
      if (ss[k] == hh[k]) continue;  // fixed point
      dd[k] = hh[k];
      if (!cut[k]) {
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          const int64_t x = min(cc[k] + u * 32 + lane, W - 1);
          stash[wid][k][u * 32 + lane] = reinterpret_cast<const T*>(pay + (int64_t)hh[k] * w)[x];
        }
      }
      act[k] = true;
      break;
    }
  };
#pragma unroll
  for (int k = 0; k < kC; ++k) refill(k);
  for (;;) {
    bool any = false;
#pragma unroll
    for (int k = 0; k < kC; ++k) any |= act[k];
    if (!any) break;
    // every slot loads unconditionally (idle slots read a valid dummy row, x is
    // clamped into the row), so the loads of all chains are in flight together
    T v[kC][CW];
    bool end[kC];
    int32_t nn[kC];
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      end[k] = cut[k] ? (ss[k] % G == 0) : (ss[k] == hh[k]);
      nn[k] = __ldg(idx + ((end[k] || !act[k]) ? 0 : ss[k]));  // successor link, in flight with the row load
      const T* src = !act[k] ? reinterpret_cast<const T*>(pay)
                     : !end[k] ? reinterpret_cast<const T*>(pay + (int64_t)ss[k] * w)
                     : cut[k] ? reinterpret_cast<const T*>(save + (int64_t)(ss[k] / G) * w)
                              : &stash[wid][k][0] - cc[k];
#pragma unroll
      for (int u = 0; u < CW; ++u) v[k][u] = src[min(cc[k] + u * 32 + lane, W - 1)];
    }
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      if (act[k]) {
        T* dst = reinterpret_cast<T*>(pay + (int64_t)dd[k] * w);
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          const int64_t x = cc[k] + u * 32 + lane;
          if (x < W) dst[x] = v[k][u];
        }
        if (end[k]) {
          refill(k);
        } else {
          dd[k] = ss[k];
          ss[k] = nn[k];
        }
      }
    }
  }
}

int grid_for(int64_t work, int num_sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + kWideThreads - 1) / kWideThreads, (int64_t)num_sms * 8));
}

int vec_bytes(int64_t w, std::initializer_list<const void*> ptrs) {
  uintptr_t acc = (uintptr_t)w;
  for (const void* p : ptrs) acc |= (uintptr_t)p;
  for (int v : {16, 8, 4, 2}) if ((acc & (uintptr_t)(v - 1)) == 0) return v;
  return 1;
}

}  // namespace

cudaError_t launch_iota(int32_t* idx, int64_t n, int num_sms, cudaStream_t st) {
  k_iota<<<grid_for(n, num_sms), kWideThreads, 0, st>>>(idx, n);
  count_launches(1);
  return cudaGetLastError();
}

#define PM_WIDE_DISPATCH(V, CALL) \
  switch (V) {                    \
    case 16: { constexpr int kV = 16; CALL; break; } \
    case 8: { constexpr int kV = 8; CALL; break; }   \
    case 4: { constexpr int kV = 4; CALL; break; }   \
    case 2: { constexpr int kV = 2; CALL; break; }   \
    default: { constexpr int kV = 1; CALL; break; }  \
  }

cudaError_t launch_gather_rows(uint8_t* out, const uint8_t* a, const uint8_t* b, const int32_t* idx, int64_t n,
                               int64_t la, int64_t w, int num_sms, cudaStream_t st) {
  const int v = vec_bytes(w, {out, a, b});
  const int64_t span = 32 * kChunkWords, nch = (w / v + span - 1) / span;
  const int grid = grid_for(n * nch * 32, num_sms);
  PM_WIDE_DISPATCH(v, (k_gather_rows<kV><<<grid, kWideThreads, 0, st>>>(out, a, b, idx, n, la, w)));
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cycle_permute(uint8_t* pay, int64_t w, const int32_t* idx, int64_t n, int32_t G, int2* dbl0,
                                 int2* dbl1, int32_t* heads, int32_t* ctl, uint8_t* unres, uint8_t* save, int num_sms,
                                 cudaStream_t st) {
  // ctl: [0] uncut heads, [1] any unresolved, [2..3] grid barrier
  cudaError_t e = cudaMemsetAsync(ctl, 0, 4 * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, num_sms);
  e = cudaMemsetAsync(unres, 0, (size_t)n, st);
  if (e != cudaSuccess) return e;
  k_cyc_mark<<<grid_for((n + G - 1) / G, num_sms), kWideThreads, 0, st>>>(idx, n, G, unres);
  k_cyc_walk<<<g, kWideThreads, 0, st>>>(idx, n, heads, ctl, unres, ctl + 1);
  int rounds = 0;
  while (((int64_t)1 << rounds) < n) ++rounds;
  {
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cyc_fallback, kWideThreads, 0);
    if (e != cudaSuccess) return e;
    const int fg = std::max(1, std::min(bps * num_sms, g));
    int32_t* cnt = ctl;
    int32_t* anyu = ctl + 1;
    unsigned* bar = reinterpret_cast<unsigned*>(ctl + 2);
    void* args[] = {(void*)&idx, (void*)&n, (void*)&G, (void*)&dbl0, (void*)&dbl1, (void*)&unres,
                    (void*)&anyu, (void*)&heads, (void*)&cnt, (void*)&bar, (void*)&rounds};
    e = cudaLaunchCooperativeKernel((const void*)k_cyc_fallback, dim3(fg), dim3(kWideThreads), args, 0, st);
    if (e != cudaSuccess) return e;
  }
  const int v = vec_bytes(w, {pay, save});
  const int64_t ncut = (n + G - 1) / G;
  PM_WIDE_DISPATCH(v, (k_cyc_save<kV><<<grid_for(ncut * (w / v), num_sms), kWideThreads, 0, st>>>(save, pay, idx, n,
                                                                                                   w, G)));
  int64_t nch = 0;
  PM_WIDE_DISPATCH(v, (nch = (w / kV + 32 * chunk_words<kV>() - 1) / (32 * chunk_words<kV>())));
  // enough warps for every cut segment's chunks; uncut heads share the grid-stride loop
  const int mgrid = grid_for(std::max<int64_t>(ncut * nch, (int64_t)num_sms * 64) * 32, num_sms);
  PM_WIDE_DISPATCH(v, (k_cyc_move<kV><<<mgrid, kWideThreads, 0, st>>>(pay, save, idx, heads, ctl, n, w, G)));
  count_launches(5);
  return cudaGetLastError();
}

}  // namespace pm
