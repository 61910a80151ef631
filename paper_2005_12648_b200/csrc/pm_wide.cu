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

#include "pm_common.cuh"
#include "pm_launch.h"
#include "pm_hostcache.h"

namespace pm {

namespace {

constexpr int kWideThreads = 256;
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
// its segment up to the next cut (the positions of cut cycles, all of them) and
// appends the segment to segs[] = {head, idx[head], end slot, 0}.  A segment
// longer than Lmax links is split: every Lmax-th position along it becomes an
// extra cut (its old row saved at save slot ncut + e, xpos[e] = its position)
// that ends one chain (end slot e) and heads the next, so no chain of the move
// walks more than Lmax links.  Slots past xcap are not cut (the chain continues).
__global__ void k_cyc_mark(const int32_t* __restrict__ idx, int64_t n, int32_t G, uint8_t* mark, int32_t Lmax,
                           int4* segs, int32_t* scnt, int32_t* xpos, int32_t* xcnt, int32_t xcap) {
  const int64_t ncut = (n + G - 1) / G;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ncut; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = (int32_t)(k * G);
    int32_t q = __ldg(idx + c);
    if (q == c) continue;
    mark[c] = 1;
    int4 pend = make_int4(c, q, -1, 0);
    bool cutting = true;
    for (int32_t step = 1; q % G != 0; ++step) {
      mark[q] = 1;
      const int32_t nq = __ldg(idx + q);
      if (step == Lmax && cutting) {
        const int32_t e = atomicAdd(xcnt, 1);
        if (e < xcap) {
          xpos[e] = q;
          pend.z = e;
          segs[atomicAdd(scnt, 1)] = pend;
          pend = make_int4(q, nq, -1, 0);
          step = 0;
        } else {
          cutting = false;
        }
      }
      q = nq;
    }
    segs[atomicAdd(scnt, 1)] = pend;
  }
}

// Uncut cycles (positions left unmarked, not fixed): walk at most kWalk steps;
// closing the cycle makes its minimum a head, heads[] = {head, idx[head]}.  A
// longer uncut cycle leaves its positions unresolved (mark = 2) and switches on
// the fallback.
constexpr int kWalk = 256;
__global__ void k_cyc_walk(const int32_t* __restrict__ idx, int64_t n, int2* heads, int32_t* cnt, uint8_t* mark,
                           int32_t* any_unres) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q0 = __ldg(idx + p);
    if (q0 == (int32_t)p || mark[p]) continue;
    int32_t q = q0, mn = (int32_t)p;
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
      heads[atomicAdd(cnt, 1)] = make_int2((int32_t)p, q0);
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
                               const int32_t* any_unres, int2* heads, int32_t* cnt, unsigned* bar, int rounds) {
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
    if (unres[p] == 2 && d0[p].x == (int32_t)p) heads[atomicAdd(cnt, 1)] = make_int2((int32_t)p, idx[p]);
}

// save[k] = row kG for every cut position kG that is not a fixed point; then
// save[ncut + e] = row xpos[e] for every extra cut e < min(*xcnt, xcap).
template <int V>
__global__ void __launch_bounds__(kWideThreads) k_cyc_save(uint8_t* __restrict__ save, const uint8_t* __restrict__ pay,
                                                           const int32_t* __restrict__ idx,
                                                           const int32_t* __restrict__ xpos, const int32_t* xcnt,
                                                           int32_t xcap, int64_t n, int64_t w, int32_t G) {
  using T = typename VecT<V>::T;
  const int64_t W = w / V, ncut = (n + G - 1) / G, nx = min(*xcnt, xcap);
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (ncut + nx) * W; t += nt) {
    const int64_t k = t / W, x = t - k * W;
    int64_t p;
    if (k < ncut) {
      p = k * G;
      if (__ldg(idx + p) == (int32_t)p) continue;
    } else {
      p = xpos[k - ncut];
    }
    reinterpret_cast<T*>(save + k * w)[x] = reinterpret_cast<const T*>(pay + p * w)[x];
  }
}

// The walk.  Items are (segment, kCycChunk-byte column chunk); segments are
// segs[0, *scnt) (cut and extra-cut heads) then heads[0, *hcnt) (uncut cycles).
// Lane k < kCycChains of every warp owns one chain and walks items k, k + C,
// k + 2C, ... (C = chains in the grid); the next item's record is prefetched,
// so a refill costs no memory round trip.  One step of all the warp's chains:
// each owner lane TMA-copies its source chunk (the 16-byte-aligned superset)
// into its shared buffer and loads its successor link, all on one mbarrier
// phase; then the warp stores the chains' chunks one after the other with
// V-byte vector stores.  Row data never sits in registers, so a warp keeps
// kCycChains x 512 B in flight for the price of a few state registers per lane.
// A step writes row d from its source s = idx[d] and the next step writes row
// s: every row is read before it is written.  A cut chain ends at the next cut
// (old row in save[q / G]) or, after Lmax links, at its extra cut (save[ncut +
// slot]); an uncut cycle ends back at its head, whose old chunk the chain copied
// into its second buffer at its first step.
#ifndef PM_CYC_CHAINS
#define PM_CYC_CHAINS 2  // tune: chains per warp (2 x 2 KB: 16 KB rows 1.12 ms vs 1.18 for 8 x 512 B, 2 GB)
#endif
#ifndef PM_CYC_CHUNK
#define PM_CYC_CHUNK 2048  // tune: row bytes per chain step
#endif
constexpr int kCycChains = PM_CYC_CHAINS;
constexpr int kCycWarps = 8;
constexpr int kCycChunk = PM_CYC_CHUNK;
constexpr int kCycBuf = kCycChunk + 32;  // superset of a chunk: <= 15 bytes of slack either side
constexpr size_t kCycWarpSmem = 2 * kCycChains * kCycBuf;
constexpr size_t kCycSmem = kCycWarps * kCycWarpSmem + kCycWarps * 16;

#ifndef PM_CYC_HINT
#define PM_CYC_HINT 0  // tune: 1 = row loads evict_last in L2 (kept until the chain's next step writes them), 2 = + stores evict_first
#endif
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t cyc_copy(uint8_t* buf, const uint8_t* src, int nbytes, uint64_t* bar, uint64_t pol) {
  const uintptr_t a = (uintptr_t)src & ~(uintptr_t)15;
  const uint32_t nb = (uint32_t)((((uintptr_t)src + nbytes + 15) & ~(uintptr_t)15) - a);
  mbar_expect_tx(bar, nb);
#if PM_CYC_HINT >= 1
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(buf)),
      "l"(a), "r"(nb), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  (void)pol;
  bulk_g2s(buf, reinterpret_cast<const void*>(a), nb, bar);
#endif
  return (uint32_t)((uintptr_t)src & 15);
}
template <typename T>
__device__ __forceinline__ void cyc_store(T* p, T v, uint64_t pol) {
#if PM_CYC_HINT >= 2
  if constexpr (sizeof(T) == 16) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
  } else if constexpr (sizeof(T) == 8) {
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
  } else if constexpr (sizeof(T) == 4) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
  } else {
    *p = v;
  }
#else
  (void)pol;
  *p = v;
#endif
}

template <int V>
__global__ void __launch_bounds__(kCycWarps * 32) k_cyc_move(uint8_t* pay, const uint8_t* __restrict__ save,
                                                           const int32_t* __restrict__ idx,
                                                           const int4* __restrict__ segs, const int32_t* scnt,
                                                           const int2* __restrict__ heads, const int32_t* hcnt,
                                                           int64_t n, int64_t w, int32_t G, int32_t Lmax) {
  using T = typename VecT<V>::T;
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool owner = lane < kCycChains;
  uint8_t* buf = sm + wid * kCycWarpSmem + (owner ? lane : 0) * kCycBuf;
  uint8_t* hbuf = buf + kCycChains * kCycBuf;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kCycWarps * kCycWarpSmem + wid * 16);
  if (lane == 0) mbar_init(bar, 32);
  __syncthreads();
  const uint64_t pol_ld = l2_policy_last(), pol_st = l2_policy_first();
  const int64_t ncut = (n + G - 1) / G, nch = (w + kCycChunk - 1) / kCycChunk;
  const int64_t cs = *scnt, items = (cs + *hcnt) * nch;
  const int64_t nchains = (int64_t)gridDim.x * kCycWarps * kCycChains;
  int64_t pj = ((int64_t)blockIdx.x * kCycWarps + wid) * kCycChains + lane;  // this chain's next item
  auto fetch = [&](int64_t j) -> int4 {
    const int64_t sg = j / nch;
    if (sg < cs) return segs[sg];
    const int2 h = heads[sg - cs];
    return make_int4(h.x, h.y, -1, 1);
  };
  int4 pf = make_int4(0, 0, -1, 0);
  if (owner && pj < items) pf = fetch(pj);
  int32_t hh = 0, dd = 0, ss = 0, xs = -1, stp = 1, kind = 0, col = 0;
  bool act = false, fresh = false;
  auto refill = [&]() {
    act = false;
    if (!owner || pj >= items) return;
    col = (int32_t)(pj % nch) * kCycChunk;
    hh = pf.x;
    ss = pf.y;
    xs = pf.z;
    kind = pf.w;
    dd = hh;
    stp = 1;
    act = fresh = true;
    pj += nchains;
    if (pj < items) pf = fetch(pj);
  };
  refill();
  uint32_t ph = 0;
  while (__any_sync(~0u, act)) {
    bool end = false;
    int32_t nn = 0;
    uint32_t soff = 0;  // shared address of this step's source chunk
    const int nb = (int)(w - col < kCycChunk ? w - col : kCycChunk);
    if (act) {
      const bool xend = kind == 0 && ss % G != 0 && xs >= 0 && stp == Lmax;
      end = kind == 0 ? (ss % G == 0 || xend) : (ss == hh);
      if (fresh && kind == 1) {
        const uint32_t o = cyc_copy(hbuf, pay + (int64_t)hh * w + col, nb, bar, pol_ld);
        if (end) soff = smem_u32(hbuf) + o;
      }
      if (!end || kind == 0) {
        const uint8_t* src = !end ? pay + (int64_t)ss * w
                             : xend ? save + (ncut + xs) * w
                                    : save + (int64_t)(ss / G) * w;
        soff = smem_u32(buf) + cyc_copy(buf, src + col, nb, bar, pol_ld);
      } else if (!fresh) {
        soff = smem_u32(hbuf) + (uint32_t)(((uintptr_t)(pay + (int64_t)hh * w + col)) & 15);
      }
      if (!end) nn = __ldg(idx + ss);
    }
    mbar_arrive(bar);
    while (!mbar_try_wait(bar, ph)) {
    }
    ph ^= 1;
#pragma unroll 1
    for (int k = 0; k < kCycChains; ++k) {
      if (!__shfl_sync(~0u, act, k)) continue;
      T* dst = reinterpret_cast<T*>(__shfl_sync(~0u, (unsigned long long)(pay + (int64_t)dd * w + col), k));
      const uint32_t so = __shfl_sync(~0u, soff, k);
      const int nv = __shfl_sync(~0u, nb, k) / V;
      for (int i = lane; i < nv; i += 32) {
        T v;
        if constexpr (V == 16) {
          uint4 r;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(so + i * 16));
          v = r;
        } else if constexpr (V == 8) {
          uint2 r;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(so + i * 8));
          v = r;
        } else if constexpr (V == 4) {
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(so + i * 4));
        } else if constexpr (V == 2) {
          uint16_t r;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(so + i * 2));
          v = r;
        } else {
          uint16_t r;
          asm volatile("ld.shared.u8 %0, [%1];" : "=h"(r) : "r"(so + i));
          v = (uint8_t)r;
        }
        cyc_store(dst + i, v, pol_st);
      }
    }
    __syncwarp();
    fence_proxy_async_smem();  // the buffers' generic reads before the next steps' bulk writes
    if (act) {
      fresh = false;
      if (end) {
        refill();
      } else {
        dd = ss;
        ss = nn;
        ++stp;
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
                                 int2* dbl1, int2* heads, int32_t* ctl, uint8_t* unres, int4* segs, int32_t* xpos,
                                 int32_t xcap, int32_t Lmax, uint8_t* save, int num_sms, cudaStream_t st) {
  // ctl: [0] uncut heads, [1] any unresolved, [2..3] grid barrier, [4] extra cuts, [5] segments
  cudaError_t e = cudaMemsetAsync(ctl, 0, 8 * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, num_sms);
  e = cudaMemsetAsync(unres, 0, (size_t)n, st);
  if (e != cudaSuccess) return e;
  int32_t* xcnt = ctl + 4;
  int32_t* scnt = ctl + 5;
  const int64_t ncut = (n + G - 1) / G;
  k_cyc_mark<<<grid_for(ncut, num_sms), kWideThreads, 0, st>>>(idx, n, G, unres, Lmax, segs, scnt, xpos, xcnt, xcap);
  k_cyc_walk<<<g, kWideThreads, 0, st>>>(idx, n, heads, ctl, unres, ctl + 1);
  int rounds = 0;
  while (((int64_t)1 << rounds) < n) ++rounds;
  {
    int bps = 0;
    e = cached_occupancy(&bps, (const void*)k_cyc_fallback, kWideThreads, 0);
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
  PM_WIDE_DISPATCH(v, (k_cyc_save<kV><<<grid_for((ncut + xcap) * (w / v), num_sms), kWideThreads, 0, st>>>(
                          save, pay, idx, xpos, xcnt, xcap, n, w, G)));
  // persistent: every SM full of walking warps
  int mgrid = 0;
  PM_WIDE_DISPATCH(v, ({
    auto kern = k_cyc_move<kV>;
    e = ensure_smem_attr((const void*)kern, kCycSmem);
    int bm = 0;
    if (e == cudaSuccess) e = cached_occupancy(&bm, (const void*)kern, kCycWarps * 32, kCycSmem);
    mgrid = std::max(1, bm) * num_sms;
    if (e == cudaSuccess)
      kern<<<mgrid, kCycWarps * 32, kCycSmem, st>>>(pay, save, idx, segs, ctl + 5, heads, ctl, n, w, G, Lmax);
  }));
  if (e != cudaSuccess) return e;
  count_launches(5);
  return cudaGetLastError();
}

}  // namespace pm
