// pm_small.cu -- small and medium in-place merges in one launch: one CTA (up to
// 32 KB of records), one cooperative grid with a shared-memory tile per SM (up to
// ~14 MB, k_merge_grid below), and the thread-block-cluster merge (kept behind
// PM_CLUSTER_MERGE; the grid merge is faster).
//
// When both runs fit in shared memory (keys + payload rows <= kSmallBytes), a
// single CTA stages A|B on chip (16-byte bulk loads), each thread finds its
// output range's stable merge-path split (A wins ties, as the reference's
// buffered_merge, _kernels.py:227-313) and merges it straight back into the
// caller's arrays -- everything was read before anything is written, so the
// in-place semantics hold with no scratch.  One launch, a few microseconds:
// the persistent engine's plan + ticket machinery costs ~50 us at these sizes.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <cstdint>

#include "pm_launch.h"
#include "pm_hostcache.h"
#include "pm_search.cuh"
#include "pm_common.cuh"

namespace pm {

namespace {

constexpr int kSmallThreads = 1024;
constexpr int64_t kClusterSmem = 216 * 1024;  // shared memory per CTA of the cluster merge (staging + window)

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

// merged records of a thread's output span go to a shared-memory output tile
// first (per-thread spans written straight to global memory would scatter every
// warp store over 32 lines); the tile then leaves with coalesced stores
template <typename KT>
__device__ __forceinline__ void merge_spans_to_tile(const KT* A, int la, const KT* B, int lb, const uint8_t* PA,
                                                    const uint8_t* PB, int64_t w, KT* ok, uint8_t* op) {
  const int no = la + lb;
  const int per = (no + blockDim.x - 1) / blockDim.x;
  const int d0 = min(no, (int)threadIdx.x * per), d1 = min(no, d0 + per);
  if (d0 >= d1) return;
  int i = split_smem(A, la, B, lb, d0), j = d0 - i;
  const bool w4 = w && ((uintptr_t)w & 3) == 0;
  for (int d = d0; d < d1; ++d) {
    const bool ta = j >= lb || (i < la && A[i] <= B[j]);
    ok[d] = ta ? A[i] : B[j];
    if (w) {
      const uint8_t* rs = ta ? PA + (int64_t)i * w : PB + (int64_t)j * w;
      uint8_t* rd = op + (int64_t)d * w;
      if (w4) {
        for (int64_t c = 0; c < w; c += 4) *reinterpret_cast<uint32_t*>(rd + c) = *reinterpret_cast<const uint32_t*>(rs + c);
      } else {
        for (int64_t c = 0; c < w; ++c) rd[c] = rs[c];
      }
    }
    if (ta) ++i;
    else ++j;
  }
}

// coalesced copy of a tile (keys ok[0, n), rows op) to keys / pay
template <typename KT>
__device__ __forceinline__ void tile_out(KT* keys, uint8_t* pay, const KT* ok, const uint8_t* op, int n, int64_t w) {
  for (int t = threadIdx.x; t < n; t += blockDim.x) keys[t] = ok[t];
  if (w) {
    if (((((uintptr_t)pay) | (uintptr_t)w) & 3) == 0) {
      const int64_t nw = (int64_t)n * (w >> 2);
      for (int64_t t = threadIdx.x; t < nw; t += blockDim.x)
        reinterpret_cast<uint32_t*>(pay)[t] = reinterpret_cast<const uint32_t*>(op)[t];
    } else {
      for (int64_t t = threadIdx.x; t < (int64_t)n * w; t += blockDim.x) pay[t] = op[t];
    }
  }
}

template <typename KT>
__global__ void __launch_bounds__(kSmallThreads) k_merge_small(KT* keys, uint8_t* pay, int64_t w, int la, int lb) {
  extern __shared__ __align__(16) uint8_t sm[];
  if (keys[la - 1] <= keys[la]) return;  // already in order (srecpar.py:56-57): nothing moves
  const int n = la + lb;
  const int64_t kreg = ((int64_t)n * sizeof(KT) + 15) & ~(int64_t)15, preg = ((int64_t)n * w + 15) & ~(int64_t)15;
  KT* sk = reinterpret_cast<KT*>(sm);
  uint8_t* sp = sm + kreg;
  KT* ok = reinterpret_cast<KT*>(sm + kreg + preg);
  uint8_t* op = sm + 2 * kreg + preg;
  // stage keys (and payload rows) -- word size chosen by alignment
  if ((((uintptr_t)keys) & 15) == 0 && ((n * sizeof(KT)) & 15) == 0) block_copy<uint4>(sk, keys, n * sizeof(KT));
  else block_copy<KT>(sk, keys, n * sizeof(KT));
  if (w) {
    if (((((uintptr_t)pay) | (uintptr_t)(n * w)) & 15) == 0) block_copy<uint4>(sp, pay, n * w);
    else if (((((uintptr_t)pay) | (uintptr_t)w) & 3) == 0) block_copy<uint32_t>(sp, pay, n * w);
    else block_copy<uint8_t>(sp, pay, n * w);
  }
  __syncthreads();
  merge_spans_to_tile<KT>(sk, la, sk + la, lb, sp, sp + (int64_t)la * w, w, ok, op);
  __syncthreads();
  tile_out<KT>(keys, pay, ok, op, n, w);
}

// ---- cluster merge: both runs spread over the shared memory of a thread-block
// cluster (up to 16 CTAs, ~1.7 MB), read across CTAs through distributed shared
// memory.  CTA k stages records [k*chunk, (k+1)*chunk) of A|B (chunk a power of
// two: a record's CTA is a shift away); after a cluster barrier two threads
// find the merge-path splits of the CTA's output range [k*chunk, (k+1)*chunk)
// over the cluster, the CTA copies its A and B windows in (consecutive threads
// read consecutive remote records), a second cluster barrier releases the
// staging, and the CTA merges the windows in local shared memory straight into
// the caller's arrays (everything was read before anything is written).
namespace cg = cooperative_groups;

// distributed shared memory: this CTA's shared address -> the same offset in CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
template <typename KT>
__device__ __forceinline__ KT ld_dsmem(uint32_t a) {
  if constexpr (sizeof(KT) == 4) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return (KT)(int32_t)v;
  } else {
    unsigned long long v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return (KT)(long long)v;
  }
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint8_t ld_dsmem_u8(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared::cluster.u8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return (uint8_t)v;
}

// record x of A|B: key / payload-row addresses in the cluster's shared memory
template <typename KT>
struct ClusterRuns {
  uint32_t sk, sp;  // this CTA's key / payload staging (shared addresses)
  int lchunk;
  __device__ __forceinline__ KT k(int x) const {
    return ld_dsmem<KT>(dsmem_addr(sk + (uint32_t)(x & ((1 << lchunk) - 1)) * (uint32_t)sizeof(KT), (uint32_t)(x >> lchunk)));
  }
  __device__ __forceinline__ uint32_t row(int x, int64_t w) const {
    return dsmem_addr(sp + (uint32_t)((int64_t)(x & ((1 << lchunk) - 1)) * w), (uint32_t)(x >> lchunk));
  }
};

template <typename KT>
__global__ void __launch_bounds__(kSmallThreads) k_merge_cluster(KT* keys, uint8_t* pay, int64_t w, int la, int lb,
                                                                 int lchunk) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int s_split[2];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int n = la + lb, chunk = 1 << lchunk;
  const int x0 = min(n, rank * chunk), x1 = min(n, x0 + chunk);
  const int64_t kreg = ((int64_t)chunk * sizeof(KT) + 15) & ~(int64_t)15, preg = ((int64_t)chunk * w + 15) & ~(int64_t)15;
  KT* sk = reinterpret_cast<KT*>(sm);  // staged records [x0, x1) of A|B
  uint8_t* sp = sm + kreg;
  KT* wk = reinterpret_cast<KT*>(sm + kreg + preg);  // this CTA's A window then B window
  uint8_t* wp = sm + 2 * kreg + preg;
  if (x1 > x0) {
    const int64_t kb = (int64_t)(x1 - x0) * sizeof(KT);
    if ((((uintptr_t)(keys + x0)) & 15) == 0 && (kb & 15) == 0) block_copy<uint4>(sk, keys + x0, kb);
    else block_copy<KT>(sk, keys + x0, kb);
    if (w) {
      const int64_t pb = (int64_t)(x1 - x0) * w;
      const uint8_t* src = pay + (int64_t)x0 * w;
      if (((((uintptr_t)src) | (uintptr_t)pb) & 15) == 0) block_copy<uint4>(sp, src, pb);
      else if (((((uintptr_t)src) | (uintptr_t)pb) & 3) == 0) block_copy<uint32_t>(sp, src, pb);
      else block_copy<uint8_t>(sp, src, pb);
    }
  }
  ClusterRuns<KT> R;
  R.lchunk = lchunk;
  R.sk = (uint32_t)__cvta_generic_to_shared(sk);
  R.sp = (uint32_t)__cvta_generic_to_shared(sp);
  cluster.sync();  // every CTA's records are staged
  // this CTA's output range [x0, x1): its A and B windows (merge-path splits over the cluster)
  if (threadIdx.x < 2) {
    const int d = threadIdx.x ? x1 : x0;
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (R.k(mid) <= R.k(la + d - 1 - mid)) lo = mid + 1;
      else hi = mid;
    }
    s_split[threadIdx.x] = lo;
  }
  __syncthreads();
  const int a0 = s_split[0], a1 = s_split[1], b0 = x0 - a0, b1 = x1 - a1;
  const int alpha = a1 - a0, beta = b1 - b0;
  // copy both windows in from distributed shared memory (consecutive threads, consecutive records)
  for (int t = threadIdx.x; t < alpha + beta; t += blockDim.x) wk[t] = R.k(t < alpha ? a0 + t : la + b0 + (t - alpha));
  if (w) {
    const bool w4 = ((uintptr_t)w & 3) == 0;
    const int64_t words = w4 ? w >> 2 : w;
    for (int64_t t = threadIdx.x; t < (int64_t)(alpha + beta) * words; t += blockDim.x) {
      const int r = (int)(t / words);
      const int64_t c = t - (int64_t)r * words;
      const uint32_t src = R.row(r < alpha ? a0 + r : la + b0 + (r - alpha), w);
      if (w4) reinterpret_cast<uint32_t*>(wp)[t] = ld_dsmem_u32(src + (uint32_t)(c * 4));
      else wp[t] = ld_dsmem_u8(src + (uint32_t)c);
    }
  }
  cluster.sync();  // every window is copied: the staging may go away
  // merge the windows into this CTA's output tile, then write it back coalesced
  KT* ok = reinterpret_cast<KT*>(sm + 2 * (kreg + preg));
  uint8_t* op = sm + 3 * kreg + 2 * preg;
  merge_spans_to_tile<KT>(wk, alpha, wk + alpha, beta, wp, wp + (int64_t)alpha * w, w, ok, op);
  __syncthreads();
  tile_out<KT>(keys + x0, w ? pay + (int64_t)x0 * w : pay, ok, op, x1 - x0, w);
}

// ---- grid merge: up to ~14 MB in one cooperative launch, no staging buffer ----
// CTA c (one per SM) owns the output range [c R, (c + 1) R): two warps find its
// stable merge-path splits over the whole job (33-ary ballot searches), the CTA
// loads its A and B pieces into shared memory (each at its source's 16-byte
// phase, so the bulk of the copy is 16-byte words), merges them into a shared
// output tile, and after one grid-wide barrier -- every CTA has read its inputs --
// stores the tile in place (TMA bulk copies both ways, tiles at the source /
// destination 16-byte phase).  One read and one write per record and a single
// launch, where the staged path takes a plan kernel, a copy-mode merge into a
// staging buffer and a copy back (2^21 records: 34 us; here 19 us).
// TMA staging of a byte range into shared memory at the source's 16-byte phase:
// the 16-byte-aligned body by one bulk copy (thread 0, completing on `bar`), the
// <= 15-byte head and tail by threads; returns the body bytes (for expect_tx).
__device__ __forceinline__ uint32_t g2s_tma(uint8_t* dst, const uint8_t* src, int64_t bytes, uint64_t* bar) {
  const int64_t head = min(bytes, (int64_t)((16 - ((uintptr_t)src & 15)) & 15));
  const int64_t body = (bytes - head) & ~(int64_t)15;
  if (threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
  const int64_t t0 = head + body;
  if (t0 + threadIdx.x < bytes) dst[t0 + threadIdx.x] = src[t0 + threadIdx.x];
  if (threadIdx.x == 0 && body) bulk_g2s(dst + head, src + head, (uint32_t)body, bar);
  return (uint32_t)body;
}
__device__ __forceinline__ uint32_t body_bytes(const uint8_t* src, int64_t bytes) {
  const int64_t head = min(bytes, (int64_t)((16 - ((uintptr_t)src & 15)) & 15));
  return (uint32_t)((bytes - head) & ~(int64_t)15);
}
// shared -> global at the same 16-byte phase: the body by one bulk store (thread 0;
// committed, waited for by the caller), head and tail by threads
__device__ __forceinline__ void s2g_tma(uint8_t* dst, const uint8_t* src, int64_t bytes) {
  const int64_t head = min(bytes, (int64_t)((16 - ((uintptr_t)dst & 15)) & 15));
  const int64_t body = (bytes - head) & ~(int64_t)15;
  if (threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
  const int64_t t0 = head + body;
  if (t0 + threadIdx.x < bytes) dst[t0 + threadIdx.x] = src[t0 + threadIdx.x];
  if (threadIdx.x == 0 && body) bulk_s2g(dst + head, src + head, (uint32_t)body);
}

template <typename KT>
__global__ void __launch_bounds__(kSmallThreads, 1) k_merge_grid(KT* keys, uint8_t* pay, int64_t w, int64_t la,
                                                                 int64_t lb, int64_t R) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int64_t s_split[2];
  __shared__ __align__(8) uint64_t bar;
  cg::grid_group grid = cg::this_grid();
  // already in order (srecpar.py:56-57): nothing moves (every CTA reads the same two
  // keys and leaves before the grid barrier, so no CTA waits there alone)
  if (keys[la - 1] <= keys[la]) return;
  const int64_t n = la + lb;
  const int64_t x0 = min(n, (int64_t)blockIdx.x * R), x1 = min(n, x0 + R);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) {
    const int64_t a = merge_path_warp<KT>(keys, la, keys + la, lb, warp ? x1 : x0, lane);
    if (lane == 0) s_split[warp] = a;
  }
  if (threadIdx.x == 64) mbar_init(&bar, 1);
  __syncthreads();
  const int64_t a0 = s_split[0], a1 = s_split[1], b0 = x0 - a0, b1 = x1 - a1;
  const int alpha = (int)(a1 - a0), beta = (int)(b1 - b0), no = (int)(x1 - x0);
  // shared layout: A keys, B keys (each at its source's 16-byte phase), A rows, B
  // rows (same), output keys and rows (at the destination's phase): TMA bulk copies
  const uint8_t* gka = reinterpret_cast<const uint8_t*>(keys + a0);
  const uint8_t* gkb = reinterpret_cast<const uint8_t*>(keys + la + b0);
  auto up16 = [](const uint8_t* p) { return reinterpret_cast<uint8_t*>(((uintptr_t)p + 15) & ~(uintptr_t)15); };
  uint8_t* ska = sm + ((uintptr_t)gka & 15);
  uint8_t* skb = up16(ska + (int64_t)alpha * sizeof(KT)) + ((uintptr_t)gkb & 15);
  uint8_t* end = skb + (int64_t)beta * sizeof(KT);
  const uint8_t* gpa = w ? pay + a0 * w : nullptr;
  const uint8_t* gpb = w ? pay + (la + b0) * w : nullptr;
  uint8_t *spa = end, *spb = end;
  if (w) {
    spa = up16(end) + ((uintptr_t)gpa & 15);
    spb = up16(spa + (int64_t)alpha * w) + ((uintptr_t)gpb & 15);
    end = spb + (int64_t)beta * w;
  }
  uint8_t* dk = reinterpret_cast<uint8_t*>(keys + x0);
  uint8_t* dp = w ? pay + x0 * w : nullptr;
  KT* ok = reinterpret_cast<KT*>(up16(end) + ((uintptr_t)dk & 15));
  uint8_t* op = w ? up16(reinterpret_cast<uint8_t*>(ok + no)) + ((uintptr_t)dp & 15) : nullptr;
  if (threadIdx.x == 0) {
    uint32_t tx = body_bytes(gka, (int64_t)alpha * sizeof(KT)) + body_bytes(gkb, (int64_t)beta * sizeof(KT));
    if (w) tx += body_bytes(gpa, (int64_t)alpha * w) + body_bytes(gpb, (int64_t)beta * w);
    mbar_expect_tx(&bar, tx);
  }
  g2s_tma(ska, gka, (int64_t)alpha * sizeof(KT), &bar);
  g2s_tma(skb, gkb, (int64_t)beta * sizeof(KT), &bar);
  if (w) {
    g2s_tma(spa, gpa, (int64_t)alpha * w, &bar);
    g2s_tma(spb, gpb, (int64_t)beta * w, &bar);
  }
  if (threadIdx.x == 0) mbar_arrive(&bar);
  while (!mbar_try_wait(&bar, 0)) {
  }
  __syncthreads();  // (head / tail bytes by threads)
  merge_spans_to_tile<KT>(reinterpret_cast<const KT*>(ska), alpha, reinterpret_cast<const KT*>(skb), beta, spa, spb,
                          w, ok, op);
  __syncthreads();
  grid.sync();  // every CTA has read its pieces: the output ranges may be overwritten
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (generic writes of the tile -> the bulk store)
  __syncthreads();
  s2g_tma(dk, reinterpret_cast<const uint8_t*>(ok), (int64_t)no * sizeof(KT));
  if (w) s2g_tma(dp, op, (int64_t)no * w);
  if (threadIdx.x == 0) {
    bulk_commit();
    bulk_wait_all();
  }
}

}  // namespace

int64_t small_merge_smem(int ks, int64_t w, int64_t n) { return 2 * (((n * ks + 15) & ~15ll) + ((n * w + 15) & ~15ll)); }

template <typename KT>
cudaError_t launch_merge_small(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                               cudaStream_t st) {
  const int64_t n = e - s;
  const size_t smem = (size_t)small_merge_smem(sizeof(KT), w, n);
  // function attributes belong to each device's context: set once per device
  static std::atomic<uint64_t> attrs_set{0};
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return ce;
  const uint64_t bit = 1ull << (dev & 63);
  if (dev >= 64 || !(attrs_set.load(std::memory_order_acquire) & bit)) {
    ce = cudaFuncSetAttribute(k_merge_small<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (ce != cudaSuccess) return ce;
    attrs_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  k_merge_small<KT><<<1, kSmallThreads, smem, st>>>(static_cast<KT*>(keys) + s,
                                                    w ? static_cast<uint8_t*>(payload) + s * w : nullptr, w,
                                                    (int)(m - s), (int)(e - m));
  count_launches(1);
  return cudaGetLastError();
}
template cudaError_t launch_merge_small<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);
template cudaError_t launch_merge_small<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);

// Cluster size and chunk for n records of (ks + w) bytes: the smallest
// power-of-two cluster (2..16) whose CTAs hold a power-of-two chunk each
// within kClusterSmem; 0 when n does not fit.
int cluster_merge_plan(int ks, int64_t w, int64_t n, int* lchunk) {
  for (int C = 2; C <= 16; C *= 2) {
    int lc = 0;
    while ((int64_t)C << lc < n) ++lc;
    const int64_t chunk = (int64_t)1 << lc;
    if (3 * (((chunk * ks + 15) & ~15ll) + ((chunk * w + 15) & ~15ll)) <= kClusterSmem) {
      *lchunk = lc;
      return C;
    }
  }
  return 0;
}

template <typename KT>
cudaError_t launch_merge_cluster(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e, int C,
                                 int lchunk, cudaStream_t st) {
  const int64_t chunk = (int64_t)1 << lchunk;
  const size_t smem = (size_t)(3 * (((chunk * (int64_t)sizeof(KT) + 15) & ~15ll) + ((chunk * w + 15) & ~15ll)));
  // function attributes belong to each device's context: set once per device
  // (each call costs host time on the launch path)
  static std::atomic<uint64_t> attrs_set{0};
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return ce;
  const uint64_t bit = 1ull << (dev & 63);
  if (dev >= 64 || !(attrs_set.load(std::memory_order_acquire) & bit)) {
    ce = cudaFuncSetAttribute(k_merge_cluster<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kClusterSmem));
    if (ce == cudaSuccess) ce = cudaFuncSetAttribute(k_merge_cluster<KT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (ce != cudaSuccess) return ce;
    attrs_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ce = cudaLaunchKernelEx(&cfg, k_merge_cluster<KT>, static_cast<KT*>(keys) + s,
                          w ? static_cast<uint8_t*>(payload) + s * w : static_cast<uint8_t*>(nullptr), w,
                          (int)(m - s), (int)(e - m), lchunk);
  count_launches(1);
  return ce != cudaSuccess ? ce : cudaGetLastError();
}
template cudaError_t launch_merge_cluster<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, int,
                                                   cudaStream_t);
template cudaError_t launch_merge_cluster<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, int,
                                                   cudaStream_t);

// Grid merge plan: the output range per CTA (R records, every SM busy once the job
// has >= 1024 records per SM) and its shared memory; 0 when the job does not fit
// one resident CTA per SM (tile bytes kGridTileBytes per CTA, inputs + output = 2x).
int64_t grid_merge_plan(int ks, int64_t w, int64_t n, int num_sms, int* ctas, size_t* smem) {
  const int64_t rec = ks + w;
  const int64_t rmax = kGridTileBytes / rec;
  if (n <= 0 || rmax < 64 || n > rmax * num_sms) return 0;
  const int64_t g = std::min<int64_t>(num_sms, std::max<int64_t>(1, (n + 1023) / 1024));
  const int64_t R = (n + g - 1) / g;
  if (R > rmax) return 0;
  *ctas = (int)((n + R - 1) / R);
  *smem = (size_t)(2 * R * rec + 256);  // (six regions, each up to 30 bytes of alignment and phase)
  return R;
}

template <typename KT>
cudaError_t launch_merge_grid(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e, int ctas,
                              int64_t R, size_t smem, cudaStream_t st) {
  cudaError_t ce = ensure_smem_attr((const void*)k_merge_grid<KT>, smem);
  if (ce != cudaSuccess) return ce;
  KT* k = static_cast<KT*>(keys) + s;
  uint8_t* p = w ? static_cast<uint8_t*>(payload) + s * w : nullptr;
  int64_t la = m - s, lb = e - m;
  void* args[] = {(void*)&k, (void*)&p, (void*)&w, (void*)&la, (void*)&lb, (void*)&R};
  ce = cudaLaunchCooperativeKernel((const void*)k_merge_grid<KT>, dim3(ctas), dim3(kSmallThreads), args, smem, st);
  count_launches(1);
  return ce != cudaSuccess ? ce : cudaGetLastError();
}
template cudaError_t launch_merge_grid<int32_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, int64_t,
                                                size_t, cudaStream_t);
template cudaError_t launch_merge_grid<int64_t>(void*, void*, int64_t, int64_t, int64_t, int64_t, int, int64_t,
                                                size_t, cudaStream_t);

}  // namespace pm
