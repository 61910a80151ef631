// Micro-benchmark: keys-only tile merge by 16-record chunks (merge-path split,
// bitonic sequence gathered into registers, bitonic merging network, rotated
// 16-byte stores) against the serial per-thread merge.
#include <cstdio>
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>
template <typename KT> __device__ __forceinline__ KT kmax();
template <> __device__ __forceinline__ int kmax<int>() { return INT_MAX; }
__device__ __forceinline__ int mp_search(const int* As, const int* Bs, int al, int bl, int o) {
  int lo = o > bl ? o - bl : 0, hi = o < al ? o : al;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (As[mid] <= Bs[o - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
template <typename KT>
__device__ __forceinline__ void cas(KT& a, KT& b) {
  const KT x = min(a, b), y = max(a, b);
  a = x;
  b = y;
}
// chunk c: outputs [16c, 16c+16) of the tile
template <typename KT>
__device__ __forceinline__ void merge_chunks(const KT* As, const KT* Bs, int al, int bl, int no, KT* ko, int gt, int GT) {
  const int nch = (no + 15) >> 4;
  const int lane = threadIdx.x & 31;
  for (int c = gt; c < nch; c += GT) {
    const int o = c << 4, oe = min(o + 16, no);
    const int i0 = mp_search(As, Bs, al, bl, o), i1 = mp_search(As, Bs, al, bl, oe);
    const int na = i1 - i0, j0 = o - i0, j1 = oe - i1;
    KT v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      // A ascending, then padding (max), then B descending: a bitonic sequence
      const int kb = 15 - k;  // position from the end
      const bool isA = k < na, isB = kb < (j1 - j0);
      const KT* p = isA ? As + i0 + k : Bs + j0 + kb;
      v[k] = (isA | isB) ? *p : kmax<KT>();
    }
#pragma unroll
    for (int d = 8; d >= 1; d >>= 1) {
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if ((k & d) == 0) cas(v[k], v[k + d]);
    }
    if (oe - o == 16 && (((uintptr_t)(ko + o)) & 15) == 0) {
      // four 16-byte stores, rotated per lane pair so a quarter warp hits 8 distinct granules
      uint4 q[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) q[s] = make_uint4(v[4 * s], v[4 * s + 1], v[4 * s + 2], v[4 * s + 3]);
      uint4* dst = reinterpret_cast<uint4*>(ko + o);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int pc = (s + (lane >> 1)) & 3;
        const uint4 val = pc == 0 ? q[0] : pc == 1 ? q[1] : pc == 2 ? q[2] : q[3];
        dst[pc] = val;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (o + k < oe) ko[o + k] = v[k];
    }
  }
}
template <typename KT, int C>
__device__ __forceinline__ void merge_chunks_shfl(const KT* As, const KT* Bs, int al, int bl, int no, KT* ko, int gt, int GT) {
  const int lane = gt & 31, wid = gt >> 5, NW = GT >> 5;
  const int nch = (no + C - 1) / C;
  for (int c0 = wid * 31; c0 < nch; c0 += NW * 31) {
    const int c = c0 + lane;  // lane 31 only supplies the end split of lane 30
    const int o = min(c * C, no);
    const int i0 = mp_search(As, Bs, al, bl, o);
    const int i1 = __shfl_down_sync(0xffffffffu, i0, 1);
    if (lane == 31 || c >= nch) continue;
    const int oe = min(o + C, no);
    const int na = i1 - i0, nb = (oe - o) - na, j0 = o - i0;
    KT v[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int kb = C - 1 - k;
      const bool isA = k < na, isB = kb < nb;
      const KT* p = isA ? As + i0 + k : Bs + j0 + kb;
      v[k] = (isA | isB) ? *p : kmax<KT>();
    }
#pragma unroll
    for (int d = C / 2; d >= 1; d >>= 1) {
#pragma unroll
      for (int k = 0; k < C; ++k)
        if ((k & d) == 0) cas(v[k], v[k + d]);
    }
    if (oe - o == C && (((uintptr_t)(ko + o)) & 15) == 0) {
      uint4* dst = reinterpret_cast<uint4*>(ko + o);
#pragma unroll
      for (int s = 0; s < C / 4; ++s) {
        const int pc = (s + (lane >> 1)) & (C / 4 - 1);
        uint4 val = make_uint4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int q = 1; q < C / 4; ++q)
          if (pc == q) val = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        dst[pc] = val;
      }
    } else {
#pragma unroll
      for (int k = 0; k < C; ++k)
        if (o + k < oe) ko[o + k] = v[k];
    }
  }
}
template <typename KT>
__device__ __forceinline__ void merge_serial(const KT* As, const KT* Bs, int al, int bl, int no, KT* ko, int gt, int GT) {
  int E = (no + GT - 1) / GT;
  E |= 1;
  int o = min(gt * E, no);
  const int oe = min(o + E, no);
  int lo = mp_search(As, Bs, al, bl, o);
  const int amax = al > 0 ? al - 1 : 0, bmax = bl > 0 ? bl - 1 : 0;
  int i = lo, jb = o - lo;
  KT va = As[min(i, amax)], vb = Bs[min(jb, bmax)];
#pragma unroll 4
  for (; o < oe; ++o) {
    const bool takeA = (jb >= bl) | ((i < al) & (va <= vb));
    ko[o] = takeA ? va : vb;
    i += takeA;
    jb += !takeA;
    const KT v = *(takeA ? As + min(i, amax) : Bs + min(jb, bmax));
    va = takeA ? v : va;
    vb = takeA ? vb : v;
  }
}
__global__ void k(int variant, int reps, int GTw, int M, int al, unsigned long long* cyc, int* bad) {
  extern __shared__ __align__(16) uint8_t dyn[];
  int* in = reinterpret_cast<int*>(dyn);
  int* out = in + M + 16;
  const int bl = M - al;
  for (int x = threadIdx.x; x < M; x += blockDim.x) in[x] = (x < al ? x : x - al) * 4 + ((x * 2654435761u) >> 30);
  __syncthreads();
  const int GT = GTw * 32;
  if ((int)threadIdx.x >= GT) return;
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    long long c0 = clock64();
    if (variant == 0) merge_serial<int>(in, in + al, al, bl, M, out, threadIdx.x, GT);
    else if (variant == 1) merge_chunks<int>(in, in + al, al, bl, M, out, threadIdx.x, GT);
    else if (variant == 2) merge_chunks_shfl<int, 16>(in, in + al, al, bl, M, out, threadIdx.x, GT);
    else merge_chunks_shfl<int, 8>(in, in + al, al, bl, M, out, threadIdx.x, GT);
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    tot += clock64() - c0;
  }
  if (threadIdx.x == 0) atomicAdd(cyc, tot);
  if (blockIdx.x == 0) {
    for (int x = threadIdx.x; x + 1 < M; x += GT)
      if (out[x] > out[x + 1]) atomicAdd(bad, 1);
    // multiset check: sum
    long long sa = 0, sb = 0;
    for (int x = threadIdx.x; x < M; x += GT) { sa += in[x]; sb += out[x]; }
    if (sa != sb) atomicAdd(bad, 1000);  // (per-thread partial sums differ only if elements moved across threads; report)
  }
}
int main() {
  unsigned long long* cyc; cudaMalloc(&cyc, 8);
  int* bad; cudaMalloc(&bad, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  int cfgs[][4] = {{0, 7, 4096, 2048}, {2, 7, 4096, 2048}, {3, 7, 4096, 2048}, {0, 4, 8192, 4096}, {2, 4, 8192, 4096}, {3, 4, 8192, 4096}, {2, 7, 4096, 1000}, {2, 7, 4090, 3000}, {3, 7, 4090, 3000}};
  for (auto& c : cfgs) {
    cudaMemset(cyc, 0, 8); cudaMemset(bad, 0, 4);
    k<<<444, 32 * c[1], 70000>>>(c[0], 64, c[1], c[2], c[3], cyc, bad);
    cudaDeviceSynchronize();
    unsigned long long h; int hb;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("variant %d warps=%d M=%d al=%d: %.0f cycles per tile (unsorted %d)\n", c[0], c[1], c[2], c[3],
           (double)h / 444 / 64, hb % 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
