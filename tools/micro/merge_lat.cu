// Micro-benchmark: cycles of the engine's shared-memory tile merge (merge_tile's
// keys-only path) for an 8192-record region, 128 merging threads per CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <typename KT>
__device__ __forceinline__ void merge_keys(const KT* As, const KT* Bs, int al, int bl, int no, KT* ko, int gt, int GT) {
  int E = (no + GT - 1) / GT;
  E |= 1;
  int o = min(gt * E, no);
  const int oe = min(o + E, no);
  int lo = o > bl ? o - bl : 0, hi = o < al ? o : al;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (As[mid] <= Bs[o - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
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
__global__ void k(int reps, int GTw, unsigned long long* cyc) {
  extern __shared__ __align__(16) uint8_t dyn[];
  int* in = reinterpret_cast<int*>(dyn);
  int* out = in + 8192 + 16;
  const int M = 8192, al = 4096, bl = 4096;
  for (int x = threadIdx.x; x < M; x += blockDim.x) {
    // two sorted runs of pseudo-random increments
    in[x] = (x < al ? x : x - al) * 4 + ((x * 2654435761u) >> 30);
  }
  __syncthreads();
  const int GT = GTw * 32;
  if ((int)threadIdx.x >= GT) return;
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    long long c0 = clock64();
    merge_keys<int>(in, in + al, al, bl, M, out, threadIdx.x, GT);
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    tot += clock64() - c0;
  }
  if (threadIdx.x == 0) atomicAdd(cyc, tot);
}
int main() {
  unsigned long long* cyc; cudaMalloc(&cyc, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  int cfgs[][2] = {{1, 4}, {148, 4}, {444, 4}, {444, 8}, {148, 8}, {148, 16}};
  for (auto& c : cfgs) {
    cudaMemset(cyc, 0, 8);
    k<<<c[0], 32 * c[1], 70000>>>(64, c[1], cyc);
    cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ctas=%d merge warps=%d: %.0f cycles per 8192-record tile\n", c[0], c[1], (double)h / c[0] / 64);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
