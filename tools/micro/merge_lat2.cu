// Micro-benchmark: tile merge variants (1 chain vs bidirectional 2 chains vs 4 chains).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ int mp_search(const int* As, const int* Bs, int al, int bl, int o) {
  int lo = o > bl ? o - bl : 0, hi = o < al ? o : al;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (As[mid] <= Bs[o - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// forward chain over outputs [o, oe) starting at A index i (B index o - i)
// backward chain over outputs [ob, oe2) ending at A index ie (B index oe2 - ie)
__device__ __forceinline__ void merge_bidir(const int* As, const int* Bs, int al, int bl, int o, int oe, int i, int ie, int* ko) {
  // forward: outputs o .. mid-1 ; backward: outputs oe-1 down to mid
  const int n = oe - o, mid = o + (n + 1) / 2;
  const int amax = al > 0 ? al - 1 : 0, bmax = bl > 0 ? bl - 1 : 0;
  int fi = i, fj = o - i;
  int va = As[min(fi, amax)], vb = Bs[min(fj, bmax)];
  int bi = ie, bj = oe - ie;  // backward: next candidates are A[bi-1], B[bj-1]
  int wa = As[max(bi - 1, 0)], wb = Bs[max(bj - 1, 0)];
  int of = o, ob = oe - 1;
  const int nb = oe - mid, nf = mid - o;
#pragma unroll 2
  for (int s = 0; s < nf; ++s) {
    // forward step
    const bool takeA = (fj >= bl) | ((fi < al) & (va <= vb));
    ko[of++] = takeA ? va : vb;
    fi += takeA;
    fj += !takeA;
    const int v = *(takeA ? As + min(fi, amax) : Bs + min(fj, bmax));
    va = takeA ? v : va;
    vb = takeA ? vb : v;
    if (s < nb) {
      // backward step: the larger goes last; ties -> B last (stable)
      const bool lastA = (bj <= 0) | ((bi > 0) & (wa > wb));
      ko[ob--] = lastA ? wa : wb;
      bi -= lastA;
      bj -= !lastA;
      const int w = *(lastA ? As + max(bi - 1, 0) : Bs + max(bj - 1, 0));
      wa = lastA ? w : wa;
      wb = lastA ? wb : w;
    }
  }
}
__global__ void k(int variant, int reps, int GTw, unsigned long long* cyc, int* outcheck) {
  extern __shared__ __align__(16) uint8_t dyn[];
  int* in = reinterpret_cast<int*>(dyn);
  int* out = in + 8192 + 16;
  const int M = 8192, al = 4096, bl = 4096;
  for (int x = threadIdx.x; x < M; x += blockDim.x) in[x] = (x < al ? x : x - al) * 4 + ((x * 2654435761u) >> 30);
  __syncthreads();
  const int GT = GTw * 32;
  if ((int)threadIdx.x >= GT) return;
  const int* As = in;
  const int* Bs = in + al;
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    long long c0 = clock64();
    const int gt = threadIdx.x;
    int E = (M + GT - 1) / GT;
    E |= 1;
    const int o = min(gt * E, M), oe = min(o + E, M);
    if (variant == 1) {
      const int i = mp_search(As, Bs, al, bl, o), ie = mp_search(As, Bs, al, bl, oe);
      merge_bidir(As, Bs, al, bl, o, oe, i, ie, out);
    } else {
      const int om = o + (oe - o) / 2;
      const int i = mp_search(As, Bs, al, bl, o), im = mp_search(As, Bs, al, bl, om), ie = mp_search(As, Bs, al, bl, oe);
      merge_bidir(As, Bs, al, bl, o, om, i, im, out);
      merge_bidir(As, Bs, al, bl, om, oe, im, ie, out);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    tot += clock64() - c0;
  }
  if (threadIdx.x == 0) atomicAdd(cyc, tot);
  if (blockIdx.x == 0) {
    asm volatile("bar.sync 1, %0;" ::"r"(GT));
    for (int x = threadIdx.x; x + 1 < M; x += GT)
      if (out[x] > out[x + 1]) atomicAdd(outcheck, 1);
  }
}
int main() {
  unsigned long long* cyc; cudaMalloc(&cyc, 8);
  int* bad; cudaMalloc(&bad, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int variant = 1; variant <= 2; ++variant) {
    int cfgs[][2] = {{148, 4}, {444, 4}};
    for (auto& c : cfgs) {
      cudaMemset(cyc, 0, 8); cudaMemset(bad, 0, 4);
      k<<<c[0], 32 * c[1], 70000>>>(variant, 64, c[1], cyc, bad);
      cudaDeviceSynchronize();
      unsigned long long h; int hb;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
      printf("variant %d ctas=%d warps=%d: %.0f cycles per tile (unsorted pairs %d)\n", variant, c[0], c[1], (double)h / c[0] / 64, hb);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
