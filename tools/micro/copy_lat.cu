// Micro-benchmark: latency of a warp-wide 8 KB global->global copy (+ fence), the
// engine's salvage move, alone and with every warp slot of the GPU copying.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void copy_warp(uint4* d4, const uint4* s4, int nvec, int lane) {
  int i = lane;
  for (; i + 224 < nvec; i += 256) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(s4 + i + 32 * k);
#pragma unroll
    for (int k = 0; k < 8; ++k) d4[i + 32 * k] = v[k];
  }
  for (; i < nvec; i += 32) d4[i] = __ldcs(s4 + i);
}
__global__ void k(uint4* buf, int64_t nunits, int reps, int warps_per_cta, unsigned long long* cyc, unsigned long long* ld_cyc) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= warps_per_cta) return;
  uint64_t x = (blockIdx.x * 131 + wid) * 0x9E3779B97F4A7C15ull;
  unsigned long long tot = 0, tl = 0;
  for (int r = 0; r < reps; ++r) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const int64_t a = (x % nunits), b = ((x >> 20) % nunits);
    long long c0 = clock64();
    copy_warp(buf + b * 512, buf + a * 512, 512, lane);
    long long c1 = clock64();
    __threadfence();
    __syncwarp();
    long long c2 = clock64();
    tot += c2 - c0;
    tl += c1 - c0;
  }
  if (lane == 0) { atomicAdd(cyc, tot); atomicAdd(ld_cyc, tl); }
}
int main() {
  const int64_t nunits = (int64_t)1 << 19;  // 4 GB of 8 KB units
  uint4* buf; cudaMalloc(&buf, nunits * 8192);
  cudaMemset(buf, 1, nunits * 8192);
  unsigned long long *cyc, *lc; cudaMalloc(&cyc, 8); cudaMalloc(&lc, 8);
  int cfgs[][3] = {{1, 1, 64}, {148, 1, 64}, {444, 4, 64}, {444, 8, 64}, {888, 8, 32}};
  for (auto& c : cfgs) {
    cudaMemset(cyc, 0, 8); cudaMemset(lc, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<c[0], 256>>>(buf, nunits, c[2], c[1], cyc, lc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h, hl; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hl, lc, 8, cudaMemcpyDeviceToHost);
    double n = (double)c[0] * c[1] * c[2];
    printf("ctas=%d warps/cta=%d: %.0f cycles/copy (loads+stores issue %.0f, fence %.0f), %.1f GB/s copied\n", c[0], c[1],
           h / n, hl / n, (h - hl) / n, n * 8192 * 2 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
