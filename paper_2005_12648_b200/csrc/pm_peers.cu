// pm_peers.cu -- searches over a block-distributed A|B read through a peer-pointer
// table (multi-GPU merge with the exchange fused into the merge's loads).
//
// The global array X = A|B of N = world * block records lives in `world`
// equal blocks, block k on GPU k; every GPU maps the others' blocks into its
// address space (CUDA IPC + NVLink peer access).  Rank r's output is the merged
// range [r*block, (r+1)*block).  The queries here (one thread each, a few dozen
// dependent peer loads) give the stable merge-path split at a diagonal and the
// output position of every block boundary inside rank r's A and B pieces; the
// host cuts r's range there, so every sub-merge reads one contiguous A piece and
// one contiguous B piece, each inside a single (possibly remote) block, and the
// copy-mode merge pipeline streams them over NVLink straight into r's output.
#include <cuda_runtime.h>

#include <cstdint>

#include "pm_launch.h"

namespace pm {

namespace {

template <typename KT>
struct Dist {
  const KT* const* tab;
  int64_t block, la, lb;
  __device__ __forceinline__ KT x(int64_t g) const { return tab[g / block][g % block]; }
  __device__ __forceinline__ KT a(int64_t i) const { return x(i); }
  __device__ __forceinline__ KT b(int64_t j) const { return x(la + j); }
};

// q = {kind, arg}: kind 0: stable split (# A among the first arg outputs, A wins
// ties); kind 1: # B < A[arg]; kind 2: # A <= B[arg].
template <typename KT>
__global__ void k_peer_queries(const KT* const* tab, int64_t block, int64_t la, int64_t lb, const int64_t* q, int nq,
                               int64_t* out) {
  const Dist<KT> D{tab, block, la, lb};
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nq; k += gridDim.x * blockDim.x) {
    const int64_t kind = q[2 * k], arg = q[2 * k + 1];
    int64_t lo, hi;
    if (kind == 0) {
      lo = arg > lb ? arg - lb : 0;
      hi = arg < la ? arg : la;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (D.a(mid) <= D.b(arg - 1 - mid)) lo = mid + 1;
        else hi = mid;
      }
    } else if (kind == 1) {  // lower bound of A[arg] in B
      const KT v = D.a(arg);
      lo = 0;
      hi = lb;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (D.b(mid) < v) lo = mid + 1;
        else hi = mid;
      }
    } else {  // upper bound of B[arg] in A
      const KT v = D.b(arg);
      lo = 0;
      hi = la;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (D.a(mid) <= v) lo = mid + 1;
        else hi = mid;
      }
    }
    out[k] = lo;
  }
}

}  // namespace

template <typename KT>
cudaError_t launch_peer_queries(const void* const* tab, int64_t block, int64_t la, int64_t lb, const int64_t* q, int nq,
                                int64_t* out, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  k_peer_queries<KT><<<(nq + 63) / 64, 64, 0, st>>>(reinterpret_cast<const KT* const*>(tab), block, la, lb, q, nq, out);
  count_launches(1);
  return cudaGetLastError();
}
template cudaError_t launch_peer_queries<int32_t>(const void* const*, int64_t, int64_t, int64_t, const int64_t*, int,
                                                  int64_t*, cudaStream_t);
template cudaError_t launch_peer_queries<int64_t>(const void* const*, int64_t, int64_t, int64_t, const int64_t*, int,
                                                  int64_t*, cudaStream_t);

}  // namespace pm
