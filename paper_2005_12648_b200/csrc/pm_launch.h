// pm_launch.h -- host launchers exported by pm_engine.cu / pm_plan.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pm_engine.cuh"

namespace pm {
// every kernel launch of the library bumps this process-wide count (pm_launch_count)
void count_launches(int n);
template <typename KT> cudaError_t launch_plan(const EngineParams& P, int grid, cudaStream_t st);
template <typename KT> cudaError_t launch_engine(const EngineParams& P, int grid, int block, size_t smem, cudaStream_t st);
template <typename KT> cudaError_t engine_occupancy(int block, size_t smem, int* blocks_per_sm);
template <typename KT> cudaError_t buffered_occupancy(size_t smem, int* blocks_per_sm);
// scheduled in-place merge (pm_flow.cu): plan kernels + pool copy + streaming merge
#ifndef PM_FLOW_STAGES
#define PM_FLOW_STAGES 2  // k_flow input stages (regions whose loads are in flight + the one merging)
#endif
#ifndef PM_FLOW_THREADS
#define PM_FLOW_THREADS 256  // k_flow CTA: one control warp + merge warps
#endif
#ifndef PM_FLOW_OUT
#define PM_FLOW_OUT 1  // k_flow output tiles (1: the leader waits for each store to read its tile)
#endif
#ifndef PM_FLOW_TILE
#define PM_FLOW_TILE (32 * 1024)  // k_flow tile bytes (keys + payload): regions of up to 8192 records
#endif
constexpr int kFlowStages = PM_FLOW_STAGES;
constexpr int kFlowOut = PM_FLOW_OUT;
constexpr int kFlowThreads = PM_FLOW_THREADS;
template <typename KT>
cudaError_t flow_occupancy(size_t smem, size_t attr_smem, int* blocks_per_sm, int* plan_blocks_per_sm);
template <typename KT>
cudaError_t launch_flow(const FlowParams& F, int grid, size_t smem, int num_sms, int plan_bps, cudaStream_t st,
                        cudaEvent_t ev, cudaEvent_t ev_merge, cudaEvent_t ev_fork);
template <typename KT>
cudaError_t launch_rotate(void* keys, void* payload, int64_t w, int64_t lo, int64_t la, int64_t lb, int num_sms,
                          cudaStream_t st, const int32_t* gate = nullptr);  // gate: run only if *gate != 0
// A|B -> B|A on [lo, lo + la + lb) by Gries-Mills block swaps, three reversals for the remainder (gated likewise)
template <typename KT>
cudaError_t launch_block_exchange(void* keys, void* payload, int64_t w, int64_t lo, int64_t la, int64_t lb,
                                  int num_sms, cudaStream_t st, const int32_t* gate = nullptr);
// equal blocks: [lo, lo + len) <-> [lo + len, lo + 2 len), keys and payload planes (gated likewise)
cudaError_t launch_swap_blocks(void* keys, int ks, void* payload, int64_t w, int64_t lo, int64_t len, int num_sms,
                               cudaStream_t st, const int32_t* gate = nullptr);
// staged path: a copy that runs only if the gate (A[m-1] > B[0], set by k_plan) is set
cudaError_t launch_copy_gated(void* dst, const void* src, int64_t n, const int32_t* gate, int num_sms, cudaStream_t st);
template <typename KT> cudaError_t launch_merge_copy(const EngineParams& P, int grid, size_t smem, cudaStream_t st);
template <typename KT>
cudaError_t launch_buffered(const EngineParams& P, int32_t buf_a, int grid, size_t smem, cudaStream_t st);
template <typename KT>
cudaError_t launch_find_median(const void* a, const void* b, int64_t la, int64_t lb, int64_t* out, cudaStream_t st);
template <typename KT>
cudaError_t launch_find_splits(const void* a, const void* b, int64_t la, int64_t lb, const int64_t* diags, int64_t nd,
                               int64_t* out_a, int grid, cudaStream_t st);
template <typename KT>
cudaError_t launch_plan_intervals(const void* keys, int64_t s, int64_t m, int64_t e, int32_t levels, int64_t* nodes,
                                  cudaStream_t st);
// wide records (pm_wide.cu): row index fill, out-of-place row gather, in-place cycle permutation
cudaError_t launch_iota(int32_t* idx, int64_t n, int num_sms, cudaStream_t st);
cudaError_t launch_gather_rows(uint8_t* out, const uint8_t* a, const uint8_t* b, const int32_t* idx, int64_t n,
                               int64_t la, int64_t w, int num_sms, cudaStream_t st);
cudaError_t launch_cycle_permute(uint8_t* pay, int64_t w, const int32_t* idx, int64_t n, int32_t G, int2* dbl0,
                                 int2* dbl1, int2* heads, int32_t* ctl, uint8_t* unres, int4* segs, int32_t* xpos,
                                 int32_t xcap, int32_t Lmax, uint8_t* save, int num_sms, cudaStream_t st);
// one-pass overlapping move of a byte plane by D bytes (pm_rotate.cu); flags: one int32 per 32 KB tile
cudaError_t launch_slide(void* plane, int64_t S0, int64_t L, int64_t D, bool right, int32_t* flags, int32_t* ticket,
                         int32_t* err, int num_sms, cudaStream_t st);
// block-distributed searches through a peer-pointer table (pm_peers.cu)
template <typename KT>
cudaError_t launch_peer_queries(const void* const* tab, int64_t block, int64_t la, int64_t lb, const int64_t* q, int nq,
                                int64_t* out, cudaStream_t st);
// small jobs (pm_small.cu): one CTA, both runs staged in shared memory
int64_t small_merge_smem(int ks, int64_t w, int64_t n);
template <typename KT>
cudaError_t launch_merge_small(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                               cudaStream_t st);
// cluster size (0: does not fit) and log2 chunk of the cluster merge; its launcher
int cluster_merge_plan(int ks, int64_t w, int64_t n, int* lchunk);
// grid merge (one cooperative launch, one CTA per SM, tiles in shared memory): R
// records per CTA, 0 when the job does not fit
int64_t grid_merge_plan(int ks, int64_t w, int64_t n, int num_sms, int* ctas, size_t* smem);
template <typename KT>
cudaError_t launch_merge_grid(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e, int ctas,
                              int64_t R, size_t smem, cudaStream_t st);
constexpr int64_t kGridTileBytes = 113 * 1024;  // records per CTA tile (in + out: 2x in shared memory, + 256 B of alignment <= 227 KB); 148 tiles hold 2^21 int32 records per side
template <typename KT>
cudaError_t launch_merge_cluster(void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e, int C,
                                 int lchunk, cudaStream_t st);
}  // namespace pm
