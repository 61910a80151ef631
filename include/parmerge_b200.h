/*
 * parmerge_b200.h -- C-ABI of the B200-native parallel in-place merge.
 *
 * Drop-in boundary for the reference package `parmerge`, whose native layer is
 * the numba module `_kernels` (/root/reference/pkg/src/parmerge/_kernels.py,
 * "every kernel takes the full keys/payload arrays plus integer offsets",
 * _kernels.py:3-7).  Each entry point below replaces one reference call site;
 * the replaced interface is cited beside it.  The Python mirror
 * (paper_2005_12648_b200/) binds these through ctypes exactly as the
 * reference's L2 wrappers call `_kernels`.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; `keys` / `payload` are DEVICE pointers to
 *     the base of the caller's arrays (record x at keys + x*key_bytes and
 *     payload + x*width), positions are absolute int64 record indices;
 *   - key_bytes is 4 (int32, the reference's KEY_DTYPE, records.py:9) or 8
 *     (int64, the skewed BASELINE config); payload rows are opaque bytes that
 *     travel with their key (records.py:15-22); width may be 0;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *     stream-ordered and asynchronous -- device-side failures are reported by
 *     pm_status(), host-side argument errors by the return code;
 *   - return value: 0 on success, else a PM_ERR_* code; pm_last_error() gives
 *     the thread's last message;
 *   - a context owns the persistent device workspace (split table, unit
 *     bookkeeping, bounded scratch); use one context per stream.
 */
#ifndef PARMERGE_B200_H
#define PARMERGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM_OK 0
#define PM_ERR_ARG 1         /* invalid argument (ValueError/IndexError in the reference wrappers) */
#define PM_ERR_CUDA 2        /* CUDA runtime failure */
#define PM_ERR_TIMEOUT 3     /* device wait bound exceeded (protocol fault) */
#define PM_ERR_NOSPACE 4     /* salvage space exhausted */
#define PM_ERR_INTERNAL 5
#define PM_ERR_UNSUPPORTED 6 /* record too wide for the staging buffers */

typedef struct pm_ctx pm_ctx;

/* library version (major*10000 + minor*100 + patch) */
int pm_version(void);
/* last error message of the calling thread ("" if none) */
const char *pm_last_error(void);

int pm_ctx_create(int device, pm_ctx **out);
int pm_ctx_destroy(pm_ctx *ctx);

/*
 * Stable in-place merge of the adjacent sorted runs [start, middle) and
 * [middle, end); ties keep A first, so the result equals the reference's
 * seq_merge_buffered (seqmerge.py:55-75 -> _kernels.buffered_merge,
 * _kernels.py:227-313), seq_merge_rotation (_kernels.py:201-223) and
 * merge_srecpar(threads=1) (srecpar.py:33-60).  Replaces the partition + shift
 * + leaf-merge pipeline of merge_srecpar / merge_soptmov (srecpar.py:63-84,
 * soptmov.py:195-240).  `scratch_records` is the caller's scratch budget in
 * records: 0 = the library default (the scheduled engine may salvage up to N/4
 * records into its pool); > 0 caps that pool -- a job whose planned salvage does
 * not fit runs the bounded-pool engine instead (decided on the device), whose
 * own pool is at least `scratch_records` records.
 */
int pm_merge(pm_ctx *ctx, void *keys, int key_bytes, void *payload, int64_t width,
             int64_t start, int64_t middle, int64_t end, int64_t scratch_records, void *stream);

/*
 * Out-of-place stable merge: src holds the sorted runs A = src[0, len_a) and
 * B = src[len_a, len_a+len_b); the merged records (A wins ties, as pm_merge)
 * go to dst[0, len_a+len_b).  src and dst must not overlap.  The partition
 * exchange of the reference's parallel merge lands a GPU's two runs in a
 * receive buffer (srecpar.py:63-84 across ranks, paper_2005_12648_b200/dist.py);
 * this merges them straight into the rank's block, one read and one write per
 * record.
 */
int pm_merge_copy(pm_ctx *ctx, const void *src_keys, const void *src_payload, void *dst_keys,
                  void *dst_payload, int key_bytes, int64_t width, int64_t len_a, int64_t len_b,
                  void *stream);

/*
 * In-place block exchange A|B -> B|A of [lo, lo+len_a) and [lo+len_a,
 * lo+len_a+len_b).  When the smaller block fits a 64 MB stash it is staged and
 * the larger block slides over it in one pass (the reference's staged exchange,
 * _kernels.py:46-90); otherwise three streaming reversals (two passes).  Replaces _kernels.linear_shift (_kernels.py:92-150) and
 * _kernels.circular_shift (_kernels.py:154-197) behind shift_region /
 * linear_shift / circular_shift (shift.py:38-55); both kinds produce the same
 * array (tests/test_srecpar.py:70-80 of the reference).
 */
int pm_shift(pm_ctx *ctx, void *keys, int key_bytes, void *payload, int64_t width,
             int64_t lo, int64_t len_a, int64_t len_b, void *stream);

/*
 * Replaces reorder_multi / reorder_cycles (soptmov.py:146-192, _kernels.py:317-369):
 * permute [start, end) into the leaf layout A_0 B_0 A_1 B_1 ... where the A run is
 * [start, start + sum|A_i|) cut into consecutive slices of the given sizes and the B
 * run follows likewise (leaf_sizes: host int64[2*nleaves] = |A_0|, |B_0|, |A_1|, ...).
 * One in-place pass of the scheduled engine (plan, salvage copy, streaming
 * gather): every record is read and written once plus the salvaged ones; no keys
 * are marked (the reference's marker offsets are not needed).
 */
int pm_reorder(pm_ctx *ctx, void *keys, int key_bytes, void *payload, int64_t width, int64_t start, int64_t end,
               const int64_t *leaf_sizes, int32_t nleaves, void *stream);

/*
 * Alg. 1 pivot pair of the sorted runs a[0, la) and b[0, lb) (DEVICE
 * pointers), exactly as find_median (median.py:23-60).  out2 is a DEVICE
 * int64[2] receiving (p_a, p_b).
 */
int pm_find_median(pm_ctx *ctx, const void *a, const void *b, int key_bytes, int64_t la, int64_t lb,
                   int64_t *out2, void *stream);

/*
 * Stable merge-path splits of the sorted runs a[0, la) and b[0, lb) (DEVICE
 * pointers): for each diagonal diags[i] (DEVICE int64[nd]),
 * out_a[i] (DEVICE) = number of A records among the first diags[i] outputs of
 * the stable merge (A wins ties).  The GPU pipeline's partition search; the
 * stable counterpart of plan_intervals' pivots (soptmov.py:93-123).
 */
int pm_find_splits(pm_ctx *ctx, const void *a, const void *b, int key_bytes, int64_t la, int64_t lb,
                   const int64_t *diags, int64_t nd, int64_t *out_a, void *stream);

/*
 * plan_intervals (soptmov.py:93-123): log2(threads) levels of Alg. 1 over run
 * pairs.  nodes (DEVICE int64[4*(2*threads-1)]) receives the level-order
 * RunPairs (a_start, a_end, b_start, b_end), level 0 first.
 */
int pm_plan_intervals(pm_ctx *ctx, const void *keys, int key_bytes, int64_t start, int64_t middle,
                      int64_t end, int32_t threads, int64_t *nodes, void *stream);

/*
 * Global stable splits of a block-distributed A|B (the distributed form of
 * median.find_median's split search, median.py:23-60, made stable): for each
 * diagonal diags[i] the number of A records among the first diags[i] outputs,
 * read through the peer-pointer table (one thread per diagonal, dependent peer
 * loads over NVLink).  Host diags / out_a; synchronises the stream.
 */
int pm_peer_splits(pm_ctx *ctx, const void *const *peer_keys, int world, int64_t block, int64_t len_a,
                   int key_bytes, const int64_t *diags, int nd, int64_t *out_a, void *stream);

/*
 * Multi-GPU merge with the partition exchange fused into the merge's loads.
 * The global array X = A|B (A = X[0, len_a), B = X[len_a, N), N = world*block)
 * is block-distributed: block k (records [k*block, (k+1)*block)) at
 * peer_keys[k] / peer_payload[k] -- a HOST array of `world` DEVICE pointers,
 * valid in this process (this GPU's own block, and the others' mapped through
 * pm_ipc_open with NVLink peer access).  Writes rank `rank`'s share of the
 * stable merge, X'[rank*block, (rank+1)*block), to out_keys / out_payload
 * (this GPU; must not alias any block).  The global splits and the output
 * positions of the block boundaries inside the rank's pieces come from merge
 * path searches over the peer table (the median/split search of srecpar.py:
 * 63-84 across GPUs); each resulting sub-range is one streaming merge whose
 * TMA loads read the remote pieces over NVLink.  The caller keeps every block
 * unmodified until all ranks have returned (a barrier), then may copy out
 * into its block.  Synchronises `stream` (the searches are read back).
 * the dist variant taking a peer-pointer table.
 */
int pm_merge_peers(pm_ctx *ctx, const void *const *peer_keys, const void *const *peer_payload, int world,
                   int rank, int64_t block, int64_t len_a, int key_bytes, int64_t width, void *out_keys,
                   void *out_payload, void *stream);
/* CUDA IPC for the peer table: a 64-byte handle of a device allocation's base,
 * its mapping in another process (NVLink peer access enabled lazily), unmap. */
int pm_ipc_handle(void *device_ptr, void *out_handle64);
int pm_ipc_open(const void *handle64, void **out_ptr);
int pm_ipc_close(void *ptr);

/*
 * Synchronise `stream`, then return (and clear) the sticky device status of the
 * context's last merges/shifts.  stats (host uint64[16], may be NULL) receives
 * the last job's counters: [0] salvaged units, [1] salvaged records, [2] merged
 * regions, [3] identity (skipped) regions, [4..9] summed per-CTA cycles in the
 * engine phases (ticket, gather issue, gather land, salvage, merge, store),
 * [10..11] spin iterations in reader / occupant waits; [13] 1 when a pure
 * rotation took the block-exchange route (three reversals) instead of the engine.
 */
int pm_status(pm_ctx *ctx, void *stream, uint64_t *stats);

/*
 * End-to-end entry point with HOST buffers (the reference's calling
 * convention: numpy arrays in host memory).  Copies keys/payload to the
 * device, merges, copies back, synchronises and returns the status.
 * Pinned host memory gives full PCIe bandwidth.  Records already on their
 * output positions (the A prefix <= B[0], the B suffix >= A[last]) never cross
 * PCIe; chunks are uploaded in merge order and written back as soon as merged
 * (through a grow-only pinned staging buffer per context, moved into place by
 * host threads once their range has been uploaded).
 */
int pm_merge_host(pm_ctx *ctx, void *keys_host, int key_bytes, void *payload_host, int64_t width,
                  int64_t start, int64_t middle, int64_t end, void *stream);
/* The host side of pm_merge_host, no device calls (CPU tests): out_span = the
 * trimmed job [start, end) or {-1, -1} when nothing moves; *out_nch chunks with
 * output boundaries out_d[0..nch] and A splits out_a[0..nch] (trimmed-job local)
 * and out_free[k] = the upload after which chunk k's output range is free. */
int pm_debug_host_plan(const void *keys_host, int key_bytes, int64_t start, int64_t middle, int64_t end,
                       int64_t min_chunk, int32_t chunks, int64_t *out_span, int64_t *out_d, int64_t *out_a,
                       int32_t *out_free, int32_t cap, int32_t *out_nch);

/*
 * Instrumentation (no reference counterpart): when enabled, the context
 * records CUDA events around the plan and engine kernels of each merge/shift;
 * pm_kernel_ms() waits for the last one and returns their device durations.
 */
int pm_set_timing(pm_ctx *ctx, int on);
/* After a timed in-place merge: out4 = {plan, salvage copy, merge kernel, total} in
 * ms (salvage copy 0 when the bounded-pool engine ran; its kernel is then "merge"). */
int pm_kernel_ms_detail(pm_ctx *ctx, float *out4);
/* Host evaluation of the engine's two-front ticket order (same source as the
 * device code): out4 = {region of ticket t, order(region), window lo, window hi}. */
int pm_debug_order(int64_t Q, int64_t qc, int64_t t, int64_t *out4);
/* Debug: on != 0 routes every in-place merge of this context through the
 * bounded-scratch engine (no one-CTA small-job or staged shortcut) and every
 * block exchange through the three reversals (no one-pass slide), so tests
 * exercise those paths at small sizes. */
int pm_debug_engine_only(pm_ctx *ctx, int on);

/* In-place merge engine selection (debug/benchmark control; default 1).
 *   0: the bounded-pool engine only (k_engine: a fixed ~175 MB salvage pool);
 *   1: the scheduled engine (pm_flow.cu), order chosen per job, falling back on
 *      the device to the bounded-pool engine if the salvage exceeds its pool;
 *   2 / 3: the scheduled engine with the two-front / itinerary-angle order forced;
 *   4: run the scheduled plan, then force the device-side fallback (tests). */
int pm_debug_flow(pm_ctx *ctx, int mode);
/* Debug: the wide-record path's in-place row permutation on its own:
 * row p of payload (DEVICE, n rows of width bytes) becomes old row idx[p]
 * (idx: DEVICE int32[n], a permutation), cycles cut every cut_every rows. */
int pm_debug_permute_rows(pm_ctx *ctx, void *payload, int64_t width, const int32_t *idx, int64_t n,
                          int32_t cut_every, void *stream);
/* Copy the first n entries of the last job's split table to host memory (debug). */
int pm_debug_splits(pm_ctx *ctx, int64_t *host_out, int64_t n);

/* Debug: the 64 device counters of the last job ([0,16) as pm_status; [16,64)
 * per-ticket-range histograms filled only by -DPM_STATS=1 tuning builds). */
int pm_debug_stats(pm_ctx *ctx, uint64_t *host_out64);
int pm_kernel_ms(pm_ctx *ctx, float *plan_ms, float *engine_ms);
/* Kernels this library has launched in this process (all contexts, since load):
 * the bench's gpu_launches claim is the difference around its timed region. */
int pm_launch_count(int64_t *out);

#ifdef __cplusplus
}
#endif
#endif /* PARMERGE_B200_H */
