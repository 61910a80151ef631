// pm_capi.cu -- extern "C" boundary (include/parmerge_b200.h) over the sm_100a
// kernels.  Validation mirrors the reference wrappers' ValueError/IndexError
// conditions (records.py:100-127, shift.py:156-162); the Python mirror maps
// PM_ERR_ARG back to those exceptions.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <vector>
#include <string>
#include <thread>
#include <map>
#include <chrono>

#include "../../include/parmerge_b200.h"
#include "pm_common.cuh"
#include "pm_engine.cuh"
#include "pm_launch.h"

using namespace pm;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(PM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define PM_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// control block layout (device, bytes)
// Words polled or hammered by every CTA live on their own 256-byte lines (distinct
// L2 slices): a spin loop on `err` must not queue up the ticket atomics.
struct alignas(256) Line32 {
  int32_t v;
  int32_t pad_[63];
};
struct Ctl {
  unsigned long long free_top;
  unsigned long long scr_top;
  unsigned long long stats[64];  // [0,16): pm_status; [16,64): tuning histograms (PM_STATS builds)
  Line32 ticket_;
  Line32 err_;
  Line32 noop_;
  Line32 need_space_;
  Line32 stage_gate_;  // staged path: the runs are out of order (computed by k_plan)
};


}  // namespace

struct pm_ctx {
  int device = 0;
  int num_sms = 148;
  std::mutex mu;
  std::mutex host_mu;  // pm_merge_host: one call at a time per context (staging buffer, its streams and events)
  void* ws = nullptr;  // split_a | state | loc | reads | next_free | next_scr
  size_t ws_bytes = 0;
  Ctl* ctl = nullptr;
  void* scr = nullptr;  // scratch keys + payload
  size_t scr_bytes = 0;
  void* stage = nullptr;  // device staging for pm_merge_host (input copy + output)
  size_t stage_bytes = 0;
  cudaStream_t hs[3] = {nullptr, nullptr, nullptr};  // pm_merge_host: H2D, merge, D2H
  cudaEvent_t hev[33] = {};                          // [0]: joins; then per-chunk events (ring)
  std::map<std::pair<int, size_t>, std::pair<int, int>> flow_occ;  // (key bytes, smem) -> k_flow, plan CTAs/SM
  uint64_t peer_on = 0;  // peer devices whose memory this context's device may access (P2P enabled)
  size_t flow_attr[2] = {0, 0};  // k_flow<int32/int64>: dynamic shared memory limit set so far
  cudaStream_t fside = nullptr;  // the scheduled engine's gated fallback runs here (forked after the plan)
  cudaEvent_t ffork = nullptr, fjoin = nullptr;  // (key bytes, smem) -> k_flow, plan CTAs/SM
  std::vector<cudaEvent_t> hup, hdn;  // pm_merge_host: per chunk, upload done / staged write-back landed
  void* hstage = nullptr;             // pm_merge_host: pinned host staging of early write-backs
  size_t hstage_bytes = 0;
  void* buf = nullptr;    // min-side buffer of the buffered mode
  size_t buf_bytes = 0;
  void* wide = nullptr;   // wide records: row indices, merged keys
  size_t wide_bytes = 0;
  void* wperm = nullptr;  // in-place row permutation: cycle tables, uncut heads, saved cut rows
  size_t wperm_bytes = 0;
  void* peer = nullptr;   // pm_merge_peers: device copy of the peer table + queries + answers
  size_t peer_bytes = 0;
  bool timing = false;  // record events around the plan and engine kernels
  bool engine_only = false;  // debug: no small-job / staged shortcuts (pm_debug_engine_only)
  int flow_mode = 1;  // scheduled engine: 0 off (bounded-pool engine), 1 auto, 2 two-front, 3 angle, 4 force fallback
  void* fws = nullptr;  // scheduled engine: plan arrays + tickets + control words
  size_t fws_bytes = 0;
  void* fpool = nullptr;  // scheduled engine: salvage pool (keys + payload, phase matched)
  size_t fpool_bytes = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // plan | engine [| merge kernel] | end
  bool ev_mid = false;  // ev[3] recorded (scheduled engine: between the salvage copy and k_flow)
  cudaStream_t last_stream = nullptr;  // the stream of the previous call (use_stream)
  bool have_last = false;
  cudaEvent_t xev = nullptr;
  bool ev_recorded = false;
};

// Every entry point runs on the context's device and restores the caller's current
// device on return (tensors on cuda:1 while cuda:0 is current must not allocate or
// launch on cuda:0).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev < 0 || cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      return;
    }
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// A context's workspace (splits, tickets, pools, control words) is shared by every
// call on it: a call on another stream than the previous one first waits for the
// previous stream's work (one event), so calls on different streams cannot race on it.
static void use_stream(pm_ctx* ctx, cudaStream_t st) {
  if (ctx->have_last && ctx->last_stream != st) {
    if (!ctx->xev) cudaEventCreateWithFlags(&ctx->xev, cudaEventDisableTiming);
    if (cudaEventRecord(ctx->xev, ctx->last_stream) == cudaSuccess) cudaStreamWaitEvent(st, ctx->xev, 0);
    else cudaGetLastError();  // (the previous stream is gone: nothing left to wait for)
  }
  ctx->last_stream = st;
  ctx->have_last = true;
}

static int ensure(void** p, size_t* have, size_t need) {
  if (*have >= need) return PM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  size_t sz = std::max(need, (size_t)1 << 20);
  cudaError_t e = cudaMalloc(p, sz);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(workspace)");
  *have = sz;
  return PM_OK;
}

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Tile geometry for a record of ks+w bytes: region M (power of two) so that the
// staged keys+payload+index map stay ~<=72 KB per CTA (3 CTAs per SM).
static bool pick_tiles(int ks, int64_t w, int64_t budget, int64_t* M, int64_t* T, int32_t* mu) {
  int64_t m = 8192;
  while (m > 16 && m * 2 * (ks + w) + 256 > budget) m >>= 1;
  if (m * 2 * (ks + w) + 256 > budget + 64 * 1024) return false;  // records too wide
  *M = m;
#ifndef PM_MU
#define PM_MU 1
#endif
  *T = std::max<int64_t>(16, m / PM_MU);
  *mu = (int32_t)(m / *T);
  return true;
}

static int run_engine(pm_ctx* ctx, void* keys, int ks, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                      int mode, int64_t scratch_records, cudaStream_t st, void* out_keys = nullptr,
                      void* out_payload = nullptr, const void* keys_b = nullptr, const void* pay_b = nullptr,
                      const int32_t* gate = nullptr, int32_t* gate_out = nullptr);

#ifndef PM_SLIDE_STASH
#define PM_SLIDE_STASH (64ll << 20)  // pm_shift: one-pass slide when the smaller block fits this stash
#endif
#ifndef PM_GRIES_MILLS
#define PM_GRIES_MILLS 0  // 1: block exchanges by Gries-Mills swaps + reversals for the remainder -- slower than the
                          // reversals alone (2^30, 1:2 blocks: 3.94 vs 2.97 ms; unaligned swaps, several launches)
#endif
#ifndef PM_CLUSTER_MERGE
#define PM_CLUSTER_MERGE 0  // 1: jobs of up to ~1 MB in one thread-block cluster (distributed shared memory) --
                            // the one-launch grid merge is faster at every such size (2^15 records per side:
                            // 26.8 vs 14.7 us, 2^17: 30.0 vs 18.4 us), so it is off by default
#endif
#ifndef PM_STAGE_WIDE
#define PM_STAGE_WIDE 1  // tune: wide rows also take the staged path (row gather + copy back; 0.20 vs 0.31-0.45 ms at 200 MB)
#endif
#ifndef PM_SMALL_BYTES
#define PM_SMALL_BYTES (64 * 1024)  // one-CTA small merge up to 32 KB of records (in + out tile in shared
                                    // memory); beyond, the grid merge is faster (2^13 per side: 19.2 vs 16.3 us)
#endif
#ifndef PM_STAGE_BYTES
#define PM_STAGE_BYTES (256ll << 20)  // in-place jobs up to this size merge via a staging buffer (a constant, below the engine pool)
#endif
static int launch_merge_small_(int ks, void* keys, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                               cudaStream_t st) {
  cudaError_t ce = ks == 4 ? launch_merge_small<int32_t>(keys, payload, w, s, m, e, st)
                           : launch_merge_small<int64_t>(keys, payload, w, s, m, e, st);
  return ce == cudaSuccess ? PM_OK : cuda_fail(ce, "k_merge_small launch");
}

// Payload rows of at least PM_WIDE_MIN bytes (or too wide for the staging tiles)
// take the wide-record path (pm_wide.cu): the stable merge of (key, row index)
// pairs in copy mode, then the row permutation -- a gather into the destination
// (copy mode) or the in-place cycle walk over segments cut every G rows.
#ifndef PM_WIDE_MIN
#define PM_WIDE_MIN 256  // tune: bytes per payload row from which the wide path runs
#endif
#ifndef PM_FLOW_TF_Q
#define PM_FLOW_TF_Q 32768  // tune: regions below which the scheduled engine plans the two-front order only (2^26/side: 336 vs 352 us; 2^27: even)
#endif
#ifndef PM_FLOW_WIDE_MAX
#define PM_FLOW_WIDE_MAX 2048  // tune: bytes per record up to which in-place wide rows take the scheduled engine
#endif
#ifndef PM_WIDE_SAVE_BYTES
#define PM_WIDE_SAVE_BYTES (256ll << 20)  // bound on the saved cut rows (G grows past 16 to respect it)
#endif
// In-place row permutation new_row[p] = old_row[idx[p]] (idx: DEVICE int32[n], a
// permutation of [0, n)), cycles cut every G rows (pm_wide.cu).
#ifndef PM_CYC_LMAX
#define PM_CYC_LMAX 32  // tune: longest chain of the cycle walk (longer segments get extra cuts)
#endif
static int permute_rows(pm_ctx* ctx, uint8_t* pay, int64_t w, const int32_t* idx, int64_t n, int32_t G,
                        cudaStream_t st) {
  const int64_t ncut = (n + G - 1) / G;
  // extra cuts: at most one per Lmax positions, and within the save budget
  const int32_t Lmax = PM_CYC_LMAX;
  const int64_t xcap = std::max<int64_t>(1, std::min<int64_t>(n / Lmax + 1, PM_WIDE_SAVE_BYTES / w));
  const size_t o_d1 = (size_t)align_up(n * 8, 256);
  const size_t o_heads = o_d1 + (size_t)align_up(n * 8, 256);
  const size_t o_unres = o_heads + (size_t)align_up(n * 8, 256);
  const size_t o_segs = o_unres + (size_t)align_up(n, 256);
  const size_t o_xpos = o_segs + (size_t)align_up((ncut + xcap) * 16, 256);
  const size_t o_ctl = o_xpos + (size_t)align_up(xcap * 4, 256);
  const size_t o_save = o_ctl + 256;
  int rc = ensure(&ctx->wperm, &ctx->wperm_bytes, o_save + (size_t)((ncut + xcap) * w));
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->wperm);
  cudaError_t ce = launch_cycle_permute(pay, w, idx, n, G, reinterpret_cast<int2*>(base), reinterpret_cast<int2*>(base + o_d1),
                                        reinterpret_cast<int2*>(base + o_heads), reinterpret_cast<int32_t*>(base + o_ctl),
                                        reinterpret_cast<uint8_t*>(base + o_unres), reinterpret_cast<int4*>(base + o_segs),
                                        reinterpret_cast<int32_t*>(base + o_xpos), (int32_t)xcap, Lmax,
                                        reinterpret_cast<uint8_t*>(base + o_save), ctx->num_sms, st);
  return ce == cudaSuccess ? PM_OK : cuda_fail(ce, "cycle permutation launch");
}

static int run_wide(pm_ctx* ctx, char* keys, int ks, uint8_t* pay, int64_t w, int64_t s, int64_t m, int64_t e,
                    cudaStream_t st, char* out_keys, uint8_t* out_pay, const char* keys_b, const uint8_t* pay_b) {
  const bool copy = out_keys != nullptr;
  const int64_t n = e - s, la = m - s;
  if (n >= INT32_MAX) return fail(PM_ERR_UNSUPPORTED, "wide-record merges index rows with 32 bits");
  const size_t o_idx = (size_t)align_up(n * 4, 256);
  const size_t o_tmpk = o_idx + (size_t)align_up(n * 4, 256);
  const size_t need = o_tmpk + (size_t)(copy ? 0 : align_up(n * ks, 256));
  int rc = ensure(&ctx->wide, &ctx->wide_bytes, need);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->wide);
  int32_t* idx0 = reinterpret_cast<int32_t*>(base);
  int32_t* idx = reinterpret_cast<int32_t*>(base + o_idx);
  cudaError_t ce = launch_iota(idx0, n, ctx->num_sms, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "k_iota launch");
  // (1) merged keys + the source row of every output position
  rc = run_engine(ctx, keys + s * ks, ks, idx0, 4, 0, la, n, MODE_MERGE, 0, st, copy ? out_keys + s * ks : base + o_tmpk,
                  idx, keys_b, keys_b ? idx0 + la : nullptr);
  if (rc) return rc;
  uint8_t* a = pay + s * w;
  if (copy) {  // (2) gather
    ce = launch_gather_rows(out_pay + s * w, a, pay_b ? pay_b : a + la * w, idx, n, la, w, ctx->num_sms, st);
    return ce == cudaSuccess ? PM_OK : cuda_fail(ce, "k_gather_rows launch");
  }
  PM_CUDA(cudaMemcpyAsync(keys + s * ks, base + o_tmpk, (size_t)(n * ks), cudaMemcpyDeviceToDevice, st));
  // (2) in-place cycle permutation of the rows; cut every G rows, G >= 16 bounded by the save budget
  int32_t G = 16;
  while (G < n && ((n + G - 1) / G) * w > PM_WIDE_SAVE_BYTES) G *= 2;
  return permute_rows(ctx, a, w, idx, n, G, st);
}

// out_keys / out_payload non-null: copy mode -- merge keys[s,m) and keys[m,e) into
// out[s,e) (the streaming pipeline of the buffered mode, nothing overlaps).
// keys_b / pay_b (copy mode only): the B run lives there instead of at keys + m.
static int run_flow(pm_ctx* ctx, void* keys, int ks, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                    cudaStream_t st, const int64_t* leaf_sizes = nullptr, int32_t nleaves = 0,
                    int64_t scratch_records = 0);

static int run_engine(pm_ctx* ctx, void* keys, int ks, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                      int mode, int64_t scratch_records, cudaStream_t st, void* out_keys, void* out_payload,
                      const void* keys_b, const void* pay_b, const int32_t* gate, int32_t* gate_out) {
  const bool copy = out_keys != nullptr;
  if (e - s <= 0 || (!copy && (m == s || m == e))) return PM_OK;
  int64_t M, T;
  int32_t mu;
  // the fallback behind the scheduled engine goes straight to the bounded-pool engine
  // (a gated copy-mode call is the staged path's merge, not a fallback)
  const bool direct = gate != nullptr && !copy;
  // small in-place jobs: one CTA with both runs in shared memory
  if (mode == MODE_MERGE && !copy && !direct && !ctx->engine_only && small_merge_smem(ks, w, e - s) <= PM_SMALL_BYTES)
    return launch_merge_small_(ks, keys, payload, w, s, m, e, st);
  // up to ~3 MB: one thread-block cluster, both runs in distributed shared memory
  if (mode == MODE_MERGE && !copy && !direct && !ctx->engine_only && w <= 64 && PM_CLUSTER_MERGE) {
    int lchunk = 0;
    const int C = cluster_merge_plan(ks, w, e - s, &lchunk);
    if (C > 0) {
      cudaError_t ce = ks == 4 ? launch_merge_cluster<int32_t>(keys, payload, w, s, m, e, C, lchunk, st)
                               : launch_merge_cluster<int64_t>(keys, payload, w, s, m, e, C, lchunk, st);
      if (ce != cudaSuccess) return cuda_fail(ce, "k_merge_cluster launch");
      return PM_OK;
    }
  }
  // up to ~14 MB (one CTA per SM holding a 100 KB output tile): one cooperative
  // launch that merges every CTA's range into shared memory and stores it in place
  // after a grid barrier (pm_small.cu, k_merge_grid)
#ifndef PM_GRID_MERGE
#define PM_GRID_MERGE 1
#endif
  if (mode == MODE_MERGE && !copy && !direct && !ctx->engine_only && w <= 64 && PM_GRID_MERGE) {
    int ctas = 0;
    size_t gsm = 0;
    const int64_t R = grid_merge_plan(ks, w, e - s, ctx->num_sms, &ctas, &gsm);
    if (R > 0) {
      cudaError_t ce = ks == 4 ? launch_merge_grid<int32_t>(keys, payload, w, s, m, e, ctas, R, gsm, st)
                               : launch_merge_grid<int64_t>(keys, payload, w, s, m, e, ctas, R, gsm, st);
      if (ce == cudaSuccess) return PM_OK;
      // not every SM free for a co-resident grid (other work / partitioned GPU):
      // the staged path below needs no co-residency
      if (ce != cudaErrorCooperativeLaunchTooLarge) return cuda_fail(ce, "k_merge_grid launch");
      cudaGetLastError();
    }
  }
  // medium in-place jobs (at most PM_STAGE_BYTES of records): the streaming merge
  // into a staging buffer, then one copy back -- both passes mostly in L2
  if (mode == MODE_MERGE && !copy && !direct && !ctx->engine_only && (e - s) * (ks + w) <= PM_STAGE_BYTES && (PM_STAGE_WIDE || w < PM_WIDE_MIN)) {
    const int64_t n = e - s;
    const size_t kb = (size_t)align_up(n * ks + 16, 256);  // + the phase offset below
    int rc = ensure(&ctx->buf, &ctx->buf_bytes, kb + (size_t)(n * w) + 256);
    if (rc) return rc;
    char* sk = static_cast<char*>(ctx->buf) + (((uintptr_t)keys + s * ks) & 15);
    uint8_t* sp = reinterpret_cast<uint8_t*>(static_cast<char*>(ctx->buf) + kb + (w ? (((uintptr_t)payload + s * w) & 15) : 0));
    char* k0 = static_cast<char*>(keys) + s * ks;
    uint8_t* p0 = w ? static_cast<uint8_t*>(payload) + s * w : nullptr;
    // runs already in order (srecpar.py:56-57): the device skips the merge and the
    // copy back (the streaming pipeline's path; the wide-row path always runs)
    int64_t Mt, Tt;
    int32_t mut;
    const bool gated = !(w > 0 && (w >= PM_WIDE_MIN || !pick_tiles(ks, w, kTileBudget, &Mt, &Tt, &mut)));
    int32_t* gate = gated ? &ctx->ctl->stage_gate_.v : nullptr;
    // (k_plan computes the gate before the gated merge and copy read it)
    rc = run_engine(ctx, k0, ks, p0, w, 0, m - s, n, MODE_MERGE, 0, st, sk, w ? sp : nullptr, nullptr, nullptr, gate,
                    gate);
    if (rc) return rc;
    if (gated) {
      cudaError_t ce2 = launch_copy_gated(k0, sk, n * ks, gate, ctx->num_sms, st);
      if (ce2 == cudaSuccess && w) ce2 = launch_copy_gated(p0, sp, n * w, gate, ctx->num_sms, st);
      if (ce2 != cudaSuccess) return cuda_fail(ce2, "k_copy_gated launch");
    } else {
      PM_CUDA(cudaMemcpyAsync(k0, sk, (size_t)(n * ks), cudaMemcpyDeviceToDevice, st));
      if (w) PM_CUDA(cudaMemcpyAsync(p0, sp, (size_t)(n * w), cudaMemcpyDeviceToDevice, st));
    }
    return PM_OK;
  }
  // in-place wide rows of up to PM_FLOW_WIDE_MAX bytes per record take the scheduled
  // engine (tiles of >= 16 records read and written sequentially beat the cycle
  // walk's random rows: 1.17 vs 1.55 ms at 508-byte rows, 2 GB); its device-side
  // fallback is the bounded-pool engine, never the (ungated) wide path
  const bool wide = mode == MODE_MERGE && w > 0 && (w >= PM_WIDE_MIN || !pick_tiles(ks, w, kTileBudget, &M, &T, &mu));
  const bool flow_wide = wide && !copy && !ctx->engine_only && ctx->flow_mode != 0 && ks + w <= PM_FLOW_WIDE_MAX &&
                         pick_tiles(ks, w, kTileBudget, &M, &T, &mu);
  if (wide && !flow_wide)
    return run_wide(ctx, static_cast<char*>(keys), ks, static_cast<uint8_t*>(payload), w, s, m, e, st,
                    static_cast<char*>(out_keys), static_cast<uint8_t*>(out_payload),
                    static_cast<const char*>(keys_b), static_cast<const uint8_t*>(pay_b));
  // buffered mode (the caller granted a min(|A|,|B|) buffer, seq_merge_buffered):
  // half-size regions, two staging + two output tiles (72 KB of shared memory)
#ifndef PM_USE_BUFFERED
#define PM_USE_BUFFERED 1  // tune: the streaming buffered pipeline when scratch >= min(|A|,|B|) (2^30 int32: 2.6 ms vs 3.0 for the engine with that pool)
#endif
  // the scheduled engine (pm_flow.cu) for in-place merges
  if (mode == MODE_MERGE && !copy && !direct && ctx->flow_mode != 0)
    return run_flow(ctx, keys, ks, payload, w, s, m, e, st, nullptr, 0, scratch_records);
  const bool buffered = copy || (!direct && PM_USE_BUFFERED && mode == MODE_MERGE && scratch_records >= std::min(m - s, e - m));
  // (the engine stages one input and one output tile; the buffered pipeline
  //  kBufStages inputs and two outputs)
  if (!pick_tiles(ks, w, buffered ? kBufBudget * 2 / (kBufStages + 2) : kTileBudget, &M, &T, &mu))
    return fail(PM_ERR_UNSUPPORTED, "payload rows too wide for the staging tiles");
  EngineParams P{};
  P.keys = static_cast<char*>(keys);
  P.pay = static_cast<uint8_t*>(payload);
  P.out_keys = static_cast<char*>(out_keys);
  P.out_pay = static_cast<uint8_t*>(out_payload);
  P.keys_b = static_cast<const char*>(keys_b);
  P.pay_b = static_cast<const uint8_t*>(pay_b);
  P.gate = gate;
  P.gate_out = gate_out;
  P.w = w;
  P.ks = ks;
  P.mode = mode;
  P.s = s;
  P.m = m;
  P.e = e;
  P.T = T;
  P.lT = 63 - __builtin_clzll((unsigned long long)T);
  P.lmu = 31 - __builtin_clz((unsigned)mu);
  if ((1ll << P.lT) != T || (1 << P.lmu) != mu) return fail(PM_ERR_INTERNAL, "unit geometry must be powers of two");
  P.mu = mu;
  if (mu > 8) return fail(PM_ERR_INTERNAL, "too many slots per region");
  P.M = M;
  P.k0 = s / T;
  P.K = (e - 1) / T - P.k0 + 1;
  P.R0 = s / M;
  P.Q = (e - 1) / M - P.R0 + 1;
  P.qc = std::min<int64_t>(std::max<int64_t>(m / M - P.R0, 0), P.Q - 1);
  if (P.K >= INT32_MAX / 2) return fail(PM_ERR_UNSUPPORTED, "job too large for 32-bit unit indices");
  // shared memory carve-up (all offsets 16-byte aligned)
  P.smem_keys = (size_t)align_up((M + 2 * kSent) * ks + 64, 128);  // + sentinel gaps (write_sentinels)
  {
    const int64_t merge_threads = buffered ? kBufferedThreads - 32 : kEngineThreads - 32 * kEngineTeam;
    if ((((M + merge_threads - 1) / merge_threads) | 1) + 1 > kSent)
      return fail(PM_ERR_INTERNAL, "tile merge span exceeds the sentinel gap");
  }
  P.smem_pay = w ? (size_t)align_up(M * w + 48, 128) : 0;
  // staged inputs (keys, payload) + merged output tile (keys, payload), same sizes;
  // the buffered pipeline double-buffers both
  const size_t smem = (buffered ? kBufStages + 2 : 2) * (P.smem_keys + P.smem_pay);
  // persistent grid: every resident CTA slot on every SM
  int bps = 0;
  cudaError_t ce;
  if (buffered)
    ce = ks == 4 ? buffered_occupancy<int32_t>(smem, &bps) : buffered_occupancy<int64_t>(smem, &bps);
  else
    ce = ks == 4 ? engine_occupancy<int32_t>(kEngineThreads, smem, &bps)
                 : engine_occupancy<int64_t>(kEngineThreads, smem, &bps);
  if (ce != cudaSuccess) return cuda_fail(ce, "engine occupancy");
  if (bps < 1) return fail(PM_ERR_UNSUPPORTED, "engine does not fit on an SM");
  int grid = (int)std::min<int64_t>((int64_t)bps * ctx->num_sms, P.Q);
  // bounded salvage pool: O(grid * tile) records, phase matched to the caller's arrays
  // every CTA may hold kRing tickets' moved-but-unread units at once
  P.reserve = (int64_t)grid * (kRing * mu + 4) + 16;
  int64_t S = std::max<int64_t>(2 * P.reserve, scratch_records / T + P.reserve);
  S = std::min<int64_t>(S, P.K + P.reserve);
  P.S = S;
  P.grid = grid;
  // half of the pool starts in the CTAs' caches (<= 32 each, the cache holds 64)
#ifndef PM_SPER_DIV
#define PM_SPER_DIV 2
#endif
  P.s_per = buffered ? 0 : std::min<int64_t>(S / (PM_SPER_DIV * (int64_t)grid), 32);
  // workspace
  const size_t off_state = (size_t)align_up((P.Q + 1) * 8, 256);
  const size_t off_loc = off_state + (size_t)align_up(P.K * 4, 256);
  const size_t off_reads = off_loc + (size_t)align_up(P.K * 4, 256);
  const size_t off_nf = off_reads + (size_t)align_up(P.K * 4, 256);
  const size_t off_ns = off_nf + (size_t)align_up(P.K * 4, 256);
  const size_t off_tops = off_ns + (size_t)align_up(S * 4, 256);
  const size_t off_tlist = off_tops + 2 * kShards * kTopStride * sizeof(unsigned long long);
  const size_t ws_need = off_tlist + (size_t)align_up((2 * P.Q + 16) * 4 + 16, 256);  // list | flags | count
  int rc = ensure(&ctx->ws, &ctx->ws_bytes, ws_need);
  if (rc) return rc;
  const size_t scr_k = (size_t)align_up(S * T * ks + 32, 256);
  const size_t scr_need = scr_k + (size_t)(w ? S * T * w + 32 : 0);
  rc = ensure(&ctx->scr, &ctx->scr_bytes, scr_need);
  if (rc) return rc;
  char* ws = static_cast<char*>(ctx->ws);
  P.split_a = reinterpret_cast<int64_t*>(ws);
  P.state = reinterpret_cast<int32_t*>(ws + off_state);
  P.loc = reinterpret_cast<int32_t*>(ws + off_loc);
  P.reads = reinterpret_cast<int32_t*>(ws + off_reads);
  P.next_free = reinterpret_cast<int32_t*>(ws + off_nf);
  P.next_scr = reinterpret_cast<int32_t*>(ws + off_ns);
  P.free_top = reinterpret_cast<unsigned long long*>(ws + off_tops);  // [64] shard tops
  P.tlist = buffered ? nullptr : reinterpret_cast<int32_t*>(ws + off_tlist);  // engine tickets (k_compact)
  P.ntick = buffered ? nullptr : P.tlist + 2 * P.Q + 12;
  P.scr_top = P.free_top + kShards * kTopStride;
  P.stats = ctx->ctl->stats;
  P.ticket = &ctx->ctl->ticket_.v;
  P.err = &ctx->ctl->err_.v;
  P.noop = &ctx->ctl->noop_.v;
  P.need_space = &ctx->ctl->need_space_.v;
  char* scr = static_cast<char*>(ctx->scr);
  P.scr_keys = scr + ((uintptr_t)keys & 15);
  P.scr_pay = reinterpret_cast<uint8_t*>(scr + scr_k + (w ? ((uintptr_t)payload & 15) : 0));
  // buffered mode: the caller granted a min(|A|,|B|) buffer (seq_merge_buffered)
  const int64_t la = m - s, lb = e - m, mn = std::min(la, lb);
  const int32_t buf_a = la <= lb ? 1 : 0;
  if (buffered && !copy) {
    const size_t bk = (size_t)align_up(mn * ks + 64, 256), bp = (size_t)(w ? mn * w + 64 : 0);
    rc = ensure(&ctx->buf, &ctx->buf_bytes, bk + bp);
    if (rc) return rc;
    const int64_t x0 = buf_a ? s : m;
    char* b = static_cast<char*>(ctx->buf);
    P.scr_keys = b + (((uintptr_t)keys + x0 * ks) & 15);
    P.scr_pay = reinterpret_cast<uint8_t*>(b + bk + (w ? (((uintptr_t)payload + x0 * w) & 15) : 0));
  }
  // plan (splits + reset) then engine
  int64_t plan_work = std::max<int64_t>(P.Q + 1, P.K);
  int plan_grid = (int)std::min<int64_t>(std::max<int64_t>((plan_work + 255) / 256, 1), (int64_t)ctx->num_sms * 8);
  const bool timed = ctx->timing && !direct;
  if (timed) PM_CUDA(cudaEventRecord(ctx->ev[0], st));
  ce = ks == 4 ? launch_plan<int32_t>(P, plan_grid, st) : launch_plan<int64_t>(P, plan_grid, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "k_plan launch");
  if (timed) PM_CUDA(cudaEventRecord(ctx->ev[1], st));
  if (copy) {
    ce = ks == 4 ? launch_merge_copy<int32_t>(P, grid, smem, st) : launch_merge_copy<int64_t>(P, grid, smem, st);
  } else if (buffered) {
    ce = ks == 4 ? launch_buffered<int32_t>(P, buf_a, grid, smem, st) : launch_buffered<int64_t>(P, buf_a, grid, smem, st);
  } else {
    ce = ks == 4 ? launch_engine<int32_t>(P, grid, kEngineThreads, smem, st)
                 : launch_engine<int64_t>(P, grid, kEngineThreads, smem, st);
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "k_engine launch");
  if (timed) {
    PM_CUDA(cudaEventRecord(ctx->ev[2], st));
    ctx->ev_recorded = true;
    ctx->ev_mid = false;
  }
  return PM_OK;
}

#ifndef PM_FLOW_POOL_DIV
#define PM_FLOW_POOL_DIV 4  // scheduled engine: salvage pool capacity N / PM_FLOW_POOL_DIV records (+ slack)
#endif
#ifndef PM_FLOW_BITS
#define PM_FLOW_BITS 12  // itinerary length of the angle order
#endif
#ifndef PM_FLOW_SYNC
#define PM_FLOW_SYNC 4  // angular-synchronisation steps refining the angle order
#endif
#ifndef PM_FLOW_SYNC_DIV
#define PM_FLOW_SYNC_DIV 10  // their phase step 2 pi / PM_FLOW_SYNC_DIV
#endif
#ifndef PM_FLOW_BINS
#define PM_FLOW_BINS 16384  // angle bins of the counting sort
#endif
// Scheduled in-place merge (pm_flow.cu), with the bounded-pool engine queued
// behind it on the device: it runs only if the plan's salvage exceeds the pool
// (FC_FAIL), so the whole call stays asynchronous.
static int run_flow(pm_ctx* ctx, void* keys, int ks, void* payload, int64_t w, int64_t s, int64_t m, int64_t e,
                    cudaStream_t st, const int64_t* leaf_sizes, int32_t nleaves, int64_t scratch_records) {
  int64_t M, T;
  int32_t mu;
  // regions: the largest power of two <= 8192 records whose keys + rows fit a tile
#ifndef PM_FLOW_MAXM
#define PM_FLOW_MAXM 8192  // tune: largest scheduled-engine region (records)
#endif
  M = PM_FLOW_MAXM;
  while (M > 16 && M * (ks + w) > PM_FLOW_TILE) M >>= 1;
  if (M * (ks + w) > PM_FLOW_TILE) return fail(PM_ERR_UNSUPPORTED, "payload rows too wide for the staging tiles");
  T = M;
  (void)mu;
  FlowParams F{};
  EngineParams& P = F.P;
  P.keys = static_cast<char*>(keys);
  P.pay = static_cast<uint8_t*>(payload);
  P.w = w;
  P.ks = ks;
  P.mode = MODE_MERGE;
  P.s = s;
  P.m = m;
  P.e = e;
  P.T = T;
  P.M = M;
  P.mu = 1;
  P.lT = 63 - __builtin_clzll((unsigned long long)T);
  P.lmu = 0;
  P.k0 = s / T;
  P.K = (e - 1) / T - P.k0 + 1;
  P.R0 = P.k0;
  P.Q = P.K;
  P.qc = std::min<int64_t>(std::max<int64_t>(m / M - P.R0, 0), P.Q - 1);
  if (P.K >= INT32_MAX / 2) return fail(PM_ERR_UNSUPPORTED, "job too large for 32-bit region indices");
  P.smem_keys = (size_t)align_up((M + 2 * kSent) * ks + 64, 128);
  if ((((M + kFlowThreads - 32 - 1) / (kFlowThreads - 32)) | 1) + 1 > kSent)
    return fail(PM_ERR_INTERNAL, "tile merge span exceeds the sentinel gap");
  P.smem_pay = w ? (size_t)align_up(M * w + 48, 128) : 0;
  const size_t smem = (kFlowStages + kFlowOut) * (P.smem_keys + P.smem_pay);
  int bps = 0, plan_bps = 0;
  cudaError_t ce;
  {
    auto it = ctx->flow_occ.find({ks, smem});
    if (it == ctx->flow_occ.end()) {
      size_t& attr = ctx->flow_attr[ks == 8];
      attr = std::max(attr, smem);
      ce = ks == 4 ? flow_occupancy<int32_t>(smem, attr, &bps, &plan_bps)
                   : flow_occupancy<int64_t>(smem, attr, &bps, &plan_bps);
      if (ce != cudaSuccess) return cuda_fail(ce, "flow occupancy");
      it = ctx->flow_occ.emplace(std::make_pair(ks, smem), std::make_pair(bps, plan_bps)).first;
    }
    bps = it->second.first;
    plan_bps = it->second.second;
  }
  if (bps < 1) return fail(PM_ERR_UNSUPPORTED, "scheduled engine does not fit on an SM");
  const int grid = (int)std::min<int64_t>((int64_t)bps * ctx->num_sms, P.Q);
  P.grid = grid;
  // workspace: splits | D | key | order | rank | slo | shi | pend | pdelta | tickets | hist | chunk | idn | fc
  const int64_t K = P.K;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (size_t)align_up((int64_t)bytes, 256);
    return o;
  };
  const size_t o_split = take((size_t)(P.Q + 1) * 8), o_D = take(K * 4), o_key = take(K * 4), o_order = take(K * 4),
               o_rank = take(K * 4), o_slo = take(K * 4), o_shi = take(K * 4), o_pend = take(K * 4),
               o_pd = take(K * 8), o_tk = take(K * sizeof(FlowTicket)), o_hist = take((PM_FLOW_BINS + 1) * 4),
               o_chunk = take((P.Q / 1024 + 2) * 4), o_idn = take(K), o_fc = take(FC_WORDS * 8);
  // split-search samples (stride S = min(256, M); S divides M)
#ifndef PM_FLOW_SAMPLE
#define PM_FLOW_SAMPLE 8192  // split-search sample stride (records; capped at the region size): 2^30 int32 plan 0.136 -> 0.127 ms vs 2048 (fewer row activations in the sample phase, the interpolation probes absorb the wider window)
#endif
  const int64_t S = std::min<int64_t>(PM_FLOW_SAMPLE, M);
  F.lS = 63 - __builtin_clzll((unsigned long long)S);
  F.phi = (int32_t)(((-(s + 1)) % S + S) % S);
  F.nsa = (m - s + S - 1) / S;
  F.nsb = (e - m) > F.phi ? (e - m - F.phi + S - 1) / S : 0;
  const size_t o_sa = take((size_t)(F.nsa + 1) * ks), o_sb = take((size_t)(F.nsb + 1) * ks);
  const size_t o_pc = take((size_t)K * 64), o_z = take((size_t)K * 24);
  const size_t o_leaf = take((size_t)(2 * nleaves + 2) * 8);
  int rc = ensure(&ctx->fws, &ctx->fws_bytes, off);
  if (rc) return rc;
  char* b = static_cast<char*>(ctx->fws);
  P.split_a = reinterpret_cast<int64_t*>(b + o_split);
  F.D = reinterpret_cast<int32_t*>(b + o_D);
  F.key = reinterpret_cast<uint32_t*>(b + o_key);
  F.order = reinterpret_cast<int32_t*>(b + o_order);
  F.rank = reinterpret_cast<int32_t*>(b + o_rank);
  F.slo = reinterpret_cast<int32_t*>(b + o_slo);
  F.shi = reinterpret_cast<int32_t*>(b + o_shi);
  F.pend = reinterpret_cast<int32_t*>(b + o_pend);
  F.pdelta = reinterpret_cast<int64_t*>(b + o_pd);
  F.tk = reinterpret_cast<FlowTicket*>(b + o_tk);
  F.hist = reinterpret_cast<int32_t*>(b + o_hist);
  F.chunk = reinterpret_cast<int32_t*>(b + o_chunk);
  F.idn = reinterpret_cast<uint8_t*>(b + o_idn);
  F.fc = reinterpret_cast<long long*>(b + o_fc);
  F.samp_a = b + o_sa;
  F.samp_b = b + o_sb;
  F.pieces = reinterpret_cast<int4*>(b + o_pc);
  F.nleaves = nleaves;
  if (nleaves) {  // prescribed layout: leaf output starts and A prefixes, job-local
    std::vector<int64_t> tab(2 * nleaves + 2);
    int64_t L = 0, Apre = 0;
    for (int32_t i = 0; i < nleaves; ++i) {
      tab[i] = L;
      tab[nleaves + 1 + i] = Apre;
      L += leaf_sizes[2 * i] + leaf_sizes[2 * i + 1];
      Apre += leaf_sizes[2 * i];
    }
    tab[nleaves] = L;
    tab[2 * nleaves + 1] = Apre;
    PM_CUDA(cudaMemcpyAsync(b + o_leaf, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, st));
    PM_CUDA(cudaStreamSynchronize(st));  // (pageable source: keep it alive until copied)
    F.leaf_l = reinterpret_cast<const int64_t*>(b + o_leaf);
    F.leaf_a = F.leaf_l + nleaves + 1;
  }
  F.z = reinterpret_cast<float2*>(b + o_z);
  F.nsync = PM_FLOW_SYNC;
  F.nsync_div = PM_FLOW_SYNC_DIV;
  F.nbits = PM_FLOW_BITS;
  F.nb = PM_FLOW_BINS;
  F.force = ctx->flow_mode == 2 ? 0 : ctx->flow_mode == 3 ? 1 : ctx->flow_mode == 4 ? 2 : -1;
  // small jobs: the two-front order with the lean plan (the itinerary phases cost
  // more than the extra salvage copy below ~PM_FLOW_TF_Q regions); its salvage is
  // ~N/3, so its default pool is N/2
  const int64_t n = e - s;
  const bool lean = F.force < 0 && !nleaves && P.Q < PM_FLOW_TF_Q && (scratch_records == 0 || scratch_records >= n / 2);
  if (lean) F.force = 0;
  // salvage pool, phase matched to the caller's (16-byte aligned) arrays
  // a prescribed layout has no fallback engine: its pool holds any salvage (<= every slot);
  // otherwise the caller's budget (scratch_records > 0) or the default N / PM_FLOW_POOL_DIV
  F.pool_cap = nleaves ? n + 32 * T + 16 * K
                       : scratch_records > 0 ? scratch_records : n / (lean ? 2 : PM_FLOW_POOL_DIV) + 32 * T;
  const size_t pk = (size_t)align_up(F.pool_cap * ks + 16, 256);
  rc = ensure(&ctx->fpool, &ctx->fpool_bytes, pk + (size_t)(w ? F.pool_cap * w + 16 : 0));
  if (rc) return rc;
  // same 16-byte phase as the caller's arrays (pool entries are 16-record aligned)
  F.pool_keys = static_cast<char*>(ctx->fpool) + ((uintptr_t)keys & 15);
  F.pool_pay = reinterpret_cast<uint8_t*>(static_cast<char*>(ctx->fpool) + pk + (w ? ((uintptr_t)payload & 15) : 0));
  P.stats = ctx->ctl->stats;
  P.ticket = &ctx->ctl->ticket_.v;
  P.err = &ctx->ctl->err_.v;
  P.noop = &ctx->ctl->noop_.v;
  P.need_space = &ctx->ctl->need_space_.v;
  // the bounded-pool engine, gated on the plan's overflow word, runs on a side
  // stream forked right after the plan: its five gated launches (~16 us of launch
  // and exit when the flow engine runs) overlap the salvage copy and the merge
  // instead of trailing them; the caller's stream joins it at the end.  The
  // flow kernels exit at once when the word is set, so the two never both move data.
  if (!ctx->fside) {
    PM_CUDA(cudaStreamCreateWithFlags(&ctx->fside, cudaStreamNonBlocking));
    PM_CUDA(cudaEventCreateWithFlags(&ctx->ffork, cudaEventDisableTiming));
    PM_CUDA(cudaEventCreateWithFlags(&ctx->fjoin, cudaEventDisableTiming));
  }
  // plan (splits, order, salvage, tickets) and merge
  if (ctx->timing) PM_CUDA(cudaEventRecord(ctx->ev[0], st));
  ce = ks == 4 ? launch_flow<int32_t>(F, grid, smem, ctx->num_sms, plan_bps, st, ctx->timing ? ctx->ev[1] : nullptr,
                                      ctx->timing ? ctx->ev[3] : nullptr, ctx->ffork)
               : launch_flow<int64_t>(F, grid, smem, ctx->num_sms, plan_bps, st, ctx->timing ? ctx->ev[1] : nullptr,
                                      ctx->timing ? ctx->ev[3] : nullptr, ctx->ffork);
  ctx->ev_mid = ctx->timing;
  if (ce == cudaErrorCooperativeLaunchTooLarge && !nleaves) {
    // the cooperative plan grid cannot be co-resident (SMs taken by other work, a
    // partitioned GPU): nothing was launched -- the bounded-pool engine needs no
    // co-residency (its persistent grid only needs forward progress)
    cudaGetLastError();
    const int fm = ctx->flow_mode;
    ctx->flow_mode = 0;
    const int rc2 = run_engine(ctx, keys, ks, payload, w, s, m, e, MODE_MERGE, scratch_records, st);
    ctx->flow_mode = fm;
    return rc2;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "k_flow launch");
  if (ctx->timing) {
    PM_CUDA(cudaEventRecord(ctx->ev[2], st));
    ctx->ev_recorded = true;
  }
  PM_CUDA(cudaStreamWaitEvent(ctx->fside, ctx->ffork, 0));
  rc = run_engine(ctx, keys, ks, payload, w, s, m, e, MODE_MERGE, scratch_records, ctx->fside, nullptr, nullptr,
                  nullptr, nullptr, reinterpret_cast<const int32_t*>(&F.fc[FC_FAIL]));
  if (rc) return rc;
  // a pure rotation (every B key below every A key) whose salvage overflows the pool
  // (N/2 for equal runs) takes a gated block exchange instead of the bounded-pool
  // engine: equal runs one block swap (2 N w of traffic), otherwise three streaming
  // reversals (4 N w); neither needs workspace
  if (!nleaves) {
    const int32_t* rg = reinterpret_cast<const int32_t*>(&F.fc[FC_ROTFAIL]);
    if (m - s == e - m)
      ce = launch_swap_blocks(keys, ks, payload, w, s, m - s, ctx->num_sms, ctx->fside, rg);
    else if (PM_GRIES_MILLS)
      ce = ks == 4 ? launch_block_exchange<int32_t>(keys, payload, w, s, m - s, e - m, ctx->num_sms, ctx->fside, rg)
                   : launch_block_exchange<int64_t>(keys, payload, w, s, m - s, e - m, ctx->num_sms, ctx->fside, rg);
    else
      ce = ks == 4 ? launch_rotate<int32_t>(keys, payload, w, s, m - s, e - m, ctx->num_sms, ctx->fside, rg)
                   : launch_rotate<int64_t>(keys, payload, w, s, m - s, e - m, ctx->num_sms, ctx->fside, rg);
    if (ce != cudaSuccess) return cuda_fail(ce, "block exchange launch (gated)");
  }
  PM_CUDA(cudaEventRecord(ctx->fjoin, ctx->fside));
  PM_CUDA(cudaStreamWaitEvent(st, ctx->fjoin, 0));
  return PM_OK;
}

static int check_common(pm_ctx* ctx, const void* keys, int ks, const void* payload, int64_t w) {
  if (!ctx) return fail(PM_ERR_ARG, "null context");
  if (ks != 4 && ks != 8) return fail(PM_ERR_ARG, "key_bytes must be 4 or 8");
  if (!keys) return fail(PM_ERR_ARG, "null keys");
  if (((uintptr_t)keys) % ks) return fail(PM_ERR_ARG, "keys pointer not aligned to key size");
  if (w < 0) return fail(PM_ERR_ARG, "negative payload width");
  if (w > 0 && !payload) return fail(PM_ERR_ARG, "null payload with nonzero width");
  return PM_OK;
}

// Stable merge path on host arrays: number of A records among the first d outputs
// (A wins ties).  Reads ~2*log2(n) records of the (pinned) host arrays.
template <typename KT>
static int64_t host_split(const KT* A, int64_t la, const KT* B, int64_t lb, int64_t d) {
  int64_t lo = std::max<int64_t>(0, d - lb), hi = std::min(d, la);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// The host side of pm_merge_host (no device calls; pm_debug_host_plan exposes it
// to the CPU tests).  The identity trim: the A prefix with keys <= B[0] and the B
// suffix with keys >= A[last] (A first on ties) are already on their output
// positions and never cross PCIe.  Then output chunks [d_k, d_{k+1}) of the
// trimmed job with their stable merge-path splits a_k (read from the host arrays
// before anything is written back), and free_at[k]: the first upload j >= k
// (uploads in merge order: upload j brings A[a_j, a_{j+1}) and B[b_j, b_{j+1}))
// after which no record of chunk k's output range is still to be uploaded.
struct HostPlan {
  bool nothing = false;
  int64_t start = 0, end = 0;
  std::vector<int64_t> dk, ak;
  std::vector<int> free_at;
};
template <typename KT>
static HostPlan host_plan_t(const KT* keys, int64_t start, int64_t middle, int64_t end, int64_t min_chunk, int chunks) {
  HostPlan p;
  if (middle == start || middle == end) {
    p.nothing = true;
    return p;
  }
  const KT* A = keys + start;
  const KT* B = keys + middle;
  const int64_t a_lo = std::upper_bound(A, A + (middle - start), B[0]) - A;
  const int64_t b_hi = std::lower_bound(B, B + (end - middle), A[middle - start - 1]) - B;
  if (a_lo == middle - start || b_hi == 0) {  // already in order (srecpar.py:56-57): nothing moves
    p.nothing = true;
    return p;
  }
  p.start = start + a_lo;
  p.end = middle + b_hi;
  const int64_t n = p.end - p.start, la = middle - p.start, lb = p.end - middle;
  const KT* X = keys + p.start;
  const int64_t chunk = std::max<int64_t>(min_chunk, (n + chunks - 1) / chunks);
  for (int64_t d = 0; d < n; d += chunk) p.dk.push_back(d);  // (geometric end ramps: no gain measured)
  p.dk.push_back(n);
  const int nch = (int)p.dk.size() - 1;
  p.ak.resize(nch + 1);
  for (int k = 0; k <= nch; ++k) p.ak[k] = host_split(X, la, X + la, lb, p.dk[k]);
  p.free_at.resize(nch);
  for (int k = 0; k < nch; ++k) {
    // A positions in the range: [d_k, min(d_{k+1}, la)); B positions: [max(d_k, la), d_{k+1}) - la
    const int64_t needA = p.dk[k] < la ? std::min(p.dk[k + 1], la) : 0;
    const int64_t needB = std::max<int64_t>(p.dk[k + 1] - la, 0);
    int j = k;
    while (j + 1 < nch && (p.ak[j + 1] < needA || (p.dk[j + 1] - p.ak[j + 1]) < needB)) ++j;
    p.free_at[k] = j;
  }
  return p;
}
static HostPlan host_plan(const void* keys, int key_bytes, int64_t start, int64_t middle, int64_t end,
                          int64_t min_chunk, int chunks) {
  return key_bytes == 4 ? host_plan_t(static_cast<const int32_t*>(keys), start, middle, end, min_chunk, chunks)
                        : host_plan_t(static_cast<const int64_t*>(keys), start, middle, end, min_chunk, chunks);
}

namespace pm {
static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace pm

extern "C" {

int pm_version(void) { return 100; }

int pm_launch_count(int64_t* out) {
  if (!out) return fail(PM_ERR_ARG, "bad arguments");
  *out = pm::g_launches.load(std::memory_order_relaxed);
  return PM_OK;
}

int pm_debug_stats(pm_ctx* ctx, uint64_t* host_out64) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !host_out64) return fail(PM_ERR_ARG, "bad arguments");
  PM_CUDA(cudaDeviceSynchronize());
  Ctl h;
  PM_CUDA(cudaMemcpy(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 64; ++i) host_out64[i] = h.stats[i];
  return PM_OK;
}

int pm_debug_splits(pm_ctx* ctx, int64_t* host_out, int64_t n) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !host_out || n < 0) return fail(PM_ERR_ARG, "bad arguments");
  PM_CUDA(cudaDeviceSynchronize());
  PM_CUDA(cudaMemcpy(host_out, ctx->ws, (size_t)n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return PM_OK;
}

// A peer block (mapped through CUDA IPC) on another device: enable P2P access to that
// device from this context's device once (the IPC mapping itself is made in the
// owning device's context, so kernels here need the peer access explicitly).
static int ensure_peer_access(pm_ctx* ctx, const void* p) {
  cudaPointerAttributes at{};
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return PM_OK;  // (not a CUDA allocation the runtime knows: the kernel's loads decide)
  }
  const int dev = at.device;
  if (at.type != cudaMemoryTypeDevice || dev == ctx->device || dev < 0 || dev >= 64) return PM_OK;
  if (ctx->peer_on & (1ull << dev)) return PM_OK;
  int can = 0;
  PM_CUDA(cudaDeviceCanAccessPeer(&can, ctx->device, dev));
  if (!can) return fail(PM_ERR_UNSUPPORTED, "a peer block lives on a device without P2P access from this one");
  const cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  cudaGetLastError();
  ctx->peer_on |= 1ull << dev;
  return PM_OK;
}

int pm_peer_splits(pm_ctx* ctx, const void* const* peer_keys, int world, int64_t block, int64_t len_a, int key_bytes,
                   const int64_t* diags, int nd, int64_t* out_a, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !peer_keys || world < 1 || block < 0 || (key_bytes != 4 && key_bytes != 8) || nd < 0 || (nd && (!diags || !out_a)))
    return fail(PM_ERR_ARG, "bad pm_peer_splits arguments");
  const int64_t N = (int64_t)world * block;
  if (len_a < 0 || len_a > N) return fail(PM_ERR_ARG, "len_a outside [0, world*block]");
  for (int i = 0; i < nd; ++i)
    if (diags[i] < 0 || diags[i] > N) return fail(PM_ERR_ARG, "diagonal outside [0, world*block]");
  for (int k = 0; k < world; ++k)
    if (block && !peer_keys[k]) return fail(PM_ERR_ARG, "null peer block");
  if (nd == 0) return PM_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> lk(ctx->mu);
  for (int k = 0; k < world && block; ++k) {
    const int prc = ensure_peer_access(ctx, peer_keys[k]);
    if (prc) return prc;
  }
  use_stream(ctx, st);
  const size_t o_q = (size_t)align_up((int64_t)world * 8, 256), o_out = o_q + (size_t)align_up((int64_t)nd * 16, 256);
  int rc = ensure(&ctx->peer, &ctx->peer_bytes, o_out + (size_t)nd * 8);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->peer);
  const void** dtab = reinterpret_cast<const void**>(base);
  int64_t* dq = reinterpret_cast<int64_t*>(base + o_q);
  int64_t* dout = reinterpret_cast<int64_t*>(base + o_out);
  std::vector<int64_t> q(2 * (size_t)nd);
  for (int i = 0; i < nd; ++i) {
    q[2 * i] = 0;  // stable split (A wins ties)
    q[2 * i + 1] = diags[i];
  }
  PM_CUDA(cudaMemcpyAsync(dtab, peer_keys, (size_t)world * sizeof(void*), cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(dq, q.data(), q.size() * 8, cudaMemcpyHostToDevice, st));
  const int64_t la = len_a, lb = N - len_a;
  cudaError_t ce = key_bytes == 4 ? launch_peer_queries<int32_t>(dtab, block, la, lb, dq, nd, dout, st)
                                  : launch_peer_queries<int64_t>(dtab, block, la, lb, dq, nd, dout, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "k_peer_queries launch");
  PM_CUDA(cudaMemcpyAsync(out_a, dout, (size_t)nd * 8, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

int pm_merge_peers(pm_ctx* ctx, const void* const* peer_keys, const void* const* peer_payload, int world, int rank,
                   int64_t block, int64_t len_a, int key_bytes, int64_t width, void* out_keys, void* out_payload,
                   void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !peer_keys || world < 1 || rank < 0 || rank >= world || block < 0 || (key_bytes != 4 && key_bytes != 8) ||
      width < 0 || !out_keys || (width && (!peer_payload || !out_payload)))
    return fail(PM_ERR_ARG, "bad pm_merge_peers arguments");
  const int64_t N = (int64_t)world * block;
  if (len_a < 0 || len_a > N) return fail(PM_ERR_ARG, "len_a outside [0, world*block]");
  for (int k = 0; k < world; ++k)
    if (block && (!peer_keys[k] || (width && !peer_payload[k]))) return fail(PM_ERR_ARG, "null peer block");
  if (block == 0) return PM_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t la = len_a, lb = N - len_a, d0 = (int64_t)rank * block, d1 = d0 + block;
  std::lock_guard<std::mutex> lk(ctx->mu);
  for (int k = 0; k < world; ++k) {
    int prc = ensure_peer_access(ctx, peer_keys[k]);
    if (!prc && width) prc = ensure_peer_access(ctx, peer_payload[k]);
    if (prc) return prc;
  }
  use_stream(ctx, st);
  const int maxq = 2 + 2 * (world + 1);
  const size_t o_q = (size_t)align_up((int64_t)world * 8, 256), o_out = o_q + (size_t)maxq * 16;
  int rc = ensure(&ctx->peer, &ctx->peer_bytes, o_out + (size_t)maxq * 8);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->peer);
  const void** dtab = reinterpret_cast<const void**>(base);
  int64_t* dq = reinterpret_cast<int64_t*>(base + o_q);
  int64_t* dout = reinterpret_cast<int64_t*>(base + o_out);
  PM_CUDA(cudaMemcpyAsync(dtab, peer_keys, (size_t)world * sizeof(void*), cudaMemcpyHostToDevice, st));
  auto run = [&](const std::vector<int64_t>& q, std::vector<int64_t>& ans) -> int {
    const int nq = (int)(q.size() / 2);
    ans.assign(nq, 0);
    if (!nq) return PM_OK;
    PM_CUDA(cudaMemcpyAsync(dq, q.data(), q.size() * 8, cudaMemcpyHostToDevice, st));
    cudaError_t ce = key_bytes == 4 ? launch_peer_queries<int32_t>(dtab, block, la, lb, dq, nq, dout, st)
                                    : launch_peer_queries<int64_t>(dtab, block, la, lb, dq, nq, dout, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "k_peer_queries launch");
    PM_CUDA(cudaMemcpyAsync(ans.data(), dout, (size_t)nq * 8, cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaStreamSynchronize(st));
    return PM_OK;
  };
  // (1) rank r's pieces: A[a0, a1), B[b0, b1)
  std::vector<int64_t> ans;
  rc = run({0, d0, 0, d1}, ans);
  if (rc) return rc;
  const int64_t a0 = ans[0], a1 = ans[1], b0 = d0 - a0, b1 = d1 - a1;
  // (2) the output position of every block boundary strictly inside a piece:
  //     A[i] lands at i + #(B < A[i]); B[j] at j + #(A <= B[j])
  std::vector<int64_t> q, ai, bj;
  for (int64_t g = (a0 / block + 1) * block; g < a1; g += block) {
    ai.push_back(g);
    q.insert(q.end(), {1, g});
  }
  for (int64_t g = ((la + b0) / block + 1) * block; g < la + b1; g += block) {
    bj.push_back(g - la);
    q.insert(q.end(), {2, g - la});
  }
  rc = run(q, ans);
  if (rc) return rc;
  struct Cut { int64_t d, a; };
  std::vector<Cut> cuts{{d0, a0}, {d1, a1}};
  for (size_t k = 0; k < ai.size(); ++k) cuts.push_back({ai[k] + ans[k], ai[k]});
  for (size_t k = 0; k < bj.size(); ++k) cuts.push_back({bj[k] + ans[ai.size() + k], ans[ai.size() + k]});
  std::sort(cuts.begin(), cuts.end(), [](const Cut& x, const Cut& y) { return x.d < y.d; });
  // (3) one copy-mode merge per sub-range: each piece inside one block
  auto at = [&](const void* const* tab, int64_t g, int64_t rb) -> const char* {
    const int64_t k = std::min<int64_t>(g / block, world - 1);
    return static_cast<const char*>(tab[k]) + (g - k * block) * rb;
  };
  for (size_t k = 0; k + 1 < cuts.size(); ++k) {
    const int64_t c0 = cuts[k].d, c1 = cuts[k + 1].d;
    if (c1 <= c0) continue;
    const int64_t sa0 = cuts[k].a, sa1 = cuts[k + 1].a, nA = sa1 - sa0, nB = (c1 - c0) - nA;
    const int64_t sb0 = c0 - sa0;
    const char* ka = at(peer_keys, nA ? sa0 : 0, key_bytes);
    const char* kb = at(peer_keys, nB ? la + sb0 : 0, key_bytes);
    const char* pa = width ? at(peer_payload, nA ? sa0 : 0, width) : nullptr;
    const char* pb = width ? at(peer_payload, nB ? la + sb0 : 0, width) : nullptr;
    rc = run_engine(ctx, const_cast<char*>(ka), key_bytes, const_cast<char*>(pa), width, 0, nA, nA + nB, MODE_MERGE, 0,
                    st, static_cast<char*>(out_keys) + (c0 - d0) * key_bytes,
                    width ? static_cast<char*>(out_payload) + (c0 - d0) * width : nullptr, kb, pb);
    if (rc) return rc;
  }
  return PM_OK;
}

int pm_ipc_handle(void* device_ptr, void* out_handle) {
  if (!device_ptr || !out_handle) return fail(PM_ERR_ARG, "bad pm_ipc_handle arguments");
  cudaIpcMemHandle_t h;
  PM_CUDA(cudaIpcGetMemHandle(&h, device_ptr));
  std::memcpy(out_handle, &h, sizeof(h));
  return PM_OK;
}

int pm_ipc_open(const void* handle, void** out_ptr) {
  if (!handle || !out_ptr) return fail(PM_ERR_ARG, "bad pm_ipc_open arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  PM_CUDA(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PM_OK;
}

int pm_ipc_close(void* ptr) {
  if (!ptr) return fail(PM_ERR_ARG, "null pointer");
  PM_CUDA(cudaIpcCloseMemHandle(ptr));
  return PM_OK;
}

int pm_debug_engine_only(pm_ctx* ctx, int on) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx) return fail(PM_ERR_ARG, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ctx->engine_only = on != 0;
  return PM_OK;
}

int pm_debug_permute_rows(pm_ctx* ctx, void* payload, int64_t width, const int32_t* idx, int64_t n, int32_t cut_every,
                          void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || (n && (!payload || !idx)) || width <= 0 || n < 0 || n >= INT32_MAX || cut_every < 1)
    return fail(PM_ERR_ARG, "bad pm_debug_permute_rows arguments");
  if (n == 0) return PM_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  use_stream(ctx, static_cast<cudaStream_t>(stream));
  return permute_rows(ctx, static_cast<uint8_t*>(payload), width, idx, n, cut_every, static_cast<cudaStream_t>(stream));
}

int pm_debug_order(int64_t Q, int64_t qc, int64_t t, int64_t* out4) {
  if (Q < 1 || qc < 0 || qc >= Q || t < 0 || t >= Q || !out4) return fail(PM_ERR_ARG, "bad order arguments");
  TwoFront tf{Q, qc};
  out4[0] = tf.region_of_ticket(t);
  out4[1] = tf.order(out4[0]);
  tf.window(t, out4[2], out4[3]);
  return PM_OK;
}

const char* pm_last_error(void) { return g_last_error.c_str(); }

int pm_ctx_create(int device, pm_ctx** out) {
  if (!out) return fail(PM_ERR_ARG, "null out");
  int ndev = 0;
  PM_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PM_ERR_ARG, "no such device");
  DeviceGuard dg_(device);  // (the caller's current device is restored)
  pm_ctx* c = new pm_ctx();
  c->device = device;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaGetDeviceProperties");
  }
  c->num_sms = prop.multiProcessorCount;
  e = cudaMalloc(reinterpret_cast<void**>(&c->ctl), sizeof(Ctl));
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(ctl)");
  }
  cudaMemset(c->ctl, 0, sizeof(Ctl));
  *out = c;
  return PM_OK;
}

int pm_ctx_destroy(pm_ctx* ctx) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx) return PM_OK;
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->xev) cudaEventDestroy(ctx->xev);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->scr) cudaFree(ctx->scr);
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->buf) cudaFree(ctx->buf);
  if (ctx->wide) cudaFree(ctx->wide);
  if (ctx->wperm) cudaFree(ctx->wperm);
  if (ctx->peer) cudaFree(ctx->peer);
  if (ctx->fws) cudaFree(ctx->fws);
  if (ctx->fpool) cudaFree(ctx->fpool);
  for (auto& x : ctx->hs)
    if (x) cudaStreamDestroy(x);
  for (auto& x : ctx->hev)
    if (x) cudaEventDestroy(x);
  if (ctx->fside) cudaStreamDestroy(ctx->fside);
  if (ctx->ffork) cudaEventDestroy(ctx->ffork);
  if (ctx->fjoin) cudaEventDestroy(ctx->fjoin);
  for (auto& x : ctx->hup) cudaEventDestroy(x);
  for (auto& x : ctx->hdn) cudaEventDestroy(x);
  if (ctx->hstage) cudaFreeHost(ctx->hstage);
  if (ctx->ctl) cudaFree(ctx->ctl);
  delete ctx;
  return PM_OK;
}

int pm_debug_flow(pm_ctx* ctx, int mode) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || mode < 0 || mode > 4) return fail(PM_ERR_ARG, "bad pm_debug_flow arguments");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ctx->flow_mode = mode;
  return PM_OK;
}

int pm_set_timing(pm_ctx* ctx, int on) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx) return fail(PM_ERR_ARG, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (on && !ctx->ev[0])
    for (auto& e : ctx->ev) PM_CUDA(cudaEventCreate(&e));
  ctx->timing = on != 0;
  ctx->ev_recorded = false;
  return PM_OK;
}

int pm_kernel_ms(pm_ctx* ctx, float* plan_ms, float* engine_ms) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !plan_ms || !engine_ms) return fail(PM_ERR_ARG, "null argument");
  if (!ctx->ev_recorded) return fail(PM_ERR_ARG, "no timed launch recorded (pm_set_timing first)");
  PM_CUDA(cudaEventSynchronize(ctx->ev[2]));
  PM_CUDA(cudaEventElapsedTime(plan_ms, ctx->ev[0], ctx->ev[1]));
  PM_CUDA(cudaEventElapsedTime(engine_ms, ctx->ev[1], ctx->ev[2]));
  return PM_OK;
}

int pm_kernel_ms_detail(pm_ctx* ctx, float* out4) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !out4) return fail(PM_ERR_ARG, "null argument");
  if (!ctx->ev_recorded) return fail(PM_ERR_ARG, "no timed launch recorded (pm_set_timing first)");
  PM_CUDA(cudaEventSynchronize(ctx->ev[2]));
  PM_CUDA(cudaEventElapsedTime(&out4[0], ctx->ev[0], ctx->ev[1]));
  PM_CUDA(cudaEventElapsedTime(&out4[3], ctx->ev[0], ctx->ev[2]));
  if (ctx->ev_mid) {
    PM_CUDA(cudaEventElapsedTime(&out4[1], ctx->ev[1], ctx->ev[3]));
    PM_CUDA(cudaEventElapsedTime(&out4[2], ctx->ev[3], ctx->ev[2]));
  } else {
    out4[1] = 0.f;
    PM_CUDA(cudaEventElapsedTime(&out4[2], ctx->ev[1], ctx->ev[2]));
  }
  return PM_OK;
}

int pm_merge_copy(pm_ctx* ctx, const void* src_keys, const void* src_payload, void* dst_keys, void* dst_payload,
                  int key_bytes, int64_t width, int64_t len_a, int64_t len_b, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  int rc = check_common(ctx, src_keys, key_bytes, src_payload, width);
  if (rc) return rc;
  rc = check_common(ctx, dst_keys, key_bytes, dst_payload, width);
  if (rc) return rc;
  if (len_a < 0 || len_b < 0) return fail(PM_ERR_ARG, "negative run length");
  const int64_t n = len_a + len_b;
  auto overlap = [n](const void* a, const void* b, int64_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + (uintptr_t)(n * bytes) && y < x + (uintptr_t)(n * bytes);
  };
  if (n && (overlap(src_keys, dst_keys, key_bytes) || (width && overlap(src_payload, dst_payload, width))))
    return fail(PM_ERR_ARG, "source and destination overlap (use pm_merge for in-place)");
  if (n == 0) return PM_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  use_stream(ctx, static_cast<cudaStream_t>(stream));
  return run_engine(ctx, const_cast<void*>(src_keys), key_bytes, const_cast<void*>(src_payload), width, 0, len_a, n,
                    MODE_MERGE, 0, static_cast<cudaStream_t>(stream), dst_keys, width ? dst_payload : nullptr);
}

int pm_merge(pm_ctx* ctx, void* keys, int key_bytes, void* payload, int64_t width, int64_t start, int64_t middle,
             int64_t end, int64_t scratch_records, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  int rc = check_common(ctx, keys, key_bytes, payload, width);
  if (rc) return rc;
  if (!(0 <= start && start <= middle && middle <= end))  // records.py:100-102
    return fail(PM_ERR_ARG, "need 0 <= start <= middle <= end");
  std::lock_guard<std::mutex> lk(ctx->mu);
  use_stream(ctx, static_cast<cudaStream_t>(stream));
  return run_engine(ctx, keys, key_bytes, payload, width, start, middle, end, MODE_MERGE, scratch_records,
                    static_cast<cudaStream_t>(stream));
}

int pm_reorder(pm_ctx* ctx, void* keys, int key_bytes, void* payload, int64_t width, int64_t start, int64_t end,
               const int64_t* leaf_sizes, int32_t nleaves, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  int rc = check_common(ctx, keys, key_bytes, payload, width);
  if (rc) return rc;
  if (start < 0 || end < start || nleaves < 1 || !leaf_sizes) return fail(PM_ERR_ARG, "bad pm_reorder arguments");
  int64_t tot = 0, ta = 0;
  for (int32_t i = 0; i < 2 * nleaves; ++i) {
    if (leaf_sizes[i] < 0) return fail(PM_ERR_ARG, "negative leaf slice");
    tot += leaf_sizes[i];
    if (!(i & 1)) ta += leaf_sizes[i];
  }
  if (tot != end - start) return fail(PM_ERR_ARG, "leaf slices do not cover [start, end)");
  if (end - start == 0 || ta == 0 || ta == end - start) return PM_OK;  // one run: already in place
  std::lock_guard<std::mutex> lk(ctx->mu);
  use_stream(ctx, static_cast<cudaStream_t>(stream));
  return run_flow(ctx, keys, key_bytes, payload, width, start, start + ta, end, static_cast<cudaStream_t>(stream),
                  leaf_sizes, nleaves);
}

int pm_shift(pm_ctx* ctx, void* keys, int key_bytes, void* payload, int64_t width, int64_t lo, int64_t len_a,
             int64_t len_b, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  int rc = check_common(ctx, keys, key_bytes, payload, width);
  if (rc) return rc;
  if (lo < 0 || len_a < 0 || len_b < 0) return fail(PM_ERR_ARG, "lengths must be non-negative");  // shift.py:157
  if (len_a == 0 || len_b == 0) return PM_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // equal blocks: one swap pass, every record read and written once
  if (len_a == len_b && !ctx->engine_only) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_stream(ctx, st);
    const cudaError_t e = launch_swap_blocks(keys, key_bytes, payload, width, lo, len_a, ctx->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_swap_blocks launch");
    return PM_OK;
  }
  // one small block: stash it, slide the big block over it in one pass, land the
  // stash at the far end (the reference's staged exchange, _kernels.py:46-90)
  const int64_t small = std::min(len_a, len_b), big = std::max(len_a, len_b);
  const int64_t rb = key_bytes + width;
  if (small * rb <= PM_SLIDE_STASH && !ctx->engine_only) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_stream(ctx, st);
    const int64_t ntk = (big * key_bytes + 32767) / 32768, ntp = (big * width + 32767) / 32768;
    const size_t sk = (size_t)align_up(small * key_bytes, 256), sp = (size_t)align_up(small * width, 256);
    const size_t fl = (size_t)align_up((ntk + ntp + 2) * 4, 256);
    rc = ensure(&ctx->buf, &ctx->buf_bytes, sk + sp + fl);
    if (rc) return rc;
    char* stash_k = static_cast<char*>(ctx->buf);
    char* stash_p = stash_k + sk;
    int32_t* flags = reinterpret_cast<int32_t*>(stash_p + sp);
    char* K = static_cast<char*>(keys);
    char* Pp = static_cast<char*>(payload);
    const bool a_small = len_a <= len_b;
    // the small block's first record, the big block's first record, where the stash lands
    const int64_t xs = a_small ? lo : lo + len_a, xb = a_small ? lo + len_a : lo;
    const int64_t xdst = a_small ? lo + len_b : lo;
    PM_CUDA(cudaMemcpyAsync(stash_k, K + xs * key_bytes, (size_t)(small * key_bytes), cudaMemcpyDeviceToDevice, st));
    if (width) PM_CUDA(cudaMemcpyAsync(stash_p, Pp + xs * width, (size_t)(small * width), cudaMemcpyDeviceToDevice, st));
    cudaError_t e = launch_slide(K, xb * key_bytes, big * key_bytes, small * key_bytes, !a_small, flags,
                                 flags + ntk + ntp, &ctx->ctl->err_.v, ctx->num_sms, st);
    if (e == cudaSuccess && width)
      e = launch_slide(Pp, xb * width, big * width, small * width, !a_small, flags + ntk, flags + ntk + ntp + 1,
                       &ctx->ctl->err_.v, ctx->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_slide launch");
    PM_CUDA(cudaMemcpyAsync(K + xdst * key_bytes, stash_k, (size_t)(small * key_bytes), cudaMemcpyDeviceToDevice, st));
    if (width) PM_CUDA(cudaMemcpyAsync(Pp + xdst * width, stash_p, (size_t)(small * width), cudaMemcpyDeviceToDevice, st));
    return PM_OK;
  }
  // Gries-Mills block swaps (the reference's linear shift) while the smaller block
  // is >= 1/16 of the exchange, three streaming reversals for the rest (pm_rotate.cu);
  // no workspace
  const cudaError_t e =
      PM_GRIES_MILLS
          ? (key_bytes == 4 ? launch_block_exchange<int32_t>(keys, payload, width, lo, len_a, len_b, ctx->num_sms, st)
                            : launch_block_exchange<int64_t>(keys, payload, width, lo, len_a, len_b, ctx->num_sms, st))
          : (key_bytes == 4 ? launch_rotate<int32_t>(keys, payload, width, lo, len_a, len_b, ctx->num_sms, st)
                            : launch_rotate<int64_t>(keys, payload, width, lo, len_a, len_b, ctx->num_sms, st));
  if (e != cudaSuccess) return cuda_fail(e, "k_reverse launch");
  return PM_OK;
}

int pm_find_median(pm_ctx* ctx, const void* a, const void* b, int key_bytes, int64_t la, int64_t lb, int64_t* out2,
                   void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx) return fail(PM_ERR_ARG, "null context");
  if (key_bytes != 4 && key_bytes != 8) return fail(PM_ERR_ARG, "key_bytes must be 4 or 8");
  if (la < 0 || lb < 0 || !out2 || (la && !a) || (lb && !b)) return fail(PM_ERR_ARG, "bad find_median arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = key_bytes == 4 ? launch_find_median<int32_t>(a, b, la, lb, out2, st)
                                 : launch_find_median<int64_t>(a, b, la, lb, out2, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_find_median launch");
  return PM_OK;
}

int pm_find_splits(pm_ctx* ctx, const void* a, const void* b, int key_bytes, int64_t la, int64_t lb,
                   const int64_t* diags, int64_t nd, int64_t* out_a, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx) return fail(PM_ERR_ARG, "null context");
  if (key_bytes != 4 && key_bytes != 8) return fail(PM_ERR_ARG, "key_bytes must be 4 or 8");
  if (la < 0 || lb < 0 || nd < 0 || (nd && (!diags || !out_a)) || (la && !a) || (lb && !b))
    return fail(PM_ERR_ARG, "bad find_splits arguments");
  if (nd == 0) return PM_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int grid = (int)std::min<int64_t>((nd * 32 + 255) / 256, (int64_t)ctx->num_sms * 8);
  cudaError_t e = key_bytes == 4 ? launch_find_splits<int32_t>(a, b, la, lb, diags, nd, out_a, grid, st)
                                 : launch_find_splits<int64_t>(a, b, la, lb, diags, nd, out_a, grid, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_find_splits launch");
  return PM_OK;
}

int pm_plan_intervals(pm_ctx* ctx, const void* keys, int key_bytes, int64_t start, int64_t middle, int64_t end,
                      int32_t threads, int64_t* nodes, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  int rc = check_common(ctx, keys, key_bytes, nullptr, 0);
  if (rc) return rc;
  if (threads < 1 || (threads & (threads - 1)))  // soptmov.py:87-90
    return fail(PM_ERR_ARG, "worker count must be a power of two >= 1");
  if (!(0 <= start && start <= middle && middle <= end) || !nodes) return fail(PM_ERR_ARG, "bad plan arguments");
  int32_t levels = 0;
  while ((1 << (levels + 1)) <= threads) ++levels;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = key_bytes == 4 ? launch_plan_intervals<int32_t>(keys, start, middle, end, levels, nodes, st)
                                 : launch_plan_intervals<int64_t>(keys, start, middle, end, levels, nodes, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_plan_intervals launch");
  return PM_OK;
}

int pm_status(pm_ctx* ctx, void* stream, uint64_t* stats) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx) return fail(PM_ERR_ARG, "null context");
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_stream(ctx, static_cast<cudaStream_t>(stream));  // the status covers the latest call on any stream
  }
  PM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  Ctl h;
  PM_CUDA(cudaMemcpy(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  if (stats)
    for (int i = 0; i < 16; ++i) stats[i] = h.stats[i];
  if (h.err_.v != 0) {
    int32_t zero = 0;
    cudaMemcpy(&ctx->ctl->err_.v, &zero, sizeof(zero), cudaMemcpyHostToDevice);
    const char* what = h.err_.v == PM_ERR_TIMEOUT   ? "device wait exceeded its bound"
                       : h.err_.v == PM_ERR_NOSPACE ? "salvage space exhausted"
                                                 : "device invariant violated";
    return fail(h.err_.v, std::string("merge engine: ") + what);
  }
  return PM_OK;
}

int pm_debug_host_plan(const void* keys_host, int key_bytes, int64_t start, int64_t middle, int64_t end,
                       int64_t min_chunk, int32_t chunks, int64_t* out_span, int64_t* out_d, int64_t* out_a,
                       int32_t* out_free, int32_t cap, int32_t* out_nch) {
  if (!keys_host || (key_bytes != 4 && key_bytes != 8) || !(0 <= start && start <= middle && middle <= end) ||
      min_chunk < 1 || chunks < 1 || !out_span || !out_nch)
    return fail(PM_ERR_ARG, "bad pm_debug_host_plan arguments");
  const HostPlan p = host_plan(keys_host, key_bytes, start, middle, end, min_chunk, chunks);
  out_span[0] = p.nothing ? -1 : p.start;
  out_span[1] = p.nothing ? -1 : p.end;
  const int nch = p.nothing ? 0 : (int)p.dk.size() - 1;
  *out_nch = nch;
  if (nch > cap) return fail(PM_ERR_ARG, "pm_debug_host_plan: more chunks than the output arrays hold");
  for (int k = 0; k <= nch && nch; ++k) {
    if (out_d) out_d[k] = p.dk[k];
    if (out_a) out_a[k] = p.ak[k];
    if (out_free && k < nch) out_free[k] = p.free_at[k];
  }
  return PM_OK;
}

// Host-buffer merge, pipelined over output chunks on three streams: H2D of
// chunk k's inputs in merge order (A[a_k, a_{k+1}) and B[b_k, b_{k+1})), the
// out-of-place device merge of chunk k (copy mode), and D2H of chunk k as soon
// as it is merged.  The in-place host semantics: chunk k's output range
// [d_k, d_{k+1}) may hold records not uploaded yet -- every such range is free
// only after upload ready_k >= k (for uniform runs the first half of the output
// frees at half the upload rate).  Writing those chunks back directly would
// stall the D2H stream or force uploads ahead of the merge (1.25 N / R for
// uniform runs); instead they land in a pinned host staging buffer and host
// threads move each into place once its range has been uploaded.  Both PCIe
// directions then run at full rate for the whole call (~N / R).
int pm_merge_host(pm_ctx* ctx, void* keys_host, int key_bytes, void* payload_host, int64_t width, int64_t start,
                  int64_t middle, int64_t end, void* stream) {
  DeviceGuard dg_(ctx ? ctx->device : -1);
  if (!ctx || !keys_host || (key_bytes != 4 && key_bytes != 8) || width < 0 || (width && !payload_host))
    return fail(PM_ERR_ARG, "bad pm_merge_host arguments");
  if (!(0 <= start && start <= middle && middle <= end)) return fail(PM_ERR_ARG, "need 0 <= start <= middle <= end");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#ifndef PM_HOST_CHUNKS
#define PM_HOST_CHUNKS 48  // output chunks of the host-buffer pipeline (48: 103 ms, 96: 104, 192: 108 at 2^30 int32)
#endif
  HostPlan plan = host_plan(keys_host, key_bytes, start, middle, end, (int64_t)1 << 21, PM_HOST_CHUNKS);
  if (plan.nothing) return PM_OK;
  start = plan.start;
  end = plan.end;
  const int64_t n = end - start, la = middle - start;
  char* hk = static_cast<char*>(keys_host) + start * key_bytes;
  char* hp = width ? static_cast<char*>(payload_host) + start * width : nullptr;
  const size_t kb = (size_t)align_up(n * key_bytes, 256), pb = (size_t)align_up(n * width, 256);
  int rc;
  // host threads calling concurrently (the reference's pool runs leaf merges in
  // parallel) share the staging buffer and the pipeline streams: one at a time
  std::lock_guard<std::mutex> host_lk(ctx->host_mu);
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    rc = ensure(&ctx->stage, &ctx->stage_bytes, 2 * (kb + pb) + 256);
    if (!rc && !ctx->hs[0]) {
      for (auto& x : ctx->hs) PM_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
      for (auto& x : ctx->hev) PM_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
  }
  if (rc) return rc;
  char* dxk = static_cast<char*>(ctx->stage);  // input copy X
  char* dxp = dxk + kb;
  char* dok = dxp + pb;                        // merged output O
  char* dop = dok + kb;
  cudaStream_t sH = ctx->hs[0], sC = ctx->hs[1], sD = ctx->hs[2];
  // order after the caller's stream
  PM_CUDA(cudaEventRecord(ctx->hev[0], st));
  PM_CUDA(cudaStreamWaitEvent(sH, ctx->hev[0], 0));
  const std::vector<int64_t>& dk = plan.dk;
  const std::vector<int64_t>& ak = plan.ak;
  const int nch = (int)dk.size() - 1;
  // ready[k]: the upload after which chunk k's D2H is issued (plan.free_at, or k
  // for a chunk that goes through the staging buffer); order: the D2H issue order
  std::vector<int> ready = plan.free_at, order(nch);
  for (int k = 0; k < nch; ++k) order[k] = k;
  // chunks whose range frees after their merge go through the pinned staging
  // buffer (one grow-only allocation per context); without it (over the cap, or
  // the pinned allocation failed) they are written back directly in ready order
#ifndef PM_HOST_STAGE_MAX
#define PM_HOST_STAGE_MAX ((size_t)16 << 30)
#endif
  const size_t rec_bytes = (size_t)key_bytes + (size_t)width;
  std::vector<size_t> soff(nch, SIZE_MAX);
  size_t staged = 0;
  for (int k = 0; k < nch; ++k)
    if (ready[k] > k) {
      soff[k] = staged;
      staged += (size_t)align_up((dk[k + 1] - dk[k]) * (int64_t)rec_bytes, 256);
    }
  bool use_stage = staged > 0 && staged <= PM_HOST_STAGE_MAX;
  if (use_stage && ctx->hstage_bytes < staged) {
    if (ctx->hstage) cudaFreeHost(ctx->hstage);
    ctx->hstage = nullptr;
    ctx->hstage_bytes = 0;
    if (cudaHostAlloc(&ctx->hstage, staged, cudaHostAllocPortable) == cudaSuccess) ctx->hstage_bytes = staged;
    else {
      cudaGetLastError();
      ctx->hstage = nullptr;
      use_stage = false;
    }
  }
  while ((int)ctx->hup.size() < nch) {
    cudaEvent_t e1, e2;
    PM_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    PM_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    ctx->hup.push_back(e1);
    ctx->hdn.push_back(e2);
  }
  const std::vector<int>& free_at = plan.free_at;  // the upload after which chunk k's range is free
  std::vector<int> stg;                    // staged chunks, in the order their ranges free
  for (int k = 0; k < nch; ++k)
    if (use_stage && ready[k] > k) {
      stg.push_back(k);
      ready[k] = k;  // its D2H (into the staging buffer) leaves right after its merge
    }
  std::stable_sort(stg.begin(), stg.end(), [&](int x, int y) { return free_at[x] < free_at[y]; });
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ready[x] < ready[y]; });
  char* hs_base = static_cast<char*>(ctx->hstage);
#ifdef PM_HOST_TRACE
  // debug timeline (tools/gpu_e2e_trace.py): per chunk, upload / merge / D2H end
  std::vector<cudaEvent_t> tr(3 * nch + 1);
  for (auto& e : tr) cudaEventCreate(&e);
  cudaEventRecord(tr[3 * nch], sH);
  std::vector<double> mv_done(nch, -1);
  auto h0 = std::chrono::steady_clock::now();
#endif
  // the pipeline proper: on any failure the three streams are drained before the
  // error returns, so no transfer still writes the caller's buffers afterwards
  auto pipeline = [&]() -> int {
    auto h2d = [&](int64_t x0, int64_t x1) -> int {
      if (x1 <= x0) return PM_OK;
      PM_CUDA(cudaMemcpyAsync(dxk + x0 * key_bytes, hk + x0 * key_bytes, (x1 - x0) * key_bytes,
                              cudaMemcpyHostToDevice, sH));
      if (width)
        PM_CUDA(cudaMemcpyAsync(dxp + x0 * width, hp + x0 * width, (x1 - x0) * width, cudaMemcpyHostToDevice, sH));
      return PM_OK;
    };
    constexpr int kEv = (int)(sizeof(((pm_ctx*)nullptr)->hev) / sizeof(cudaEvent_t)) - 1;
    int next = 0;  // next chunk (in `order`) to write back
    for (int k = 0; k < nch; ++k) {
      const int64_t d0 = dk[k], a0 = ak[k], b0 = d0 - a0, d1 = dk[k + 1], a1 = ak[k + 1], b1 = d1 - a1;
      rc = h2d(a0, a1);
      if (!rc) rc = h2d(la + b0, la + b1);
      if (rc) return rc;
      PM_CUDA(cudaEventRecord(ctx->hup[k], sH));
      PM_CUDA(cudaStreamWaitEvent(sC, ctx->hup[k], 0));
#ifdef PM_HOST_TRACE
      cudaEventRecord(tr[3 * k], sH);
#endif
      {
        std::lock_guard<std::mutex> lk(ctx->mu);
        use_stream(ctx, sC);  // (the copy merges share the context's workspace with calls on other streams)
        rc = run_engine(ctx, dxk + a0 * key_bytes, key_bytes, width ? dxp + a0 * width : nullptr, width, 0, a1 - a0,
                        d1 - d0, MODE_MERGE, 0, sC, dok + d0 * key_bytes, width ? dop + d0 * width : nullptr,
                        dxk + (la + b0) * key_bytes, width ? dxp + (la + b0) * width : nullptr);
      }
      if (rc) return rc;
#ifdef PM_HOST_TRACE
      cudaEventRecord(tr[3 * k + 1], sC);
#endif
      if (next < nch && ready[order[next]] == k) {
        // merges run in order on sC: chunk k merged => uploads 0..k and merges 0..k done;
        // the event is waited on right after it is recorded, so the ring can be reused
        cudaEvent_t ec = ctx->hev[1 + k % kEv];
        PM_CUDA(cudaEventRecord(ec, sC));
        PM_CUDA(cudaStreamWaitEvent(sD, ec, 0));
        for (; next < nch && ready[order[next]] == k; ++next) {
          const int c = order[next];
          const int64_t e0 = dk[c], e1 = dk[c + 1];
          char* tk = soff[c] != SIZE_MAX && use_stage ? hs_base + soff[c] : hk + e0 * key_bytes;
          char* tp = soff[c] != SIZE_MAX && use_stage ? tk + (e1 - e0) * key_bytes : hp + e0 * width;
          PM_CUDA(cudaMemcpyAsync(tk, dok + e0 * key_bytes, (e1 - e0) * key_bytes, cudaMemcpyDeviceToHost, sD));
          if (width) PM_CUDA(cudaMemcpyAsync(tp, dop + e0 * width, (e1 - e0) * width, cudaMemcpyDeviceToHost, sD));
          if (soff[c] != SIZE_MAX && use_stage) PM_CUDA(cudaEventRecord(ctx->hdn[c], sD));
#ifdef PM_HOST_TRACE
          cudaEventRecord(tr[3 * c + 2], sD);
#endif
        }
      }
    }
    if (next != nch) return fail(PM_ERR_INTERNAL, "pm_merge_host: write-back schedule incomplete");
    PM_CUDA(cudaEventRecord(ctx->hev[0], sD));
    PM_CUDA(cudaStreamWaitEvent(st, ctx->hev[0], 0));
    if (!stg.empty()) {
      // host threads move the staged chunks into place, each once its range has
      // been uploaded and its D2H has landed.  The work is cut into pieces of at most
      // PM_HOST_PIECE bytes, taken in order from one counter: a thread that the OS
      // deschedules delays only its current piece (fixed per-thread stripes made
      // the slowest thread the critical path: 102 ms median, 129 ms outliers)
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
#ifndef PM_HOST_MOVERS
#define PM_HOST_MOVERS 4u  // more threads take host memory bandwidth from the DMA (tools/gpu_pcie_chunks.py)
#endif
#ifndef PM_HOST_PIECE
#define PM_HOST_PIECE ((int64_t)16 << 20)  // 4 MB: 103.8 ms mean, 16 MB: 102.6 (2^30 int32)
#endif
      const int nt = (int)std::min<unsigned>(PM_HOST_MOVERS, std::max(1u, hw / 2));
      struct Piece {
        int c;          // staged chunk
        char* dst;
        const char* src;
        int64_t bytes;
      };
      std::vector<Piece> pieces;
      for (int c : stg) {
        const int64_t e0 = dk[c], e1 = dk[c + 1];
        const char* src = hs_base + soff[c];
        auto cut = [&](char* dst, const char* from, int64_t bytes) {
          for (int64_t x = 0; x < bytes; x += PM_HOST_PIECE)
            pieces.push_back({c, dst + x, from + x, std::min<int64_t>(PM_HOST_PIECE, bytes - x)});
        };
        cut(hk + e0 * key_bytes, src, (e1 - e0) * key_bytes);
        if (width) cut(hp + e0 * width, src + (e1 - e0) * key_bytes, (e1 - e0) * width);
      }
      std::atomic<size_t> next_piece{0};
      std::atomic<int> err{0};
      auto mover = [&](int t) {
        int ready_c = -1;  // the chunk whose events this thread has seen complete
        for (size_t i; (i = next_piece.fetch_add(1)) < pieces.size();) {
          const Piece& pc = pieces[i];
          if (pc.c != ready_c) {
            if (cudaEventSynchronize(ctx->hup[free_at[pc.c]]) != cudaSuccess ||
                cudaEventSynchronize(ctx->hdn[pc.c]) != cudaSuccess) {
              err.store(1);
              return;
            }
            ready_c = pc.c;
          }
          std::memcpy(pc.dst, pc.src, (size_t)pc.bytes);
#ifdef PM_HOST_TRACE
          if (i + 1 == pieces.size() || pieces[i + 1].c != pc.c)
            mv_done[pc.c] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
#endif
        }
        (void)t;
      };
      std::vector<std::thread> pool;
      for (int t = 1; t < nt; ++t) pool.emplace_back(mover, t);
      mover(0);
      for (auto& th : pool) th.join();
      if (err.load()) return cuda_fail(cudaGetLastError(), "pm_merge_host: staged write-back");
    }
#ifdef PM_HOST_TRACE
    {
      cudaStreamSynchronize(sD);
      const double hend = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
      float t0h;  // host offset of the device origin is unknown: report device times from the first record
      (void)t0h;
      fprintf(stderr, "TRACE nch=%d staged=%zu use_stage=%d host_end=%.2f\n", nch, stg.size(), (int)use_stage, hend);
      for (int k = 0; k < nch; ++k) {
        float u = -1, m = -1, d = -1;
        cudaEventElapsedTime(&u, tr[3 * nch], tr[3 * k]);
        cudaEventElapsedTime(&m, tr[3 * nch], tr[3 * k + 1]);
        cudaEventElapsedTime(&d, tr[3 * nch], tr[3 * k + 2]);
        fprintf(stderr, "TRACE k=%d free=%d up=%.2f merge=%.2f d2h=%.2f moved=%.2f\n", k, free_at[k], u, m, d,
                mv_done[k]);
      }
      for (auto& e : tr) cudaEventDestroy(e);
    }
#endif
    return PM_OK;
  };
  rc = pipeline();
  if (rc) {
    for (cudaStream_t x : {sH, sC, sD}) cudaStreamSynchronize(x);
    return rc;
  }
  return pm_status(ctx, stream, nullptr);
}

}  // extern "C"
