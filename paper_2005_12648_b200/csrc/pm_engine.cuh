// pm_engine.cuh -- the in-place merge/rotation engine (shared declarations).
//
// One persistent kernel realises, on the caller's buffer and with bounded
// scratch, either
//   MODE_MERGE : the stable (A-first) merge of runs A=[s,m) and B=[m,e)
//                -- the result of the reference's seq_merge_buffered /
//                merge_srecpar at t=1 (seqmerge.py:55-75, srecpar.py:33-84),
//   MODE_ROTATE: the block exchange A|B -> B|A of linear/circular shifting
//                (shift.py:38-55, _kernels.py:92-197).
// The output is cut into regions of M = mu*T records ("pairs"); region q's
// inputs are the A and B ranges the stable merge path assigns to it.  The
// array is also cut into slots of T records ("units").  Regions are processed
// in ticket order (two fronts growing out of the A/B boundary).  A region
// gathers its inputs from wherever their units currently live, merges them in
// shared memory, and writes its slots.  A unit still needed by a later region
// is first "salvaged" into a free slot (a slot whose unit is fully consumed)
// or into the bounded scratch pool.  DESIGN.md section 3 has the protocol and
// its progress/space argument.
#pragma once
#include <cstdint>

namespace pm {

enum : int32_t { MODE_MERGE = 0, MODE_ROTATE = 1 };
enum : int32_t { ST_FREE = -1, ST_CLOSED = -2 };
constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;

// k_engine shape: kEngineTeam salvage-worker warps + kDataWarps data-team warps,
// kEngineMinBlocks resident CTAs per SM, staging tiles sized to kTileBudget bytes
// of shared memory per CTA.
#ifndef PM_ENGINE_TEAM
#define PM_ENGINE_TEAM 2
#endif
#ifndef PM_DATA_WARPS
#define PM_DATA_WARPS 6
#endif
#ifndef PM_ENGINE_MINB
#define PM_ENGINE_MINB 3
#endif
#ifndef PM_TILE_BUDGET
#define PM_TILE_BUDGET (72 * 1024)
#endif
constexpr int kEngineTeam = PM_ENGINE_TEAM;
// staged runs are followed by kSent slots of +max sentinels (keys-only merges
// then need no bound checks in their dependent chain); kSent > the longest
// per-thread output span of any tile merge (checked on the host)
constexpr int kSent = 80;
constexpr int kDataWarps = PM_DATA_WARPS;
constexpr int kEngineThreads = 32 * (PM_ENGINE_TEAM + PM_DATA_WARPS);
constexpr int kEngineMinBlocks = PM_ENGINE_MINB;
constexpr int64_t kTileBudget = PM_TILE_BUDGET;
#ifndef PM_BUF_THREADS
#define PM_BUF_THREADS 256
#endif
constexpr int kBufferedThreads = PM_BUF_THREADS;
// k_buffered (buffered / copy modes): staging ring depth and the shared-memory
// budget its (stages + 2 output) tiles are sized to
#ifndef PM_BUF_STAGES
#define PM_BUF_STAGES 2
#endif
#ifndef PM_BUF_BUDGET
#define PM_BUF_BUDGET (72 * 1024)
#endif
constexpr int kBufStages = PM_BUF_STAGES;
constexpr int64_t kBufBudget = PM_BUF_BUDGET;
// free-list shards: each tagged top word on its own 256-byte line (its own L2
// slice), so CAS traffic on one shard does not queue behind another's
constexpr int kShards = 64;
constexpr int kTopStride = 32;  // unsigned long long words between shard tops
// tickets a k_engine CTA holds at once (its salvage workers run ahead of its data team)
#ifndef PM_RING
#define PM_RING 2
#endif
constexpr int kRing = PM_RING;
static_assert(kRing >= 2, "the data team opens the next entry before finishing the current one");

// Two-front ticket order around the centre region qc (regions 0..Q-1): ticket 0
// is qc, then qc-1, qc+1, qc-2, qc+2, ... until one side runs out, then the
// rest of the longer side.  __host__ __device__ so tests can check the exact
// device formulas on the CPU (pm_debug_order).
struct TwoFront {
  int64_t Q, qc;
  __host__ __device__ int64_t nleft() const { return qc; }
  __host__ __device__ int64_t nright() const { return Q - 1 - qc; }
  __host__ __device__ static int64_t mn(int64_t a, int64_t b) { return a < b ? a : b; }
  __host__ __device__ int64_t region_of_ticket(int64_t t) const {
    if (t == 0) return qc;
    int64_t nl = nleft(), nr = nright(), m2 = mn(nl, nr);
    if (t <= 2 * m2) return (t & 1) ? qc - (t + 1) / 2 : qc + t / 2;
    return nl > nr ? qc - (t - nr) : qc + (t - nl);
  }
  __host__ __device__ int64_t order(int64_t q) const {
    if (q == qc) return 0;
    int64_t nl = nleft(), nr = nright(), m2 = mn(nl, nr);
    if (q < qc) {
      int64_t i = qc - q;
      return i <= m2 ? 2 * i - 1 : i + nr;
    }
    int64_t i = q - qc;
    return i <= m2 ? 2 * i : i + nl;
  }
  // regions with order <= t form the window [lo, hi]
  __host__ __device__ void window(int64_t t, int64_t& lo, int64_t& hi) const {
    int64_t nl = nleft(), nr = nright(), m2 = mn(nl, nr), a, b;
    if (t <= 2 * m2) {
      a = (t + 1) / 2;
      b = t / 2;
    } else if (nl > nr) {
      a = t - nr;
      b = nr;
    } else {
      a = nl;
      b = t - nl;
    }
    lo = qc - mn(a, nl);
    hi = qc + mn(b, nr);
  }
};

struct EngineParams {
  char* keys;          // element x lives at keys + x*ks
  uint8_t* pay;        // row x lives at pay + x*w (unused when w == 0)
  int64_t w;           // payload bytes per record
  int32_t ks;          // key bytes (4 or 8)
  int32_t mode;
  int64_t s, m, e;     // job, absolute element indices
  int64_t T;           // unit (slot) size, records
  int32_t mu;          // slots per region
  int32_t lT, lmu;     // log2 T, log2 mu (both powers of two)
  int64_t M;           // region size = mu*T
  int64_t k0, K;       // first absolute slot, number of slots
  int64_t R0, Q;       // first absolute region, number of regions
  int64_t qc;          // centre region (local) for the two-front order
  int64_t* split_a;    // [Q+1] A-count at each region diagonal
  int32_t* state;      // [K] slot state: occupant unit, ST_FREE or ST_CLOSED
  int32_t* loc;        // [K] unit location: slot index or -(scratch index + 1)
  int32_t* reads;      // [K] records of the unit already gathered by consumers
  int32_t* tlist;      // engine: [Q] the tickets with work (identity regions left out), k_compact
  int32_t* ntick;      // engine: number of entries in tlist
  int32_t* next_free;  // [K] free-slot stack links
  int32_t* next_scr;   // [S] scratch stack links
  unsigned long long* free_top;  // tagged stack tops (tag<<32 | index)
  unsigned long long* scr_top;
  int64_t S;           // scratch units
  int32_t grid;        // engine CTAs
  int64_t s_per;       // scratch units each engine CTA starts with in its cache
  int64_t reserve;     // minimum pool: units the CTAs may hold moved-but-unread at once
  char* scr_keys;      // phase-matched scratch bases
  uint8_t* scr_pay;
  int32_t* ticket;
  int32_t* err;
  int32_t* noop;       // set by the plan kernel when the job needs no work
  int32_t* need_space; // > 0 while some CTA is blocked on salvage space: CTAs flush their caches
  unsigned long long* stats;  // [4]: salvaged units, salvaged records, regions, identity regions
  size_t smem_keys;    // bytes reserved for staged keys
  size_t smem_pay;     // bytes reserved for staged payload
  char* out_keys;      // out-of-place merge (k_buffered copy mode): destination, else null
  uint8_t* out_pay;
  const char* keys_b;  // copy mode: B run base (record j at keys_b + j*ks), else null (B = keys + m)
  const uint8_t* pay_b;
  // device-side routing: when non-null the kernel runs only if *gate != 0 (the
  // bounded-pool engine behind the scheduled engine, taken when the latter's plan
  // does not fit its pool -- pm_flow.cu)
  const int32_t* gate;
  int32_t* gate_out;   // staged path: k_plan computes the order gate (A[m-1] > B[0]) into it first
};

// Scheduled in-place merge (pm_flow.cu).  Per region ("ticket") of the plan's
// processing order, what the streaming kernel needs in one 80-byte load: the
// region, its splits, and for each of its (at most two) A and B pieces whether it
// is read from the original slot or from the slot's salvage entry in the pool
// (pool address of record x = pool + (x + delta) * bytes).
struct FlowTicket {
  int32_t r;      // region (== slot it writes)
  int32_t flags;  // bit 1+k: A piece k from the pool; bit 3+k: B piece k from the pool
  int32_t ja[2];  // slot of A piece k (-1: none)
  int32_t jb[2];  // slot of B piece k
  int32_t pad_[2];
  int64_t a0, a1;  // A-local split at the region's two diagonals
  int64_t dA[2], dB[2];
};
static_assert(sizeof(FlowTicket) == 80, "FlowTicket is loaded as five 16-byte vectors");

// flow control words (int64, one 256-byte line)
// FC_ROT: the job is a pure rotation (every B key below every A key; set by the
// sample phase); FC_ROTFAIL: its salvage overflowed the pool, so the gated block
// exchange (three reversals, pm_rotate.cu) runs instead of the bounded-pool engine
enum : int { FC_SAL_ANGLE = 0, FC_SAL_TF = 1, FC_POOL = 2, FC_NIDENT = 3, FC_MODE = 4, FC_FAIL = 5, FC_NTICK = 6,
             FC_NSALV = 7, FC_ROT = 8, FC_ROTFAIL = 9, FC_WORDS = 32 };

struct FlowParams {
  EngineParams P;       // geometry (T == M, one slot per region, Q == K), splits, ticket/err/noop/stats
  int32_t* D;           // [K] region reading the slot's middle record | (record in B) << 31
  uint8_t* idn;         // [K] identity region (inputs already on its outputs)
  uint32_t* key;        // [K] angle-order key (bin)
  int32_t* order;       // [K] ticket -> region
  int32_t* rank;        // [K] region -> ticket (INT32_MAX: identity, never processed)
  int32_t* hist;        // [nb + 1] angle bins: counts, then cursors
  int32_t* chunk;       // [Q / 1024 + 2] identity regions per 1024 two-front tickets, then prefix
  int32_t* slo;         // [K] salvage hull of the slot (record offsets in the slot), slo >= shi: none
  int32_t* shi;
  int32_t* pend;        // [K] lower-ranked readers of the slot that have not read it yet
  int64_t* pdelta;      // [K] pool delta of the slot's salvage entry
  FlowTicket* tk;       // [K]
  long long* fc;        // control words (FC_*)
  char* pool_keys;      // phase-matched to keys (16-byte) / payload
  uint8_t* pool_pay;
  int64_t pool_cap;     // records
  int4* pieces;         // [4 K] per region: (slot, lo, hi, 2 side + k) of each piece, slot -1: none
  float2* z;            // [3 K] itinerary vectors / synchronisation buffers
  int32_t nsync;        // synchronisation steps
  int32_t nsync_div;    // their phase step delta = 2 pi / nsync_div
  int32_t nbits;        // itinerary length of the angle key
  int32_t nb;           // angle bins
  int32_t force;        // -1: choose per job, 0: two-front, 1: angle order, 2: force the fallback
  // prescribed layout (pm_reorder, reorder_multi): nleaves > 0 leaves, leaf i = the
  // A slice of size leafpre[..] then the B slice; the output is their concatenation
  const int64_t* leaf_l;  // [nleaves + 1] output start of each leaf (job-local), leaf_l[nleaves] = N
  const int64_t* leaf_a;  // [nleaves + 1] A records before each leaf
  int32_t nleaves;
  int32_t lS;           // log2 of the split-search sample stride S (S divides M)
  int32_t phi;          // B samples sit at B[k S + phi], phi = (-s - 1) mod S
  void* samp_a;         // A[k S]            k < ceil(LA / S)
  void* samp_b;         // B[k S + phi]      k S + phi < LB
  int64_t nsa, nsb;
};

}  // namespace pm
