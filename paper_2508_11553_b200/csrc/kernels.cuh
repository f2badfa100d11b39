// Device side of the tmstore: session-history arena, branch index, and the three
// hot kernels (K1 prefix-match walk, K2 record/commit, K3 trajectory assembly).
// sm_100a; integer and HBM-bound — no tensor cores.  See DESIGN.md.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tms {

constexpr int kAlignWords = 32;  // 128-byte lines: sequence positions are stored congruent mod 32
constexpr int kPathCopyDepth = 4;  // rows at this chain depth or deeper get a session path copy
constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kRootTag = 1ull << 62;

// Device view of the store (passed by value to every kernel).
struct DevView {
  int32_t *arena;  // token arena; row r's position p lives at arena[row_vb[r] + p]
  // row table (global row id)
  int64_t *row_vb;     // virtual base, multiple of 32 words
  int32_t *row_m;      // matched length = first own position
  int32_t *row_len;    // sequence length
  int64_t *row_parent; // -1 for none
  int32_t *row_sess;
  int32_t *row_local;
  int32_t *row_depth;
  int64_t *row_run0;   // first metadata run
  int32_t *row_nrun;
  // navigation hints (written once, at the child's commit)
  int64_t *row_ext;      // first child extending this row exactly at its end (-1: none) ...
  int32_t *row_ext_tok;  // ... its first own token,
  int32_t *row_ext_len;  // ... its length,
  int64_t *row_ext_vb;   // ... its virtual base: a multi-turn walk hops without a hash probe
  int64_t *row_jump;     // skew-binary jump pointer to an ancestor (O(log depth) ancestor search)
  // metadata runs (absolute start positions within the row's sequence)
  int32_t *run_start;
  int32_t *run_version;
  uint8_t *run_origin;
  // branch index: open addressing, key (owner, depth|term|token) -> child row
  uint64_t *hk0;
  uint64_t *hk1;
  int64_t *hval;
  uint64_t ht_mask;
  // sessions
  int32_t *s_nrows;
  int64_t *s_stored;
  int64_t *s_naive;
  // session path copy (long turn-by-turn chains): the newest row at depth >= kPathCopyDepth
  // keeps its FULL sequence contiguous in the arena, so a walk compares the shared history
  // in one streaming segment and resumes in the row tree with an O(log depth) ancestor
  // search instead of one hop per turn
  int64_t *s_pc_row;  // -1: none
  int64_t *s_pc_vb;   // position p of the copy at arena[s_pc_vb + p] (multiple of 32)
  int64_t *s_pc_cap;  // positions the copy can hold before it is reallocated
  // allocation counters (device-resident, advanced by the commit planner)
  int64_t *ctr;  // [0]=arena_used [1]=n_rows [2]=n_runs [3]=first device error code
  // capacities (device-side bounds checks)
  int64_t arena_cap, row_cap, run_cap;
  int64_t n_sess;  // sessions created: device-buffer matches treat any other id as unknown (matched 0)
  // record launches: rows committed in the launch are read from their entry's query until
  // the chain's copy moves them into the arena; their virtual bases fall in [qv_lo, qv_hi)
  // (debug bounds checks only)
  int64_t qv_lo, qv_hi;
};

// Device error codes (ctr[3]; first one wins; the host turns a nonzero code into TM_ECUDA).
enum : long long {
  kErrTableFull = 1,   // branch index probe wrapped the whole table (never expected: load <= 1/2)
  kErrArena = 2,       // arena access outside its capacity
  kErrRow = 3,         // row id outside the row table
  kErrRun = 4,         // metadata run outside the run table
  kErrPeerTimeout = 5, // a peer rank never signalled (routed match, device-side barrier)
};

__device__ __forceinline__ void dev_error(const DevView &v, long long code) {
  atomicCAS(reinterpret_cast<unsigned long long *>(&v.ctr[3]), 0ull, (unsigned long long)code);
}

// TM_DCHECK: bounds checks compiled into the debug build (-DTM_DEBUG, libtmstore_debug.so)
// — compute-sanitizer is not available on this pool, so the debug library records the
// first violated invariant in ctr[3] instead of faulting.
#ifdef TM_DEBUG
#define TM_DCHECK(v, cond, code) \
  do {                             \
    if (!(cond)) dev_error(v, code); \
  } while (0)
#else
#define TM_DCHECK(v, cond, code) \
  do {                             \
  } while (0)
#endif

// Walk scheduler block (one per store, zeroed once at creation): planner bucket counts,
// the walk's work counter and an exit counter; the last walk CTA re-zeroes it.
constexpr int kPlanNB = 128;
struct Sched {
  int count[kPlanNB];
  unsigned long long work;
  unsigned long long work2;  // second queue (routed walk: remote queries)
  unsigned int exit;
};

// Routing descriptor at the start of every rank's IPC-shared region (byte offsets are
// relative to the region base; arrays hold the rank's query batch and its results).
constexpr int kMaxRanks = 16;
// The header fields tm_route_prepare sets (k_route writes them into the
// region: no host-to-device copy per batch); RouteDesc starts with the same members.
struct RouteHead {
  int64_t n;        // queries in this rank's batch
  int64_t sid_off;  // int64 global session id per query
  int64_t qoff_off; // int64 token offset per query (multiple of 32)
  int64_t len_off;  // int64 length per query
  int64_t tok_off;  // int32 tokens
  int64_t idx_off;  // int32 query indices grouped by owner (written by k_route)
  int64_t m_off, par_off, dup_off;  // int64 results, written by the owners
  int64_t lo_off, hi_off;           // 18-bit planes of tok (remote owners read these), 0: not packed
  int64_t pkf_off;                  // int32[n+1]: 4096-position pack blocks before each remote query (k_route)
  int64_t rec_off;                  // RouteRec[n] at the idx positions of remote queries (pack): 0 none
  int32_t pk_bad;                   // a token outside [0, 2^18): owners read tok instead
  int32_t rank;                     // the rank whose batch this is (its own queries stay unpacked)
  int32_t nranks;
  int32_t pad_;
};

struct RouteDesc {
  int64_t n;        // queries in this rank's batch
  int64_t sid_off;  // int64 global session id per query
  int64_t qoff_off; // int64 token offset per query (multiple of 32)
  int64_t len_off;  // int64 length per query
  int64_t tok_off;  // int32 tokens
  int64_t idx_off;  // int32 query indices grouped by owner (written by k_route)
  int64_t m_off, par_off, dup_off;  // int64 results, written by the owners
  int64_t lo_off, hi_off;           // 18-bit planes of tok (remote owners read these), 0: not packed
  int64_t pkf_off;                  // int32[n+1]: 4096-position pack blocks before each remote query (k_route)
  int64_t rec_off;                  // RouteRec[n] at the idx positions of remote queries (pack): 0 none
  int32_t pk_bad;                   // a token outside [0, 2^18): owners read tok instead
  int32_t rank;                     // the rank whose batch this is (its own queries stay unpacked)
  int32_t nranks;
  int32_t pad_;
  int32_t count[kMaxRanks];  // queries owned by each rank (written by k_route)
  int32_t start[kMaxRanks];
  // per (owner, length bucket; longest first) counts and starts in idx[], so owners can
  // process every requester's queries in one global longest-first order
  int32_t bcount[kMaxRanks * kPlanNB];
  int32_t bstart[kMaxRanks * kPlanNB];
  // device-side barrier flags (epochs), written by the peers over NVLink: arrive[p] =
  // peer p has bucketed its batch for epoch e; done[p] = owner p has finished every query
  // of this rank's batch for epoch e (its results are visible).  Never rewritten by
  // tm_route_prepare; zero at allocation.
  int64_t arrive[kMaxRanks];
  int64_t done[kMaxRanks];
};
static_assert(offsetof(RouteDesc, count) == sizeof(RouteHead) && offsetof(RouteDesc, nranks) == offsetof(RouteHead, nranks),
              "RouteHead must be RouteDesc's prefix");

// What an owner needs to start a remote query, at the query's idx position: written by
// the CTA that packs the query's first block (k_route for an empty query), read with one
// 32-byte load over NVLink instead of idx -> gsid / offset / length -> first token
struct RouteRec {
  int64_t gsid;
  int64_t off;
  int32_t len;
  int32_t qi;
  int32_t q0;      // first token (0 if len == 0)
  int32_t has_q0;  // 0: q0 not filled in (the owner reads the query's first token itself)
};
static_assert(sizeof(RouteRec) == 32, "two 16-byte loads");

// Push routing (tm_route_prepare_push): the requester writes each remote query's planes and
// record straight into its owner's region (P2P stores), slice `rank` of the owner's inbox
// at + rank * stride from the layout's lo / hi / rec offsets, so the owner's walk reads
// them from its own HBM.  stride 0: the planes stay in the requester's region.
struct PushArgs {
  char *peer[kMaxRanks];  // every rank's region as mapped on this GPU (own included)
  int64_t stride;
};

struct RoutedArgs {
  int nranks, rank;
  const char *peer[kMaxRanks];  // every rank's region as mapped on this GPU (own included)
  const int32_t *g2l;           // global session id -> local session id (-1: not owned)
  int64_t g2l_len;              // entries of g2l; ids outside it are not owned here
  Sched *sched;
  int64_t push_stride;          // > 0: requesters pushed their remote queries' planes and records
                                // into this rank's region, source p's slice at + p * push_stride
  int64_t epoch;                // > 0: device-side barriers (wait for arrive, signal done)
  uint64_t timeout_ns;          // a peer silent this long is a device error, not a hang
  int tail_every;               // > 0: every tail_every-th CTA takes items from the SHORT end of its
                                // queue (latency-bound short queries overlap the long ones instead of
                                // forming a tail after them)
  long long *trace;             // diagnostics (TM_ROUTED_TRACE): per item {t0, t1, len | remote << 40, cta}
  long long trace_cap;
};

// one batch of sequences resident on the device
struct Batch {
  int64_t n;
  const int32_t *sids;
  const int32_t *tok;     // tokens; sequence w starts at tok + off[w] (multiple of 32)
  const int64_t *off;
  const int64_t *len;
  const int64_t *root;    // optional pre-resolved root row per entry (-1: none)
  int *bucket_items;      // optional planner output: entries of each length bucket (stride n;
                          // counts in sched->count), longest first
  Sched *sched;           // scheduler block (clean on entry, left clean on exit)
  // walk outputs
  int64_t *o_m;
  int64_t *o_parent;
  int64_t *o_dup;
  int32_t *o_tnext;  // query token at the mismatch (-1 if the query ended)
  int32_t *o_spar;   // parent's token at the mismatch (-1 if the parent ended)
  // metadata runs (record only)
  const int64_t *run_off;
  const int32_t *run_start;
  const uint8_t *run_origin;
  const int32_t *run_version;
  // commit plan outputs (record only)
  int64_t *c_row;
  int64_t *c_vb;
  int64_t *c_run0;
  int32_t *c_firstrun;
  int32_t *c_local;
};

struct RecordArgs {
  Batch b;                    // entries grouped by session chain, batch order inside a chain
  const int64_t *chains;      // per chain in processing order (longest first): first entry, end, session
  int64_t *ctr_out;           // non-null: the last CTA out copies the 4 counters here (one D2H for the host)
  int64_t nchains;
  unsigned long long *work;   // [0] chain counter, [1] CTAs done: zeroed by the call's staging copy
  // chain 0 handed over in the launch parameters (host batches: no dependent loads for the
  // first chain's table entry, its session id and its first entry): c0_e1 < 0 = not given
  int64_t c0_e1, c0_off;
  int32_t c0_sid, c0_len, c0_q0;
  // small host calls: the last CTA copies the results region [out_src, out_src + out_len)
  // straight into page-locked host memory (no device-to-host copy call); out_dst null: none
  const int4 *out_src;
  int4 *out_dst;
  int64_t out_len;  // int4 units
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint64_t dt_key(int64_t depth, int32_t token, bool term) {
  return ((uint64_t)depth << 33) | ((uint64_t)(term ? 1 : 0) << 32) | (uint64_t)(uint32_t)token;
}

__device__ __forceinline__ uint64_t slot_of(uint64_t owner, uint64_t dt, uint64_t mask) {
  return mix64(owner * 0x9e3779b97f4a7c15ull ^ mix64(dt + 0x632be59bd9b4e019ull)) & mask;
}

// Probes are bounded by the table size (always on): a full table reports an error
// instead of spinning forever.
__device__ __forceinline__ int64_t ht_find(const DevView &v, uint64_t owner, uint64_t dt) {
  uint64_t s = slot_of(owner, dt, v.ht_mask);
  for (uint64_t probes = 0; probes <= v.ht_mask; probes++) {
    // all three words of the slot in one round trip (the value is read speculatively)
    const uint64_t k0 = v.hk0[s], k1 = v.hk1[s];
    const int64_t r = v.hval[s];
    if (k0 == kEmpty) return -1;
    if (k0 == owner && k1 == dt) {
      TM_DCHECK(v, r >= 0 && r < v.row_cap, kErrRow);
      return r;
    }
    s = (s + 1) & v.ht_mask;
  }
  dev_error(v, kErrTableFull);
  return -1;
}

__device__ __forceinline__ void ht_insert(const DevView &v, uint64_t owner, uint64_t dt, int64_t val) {
  uint64_t s = slot_of(owner, dt, v.ht_mask);
  for (uint64_t probes = 0; probes <= v.ht_mask; probes++) {
    unsigned long long prev = atomicCAS((unsigned long long *)&v.hk0[s], (unsigned long long)kEmpty,
                                        (unsigned long long)owner);
    if (prev == kEmpty) {
      v.hk1[s] = dt;
      v.hval[s] = val;
      return;
    }
    s = (s + 1) & v.ht_mask;
  }
  dev_error(v, kErrTableFull);
}

__device__ __forceinline__ int4 ldg_stream(const int4 *p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Coherent 16-byte load (L2, no .nc): for arena lines written earlier in the SAME launch
// (k_record: entry e+1 of a chain compares against the suffix / path copy entry e wrote;
// .nc loads are only defined for data that stays read-only for the whole kernel).
__device__ __forceinline__ int4 ldg_coh(const int4 *p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}

// predicated streaming load / store (no branch, so the value stays in registers)
__device__ __forceinline__ int4 ldg_stream_if(const int4 *p, bool pred) {
  int4 r = make_int4(0, 0, 0, 0);
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n"
               " @p ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];\n}"
               : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
               : "l"(p), "r"((int)pred));
  return r;
}
__device__ __forceinline__ void stg_if(int4 *p, int4 x, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n @p st.global.v4.s32 [%0], {%1,%2,%3,%4};\n}"
               ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w), "r"((int)pred) : "memory");
}

// Whole-CTA int4 copy dst[i] = src[i], i in [i0, i1): every thread issues UC loads before
// its stores, so NT*UC*16 bytes are in flight per round (a 2,048-token suffix moves in one
// round at NT=128, UC=4; one load per thread and round was a chain of dependent round trips).
// src must stay read-only for the launch (streaming .nc loads).
template <int NT, int UC>
__device__ __forceinline__ void block_copy4(int4 *__restrict__ dst, const int4 *__restrict__ src, int64_t i0, int64_t i1) {
  for (int64_t base = i0 + threadIdx.x; base < i1; base += (int64_t)NT * UC) {
    int4 x[UC];
#pragma unroll
    for (int k = 0; k < UC; k++) x[k] = ldg_stream_if(src + base + k * NT, base + k * NT < i1);
#pragma unroll
    for (int k = 0; k < UC; k++) stg_if(dst + base + k * NT, x[k], base + k * NT < i1);
  }
}

// First mismatch position in [lo, hi) between q[] and a[] (both indexed by absolute
// position, 16-byte congruent), or hi.  Whole-block call; all threads get the result.
// Each warp owns 32*U consecutive int4 per chunk; the next chunk is prefetched into
// registers while the current one is checked; __syncthreads_or gates early exit.
// COH: a[] may have been written earlier in this launch (k_record) -> coherent loads.
template <int NT, int U, bool COH = false>
__device__ __forceinline__ int block_first_mismatch(const int32_t *__restrict__ q, const int32_t *__restrict__ a,
                                                    int lo, int hi, int *s_red) {
  if (lo >= hi) return hi;
  const int4 *q4 = reinterpret_cast<const int4 *>(q);
  const int4 *a4 = reinterpret_cast<const int4 *>(a);
  const int v0 = lo >> 2, v1 = (hi + 3) >> 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CH = NT * U;
  const int tb = warp * (32 * U) + lane;
  int4 qa[U], aa[U], qb[U], ab[U];
  int base = v0;
#pragma unroll
  for (int k = 0; k < U; k++) {
    int idx = base + tb + k * 32;
    if (idx < v1) { qa[k] = ldg_stream(q4 + idx); aa[k] = COH ? ldg_coh(a4 + idx) : ldg_stream(a4 + idx); }
    else { qa[k] = make_int4(0, 0, 0, 0); aa[k] = qa[k]; }
  }
  for (;;) {
    const int nb = base + CH;
    const bool more = nb < v1;
    if (more) {
#pragma unroll
      for (int k = 0; k < U; k++) {
        int idx = nb + tb + k * 32;
        if (idx < v1) { qb[k] = ldg_stream(q4 + idx); ab[k] = COH ? ldg_coh(a4 + idx) : ldg_stream(a4 + idx); }
        else { qb[k] = make_int4(0, 0, 0, 0); ab[k] = qb[k]; }
      }
    }
    int first = 0x7fffffff;
#pragma unroll
    for (int k = U - 1; k >= 0; k--) {
      int p = (base + tb + k * 32) * 4;
      unsigned ne = (qa[k].x != aa[k].x ? 1u : 0u) | (qa[k].y != aa[k].y ? 2u : 0u) |
                    (qa[k].z != aa[k].z ? 4u : 0u) | (qa[k].w != aa[k].w ? 8u : 0u);
      // mask positions outside [lo, hi)
      unsigned valid = 0xfu;
      if (p < lo) valid &= (0xfu << (lo - p)) & 0xfu;
      if (p + 4 > hi) valid &= (hi - p) <= 0 ? 0u : (0xfu >> (4 - (hi - p)));
      ne &= valid;
      if (ne) first = p + __ffs(ne) - 1;
    }
    if (__syncthreads_or(first != 0x7fffffff)) {
      unsigned wmin = __reduce_min_sync(0xffffffffu, (unsigned)first);
      if (lane == 0) s_red[warp] = (int)wmin;
      __syncthreads();
      int r = 0x7fffffff;
#pragma unroll
      for (int w = 0; w < NT / 32; w++) r = min(r, s_red[w]);
      __syncthreads();
      return r;
    }
    if (!more) return hi;
    base = nb;
#pragma unroll
    for (int k = 0; k < U; k++) { qa[k] = qb[k]; aa[k] = ab[k]; }
  }
}

// ---- barriers over a subset of the CTA ---------------------------------------------------
// BAR == 0: the whole CTA (__syncthreads); otherwise named barrier BAR over the first NT
// threads - a warp-specialised kernel keeps its other warps out of the compare's barriers.
template <int NT, int BAR>
__device__ __forceinline__ void group_sync() {
  if constexpr (BAR == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}
template <int NT, int BAR>
__device__ __forceinline__ int group_or(int pred) {
  if constexpr (BAR == 0) {
    return __syncthreads_or(pred);
  } else {
    int r;
    asm volatile("{ .reg .pred p, q; setp.ne.s32 p, %1, 0; bar.red.or.pred q, %2, %3, p; selp.s32 %0, 1, 0, q; }"
                 : "=r"(r) : "r"(pred), "n"(BAR), "n"(NT) : "memory");
    return r;
  }
}

// ---- TMA (cp.async.bulk) staged compare ---------------------------------------------------
// Same contract as block_first_mismatch, but the query and history chunks are moved into a
// ring of shared-memory stages by the bulk-copy engine (one elected thread issues, an
// mbarrier per stage counts the landed bytes), and the CTA compares out of shared memory.
// Registers stay free of load buffers; S stages of 2 x CHV int4 are in flight per CTA.

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{ .reg .pred P; WAIT%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT%=; }" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int NT, int S, int CHV>
struct TmaRing {
  int4 q[S][CHV];
  int4 a[S][CHV];
  uint64_t bar[S];
  uint32_t chunks;  // chunks consumed by this CTA so far (stage / phase bookkeeping)
};

template <int NT, int S, int CHV>
__device__ __forceinline__ void tma_ring_init(TmaRing<NT, S, CHV> &rg) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&rg.bar[s], 1);
    rg.chunks = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
}

// s_cap (optional, int[2 * NT / 32 + 2]): also capture the query's and the history's token
// at the first mismatch (out of the shared-memory stage that held it) into s_cap[2 * NT / 32]
// and s_cap[2 * NT / 32 + 1], so the caller needs no global load for them.
template <int NT, int S, int CHV, int BAR = 0>
__device__ __forceinline__ int block_first_mismatch_tma(const int32_t *__restrict__ q, const int32_t *__restrict__ a,
                                                        int lo, int hi, int *s_red, TmaRing<NT, S, CHV> &rg,
                                                        int *s_cap = nullptr) {
  static_assert(NT % 32 == 0 && NT <= CHV, "whole warps, at least one int4 per thread and chunk");
  static_assert(CHV % NT == 0, "chunk must split evenly over the CTA");
  if (lo >= hi) return hi;
  const int4 *q4 = reinterpret_cast<const int4 *>(q);
  const int4 *a4 = reinterpret_cast<const int4 *>(a);
  const int v0 = lo >> 2, v1 = (hi + 3) >> 2;
  const int nch = (v1 - v0 + CHV - 1) / CHV;
  const uint32_t base = rg.chunks;  // uniform: read before anyone updates it
  auto issue = [&](int c) {
    const int s = (int)((base + c) % S);
    const int i0 = v0 + c * CHV;
    const int n = min(CHV, v1 - i0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the stage -> async writes
    mbar_expect_tx(&rg.bar[s], 2u * 16u * (uint32_t)n);
    bulk_g2s(rg.q[s], q4 + i0, 16u * (uint32_t)n, &rg.bar[s]);
    bulk_g2s(rg.a[s], a4 + i0, 16u * (uint32_t)n, &rg.bar[s]);
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < S && c < nch; c++) issue(c);
  int result = hi;
  int c = 0;
  for (; c < nch; c++) {
    const int s = (int)((base + c) % S);
    mbar_wait(&rg.bar[s], ((base + c) / S) & 1);
    const int i0 = v0 + c * CHV;
    int first = 0x7fffffff;
    int fq = 0, fa = 0;  // tokens at `first` (capture)
    if (4 * i0 >= lo && 4 * (i0 + CHV) <= hi) {  // a full chunk inside [lo, hi): no masking (uniform)
#pragma unroll
      for (int k = CHV / NT - 1; k >= 0; k--) {
        const int li = k * NT + threadIdx.x;
        const int4 x = rg.q[s][li], y = rg.a[s][li];
        const unsigned ne =
            (x.x != y.x ? 1u : 0u) | (x.y != y.y ? 2u : 0u) | (x.z != y.z ? 4u : 0u) | (x.w != y.w ? 8u : 0u);
        if (ne) {
          const int c = __ffs(ne) - 1;
          first = (i0 + li) * 4 + c;
          if (s_cap) {
            fq = c == 0 ? x.x : c == 1 ? x.y : c == 2 ? x.z : x.w;
            fa = c == 0 ? y.x : c == 1 ? y.y : c == 2 ? y.z : y.w;
          }
        }
      }
    } else
#pragma unroll
    for (int k = CHV / NT - 1; k >= 0; k--) {
      const int li = k * NT + threadIdx.x;
      const int idx = i0 + li;
      if (idx >= v1) continue;
      const int4 x = rg.q[s][li], y = rg.a[s][li];
      const int p = idx * 4;
      unsigned ne = (x.x != y.x ? 1u : 0u) | (x.y != y.y ? 2u : 0u) | (x.z != y.z ? 4u : 0u) | (x.w != y.w ? 8u : 0u);
      unsigned valid = 0xfu;
      if (p < lo) valid &= (0xfu << (lo - p)) & 0xfu;
      if (p + 4 > hi) valid &= (hi - p) <= 0 ? 0u : (0xfu >> (4 - (hi - p)));
      ne &= valid;
      if (ne) {  // k runs downwards, so the last hit is this thread's lowest position
        const int c = __ffs(ne) - 1;
        first = p + c;
        if (s_cap) {
          fq = c == 0 ? x.x : c == 1 ? x.y : c == 2 ? x.z : x.w;
          fa = c == 0 ? y.x : c == 1 ? y.y : c == 2 ? y.z : y.w;
        }
      }
    }
    if (group_or<NT, BAR>(first != 0x7fffffff)) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      unsigned wmin = __reduce_min_sync(0xffffffffu, (unsigned)first);
      if (lane == 0) s_red[warp] = (int)wmin;
      if (s_cap && first != 0x7fffffff && (unsigned)first == wmin) {  // the one thread holding it
        s_cap[2 * warp] = fq;
        s_cap[2 * warp + 1] = fa;
      }
      group_sync<NT, BAR>();
      int r = 0x7fffffff, rw = 0;
#pragma unroll
      for (int w = 0; w < NT / 32; w++)
        if (s_red[w] < r) { r = s_red[w]; rw = w; }
      if (s_cap && threadIdx.x == 0) {
        s_cap[2 * (NT / 32)] = s_cap[2 * rw];
        s_cap[2 * (NT / 32) + 1] = s_cap[2 * rw + 1];
      }
      result = r;
      c++;
      break;
    }
    if (threadIdx.x == 0 && c + S < nch) issue(c + S);
  }
  // drain chunks issued but not consumed (keeps stage phases aligned; no copy may land
  // in a stage after it is reused)
  const int issued = min(nch, c - 1 + S);  // prologue issued S, each consumed chunk one more
  for (int d = c; d < issued; d++) mbar_wait(&rg.bar[(base + d) % S], ((base + d) / S) & 1);
  group_sync<NT, BAR>();
  if (threadIdx.x == 0) rg.chunks = base + (uint32_t)issued;
  group_sync<NT, BAR>();
  return result;
}

// ---- TMA compare against a PACKED query (routed match: remote queries cross NVLink as
// 18-bit split planes, hostpack.h layout: a uint16 low plane + one byte per 4 positions of
// 2-bit high parts, byte (p & 7) of a 32-position group holding p, p+8, p+16, p+24) ------
// Chunks are CHP positions; each plane is copied from its own aligned base (low plane: 8
// positions = 16 B, high plane: 64 positions = 16 B, history: 4 positions), so a chunk
// moves 2.25 B of query per position instead of 4.
template <int S, int CHP>
struct PackedRing {
  uint16_t lo[S][CHP + 16];
  uint8_t hi[S][CHP / 4 + 64];
  int4 a[S][CHP / 4 + 4];
  uint64_t bar[S];
  uint32_t chunks;
};

template <int S, int CHP>
__device__ __forceinline__ void packed_ring_init(PackedRing<S, CHP> &rg) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&rg.bar[s], 1);
    rg.chunks = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
}

// plo / phi: the requester's planes (whole buffer); the query starts at plane position
// qoff (a multiple of 32).  Same contract as block_first_mismatch_tma for positions [lo, hi)
// of the query.
template <int NT, int S, int CHP>
__device__ __forceinline__ int block_first_mismatch_packed(const uint16_t *__restrict__ plo,
                                                           const uint8_t *__restrict__ phi, int64_t qoff,
                                                           const int32_t *__restrict__ a, int lo, int hi,
                                                           int *s_red, PackedRing<S, CHP> &rg) {
  static_assert(NT == 64, "written for 64-thread CTAs");
  static_assert(CHP % (4 * NT) == 0 && CHP % 64 == 0, "chunk must split evenly over the CTA");
  if (lo >= hi) return hi;
  const int p0 = lo & ~3;  // chunk c covers positions [p0 + c*CHP, min(p0 + (c+1)*CHP, hi4))
  const int hi4 = (hi + 3) & ~3;
  const int nch = (hi4 - p0 + CHP - 1) / CHP;
  const uint32_t base = rg.chunks;
  auto issue = [&](int c) {
    const int st = (int)((base + c) % S);
    const int s0 = p0 + c * CHP, e0 = min(s0 + CHP, hi4);
    const int64_t S0 = qoff + s0, E0 = qoff + e0;        // plane positions
    const int64_t l0 = S0 & ~7ll, l1 = (E0 + 7) & ~7ll;  // low plane: 16-byte granules
    const int64_t h0 = S0 & ~63ll, h1 = (E0 + 63) & ~63ll;  // high plane: 16-byte granules
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bl = 2u * (uint32_t)(l1 - l0), bh = (uint32_t)(h1 - h0) / 4u, ba = 4u * (uint32_t)(e0 - s0);
    mbar_expect_tx(&rg.bar[st], bl + bh + ba);
    bulk_g2s(rg.lo[st], plo + l0, bl, &rg.bar[st]);
    bulk_g2s(rg.hi[st], phi + h0 / 4, bh, &rg.bar[st]);
    bulk_g2s(rg.a[st], a + s0, ba, &rg.bar[st]);
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < S && c < nch; c++) issue(c);
  int result = hi;
  int c = 0;
  for (; c < nch; c++) {
    const int st = (int)((base + c) % S);
    mbar_wait(&rg.bar[st], ((base + c) / S) & 1);
    const int s0 = p0 + c * CHP;
    const int64_t S0 = qoff + s0;
    const int l0 = (int)(S0 & 7), h0 = (int)(S0 & 63);  // plane offsets of position s0 in the stage
    int first = 0x7fffffff;
#pragma unroll
    for (int k = CHP / (4 * NT) - 1; k >= 0; k--) {
      const int li = k * NT + threadIdx.x;  // int4 slot of the chunk
      const int p = s0 + 4 * li;
      if (p >= hi4) continue;
      const int d = 4 * li;  // p - s0
      const uint2 l = *reinterpret_cast<const uint2 *>(&rg.lo[st][l0 + d]);
      const uint32_t hw = *reinterpret_cast<const uint32_t *>(&rg.hi[st][((h0 + d) >> 5) * 8 + ((h0 + d) & 7)]) >>
                          (2 * (((h0 + d) >> 3) & 3));
      int4 x;
      x.x = (int)((l.x & 0xFFFFu) | ((hw & 3u) << 16));
      x.y = (int)((l.x >> 16) | (((hw >> 8) & 3u) << 16));
      x.z = (int)((l.y & 0xFFFFu) | (((hw >> 16) & 3u) << 16));
      x.w = (int)((l.y >> 16) | (((hw >> 24) & 3u) << 16));
      const int4 y = rg.a[st][li];
      unsigned ne = (x.x != y.x ? 1u : 0u) | (x.y != y.y ? 2u : 0u) | (x.z != y.z ? 4u : 0u) | (x.w != y.w ? 8u : 0u);
      unsigned valid = 0xfu;
      if (p < lo) valid &= (0xfu << (lo - p)) & 0xfu;
      if (p + 4 > hi) valid &= (hi - p) <= 0 ? 0u : (0xfu >> (4 - (hi - p)));
      ne &= valid;
      if (ne) first = min(first, p + __ffs(ne) - 1);
    }
    if (__syncthreads_or(first != 0x7fffffff)) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      unsigned wmin = __reduce_min_sync(0xffffffffu, (unsigned)first);
      if (lane == 0) s_red[warp] = (int)wmin;
      __syncthreads();
      int r = 0x7fffffff;
#pragma unroll
      for (int w = 0; w < NT / 32; w++) r = min(r, s_red[w]);
      result = r;
      c++;
      break;
    }
    if (threadIdx.x == 0 && c + S < nch) issue(c + S);
  }
  const int issued = min(nch, c - 1 + S);
  for (int d = c; d < issued; d++) mbar_wait(&rg.bar[(base + d) % S], ((base + d) / S) & 1);
  __syncthreads();
  if (threadIdx.x == 0) rg.chunks = base + (uint32_t)issued;
  __syncthreads();
  return result;
}

}  // namespace tms
