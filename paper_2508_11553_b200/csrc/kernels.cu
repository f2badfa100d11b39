// Kernels of the tmstore (see kernels.cuh for the data layout).
//
//  k_plan_lpt      single CTA: longest-first processing order (counting sort on length)
//  k_walk          K1: longest-prefix-match walk, one CTA per query, vectorised compare
//  k_commit_plan   single CTA: allocation scan (row ids, arena slots, run slots)
//  k_commit        K2: append novel suffixes + metadata runs, branch-index insert, stats
//  k_export        K3: chain walk + gather into packed tokens / loss_mask / versions
//  k_rehash        branch-index growth
#include "kernels.cuh"

#include <algorithm>
#include <type_traits>

#include "launch.h"

#include <cstdlib>
#include <cstring>

namespace tms {

// ----------------------------------------------------------------------------------
// Planner (one grid-wide pass, one thread per entry): resolve each entry's root row
// (session, first token) in the branch index, and drop the entry into one of kPlanNB
// length buckets (longest first, 1024-token granularity).  The walk grabs items by
// rank and maps rank -> (bucket, slot) with a 128-entry scan in shared memory, so the
// tail of the grid is left with the shortest items (longest-processing-time order).
constexpr int kPlanNT = 256;

__device__ __forceinline__ int len_bucket(int64_t L) {
  const int64_t k = L >> 10;
  return kPlanNB - 1 - (int)(k < kPlanNB - 1 ? k : kPlanNB - 1);
}

__global__ void __launch_bounds__(kPlanNT) k_plan(DevView v, Batch b, int64_t *root, int *count, int *items) {
  const int64_t w = blockIdx.x * (int64_t)kPlanNT + threadIdx.x;
  if (w >= b.n) return;
  const int64_t L = b.len[w];
  if (root) root[w] = L > 0 ? ht_find(v, kRootTag | (uint64_t)(uint32_t)b.sids[w], dt_key(0, b.tok[b.off[w]], false)) : -1;
  // warp-aggregated slot allocation: most entries of a batch share a few buckets, and
  // per-thread atomics on one address serialise
  const int bk = len_bucket(L);
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, bk);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&count[bk], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  items[(int64_t)bk * b.n + base + rank] = (int)w;
}

// ----------------------------------------------------------------------------------
// K1 walk.  Per query: root lookup (session, q[0]) -> row; compare the row's own
// segment from the current position; at the first mismatch j look up the child
// branching at (row, j, q[j]); continue in the child or finish.

// Where one query's results go (element pointers; tnext/spar only when recording).
struct WalkOut {
  int64_t *m, *parent, *dup;
  int32_t *tnext, *spar;
};

struct WalkShared {
  int red[32];
  long long row;
  long long nvb;  // next row's virtual base / length (from the hint or one probe)
  int nlen;
  int lo;
  long long pc_vb;  // session path copy (kPathCopyDepth): virtual base / length, or pc_len 0
  int pc_len;
};

constexpr int kTmaStages = 4;
constexpr int kTmaChunk = 256;  // int4 per stream per stage (4 KB)
using Ring = TmaRing<64, kTmaStages, kTmaChunk>;

struct NoRing {};

// a remote query's 18-bit planes (routed match): whole-buffer plane bases + the query's start
struct PackedQuery {
  const uint16_t *lo;
  const uint8_t *hi;
  int64_t off;
};
template <class R>
struct IsPackedRing : std::false_type {};
template <int S, int CHP>
struct IsPackedRing<PackedRing<S, CHP>> : std::true_type {};
constexpr int kPackedChunk = 1024;  // positions per stage of the packed compare
using RoutedPackedRing = PackedRing<kTmaStages, kPackedChunk>;

// Whole-CTA walk of one query q[0:L) (q may live in a peer GPU's memory).  With a TmaRing
// the compare goes through the TMA-staged path, otherwise through registers.
template <int NT, int U, class R = NoRing, bool COH = false>
__device__ __forceinline__ void walk_query(const DevView &v, const int32_t *q, int L, int32_t sid, const int64_t *root_hint,
                                           WalkOut o, WalkShared &sh, R *rg = nullptr,
                                           const PackedQuery *pk = nullptr, const int32_t *q0 = nullptr) {
  // A session with a path copy (a long turn-by-turn chain): compare the query against the
  // copy in one streaming segment, then resume the walk at the row that owns the last
  // matched position - exactly the state the hop-by-hop walk would reach there (every
  // position of the copy's sequence is owned by the deepest ancestor starting at or
  // before it).
  if (threadIdx.x == 0) {
    sh.pc_len = 0;
    int64_t r = -1;
    if (root_hint) {
      r = *root_hint;
    } else if (L > 0 && sid >= 0 && sid < v.n_sess) {  // unknown session ids: matched 0
      const int64_t pc = v.s_pc_row[sid];  // in flight with the root probe
      r = ht_find(v, kRootTag | (uint64_t)(uint32_t)sid, dt_key(0, q0 ? *q0 : q[0], false));  // q0: known first token
      if (pc >= 0 && r >= 0) {
        sh.pc_vb = v.s_pc_vb[sid];
        sh.pc_len = min(L, v.row_len[pc]);
        sh.nvb = pc;
      }
    }
    sh.row = r;
  }
  __syncthreads();
  int jpc = 0;
  if (sh.pc_len > 0) {
    const int32_t *pcq = v.arena + sh.pc_vb;
    if constexpr (std::is_same<R, NoRing>::value) {
      jpc = block_first_mismatch<NT, U, COH>(q, pcq, 0, sh.pc_len, sh.red);
    } else {
      if constexpr (IsPackedRing<R>::value) {
        jpc = block_first_mismatch_packed<NT>(pk->lo, pk->hi, pk->off, pcq, 0, sh.pc_len, sh.red, *rg);
      } else {
        jpc = block_first_mismatch_tma(q, pcq, 0, sh.pc_len, sh.red, *rg);
      }
    }
  }
  if (threadIdx.x == 0) {
    int64_t r = sh.row;  // the root row (or -1)
    int lo = 1;
    if (jpc > 0) {  // owner of position jpc-1 on the copy's path: O(log depth) ancestor search
      r = sh.nvb;
      while (v.row_m[r] > jpc - 1) {
        const int64_t jp = v.row_jump[r];
        r = (jp >= 0 && v.row_m[jp] > jpc - 1) ? jp : v.row_parent[r];
      }
      lo = jpc;
    }
    if (r < 0) {  // nothing shares the first token: matched 0
      *o.m = 0;
      *o.parent = -1;
      *o.dup = -1;
      if (o.tnext) { *o.tnext = L > 0 ? q[0] : -1; *o.spar = -1; }
    }
    sh.row = r;
    sh.lo = lo;
  }
  __syncthreads();
  int64_t r = sh.row;
  int lo = sh.lo;
  __syncthreads();
  int Lr = 0;
  int64_t vb = 0;
  if (r >= 0) {
    Lr = v.row_len[r];
    vb = v.row_vb[r];
  }
  while (r >= 0) {
    TM_DCHECK(v, r < v.row_cap, kErrRow);
    const int hi = min(Lr, L);
    TM_DCHECK(v, (vb + v.row_m[r] >= 0 && vb + ((Lr + 3) & ~3) <= v.arena_cap) ||
                     (vb + v.row_m[r] >= v.qv_lo && vb + ((Lr + 3) & ~3) <= v.qv_hi), kErrArena);
    const int32_t *a = v.arena + vb;
    // the extension hint is read before the compare so a turn-by-turn chain hops for free
    int64_t ext = -1;
    int32_t ext_tok = 0, ext_len = 0;
    int64_t ext_vb = 0;
    if (threadIdx.x == 0) {  // one round trip: the hint's fields are read speculatively
      ext = v.row_ext[r];
      ext_tok = v.row_ext_tok[r];
      ext_len = v.row_ext_len[r];
      ext_vb = v.row_ext_vb[r];
    }
    int j;
    if constexpr (std::is_same<R, NoRing>::value) {
      j = block_first_mismatch<NT, U, COH>(q, a, lo, hi, sh.red);
    } else {
      if constexpr (IsPackedRing<R>::value) {
        j = block_first_mismatch_packed<NT>(pk->lo, pk->hi, pk->off, a, lo, hi, sh.red, *rg);
      } else {
        j = block_first_mismatch_tma(q, a, lo, hi, sh.red, *rg);
      }
    }
    if (threadIdx.x == 0) {
      int64_t next = -1;
      if (j < L) {
        const int32_t t = q[j];
        if (j == Lr && ext >= 0 && t == ext_tok) {
          next = ext;
          sh.nlen = ext_len;
          sh.nvb = ext_vb;
        } else {
          next = ht_find(v, (uint64_t)r, dt_key(j, t, false));
          if (next >= 0) { sh.nlen = v.row_len[next]; sh.nvb = v.row_vb[next]; }
        }
        if (next < 0) {
          *o.m = j;
          *o.parent = r;
          *o.dup = -1;
          if (o.tnext) { *o.tnext = t; *o.spar = j < Lr ? a[j] : -1; }
        }
      } else {  // the query ended inside (or at the end of) row r
        int64_t dup = (L == Lr) ? r : ht_find(v, (uint64_t)r, dt_key(L, 0, true));
        *o.m = L;
        *o.parent = r;
        *o.dup = dup;
        if (o.tnext) { *o.tnext = -1; *o.spar = L < Lr ? a[L] : -1; }
      }
      sh.row = next;
      sh.lo = j + 1;
    }
    __syncthreads();
    r = sh.row;
    lo = sh.lo;
    Lr = sh.nlen;
    vb = sh.nvb;
    __syncthreads();
  }
}

// The last CTA out leaves the scheduler block zeroed for the next launch, so a steady
// stream of batches needs no memset.
__device__ __forceinline__ bool sched_exit(Sched *sc) {  // thread 0: true in the last CTA out
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&sc->exit, 1u) == gridDim.x - 1) {
      for (int i = 0; i < kPlanNB; i++) sc->count[i] = 0;
      sc->work = 0;
      sc->work2 = 0;
      sc->exit = 0;
      __threadfence();
      return true;
    }
  }
  return false;
}

// 64-thread CTAs: ask for 6 resident per SM (<= 170 registers) so the walk keeps 6 CTAs
// of loads in flight per SM
template <int NT, int U>
__global__ void __launch_bounds__(NT, NT == 64 ? 6 : 1) k_walk(DevView v, Batch b) {
  __shared__ WalkShared sh;
  __shared__ long long s_item;
  __shared__ int s_base[kPlanNB + 1];
  if (b.bucket_items) {  // exclusive scan of the planner's bucket sizes
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int i = 0; i < kPlanNB; i++) { s_base[i] = acc; acc += b.sched->count[i]; }
      s_base[kPlanNB] = acc;
    }
    __syncthreads();
  }
  for (;;) {
    if (threadIdx.x == 0) {
      long long it = (long long)atomicAdd(&b.sched->work, 1ull);
      if (b.bucket_items && it < b.n) {
        int lo = 0, hi = kPlanNB;  // last bucket with base <= it
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (s_base[mid] <= it) lo = mid; else hi = mid;
        }
        it = b.bucket_items[(int64_t)lo * b.n + (it - s_base[lo])];
      }
      s_item = it;
    }
    __syncthreads();
    const int64_t w = s_item;
    if (w >= b.n) {
      sched_exit(b.sched);
      return;
    }
    WalkOut o{b.o_m + w, b.o_parent + w, b.o_dup + w, b.o_tnext ? b.o_tnext + w : nullptr,
              b.o_spar ? b.o_spar + w : nullptr};
    walk_query<NT, U>(v, b.tok + b.off[w], (int)b.len[w], b.sids[w], b.root ? b.root + w : nullptr, o, sh);
  }
}

// K1 with the TMA-staged compare: same scheduling as k_walk; S stages of CHV int4 per
// stream in shared memory.
template <int S, int CHV>
__global__ void __launch_bounds__(64) k_walk_tma(DevView v, Batch b) {
  __shared__ WalkShared sh;
  __shared__ long long s_item;
  __shared__ TmaRing<64, S, CHV> rg;
  tma_ring_init(rg);
  for (;;) {
    if (threadIdx.x == 0) s_item = (long long)atomicAdd(&b.sched->work, 1ull);
    __syncthreads();
    const int64_t w = s_item;
    if (w >= b.n) {
      sched_exit(b.sched);
      return;
    }
    WalkOut o{b.o_m + w, b.o_parent + w, b.o_dup + w, b.o_tnext ? b.o_tnext + w : nullptr,
              b.o_spar ? b.o_spar + w : nullptr};
    walk_query<64, 8>(v, b.tok + b.off[w], (int)b.len[w], b.sids[w], b.root ? b.root + w : nullptr, o, sh, &rg);
  }
}

template <int S, int CHV>
static cudaError_t walk_tma_variant(const DevView &v, const Batch &b, int num_sms, cudaStream_t s) {
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_walk_tma<S, CHV>, 64, 0);
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)num_sms * occ;
  if (grid > b.n) grid = b.n;
  if (grid < 1) grid = 1;
  k_walk_tma<S, CHV><<<(int)grid, 64, 0, s>>>(v, b);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------
// Cross-GPU routing on one node (config 5).  Every rank publishes its query batch in
// an IPC-shared region (RouteDesc + arrays); k_route buckets the batch by owner rank
// (session-hash sharding); after a cross-rank barrier each owner runs k_walk_routed,
// which reads its queries straight out of the requesters' HBM over NVLink (P2P loads)
// and writes the results back into the requesters' output arrays (P2P stores): the
// exchange is fused into the match kernel — no staging copies, no reverse collective.

__device__ __forceinline__ int owner_of(int64_t gsid, int nranks) {
  return (int)(mix64((uint64_t)gsid + 0x9e3779b97f4a7c15ull) % (uint64_t)nranks);
}

constexpr int kRouteNT = 1024;
constexpr int kPackBlock = 4096;  // positions per k_route_pack work item

// One CTA buckets the batch by (owner, length bucket) — owner-major, longest first — and,
// when the planes are packed, builds the pack work list.  Latency-bound (one CTA), so
// every pass issues all of a thread's loads of a chunk before using any of them: the
// whole kernel is a handful of dependent global round trips for a 4096-query batch.
constexpr int kRouteU = 4;  // queries per thread per chunk
__global__ void __launch_bounds__(kRouteNT) k_route(char *region, RouteHead head, PushArgs pa) {
  RouteDesc *d = reinterpret_cast<RouteDesc *>(region);
  if (threadIdx.x == 0) *reinterpret_cast<RouteHead *>(region) = head;
  const int nranks = head.nranks;
  const int64_t n = head.n;
  const int64_t *gsid = reinterpret_cast<const int64_t *>(region + head.sid_off);
  const int64_t *len = reinterpret_cast<const int64_t *>(region + head.len_off);
  int32_t *idx = reinterpret_cast<int32_t *>(region + head.idx_off);
  constexpr int NC = kMaxRanks * kPlanNB;
  constexpr int CH = kRouteNT * kRouteU;
  __shared__ int cnt[NC];
  __shared__ int wsum[kRouteNT / 32];
  for (int i = threadIdx.x; i < NC; i += kRouteNT) cnt[i] = 0;
  __syncthreads();
  auto load_keys = [&](int64_t c0, int key[kRouteU], int64_t L[kRouteU], int64_t g[kRouteU]) {
#pragma unroll
    for (int u = 0; u < kRouteU; u++) {
      const int64_t i = c0 + u * kRouteNT + threadIdx.x;
      g[u] = i < n ? gsid[i] : 0;
      L[u] = i < n ? len[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kRouteU; u++) key[u] = owner_of(g[u], nranks) * kPlanNB + len_bucket(L[u]);
  };
  for (int64_t c0 = 0; c0 < n; c0 += CH) {
    int key[kRouteU];
    int64_t L[kRouteU], g[kRouteU];
    load_keys(c0, key, L, g);
#pragma unroll
    for (int u = 0; u < kRouteU; u++)
      if (c0 + u * kRouteNT + threadIdx.x < n) atomicAdd(&cnt[key[u]], 1);
  }
  __syncthreads();
  // exclusive scan of the 2048 counters (2 per thread)
  constexpr int PER = NC / kRouteNT;
  int loc[PER], acc = 0;
#pragma unroll
  for (int j = 0; j < PER; j++) { loc[j] = acc; acc += cnt[threadIdx.x * PER + j]; }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = acc;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, s);
    if (lane >= s) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int pre = 0;
  for (int w = 0; w < warp; w++) pre += wsum[w];
  const int excl = pre + x - acc;
  __syncthreads();
  __shared__ int s_own0, s_nown;
#pragma unroll
  for (int j = 0; j < PER; j++) {
    const int c = threadIdx.x * PER + j;
    d->bcount[c] = cnt[c];
    d->bstart[c] = excl + loc[j];
    cnt[c] = excl + loc[j];  // cursors
  }
  __syncthreads();
  if (threadIdx.x < kMaxRanks) {
    const int r = threadIdx.x;
    const int st = cnt[r * kPlanNB];
    const int tot = (r + 1 < kMaxRanks ? cnt[(r + 1) * kPlanNB] : (int)n) - st;
    d->count[r] = tot;
    d->start[r] = st;
    if (r == head.rank) { s_own0 = st; s_nown = tot; }
  }
  __syncthreads();
  // scatter; with planes, also the pack blocks of every remote query at its place in the
  // remote order (idx minus this rank's own range)
  const bool pk = head.lo_off != 0;
  int32_t *pkf = reinterpret_cast<int32_t *>(region + head.pkf_off);
  const int own0 = s_own0, nown = s_nown;
  const int64_t *qoff = reinterpret_cast<const int64_t *>(region + head.qoff_off);
  for (int64_t c0 = 0; c0 < n; c0 += CH) {
    int key[kRouteU];
    int64_t L[kRouteU], g[kRouteU], qo[kRouteU];
#pragma unroll
    for (int u = 0; u < kRouteU; u++) {  // in flight with the keys
      const int64_t i = c0 + u * kRouteNT + threadIdx.x;
      qo[u] = (head.rec_off && i < n) ? qoff[i] : 0;
    }
    load_keys(c0, key, L, g);
#pragma unroll
    for (int u = 0; u < kRouteU; u++) {
      const int64_t i = c0 + u * kRouteNT + threadIdx.x;
      if (i >= n) continue;
      const int pos = atomicAdd(&cnt[key[u]], 1);
      idx[pos] = (int32_t)i;
      if (head.rec_off && key[u] / kPlanNB == head.rank) {  // own query: its record for the walk
        char *rb = pa.stride ? region + pa.stride * head.rank : region;
        reinterpret_cast<RouteRec *>(rb + head.rec_off)[pos] = RouteRec{g[u], qo[u], (int32_t)L[u], (int32_t)i, 0, 0};
      }
      if (pk && key[u] / kPlanNB != head.rank) {
        pkf[pos < own0 ? pos : pos - nown] = (int)((L[u] + kPackBlock - 1) / kPackBlock);
        if (L[u] == 0 && head.rec_off) {  // no block to pack: its record is written here
          char *rb = pa.stride ? pa.peer[key[u] / kPlanNB] + pa.stride * head.rank : region;
          reinterpret_cast<RouteRec *>(rb + head.rec_off)[pos] = RouteRec{g[u], 0, 0, (int32_t)i, 0, 0};
        }
      }
    }
  }
  if (!pk) return;
  // pkf[j] = blocks before remote query j (exclusive scan in place), pkf[nrem] = total
  __syncthreads();
  const int64_t nrem = n - nown;
  int running = 0;
  for (int64_t c0 = 0; c0 < nrem; c0 += CH) {
    int v[kRouteU], sum = 0;
#pragma unroll
    for (int u = 0; u < kRouteU; u++) {
      const int64_t j = c0 + (int64_t)threadIdx.x * kRouteU + u;
      v[u] = j < nrem ? pkf[j] : 0;
      sum += v[u];
    }
    int y = sum;  // inclusive warp scan, then across warps
#pragma unroll
    for (int s2 = 1; s2 < 32; s2 <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, s2);
      if (lane >= s2) y += t;
    }
    if (lane == 31) wsum[warp] = y;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int w = 0; w < kRouteNT / 32; w++) {
      if (w < warp) wpre += wsum[w];
      tot += wsum[w];
    }
    int e = running + wpre + y - sum;
#pragma unroll
    for (int u = 0; u < kRouteU; u++) {
      const int64_t j = c0 + (int64_t)threadIdx.x * kRouteU + u;
      if (j < nrem) pkf[j] = e;
      e += v[u];
    }
    running += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) pkf[nrem] = running;
}

// ---- device-side cross-rank barriers (epoch flags in the RouteDesc headers) ----------
__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until flags[0..nranks) >= epoch in this rank's own header.  false on timeout
// (the error word is set; callers stop waiting so the stream drains).
__device__ bool wait_flags(const DevView &v, const int64_t *flags, int nranks, int64_t epoch, uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer_ns();
  for (int p = 0; p < nranks; p++) {
    while (ld_acquire_sys(flags + p) < epoch) {
      if (*(volatile long long *)&v.ctr[3] != 0) return false;  // already failed (e.g. an earlier wait timed out)
      if (globaltimer_ns() - t0 > timeout_ns) {
        dev_error(v, kErrPeerTimeout);
        return false;
      }
      __nanosleep(256);
    }
  }
  return true;
}

// This rank's batch is bucketed (stream order: k_route ran before): tell every owner.
__global__ void k_route_arrive(RoutedArgs a) {
  if (threadIdx.x == 0) __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.nranks) {
    RouteDesc *d = reinterpret_cast<RouteDesc *>(const_cast<char *>(a.peer[threadIdx.x]));
    st_release_sys(&d->arrive[a.rank], a.epoch);
  }
}

// Requester side: every owner has written this rank's results (they are visible to the
// work queued after this kernel).
__global__ void k_route_wait_done(DevView v, RoutedArgs a) {
  if (threadIdx.x == 0) {
    const RouteDesc *d = reinterpret_cast<const RouteDesc *>(a.peer[a.rank]);
    wait_flags(v, d->done, a.nranks, a.epoch, a.timeout_ns);
    __threadfence_system();
  }
}

// Requester side (nranks > 1): pack this rank's query tokens into the region's 18-bit
// planes (hostpack.h layout) for the owners to pull over NVLink.  Work item = a
// 4096-position block of a query owned by ANOTHER rank (queries this rank owns itself are
// read from HBM as int32), located through k_route's block prefix pkf.  Each thread packs
// 8 consecutive positions per slot (two 16-byte loads, one 16-byte store of the low
// plane); the 4 threads of a 32-position group OR their 2-bit parts into the group's 8
// high-plane bytes (one 8-byte store).  All of a thread's loads are issued before any
// packing so a 64-thread CTA keeps 8 x 32 B in flight per thread.  Positions past a
// query's end pack as 0 (never compared).  Returns nonzero if any id is outside [0, 2^18)
// (the owners then read the int32 tokens instead).
constexpr int kPackNT = 256;
struct PackView {
  const int64_t *qoff, *qlen, *gsid;
  const int32_t *tok, *idx, *pkf;
  int64_t lo_off, hi_off, rec_off;  // planes / records at these offsets of the destination region
  int own0, nown;
  int64_t nrem, nblk;
};
__device__ __forceinline__ PackView pack_view(char *region) {
  RouteDesc *d = reinterpret_cast<RouteDesc *>(region);
  PackView w;
  w.qoff = reinterpret_cast<const int64_t *>(region + d->qoff_off);
  w.qlen = reinterpret_cast<const int64_t *>(region + d->len_off);
  w.tok = reinterpret_cast<const int32_t *>(region + d->tok_off);
  w.idx = reinterpret_cast<const int32_t *>(region + d->idx_off);
  w.gsid = reinterpret_cast<const int64_t *>(region + d->sid_off);
  w.pkf = reinterpret_cast<const int32_t *>(region + d->pkf_off);
  w.lo_off = d->lo_off;
  w.hi_off = d->hi_off;
  w.rec_off = d->rec_off;
  w.own0 = d->start[d->rank];
  w.nown = d->count[d->rank];
  w.nrem = d->n - w.nown;
  w.nblk = w.pkf[w.nrem];
  return w;
}
// block blk of remote query j (pkf[j] <= blk < pkf[j + 1]); bj = pkf[j].  The planes and
// the record go to the region at db: this rank's own (owners pull), or with push routing
// the owner's inbox slice for this rank (P2P stores over NVLink).
template <int NT>
__device__ __forceinline__ unsigned pack_block(const PackView &w, int64_t j, int64_t bj, int64_t blk, char *db) {
  constexpr int SL = kPackBlock / (8 * NT);  // 8-position slots per thread
  const int64_t pos = j < w.own0 ? j : j + w.nown;
  const int64_t q = w.idx[pos];
  uint16_t *plo = reinterpret_cast<uint16_t *>(db + w.lo_off);
  uint8_t *phi = reinterpret_cast<uint8_t *>(db + w.hi_off);
  RouteRec *rec = w.rec_off ? reinterpret_cast<RouteRec *>(db + w.rec_off) : nullptr;
  const int64_t off = w.qoff[q], len = w.qlen[q];
  const int64_t r0 = (blk - bj) * kPackBlock;
  const int64_t g = (rec && blk == bj && threadIdx.x == 0) ? w.gsid[q] : 0;  // in flight with the tokens
  const int k = threadIdx.x & 3;  // this thread's 8 positions within the 32-position group
  int4 a[SL], b[SL];
#pragma unroll
  for (int u = 0; u < SL; u++) {
    const int64_t r = r0 + 8 * (u * NT + (int64_t)threadIdx.x), p = off + r;
    if (r + 8 <= len) {
      a[u] = ldg_stream(reinterpret_cast<const int4 *>(w.tok + p));
      b[u] = ldg_stream(reinterpret_cast<const int4 *>(w.tok + p + 4));
    } else {
      int t[8];
#pragma unroll
      for (int e = 0; e < 8; e++) t[e] = r + e < len ? w.tok[p + e] : 0;
      a[u] = make_int4(t[0], t[1], t[2], t[3]);
      b[u] = make_int4(t[4], t[5], t[6], t[7]);
    }
  }
  if (rec && blk == bj && threadIdx.x == 0)  // the query's first block: its record
    rec[pos] = RouteRec{g, off, (int32_t)len, (int32_t)q, a[0].x, 1};
  unsigned bad = 0;
#pragma unroll
  for (int u = 0; u < SL; u++) {
    const int64_t r = r0 + 8 * (u * NT + (int64_t)threadIdx.x), p = off + r;
    if (r >= (len + 31) / 32 * 32) continue;  // (uniform per 32-position group)
    const int t[8] = {a[u].x, a[u].y, a[u].z, a[u].w, b[u].x, b[u].y, b[u].z, b[u].w};
    uint4 lo4;
    lo4.x = ((uint32_t)t[0] & 0xFFFFu) | ((uint32_t)t[1] << 16);
    lo4.y = ((uint32_t)t[2] & 0xFFFFu) | ((uint32_t)t[3] << 16);
    lo4.z = ((uint32_t)t[4] & 0xFFFFu) | ((uint32_t)t[5] << 16);
    lo4.w = ((uint32_t)t[6] & 0xFFFFu) | ((uint32_t)t[7] << 16);
    *reinterpret_cast<uint4 *>(plo + p) = lo4;
    unsigned long long h = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) {
      bad |= (uint32_t)t[e] >> 18;
      h |= (unsigned long long)(((uint32_t)t[e] >> 16) & 3u) << (8 * e + 2 * k);
    }
    const unsigned quad = __activemask();  // whole 32-position groups are active together
    h |= __shfl_xor_sync(quad, h, 1);
    h |= __shfl_xor_sync(quad, h, 2);
    if (k == 0) *reinterpret_cast<unsigned long long *>(phi + (p >> 5) * 8) = h;
  }
  return bad;
}

// tm_route_prepare with peers: every CTA packs one contiguous range of blocks (one
// binary search for its first query, then it steps through the queries in order)
__global__ void __launch_bounds__(kPackNT) k_route_pack(char *region, PushArgs pa) {
  const PackView w = pack_view(region);
  const int64_t per = (w.nblk + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(w.nblk, b0 + per);
  if (b0 >= b1) return;
  int64_t lo = 0, hi = w.nrem;  // last remote query j with pkf[j] <= b0
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (w.pkf[mid] <= b0) lo = mid; else hi = mid;
  }
  const RouteDesc *d = reinterpret_cast<const RouteDesc *>(region);
  // destination of query j: its owner's inbox slice (push) or this region
  auto dest = [&](int64_t j) -> char * {
    if (!pa.stride) return region;
    const int64_t pos = j < w.own0 ? j : j + w.nown;
    int o = 0;
    while (o + 1 < d->nranks && pos >= d->start[o + 1]) o++;
    return pa.peer[o] + pa.stride * d->rank;
  };
  int64_t j = lo, bj = w.pkf[j], bn = w.pkf[j + 1];
  char *db = dest(j);
  unsigned bad = 0;
  for (int64_t blk = b0; blk < b1; blk++) {
    if (blk >= bn) {
      while (blk >= bn) { j++; bj = bn; bn = w.pkf[j + 1]; }
      db = dest(j);
    }
    bad |= pack_block<kPackNT>(w, j, bj, blk, db);
  }
  if (bad) atomicOr(&reinterpret_cast<RouteDesc *>(region)->pk_bad, 1);
  if (pa.stride) __threadfence_system();  // P2P stores ordered before the arrive flag
}

// Owner side.  Two work queues, each longest first: this rank's own queries (HBM only)
// and the other ranks' (query bytes over NVLink).  1/np of the CTAs start on the local
// queue and the rest on the remote one, each falling back to the other when its queue
// runs dry, so HBM and the links are busy at the same time instead of in phases.
// Dynamic shared memory: [TmaRing (only when nranks > 1)][3 x kPlanNB x nranks + 2 ints
// of routing tables], sized by routed_smem_bytes so a single rank keeps full occupancy.
template <class RG>
__host__ __device__ constexpr size_t routed_smem_bytes(int nranks, bool packed) {
  return (packed ? (sizeof(RG) + 15) / 16 * 16 : 0) + sizeof(int) * (3 * (size_t)kPlanNB * nranks + 2);
}

template <int NT, int U, bool PACKED, class RG = RoutedPackedRing, int MINB = 6>
__global__ void __launch_bounds__(NT, NT == 64 ? MINB : 1) k_walk_routed(DevView v, RoutedArgs a) {
  extern __shared__ __align__(16) char dyn[];
  __shared__ WalkShared sh;
  __shared__ long long s_item;
  __shared__ int s_cell;
  __shared__ int s_nloc;  // cells in the local queue
  __shared__ RouteRec s_rec;
  __shared__ bool s_has_rec;
  __shared__ long long s_trace;
  const int np = a.nranks;
  const int ncell = kPlanNB * np;
  // TMA-staged compare for remote queries: bulk copies pull the query's 18-bit planes
  // over NVLink (2.25 B per position instead of 4)
  RG *rg = PACKED ? reinterpret_cast<RG *>(dyn) : nullptr;
  if constexpr (PACKED) packed_ring_init(*rg);
  int *s_pre = reinterpret_cast<int *>(dyn + (PACKED ? (sizeof(RG) + 15) / 16 * 16 : 0));  // ncell + 2
  int *s_bs = s_pre + ncell + 2;
  int *s_peer = s_bs + ncell;
  RouteDesc *own = reinterpret_cast<RouteDesc *>(const_cast<char *>(a.peer[a.rank]));
  if (a.epoch > 0) {  // device-side barrier: every requester has bucketed its batch
    if (threadIdx.x == 0) wait_flags(v, own->arrive, np, a.epoch, a.timeout_ns);
    __syncthreads();
  }
  // cell c: local cells first (bucket order), then remote cells (bucket, peer) order
  for (int c = threadIdx.x; c < ncell; c += NT) {
    int bk, p;
    if (c < kPlanNB) { bk = c; p = a.rank; }
    else { const int r = c - kPlanNB; bk = r / (np - 1); const int q = r % (np - 1); p = q < a.rank ? q : q + 1; }
    const RouteDesc *d = reinterpret_cast<const RouteDesc *>(a.peer[p]);
    s_pre[c] = d->bcount[a.rank * kPlanNB + bk];
    s_bs[c] = d->bstart[a.rank * kPlanNB + bk];
    s_peer[c] = p;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // separate exclusive scans for the two queues
    int acc = 0;
    for (int c = 0; c < kPlanNB; c++) { int t = s_pre[c]; s_pre[c] = acc; acc += t; }
    s_pre[ncell] = acc;  // local total
    acc = 0;
    for (int c = kPlanNB; c < ncell; c++) { int t = s_pre[c]; s_pre[c] = acc; acc += t; }
    s_pre[ncell + 1] = acc;  // remote total
    s_nloc = kPlanNB;
  }
  __syncthreads();
  const long long tot[2] = {s_pre[ncell], s_pre[ncell + 1]};
  // per-source views (read once per launch, after the arrive barrier: the requesters'
  // headers and pack flags are final for this batch)
  struct PeerInfo {
    const int32_t *tok;
    int64_t *m, *par, *dup;
    const uint16_t *plo;
    const uint8_t *phi;
    const int4 *rec;  // RouteRec per idx position (nullptr: none)
    const int32_t *idx;
    const int64_t *gsid, *qoff, *qlen;
    int packed;  // remote queries of this source compare through the 18-bit planes
  };
  __shared__ PeerInfo s_pi[kMaxRanks];
  __shared__ int32_t s_sid;
  if (threadIdx.x < np) {
    const int p = threadIdx.x;
    char *reg = const_cast<char *>(a.peer[p]);
    const RouteDesc *d = reinterpret_cast<const RouteDesc *>(reg);
    // push routing: planes and records of source p sit in this rank's inbox slice p
    const char *ib = a.push_stride ? reinterpret_cast<const char *>(own) + a.push_stride * p : reg;
    const RouteDesc *id = a.push_stride ? own : d;
    PeerInfo pi;
    pi.tok = reinterpret_cast<const int32_t *>(reg + d->tok_off);
    pi.m = reinterpret_cast<int64_t *>(reg + d->m_off);
    pi.par = reinterpret_cast<int64_t *>(reg + d->par_off);
    pi.dup = reinterpret_cast<int64_t *>(reg + d->dup_off);
    pi.plo = reinterpret_cast<const uint16_t *>(ib + id->lo_off);
    pi.phi = reinterpret_cast<const uint8_t *>(ib + id->hi_off);
    pi.rec = id->rec_off ? reinterpret_cast<const int4 *>(ib + id->rec_off) : nullptr;
    pi.idx = reinterpret_cast<const int32_t *>(reg + d->idx_off);
    pi.gsid = reinterpret_cast<const int64_t *>(reg + d->sid_off);
    pi.qoff = reinterpret_cast<const int64_t *>(reg + d->qoff_off);
    pi.qlen = reinterpret_cast<const int64_t *>(reg + d->len_off);
    pi.packed = PACKED && p != a.rank && d->lo_off && !*reinterpret_cast<const volatile int32_t *>(&d->pk_bad);
    s_pi[p] = pi;
  }
  __syncthreads();
  // tail CTAs take the shortest remaining items (and prefer the remote queue): each queue
  // counter holds head claims in its low and tail claims in its high 32 bits, so one
  // atomic hands out every item exactly once from either end
  const bool tail = a.tail_every > 0 && blockIdx.x % a.tail_every == (unsigned)a.tail_every - 1;
  int q = (np > 1 && (tail || blockIdx.x % np != 0)) ? 1 : 0;  // queue this CTA prefers
  bool dry[2] = {false, false};
  // thread 0: claim the next item; `left` = items still unclaimed in its queue after it
  auto claim = [&](long long &it, int &cell, long long &left) {
    it = -1;
    cell = -1;
    left = 0;
    while (it < 0 && !(dry[0] && dry[1])) {
      const int qq = dry[q] ? 1 - q : q;
      const unsigned long long old = atomicAdd(qq ? &a.sched->work2 : &a.sched->work, tail ? (1ull << 32) : 1ull);
      const long long h = (long long)(old & 0xffffffffull), t = (long long)(old >> 32);
      if (h + t >= tot[qq]) { dry[qq] = true; continue; }
      const long long x = tail ? tot[qq] - 1 - t : h;
      int lo = qq ? kPlanNB : 0, hi = qq ? ncell : kPlanNB;  // last cell with prefix <= x
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (s_pre[mid] <= x) lo = mid; else hi = mid;
      }
      it = x;
      cell = lo;
      left = tot[qq] - 1 - h - t;
    }
  };
  // The item's record (one load, over NVLink for a pulled remote query) is requested one
  // item ahead while the queue still holds more than one item per CTA, so its latency
  // hides under the current walk (near the end items are claimed only when a CTA is free).
  // Thread 0's look-ahead state lives in shared memory and the record is copied by
  // cp.async straight into it: nothing stays live in registers across the walk.
  __shared__ long long s_nit;
  __shared__ int s_ncell, s_nready;
  __shared__ __align__(16) int4 s_nrec[2];
  auto request = [&]() {  // thread 0, s_nit >= 0
    const int4 *rp = s_pi[s_peer[s_ncell]].rec;
    s_nready = rp != nullptr;
    if (rp) {
      rp += 2 * (s_bs[s_ncell] + (s_nit - s_pre[s_ncell]));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&s_nrec[0])), "l"(rp) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&s_nrec[1])), "l"(rp + 1) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  constexpr long long kClaimLater = -2;
  constexpr int kLookaheadLen = 8192;
  if (threadIdx.x == 0) s_nit = kClaimLater;
  for (;;) {
    if (threadIdx.x == 0) {
      if (s_nit == kClaimLater) {
        long long nit, left;
        int ncell;
        claim(nit, ncell, left);
        s_nit = nit;
        s_ncell = ncell;
        s_nready = 0;
      }
      const long long it = s_nit;
      const int cell = s_ncell;
      s_item = it;
      s_cell = cell;
      if (it >= 0) {
        if (!s_nready) request();
        const PeerInfo &pi = s_pi[s_peer[cell]];
        if (pi.rec) {
          asm volatile("cp.async.wait_all;" ::: "memory");
          const int4 n0 = s_nrec[0], n1 = s_nrec[1];
          s_rec.gsid = (int64_t)(uint32_t)n0.x | ((int64_t)n0.y << 32);
          s_rec.off = (int64_t)(uint32_t)n0.z | ((int64_t)n0.w << 32);
          s_rec.len = n1.x;
          s_rec.qi = n1.y;
          s_rec.q0 = n1.z;
          s_rec.has_q0 = n1.w;
        } else {  // no records (routing without planes): the batch arrays
          const int32_t qi = pi.idx[s_bs[cell] + (it - s_pre[cell])];
          s_rec.qi = qi;
          s_rec.gsid = pi.gsid[qi];
          s_rec.off = pi.qoff[qi];
          s_rec.len = (int32_t)pi.qlen[qi];
          s_rec.q0 = 0;
          s_rec.has_q0 = 0;
        }
        const int64_t g = s_rec.gsid;
        s_sid = (g >= 0 && g < a.g2l_len) ? a.g2l[g] : -1;
        // the next item is claimed (and its record requested) now only for a short current
        // item while the queue is far from empty: claiming ahead of a long item would pair
        // long items on one CTA and break the longest-first balance
        s_nit = kClaimLater;
        if (s_rec.len <= kLookaheadLen) {
          long long nit, left;
          int ncell;
          claim(nit, ncell, left);
          s_nit = nit;
          s_ncell = ncell;
          s_nready = 0;
          if (nit >= 0 && left > (long long)gridDim.x) request();
        }
      }
    }
    __syncthreads();
    const long long it = s_item;
    const int cell = s_cell;
    if (a.trace && threadIdx.x == 0 && it >= 0) {  // diagnostics: item start
      const long long k = atomicAdd(reinterpret_cast<unsigned long long *>(a.trace), 1ull);
      s_trace = k < a.trace_cap ? k : -1;
      if (s_trace >= 0) a.trace[4 + 4 * s_trace] = (long long)globaltimer_ns();
    }
    if (it < 0) {
      if (sched_exit(a.sched) && a.epoch > 0) {  // last CTA out: results are written, tell every requester
        __threadfence_system();
        for (int p = 0; p < np; p++)
          st_release_sys(&reinterpret_cast<RouteDesc *>(const_cast<char *>(a.peer[p]))->done[a.rank], a.epoch);
      }
      return;
    }
    const int p = s_peer[cell];
    const PeerInfo &pi = s_pi[p];
    const int32_t qi = s_rec.qi;
    const int64_t off = s_rec.off;
    const int L = s_rec.len;
    const int32_t sid = s_sid;
    const int32_t *q0p = s_rec.has_q0 ? &s_rec.q0 : nullptr;  // read by thread 0 before s_rec changes
    WalkOut o{pi.m + qi, pi.par + qi, pi.dup + qi, nullptr, nullptr};
    __syncthreads();  // s_rec / s_sid are read: thread 0 may overwrite them for the next item
    if (sid < 0) {  // unknown id, or routed to the wrong owner: flag it, never guess
      if (threadIdx.x == 0) { *o.m = -1; *o.parent = -1; *o.dup = -1; }
      continue;
    }
    const int32_t *q = pi.tok + off;
    if (PACKED && pi.packed) {
      // remote query: packed planes, TMA bulk copies over NVLink (or out of this rank's
      // inbox when the requester pushed them)
      const PackedQuery pk{pi.plo, pi.phi, off};
      if constexpr (PACKED) walk_query<NT, U>(v, q, L, sid, nullptr, o, sh, rg, &pk, q0p);
    } else {  // local (or ids beyond 18 bits): int32, registers
      walk_query<NT, U, NoRing>(v, q, L, sid, nullptr, o, sh, nullptr, nullptr, q0p);
    }
    if (a.trace && threadIdx.x == 0 && s_trace >= 0) {
      long long *t = a.trace + 4 + 4 * s_trace;
      t[1] = (long long)globaltimer_ns();
      t[2] = (long long)L | ((long long)(p != a.rank) << 40) | ((long long)max(0, (int)*o.m) << 41);
      t[3] = blockIdx.x;
    }
  }
}

// ----------------------------------------------------------------------------------
// K2 record: one persistent launch per batch.  Work item = a session's CHAIN of entries
// (its inserts in batch order: the sequential semantics of lpm_insert, trie.py:120-179,
// only bind entries of the same session — sessions never share rows or branch keys).
// The CTA owning a chain walks and commits each entry in order; chains run in parallel,
// longest first.  Row ids are reserved by the host in batch order (deterministic; an entry
// that re-records an existing sequence leaves its slot to be reused).
//
// A chain is serial, so its cost is the latency of each entry's dependent steps, not its
// bytes: k_record keeps only the steps the NEXT entry of the chain depends on (the walk,
// the row table, the branch index, the session counters) and leaves everything else to
// the chain's end (or a copy warp beside the chain): arena / run-table
// allocation, the novel suffix copy, the metadata runs.  Until then a committed row is
// read where its tokens already are - in its entry's query (read-only for the launch).
// Inside an entry, the session's counters and path-copy state live in shared memory for
// the whole chain, the entries' offsets / lengths / first tokens are fetched 64 at a time,
// a row's fields are read in one round trip, and the compare hands back the two tokens at
// the mismatch out of the shared-memory stage that held them.

__device__ __forceinline__ int first_run_at(const Batch &b, int64_t w, int64_t m) {
  // index (relative) of the run containing position m (runs start at 0, ascending)
  int64_t r0 = b.run_off[w], r1 = b.run_off[w + 1];
  int64_t lo = r0, hi = r1;  // last run with start <= m
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (b.run_start[mid] <= m) lo = mid; else hi = mid;
  }
  return (int)(lo - r0);
}

constexpr int kCopyU = 4;      // int4 loads in flight per thread in K2's copies
constexpr int kRecPre = 64;    // entries whose offset / length / first token are fetched at once
constexpr int kRecCache = 4;   // per-chain root-row and row-field cache entries
constexpr int kRecQ = 32;      // copy queue slots (warp-specialised K2)

struct RowFields {  // what the walk and the commit need of a row, read in one round trip
  long long vb, ext, ext_vb, jump;
  int len, m, ext_tok, ext_len, depth;
};

__device__ __forceinline__ void load_row(const DevView &v, int64_t r, RowFields &f) {
  f.vb = v.row_vb[r];
  f.len = v.row_len[r];
  f.m = v.row_m[r];
  f.ext = v.row_ext[r];
  f.ext_tok = v.row_ext_tok[r];
  f.ext_len = v.row_ext_len[r];
  f.ext_vb = v.row_ext_vb[r];
  f.depth = v.row_depth[r];
  f.jump = v.row_jump[r];
}

struct RecShared {
  int red[4];
  int cap[10];  // compare capture: per-warp (q, a) tokens, then the CTA's (<= 4 warps)
  // the current entry
  long long off;
  int len, q0;
  // the walk
  long long row;
  int lo, pc_len;
  RowFields f;       // the current row's fields
  long long m, parent, dup;
  int tnext, spar;
  RowFields pf;      // the parent's fields (commit)
  // the chain's session (cached for the whole chain, written back at its end)
  int sid, nrows;
  long long stored, naive;
  long long pc_row, pc_vb, pc_cap;
  int pc_rlen, pc_depth;  // the path copy's row: length, depth
  // path-copy upkeep of the current entry
  long long pcw_vb;
  int pcw_from, pcw_len;
  // per-chain caches (thread 0): root rows by first token and row fields.  Valid for the
  // whole chain: root keys never change, and the only fields of this session's rows that
  // change inside the launch are extension hints, which this CTA's commits set (and update
  // here).  A 16-branch session walks root -> shared-prefix row without a global load.
  int rc_tok[kRecCache];
  long long rc_row[kRecCache];
  long long fc_row[kRecCache];
  RowFields fc[kRecCache];
  int rc_next, fc_next;
  // copy warp queue (warp-specialised k_record_tma): committed entries whose novel suffix the
  // copy warp moves into the arena while the walk warps go on with the chain
  int q_e[kRecQ], q_m[kRecQ], q_L[kRecQ];
  long long q_off[kRecQ];
  int q_head, q_read, q_closed, q_done;
  // entry prefetch
  long long pre_off[kRecPre];
  int pre_len[kRecPre], pre_q0[kRecPre];
  // the chain's results for its end (chains of <= kRecPre entries): matched, new row
  int win_m[kRecPre];
  unsigned char win_new[kRecPre];
};

__device__ __forceinline__ void rec_cache_row(RecShared &sh, int64_t r, const RowFields &f) {
  for (int i = 0; i < kRecCache; i++)
    if (sh.fc_row[i] == r) { sh.fc[i] = f; return; }
  const int i = sh.fc_next++ % kRecCache;
  sh.fc_row[i] = r;
  sh.fc[i] = f;
}

__device__ __forceinline__ void rec_row(const DevView &v, RecShared &sh, int64_t r, RowFields &f) {
  for (int i = 0; i < kRecCache; i++)
    if (sh.fc_row[i] == r) { f = sh.fc[i]; return; }
  load_row(v, r, f);
  rec_cache_row(sh, r, f);
}

__device__ __forceinline__ int64_t rec_root(const DevView &v, RecShared &sh, int32_t t) {
  for (int i = 0; i < kRecCache; i++)
    if (sh.rc_row[i] >= 0 && sh.rc_tok[i] == t) return sh.rc_row[i];
  const int64_t r = ht_find(v, kRootTag | (uint64_t)(uint32_t)sh.sid, dt_key(0, t, false));
  if (r >= 0) {
    const int i = sh.rc_next++ % kRecCache;
    sh.rc_tok[i] = t;
    sh.rc_row[i] = r;
  }
  return r;
}

// Whole-CTA walk of the chain's current entry (sh.off / sh.len / sh.q0), the LPM walk of
// trie.py:136-158 over rows (see walk_query): results into sh.m / parent / dup / tnext /
// spar and the parent's fields into sh.pf.
template <int NT, int BAR, int S, int CHV>
__device__ __forceinline__ void record_walk(const DevView &v, const Batch &b, RecShared &sh,
                                            TmaRing<NT, S, CHV> &rg) {
  static_assert(NT <= 128, "RecShared holds the compare scratch of <= 4 warps");
  constexpr int kCapQ = 2 * (NT / 32);  // where the compare leaves the tokens at the mismatch
  const int32_t *q = b.tok + sh.off;
  const int L = sh.len;
  if (threadIdx.x == 0) {
    sh.pc_len = 0;
    const int64_t r = rec_root(v, sh, sh.q0);
    if (sh.pc_row >= 0 && r >= 0) sh.pc_len = min(L, sh.pc_rlen);
    sh.row = r;
  }
  group_sync<NT, BAR>();
  int jpc = 0;
  if (sh.pc_len > 0) jpc = block_first_mismatch_tma<NT, S, CHV, BAR>(q, v.arena + sh.pc_vb, 0, sh.pc_len, sh.red, rg);
  if (threadIdx.x == 0) {
    int64_t r = sh.row;
    int lo = 1;
    if (jpc > 0) {  // owner of position jpc-1 on the copy's path: O(log depth) ancestor search
      r = sh.pc_row;
      while (v.row_m[r] > jpc - 1) {
        const int64_t jp = v.row_jump[r];
        r = (jp >= 0 && v.row_m[jp] > jpc - 1) ? jp : v.row_parent[r];
      }
      lo = jpc;
    }
    if (r < 0) {  // nothing shares the first token: matched 0
      sh.m = 0;
      sh.parent = -1;
      sh.dup = -1;
      sh.tnext = sh.q0;
      sh.spar = -1;
    } else {
      rec_row(v, sh, r, sh.f);
    }
    sh.row = r;
    sh.lo = lo;
  }
  group_sync<NT, BAR>();
  while (sh.row >= 0) {
    const int64_t r = sh.row;
    const int lo = sh.lo, Lr = sh.f.len;
    const int hi = min(Lr, L);
    TM_DCHECK(v, (sh.f.vb + sh.f.m >= 0 && sh.f.vb + ((Lr + 3) & ~3) <= v.arena_cap) ||
                     (sh.f.vb + sh.f.m >= v.qv_lo && sh.f.vb + ((Lr + 3) & ~3) <= v.qv_hi), kErrArena);
    const int32_t *a = v.arena + sh.f.vb;
    const int j = block_first_mismatch_tma<NT, S, CHV, BAR>(q, a, lo, hi, sh.red, rg, sh.cap);
    if (threadIdx.x == 0) {
      int64_t next = -1;
      if (j < L) {
        const int32_t t = j < hi ? sh.cap[kCapQ] : q[j];  // j == hi == Lr: the row ended before the query
        if (j == Lr && sh.f.ext >= 0 && t == sh.f.ext_tok) next = sh.f.ext;
        else next = ht_find(v, (uint64_t)r, dt_key(j, t, false));
        if (next < 0) {
          sh.m = j;
          sh.parent = r;
          sh.dup = -1;
          sh.tnext = t;
          sh.spar = j < Lr ? sh.cap[kCapQ + 1] : -1;
          sh.pf = sh.f;
        } else {
          rec_row(v, sh, next, sh.f);
        }
      } else {  // the query ended inside (or at the end of) row r
        sh.m = L;
        sh.parent = r;
        sh.dup = (L == Lr) ? r : ht_find(v, (uint64_t)r, dt_key(L, 0, true));
        sh.tnext = -1;
        sh.spar = L < Lr ? a[L] : -1;
        sh.pf = sh.f;
      }
      sh.row = next;
      sh.lo = j + 1;
    }
    group_sync<NT, BAR>();
  }
}

// Commit the walked entry e (thread 0): row table, the parent's extension hint, the
// branch index, the session counters (shared memory).  Arena / run slots: the chain's copy.
__device__ __forceinline__ void record_commit(const DevView &v, const Batch &b, int64_t e, RecShared &sh) {
  const int64_t m = sh.m, L = sh.len, par = sh.parent;
  sh.pcw_len = 0;  // no path-copy write unless this entry's row takes the copy (below)
  b.o_m[e] = m;
  b.o_parent[e] = par;
  b.o_dup[e] = sh.dup;
  b.o_tnext[e] = sh.tnext;
  b.o_spar[e] = sh.spar;
  sh.naive += L;
  const int64_t row = b.c_row[e];
  TM_DCHECK(v, row >= 0 && row < v.row_cap, kErrRow);
  if (sh.dup >= 0) {  // re-recorded sequence: its reserved slot stays an empty hole
    v.row_len[row] = 0;
    v.row_sess[row] = -1;
    b.c_row[e] = sh.dup;
    b.c_local[e] = v.row_local[sh.dup];
    return;
  }
  const int64_t vbq = (int64_t)((b.tok + sh.off) - v.arena);  // the row's positions, in its query
  // skew-binary jump pointer (Myers): O(1) here, O(log depth) ancestor searches
  int64_t jmp = -1;
  if (par >= 0) {
    const int64_t j1 = sh.pf.jump;
    int64_t j2 = -1;
    int32_t d1 = -1, d2 = -1;
    if (j1 >= 0) {
      j2 = v.row_jump[j1];
      d1 = v.row_depth[j1];
      d2 = j2 >= 0 ? v.row_depth[j2] : -1;
    }
    jmp = (j1 >= 0 && sh.pf.depth - d1 == d1 - d2) ? j2 : par;
  }
  const int32_t local = sh.nrows++;
  const int32_t depth = par >= 0 ? sh.pf.depth + 1 : 0;
  sh.stored += L - m;
  v.row_vb[row] = vbq;
  v.row_m[row] = (int32_t)m;
  v.row_len[row] = (int32_t)L;
  v.row_parent[row] = par;
  v.row_sess[row] = sh.sid;
  v.row_local[row] = local;
  v.row_depth[row] = depth;
  v.row_ext[row] = -1;
  v.row_jump[row] = jmp;
  // the parent's extension hint; its only readers are this CTA's later entries (same
  // session chain) and later launches, so program order suffices
  if (par >= 0 && L > m && m == sh.pf.len && sh.pf.ext < 0) {
    v.row_ext_tok[par] = sh.tnext;
    v.row_ext_len[par] = (int32_t)L;
    v.row_ext_vb[par] = vbq;
    v.row_ext[par] = row;
    for (int i = 0; i < kRecCache; i++)
      if (sh.fc_row[i] == par) {
        sh.fc[i].ext = row;
        sh.fc[i].ext_tok = sh.tnext;
        sh.fc[i].ext_len = (int32_t)L;
        sh.fc[i].ext_vb = vbq;
      }
  }
  {
    RowFields nf;
    nf.vb = vbq;
    nf.len = (int)L;
    nf.m = (int)m;
    nf.ext = -1;
    nf.ext_tok = 0;
    nf.ext_len = 0;
    nf.ext_vb = 0;
    nf.depth = depth;
    nf.jump = jmp;
    rec_cache_row(sh, row, nf);
    if (m == 0 && L > 0) {  // a new root row, keyed by its first token (tnext = q[0])
      const int i = sh.rc_next++ % kRecCache;
      sh.rc_tok[i] = sh.tnext;
      sh.rc_row[i] = row;
    }
  }
  const uint64_t owner = m > 0 ? (uint64_t)par : (kRootTag | (uint64_t)(uint32_t)sh.sid);
  if (L > m) ht_insert(v, owner, dt_key(m, sh.tnext, false), row);  // tnext = q[m]
  else ht_insert(v, owner, dt_key(m, 0, true), row);
  b.c_local[e] = local;
  // session path copy upkeep (rows at chain depth >= kPathCopyDepth): a turn that extends
  // the copy's row exactly at its end appends only its new tokens (2x headroom); a row
  // deeper than the copy's re-seats the copy (in place when it fits, else a fresh buffer
  // of twice its length); siblings and shallower rows leave it alone, so sampling many
  // completions of one deep turn costs no copies and a session's copy buffers total
  // <= 4x its longest sequence.
  if (depth >= kPathCopyDepth) {
    int64_t vb = sh.pc_vb, cap = sh.pc_cap, from = m;
    bool write = true;
    if (sh.pc_row >= 0 && par == sh.pc_row && m == sh.pc_rlen && L <= cap) {
      // the next turn of the copy's own chain: append
    } else if (sh.pc_row < 0 || depth > sh.pc_depth) {
      from = 0;
      if (sh.pc_row < 0 || L > cap) {
        cap = (2 * L + kAlignWords - 1) / kAlignWords * kAlignWords;
        vb = (long long)atomicAdd((unsigned long long *)&v.ctr[0], (unsigned long long)cap);
      }
    } else {
      write = false;
    }
    if (write) {
      TM_DCHECK(v, vb >= 0 && vb + cap <= v.arena_cap, kErrArena);
      sh.pc_row = row;
      sh.pc_vb = vb;
      sh.pc_cap = cap;
      sh.pc_rlen = (int)L;
      sh.pc_depth = depth;
      sh.pcw_vb = vb;
      sh.pcw_from = (int)from;
      sh.pcw_len = (int)L;
    }
  }
}

// The copy warp of the warp-specialised K2: takes committed entries from the queue in
// order, allocates their arena lines and run slots (atomics off the chain's serial path),
// moves the novel suffix [m, L) from the query into the arena (8 int4 loads in flight per
// lane) and the runs (first clamped to m) into the run table.  The row keeps reading its
// query until the chain's end switches its virtual base.
__device__ void record_copy_warp(const DevView &v, const Batch &b, RecShared &sh) {
  const int lane = threadIdx.x & 31;
  for (int i = 0;; i++) {
    int e = -1, m = 0, L = 0;
    long long off = 0;
    if (lane == 0) {
      for (;;) {
        const int head = *(volatile int *)&sh.q_head;
        if (i < head) break;
        if (*(volatile int *)&sh.q_closed && i >= *(volatile int *)&sh.q_head) { i = -1; break; }
        __nanosleep(100);
      }
      if (i >= 0) {
        __threadfence_block();
        const int slot = i % kRecQ;
        e = *(volatile int *)&sh.q_e[slot];
        m = *(volatile int *)&sh.q_m[slot];
        L = *(volatile int *)&sh.q_L[slot];
        off = *(volatile long long *)&sh.q_off[slot];
        __threadfence_block();
        *(volatile int *)&sh.q_read = i + 1;  // the slot may be reused (one reader, in order)
      }
    }
    e = __shfl_sync(0xffffffffu, e, 0);
    if (__shfl_sync(0xffffffffu, i, 0) < 0) return;
    m = __shfl_sync(0xffffffffu, m, 0);
    L = __shfl_sync(0xffffffffu, L, 0);
    off = __shfl_sync(0xffffffffu, off, 0);
    // the arena atomic, the run table's offsets, the suffix's first round and up to 32 run
    // starts are all in flight together; only the stores wait for the allocations
    long long vb = 0, run0 = 0;
    if (lane == 0) {
      const long long words = ((L + kAlignWords - 1) / kAlignWords) * kAlignWords - ((long long)m / kAlignWords) * kAlignWords;
      vb = (long long)atomicAdd((unsigned long long *)&v.ctr[0], (unsigned long long)words) - (m / kAlignWords) * kAlignWords;
    }
    const int64_t ra = b.run_off[e], rb = b.run_off[e + 1];
    const int4 *src = reinterpret_cast<const int4 *>(b.tok + off);
    const int64_t i1 = (L + 3) >> 2;
    const int64_t base0 = (m >> 2) + lane;
    int4 t[8];
#pragma unroll
    for (int k = 0; k < 8; k++) t[k] = ldg_stream_if(src + base0 + 32 * k, base0 + 32 * k < i1);
    int fr;
    int32_t rst = 0, rver = 0;
    uint8_t rorg = 0;
    const bool few = rb - ra <= 32;
    if (few) {  // the run containing m: one round of loads and a ballot
      const bool have = lane < rb - ra;
      if (have) {
        rst = b.run_start[ra + lane];
        rorg = b.run_origin[ra + lane];
        rver = b.run_version[ra + lane];
      }
      fr = __popc(__ballot_sync(0xffffffffu, have && lane > 0 && rst <= m));
    } else {
      fr = lane == 0 ? first_run_at(b, e, m) : 0;
      fr = __shfl_sync(0xffffffffu, fr, 0);
    }
    const int nr = (int)(rb - ra) - fr;
    if (lane == 0) run0 = (long long)atomicAdd((unsigned long long *)&v.ctr[2], (unsigned long long)nr);
    vb = __shfl_sync(0xffffffffu, vb, 0);
    run0 = __shfl_sync(0xffffffffu, run0, 0);
    TM_DCHECK(v, vb + (m & ~31ll) >= 0 && vb + ((L + 31) & ~31ll) <= v.arena_cap, kErrArena);
    TM_DCHECK(v, run0 >= 0 && run0 + nr <= v.run_cap, kErrRun);
    int4 *dst = reinterpret_cast<int4 *>(v.arena + vb);
#pragma unroll
    for (int k = 0; k < 8; k++) stg_if(dst + base0 + 32 * k, t[k], base0 + 32 * k < i1);
    for (int64_t base = base0 + 32 * 8; base < i1; base += 32 * 8) {
#pragma unroll
      for (int k = 0; k < 8; k++) t[k] = ldg_stream_if(src + base + 32 * k, base + 32 * k < i1);
#pragma unroll
      for (int k = 0; k < 8; k++) stg_if(dst + base + 32 * k, t[k], base + 32 * k < i1);
    }
    if (few) {
      if (lane >= fr && lane < rb - ra) {
        v.run_start[run0 + lane - fr] = rst > m ? rst : m;
        v.run_origin[run0 + lane - fr] = rorg;
        v.run_version[run0 + lane - fr] = rver;
      }
    } else {
      const int64_t r0 = ra + fr;
      for (int k = lane; k < nr; k += 32) {
        const int32_t st = b.run_start[r0 + k];
        v.run_start[run0 + k] = st > m ? st : m;
        v.run_origin[run0 + k] = b.run_origin[r0 + k];
        v.run_version[run0 + k] = b.run_version[r0 + k];
      }
    }
    if (lane == 0) {
      b.c_vb[e] = vb;
      b.c_run0[e] = run0;
      b.c_firstrun[e] = fr;
      __threadfence_block();
      *(volatile int *)&sh.q_done = i + 1;  // records complete in queue order (one copy warp)
    }
  }
}

// A committed row switches to its arena copy (virtual base, runs; a prefix row has none),
// and a parent's extension hint pointing at it follows.
__device__ __forceinline__ void record_finish_entry(const DevView &v, const Batch &b, int64_t e) {
  if (b.o_dup[e] >= 0) return;
  const int64_t m = b.o_m[e], L = b.len[e], row = b.c_row[e];
  const bool own = L > m;
  const int64_t vb = own ? b.c_vb[e] : -m;
  v.row_vb[row] = vb;
  v.row_run0[row] = own ? b.c_run0[e] : 0;
  v.row_nrun[row] = own ? (int32_t)(b.run_off[e + 1] - b.run_off[e] - b.c_firstrun[e]) : 0;
  const int64_t par = b.o_parent[e];
  if (par >= 0 && v.row_ext[par] == row) v.row_ext_vb[par] = vb;
}

// Chain end without a copy warp: the walk group allocates the chain's arena lines and run
// slots (one scan, one atomic per counter), moves every suffix and its runs, and switches
// the rows.  Only this CTA ever reads the session's rows inside the launch, so switching
// here is safe; chains that finish early overlap their copies with the walks of others.
template <int NT, int BAR>
__device__ void record_chain_copy(const DevView &v, const Batch &b, int64_t e0, int64_t e1, long long *s_scan,
                                  const RecShared &sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool win = e1 - e0 <= kRecPre;  // the chain's results are still in shared memory
  for (int64_t base = e0; base < e1; base += NT) {
    const int64_t e = base + threadIdx.x;
    long long words = 0, runs = 0;
    int fr = 0;
    int64_t m = 0;
    const bool isnew = e < e1 && (win ? sh.win_new[e - e0] != 0 : b.o_dup[e] < 0);
    if (isnew) {
      m = win ? sh.win_m[e - e0] : b.o_m[e];
      const int64_t L = win ? sh.pre_len[e - e0] : b.len[e];
      if (L > m) {
        words = ((L + kAlignWords - 1) / kAlignWords) * kAlignWords - (m / kAlignWords) * kAlignWords;
        const int64_t r0 = b.run_off[e], r1 = b.run_off[e + 1];
        if (r1 - r0 <= 4) {  // a few runs: read them at once (one round trip, no search chain)
          int32_t st[4];
#pragma unroll
          for (int k = 0; k < 4; k++) st[k] = r0 + k < r1 ? b.run_start[r0 + k] : 0x7fffffff;
#pragma unroll
          for (int k = 1; k < 4; k++) fr += st[k] <= m ? 1 : 0;
        } else {
          fr = first_run_at(b, e, m);
        }
        runs = (r1 - r0) - fr;
      }
    }
    long long iw = words, ir = runs;  // inclusive scans within the warp, then across warps
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long tw = __shfl_up_sync(0xffffffffu, iw, d), tr = __shfl_up_sync(0xffffffffu, ir, d);
      if (lane >= d) { iw += tw; ir += tr; }
    }
    if (lane == 31) { s_scan[2 * warp] = iw; s_scan[2 * warp + 1] = ir; }
    group_sync<NT, BAR>();
    if (threadIdx.x == 0) {
      long long tw = 0, tr = 0;
      for (int w = 0; w < NT / 32; w++) {
        const long long x = s_scan[2 * w], y = s_scan[2 * w + 1];
        s_scan[2 * w] = tw;
        s_scan[2 * w + 1] = tr;
        tw += x;
        tr += y;
      }
      s_scan[8] = tw ? (long long)atomicAdd((unsigned long long *)&v.ctr[0], (unsigned long long)tw) : 0;
      s_scan[9] = tr ? (long long)atomicAdd((unsigned long long *)&v.ctr[2], (unsigned long long)tr) : 0;
    }
    group_sync<NT, BAR>();
    if (words) {
      const long long vb = s_scan[8] + s_scan[2 * warp] + iw - words - (m / kAlignWords) * kAlignWords;
      const long long run0 = s_scan[9] + s_scan[2 * warp + 1] + ir - runs;
      TM_DCHECK(v, vb + (m & ~31ll) >= 0 && vb + ((b.len[e] + 31) & ~31ll) <= v.arena_cap, kErrArena);
      TM_DCHECK(v, run0 >= 0 && run0 + runs <= v.run_cap, kErrRun);
      b.c_vb[e] = vb;
      b.c_run0[e] = run0;
      b.c_firstrun[e] = fr;
    }
    group_sync<NT, BAR>();
  }
  for (int64_t e = e0; e < e1; e++) {  // the whole group on each entry's suffix and runs
    if (win ? !sh.win_new[e - e0] : b.o_dup[e] >= 0) continue;
    const int64_t m = win ? sh.win_m[e - e0] : b.o_m[e], L = win ? sh.pre_len[e - e0] : b.len[e];
    if (L <= m) continue;
    const int64_t off = win ? sh.pre_off[e - e0] : b.off[e];
    block_copy4<NT, (NT <= 32 ? 2 * kCopyU : kCopyU)>(reinterpret_cast<int4 *>(v.arena + b.c_vb[e]), reinterpret_cast<const int4 *>(b.tok + off),
                            m >> 2, (L + 3) >> 2);
    const int64_t r0 = b.run_off[e] + b.c_firstrun[e], nr = b.run_off[e + 1] - r0, d0 = b.c_run0[e];
    for (int64_t k = threadIdx.x; k < nr; k += NT) {
      const int32_t st = b.run_start[r0 + k];
      v.run_start[d0 + k] = (int32_t)(st > m ? (int64_t)st : m);
      v.run_origin[d0 + k] = b.run_origin[r0 + k];
      v.run_version[d0 + k] = b.run_version[r0 + k];
    }
  }
  group_sync<NT, BAR>();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += NT) record_finish_entry(v, b, e);
}

// K2: the chains.  NCW = 0: NT walk threads; at each chain's end they copy its suffixes
// and switch its rows (record_chain_copy).  NCW = 1: a 32-thread copy warp beside the NT
// walk threads (named barrier 1 keeps it out of theirs) moves each committed entry's
// suffix while the chain goes on; at the chain's end the walk threads wait for its last
// record and switch the rows.  Either way one launch records the whole batch; the last CTA
// out snapshots the counters for the host.
template <int NT, int NCW, int S, int CHV, int MINB>
__global__ void __launch_bounds__(NT + 32 * NCW, MINB) k_record_tma(DevView v, RecordArgs a) {
  static_assert(NCW == 0 || NCW == 1, "one copy warp: the queue has one reader");
  static_assert(NT <= 128, "scan scratch for <= 4 warps");
  constexpr int BAR = NCW ? 1 : 0;
  const Batch &b = a.b;
  __shared__ RecShared sh;
  __shared__ long long s_item;
  __shared__ long long s_scan[10];
  __shared__ TmaRing<NT, S, CHV> rg;
  tma_ring_init(rg);  // every thread: __syncthreads inside
  if (NCW && threadIdx.x == 0) {
    sh.q_head = sh.q_read = sh.q_closed = sh.q_done = 0;
  }
  __syncthreads();
  if (NCW && threadIdx.x >= NT) {
    record_copy_warp(v, b, sh);
  } else {
    // the first wave takes chains by CTA index; later chains come from the work counter
    long long it = blockIdx.x;
    long long next_it = 0;  // thread 0: the next chain, claimed at this chain's start (used at its end)
    for (;;) {
      if (it >= a.nchains) break;
      const bool given = it == 0 && a.c0_e1 >= 0;  // chain 0 in the parameters
      const int64_t e0 = given ? 0 : a.chains[3 * it], e1 = given ? a.c0_e1 : a.chains[3 * it + 1];
      for (int t = threadIdx.x; t < kRecPre && e0 + t < e1; t += NT) {  // the first entries, beside the session
        if (given && t == 0) {
          sh.pre_off[0] = a.c0_off;
          sh.pre_len[0] = a.c0_len;
          sh.pre_q0[0] = a.c0_q0;
          continue;
        }
        const int64_t off = b.off[e0 + t];
        sh.pre_off[t] = off;
        sh.pre_len[t] = (int)b.len[e0 + t];
        sh.pre_q0[t] = b.tok[off];
      }
      if (threadIdx.x == 0) {  // the session, cached for the whole chain
        if (a.nchains > (int64_t)gridDim.x) next_it = (long long)gridDim.x + (long long)atomicAdd(&a.work[0], 1ull);
        else next_it = a.nchains;  // every chain has its own CTA: nothing to claim
        const int32_t sid = given ? a.c0_sid : (int32_t)a.chains[3 * it + 2];
        sh.sid = sid;
        sh.nrows = v.s_nrows[sid];
        sh.stored = v.s_stored[sid];
        sh.naive = v.s_naive[sid];
        sh.pc_row = v.s_pc_row[sid];
        sh.pc_vb = v.s_pc_vb[sid];
        sh.pc_cap = v.s_pc_cap[sid];
        if (sh.pc_row >= 0) {
          sh.pc_rlen = v.row_len[sh.pc_row];
          sh.pc_depth = v.row_depth[sh.pc_row];
        }
        for (int i = 0; i < kRecCache; i++) {
          sh.rc_row[i] = -1;
          sh.fc_row[i] = -1;
        }
        sh.rc_next = sh.fc_next = 0;
      }
      for (int64_t e = e0; e < e1; e++) {
        const int k = (int)((e - e0) % kRecPre);
        if (k == 0 && e != e0) {  // the next kRecPre entries' offsets, lengths and first tokens
          group_sync<NT, BAR>();
          for (int t = threadIdx.x; t < kRecPre && e + t < e1; t += NT) {
            const int64_t off = b.off[e + t];
            sh.pre_off[t] = off;
            sh.pre_len[t] = (int)b.len[e + t];
            sh.pre_q0[t] = b.tok[off];
          }
        }
        group_sync<NT, BAR>();
        if (threadIdx.x == 0) {
          sh.off = sh.pre_off[k];
          sh.len = sh.pre_len[k];
          sh.q0 = sh.pre_q0[k];
        }
        group_sync<NT, BAR>();
        record_walk<NT, BAR>(v, b, sh, rg);
        if (threadIdx.x == 0) {
          record_commit(v, b, e, sh);
          if (e - e0 < kRecPre) {
            sh.win_m[e - e0] = (int)sh.m;
            sh.win_new[e - e0] = sh.dup < 0 ? 1 : 0;
          }
          if (NCW && sh.dup < 0 && sh.len > sh.m) {  // hand the suffix copy to the copy warp
            const int head = sh.q_head;
            while (head - *(volatile int *)&sh.q_read >= kRecQ) __nanosleep(100);
            const int slot = head % kRecQ;
            sh.q_e[slot] = (int)e;
            sh.q_m[slot] = (int)sh.m;
            sh.q_L[slot] = sh.len;
            sh.q_off[slot] = sh.off;
            __threadfence_block();
            *(volatile int *)&sh.q_head = head + 1;
          }
        }
        group_sync<NT, BAR>();
        if (sh.pcw_len > 0) {  // path copy: [from, L) of the entry's query (congruent layout)
          block_copy4<NT, kCopyU>(reinterpret_cast<int4 *>(v.arena + sh.pcw_vb),
                                  reinterpret_cast<const int4 *>(b.tok + sh.off), sh.pcw_from >> 2, (sh.pcw_len + 3) >> 2);
          // generic-proxy arena writes -> visible to the next entry's cp.async.bulk reads
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
      }
      if (threadIdx.x == 0) {  // write the session back
        const int32_t sid = sh.sid;
        v.s_nrows[sid] = sh.nrows;
        v.s_stored[sid] = sh.stored;
        v.s_naive[sid] = sh.naive;
        v.s_pc_row[sid] = sh.pc_row;
        v.s_pc_vb[sid] = sh.pc_vb;
        v.s_pc_cap[sid] = sh.pc_cap;
        if (NCW) {  // the copy warp has finished every record of this chain
          const int target = sh.q_head;
          while (*(volatile int *)&sh.q_done < target) __nanosleep(64);
          __threadfence_block();
        }
      }
      group_sync<NT, BAR>();
      if (NCW) {
        for (int64_t e = e0 + threadIdx.x; e < e1; e += NT) record_finish_entry(v, b, e);
      } else {
        record_chain_copy<NT, BAR>(v, b, e0, e1, s_scan, sh);
      }
      if (threadIdx.x == 0) s_item = next_it;
      group_sync<NT, BAR>();
      it = s_item;
      group_sync<NT, BAR>();
    }
    if (NCW && threadIdx.x == 0) {
      __threadfence_block();
      *(volatile int *)&sh.q_closed = 1;
    }
  }
  if (a.ctr_out) {  // the last CTA out: every counter update of the launch is done
    __syncthreads();
    if (gridDim.x == 1) {  // the only CTA: its own updates are ordered by the barrier
      s_item = 1;
    } else if (threadIdx.x == 0) {
      __threadfence();
      s_item = atomicAdd(&a.work[1], 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_item && threadIdx.x < 4) {
      __threadfence();
      a.ctr_out[threadIdx.x] = *(volatile long long *)&v.ctr[threadIdx.x];
    }
    if (a.out_dst) {  // results (ctr snapshot included) into the caller's pinned buffer
      __syncthreads();
      if (s_item) {
        for (int64_t i = threadIdx.x; i < a.out_len; i += blockDim.x) a.out_dst[i] = ldg_coh(a.out_src + i);
        __threadfence_system();
      }
    }
  }
}

// ----------------------------------------------------------------------------------
// K3 export: one CTA per (row, 4096-position tile).  Walk the parent chain from the
// row; each ancestor owns positions [m_x, upper); copy tokens and expand runs.
constexpr int kExportNT = 256;
constexpr int kExportTile = 4096;

struct ExportPiece {        // one ancestor's share of an output tile
  int64_t vb;                // owner's arena virtual base
  int64_t run0;              // owner's first metadata run ...
  int32_t pa, pb;            // positions [pa, pb) of the output row
  int32_t nrun, first_run;   // ... its run count, and the run containing pa
  int32_t len;               // owner's length (end of its last run)
  int32_t pad;
};
constexpr int kMaxPieces = 16;  // per tile; deeper chains fall back to an in-kernel walk

struct TileHdr {            // planner output per tile: everything the copy CTA needs up front
  int64_t o;                 // output word of the tile's row start
  int32_t a, b;              // tile positions [a, b) of that row
  int32_t row;               // output row index (resp-start atomics, fallback walk)
  int32_t np;                // pieces, or -1: chain deeper than kMaxPieces, walk in-kernel
  int64_t pad;
};
struct TilePlan {            // 672 bytes: fetched into shared memory with 42 16-byte cp.async
  TileHdr h;
  ExportPiece p[kMaxPieces];
};
static_assert(sizeof(TilePlan) % 16 == 0, "TilePlan is copied in 16-byte chunks");

struct ExportArgs {
  int64_t n;
  const int64_t *rows;
  const int64_t *out_off;   // n+1
  const int64_t *tile_off;  // n+1
  int64_t ntiles;
  int32_t *tokens;
  uint8_t *mask;
  int32_t *versions;
  unsigned long long *resp;  // n (atomicMax), may be null
  TilePlan *plan;            // ntiles (planner output); pieces by descending position
};

// Copy / fill helpers for one piece [pa, pb) of an output row starting at word o.  When
// o is a multiple of 4 every output position is 16-byte congruent with its arena
// position (arena rows are 128-byte aligned), so the body moves int4 / uchar4 vectors.
template <int NT = kExportNT>
__device__ __forceinline__ void copy_tokens(int32_t *__restrict__ out, const int32_t *__restrict__ src, int64_t o,
                                            int64_t pa, int64_t pb) {
  if ((o & 3) == 0) {
    const int64_t va = (pa + 3) >> 2, vb = pb >> 2;  // int4 body [4va, 4vb)
    if (va < vb) {
      for (int64_t p = pa + threadIdx.x; p < 4 * va; p += NT) out[o + p] = src[p];
      for (int64_t p = 4 * vb + threadIdx.x; p < pb; p += NT) out[o + p] = src[p];
      const int4 *s4 = reinterpret_cast<const int4 *>(src);
      int4 *d4 = reinterpret_cast<int4 *>(out + o);
      for (int64_t q = va + threadIdx.x; q < vb; q += NT) d4[q] = ldg_stream(s4 + q);
      return;
    }
  }
  for (int64_t p = pa + threadIdx.x; p < pb; p += NT) out[o + p] = src[p];
}

template <int NT = kExportNT>
__device__ __forceinline__ void fill_meta(uint8_t *__restrict__ mask, int32_t *__restrict__ vers, int64_t o,
                                          int64_t xa, int64_t xb, uint8_t org, int32_t ver) {
  if ((o & 3) == 0) {
    const int64_t va = (xa + 3) >> 2, vb = xb >> 2;
    if (va < vb) {
      for (int64_t p = xa + threadIdx.x; p < 4 * va; p += NT) { mask[o + p] = org; vers[o + p] = ver; }
      for (int64_t p = 4 * vb + threadIdx.x; p < xb; p += NT) { mask[o + p] = org; vers[o + p] = ver; }
      const uint32_t m4 = 0x01010101u * org;
      const int4 v4 = make_int4(ver, ver, ver, ver);
      uint32_t *dm = reinterpret_cast<uint32_t *>(mask + o);
      int4 *dv = reinterpret_cast<int4 *>(vers + o);
      for (int64_t q = va + threadIdx.x; q < vb; q += NT) {
        dm[q] = m4;
        dv[q] = v4;
      }
      return;
    }
  }
  for (int64_t p = xa + threadIdx.x; p < xb; p += NT) { mask[o + p] = org; vers[o + p] = ver; }
}

__device__ __forceinline__ int first_run_of(const DevView &v, int64_t run0, int nrun, int64_t pa) {
  int lo = 0, hi = nrun;  // last run with start <= pa
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (v.run_start[run0 + mid] <= pa) lo = mid; else hi = mid;
  }
  return lo;
}

// Export planner: resolves the dependent lookups of every tile (parent chain, first run
// of each piece) in parallel, so the copy kernel's CTAs start streaming immediately
// instead of chasing pointers per tile.  One warp per output row, one lane per tile of
// the row: the tile -> row mapping needs no search.
__device__ __forceinline__ void plan_tile(const DevView &v, const ExportArgs &e, int64_t t, int64_t i, int64_t row,
                                          int64_t len, int64_t o, int64_t a) {
  const int64_t b = min((int64_t)(a + kExportTile), len);
  int64_t cur = row, upper = len;
  // climb to the owner of position b-1 with jump pointers (O(log depth)); its range
  // ends at or after b, so the tile's first piece ends at b
  while (v.row_m[cur] > b - 1) {
    const int64_t jp = v.row_jump[cur];
    cur = (jp >= 0 && v.row_m[jp] > b - 1) ? jp : v.row_parent[cur];
    upper = b;
  }
  int np = 0;
  ExportPiece *out = e.plan[t].p;
  while (cur >= 0 && upper > a) {
    const int64_t mx = v.row_m[cur];
    const int64_t pa = max(mx, a), pb = min(upper, b);
    if (pa < pb) {
      TM_DCHECK(v, cur < v.row_cap && v.row_vb[cur] + pb <= v.arena_cap, kErrArena);
      if (np == kMaxPieces) { np = -1; break; }
      ExportPiece p;
      p.vb = v.row_vb[cur];
      p.run0 = v.row_run0[cur];
      p.pa = (int32_t)pa;
      p.pb = (int32_t)pb;
      p.nrun = v.row_nrun[cur];
      p.len = v.row_len[cur];
      p.first_run = first_run_of(v, p.run0, p.nrun, pa);
      p.pad = 0;
      out[np++] = p;
    }
    upper = mx;
    cur = v.row_parent[cur];
  }
  TileHdr h;
  h.o = o;
  h.a = (int32_t)a;
  h.b = (int32_t)b;
  h.row = (int32_t)i;
  h.np = np;
  h.pad = 0;
  e.plan[t].h = h;
}

__global__ void k_export_plan(DevView v, ExportArgs e) {
  asm volatile("griddepcontrol.launch_dependents;");  // k_export_tma may start its prologue
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < e.n; i += nwarps) {
    const int64_t t0 = e.tile_off[i], t1 = e.tile_off[i + 1];
    const int64_t row = e.rows[i];
    const int64_t len = v.row_len[row], o = e.out_off[i];
    if (lane == 0 && e.resp) e.resp[i] = 0;  // the export kernel atomicMax-es into it (stream order)
    for (int64_t t = t0 + lane; t < t1; t += 32) plan_tile(v, e, t, i, row, len, o, (t - t0) * kExportTile);
  }
}

template <int NT = kExportNT>
__device__ __forceinline__ void export_runs(const DevView &v, const ExportArgs &e, const ExportPiece &p, int64_t o,
                                            long long &respmax) {
  for (int k = p.first_run; k < p.nrun; k++) {
    const int64_t rs = v.run_start[p.run0 + k];
    if (rs >= p.pb) break;
    const int64_t re = (k + 1 < p.nrun) ? v.run_start[p.run0 + k + 1] : p.len;
    const int64_t xa = max(rs, (int64_t)p.pa), xb = min(re, (int64_t)p.pb);
    const uint8_t org = v.run_origin[p.run0 + k];
    fill_meta<NT>(e.mask, e.versions, o, xa, xb, org, v.run_version[p.run0 + k]);
    if (org == 0 && xb > respmax) respmax = xb;
  }
}

// pieces are ordered by descending position and partition the tile [a, b)
__device__ __forceinline__ int piece_at(const ExportPiece *sp, int np, int32_t p) {
  int k = 0;
  while (k + 1 < np && sp[k].pa > p) k++;
  return k;
}

// Tiles the vector paths do not take: an output row that starts off a 16-byte boundary
// (scalar copies), or a chain deeper than kMaxPieces inside the tile (walked here).
template <int NT>
__device__ __forceinline__ void export_tile_generic(const DevView &v, const ExportArgs &e, const TileHdr &h, const ExportPiece *P,
                                    long long &respmax) {
  const int64_t o = h.o;
  if (h.np > 0) {  // unaligned row start
    for (int k = 0; k < h.np; k++) {
      copy_tokens<NT>(e.tokens, v.arena + P[k].vb, o, P[k].pa, P[k].pb);
      export_runs<NT>(v, e, P[k], o, respmax);
    }
  } else if (h.np < 0) {  // chain deeper than kMaxPieces inside this tile: walk it here
    const int64_t row = e.rows[h.row];
    const int64_t a = h.a, b = h.b;
    int64_t cur = row, upper = v.row_len[row];
    while (v.row_m[cur] > b - 1) {  // skip the rows above the tile (jump pointers, as the planner)
      const int64_t jp = v.row_jump[cur];
      cur = (jp >= 0 && v.row_m[jp] > b - 1) ? jp : v.row_parent[cur];
      upper = b;
    }
    while (cur >= 0 && upper > a) {
      const int64_t mx = v.row_m[cur];
      const int64_t pa = max(mx, a), pb = min(upper, b);
      if (pa < pb) {
        ExportPiece p;
        p.vb = v.row_vb[cur];
        p.run0 = v.row_run0[cur];
        p.pa = (int32_t)pa;
        p.pb = (int32_t)pb;
        p.nrun = v.row_nrun[cur];
        p.len = v.row_len[cur];
        p.first_run = first_run_of(v, p.run0, p.nrun, pa);
        copy_tokens<NT>(e.tokens, v.arena + p.vb, o, p.pa, p.pb);
        export_runs<NT>(v, e, p, o, respmax);
      }
      upper = mx;
      cur = v.row_parent[cur];
    }
  }
}

constexpr int kExportSlots = kExportTile / 4 / kExportNT;  // int4 output slots per thread per tile
constexpr int kExportCtas = 4;                             // resident CTAs per SM (64 registers)

// K3 copy: persistent CTAs over planner tiles.  Tile-centric: the mask / version fills
// (stores only) go first, then each thread issues the loads of all kExportSlots int4
// slots it owns before storing them - 4 loads in flight per thread however the tile
// splits into ancestor pieces.  The next tile's plan is fetched into the other half of
// a double-buffered shared-memory table with cp.async while this tile is processed;
// one barrier per tile.
__device__ __forceinline__ void fetch_plan(TilePlan *dst, const TilePlan *src) {
  constexpr int kChunks = (int)(sizeof(TilePlan) / 16);
  if (threadIdx.x < kChunks) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(reinterpret_cast<char *>(dst) + 16 * threadIdx.x);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(reinterpret_cast<const char *>(src) + 16 * threadIdx.x)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(kExportNT, kExportCtas) k_export(DevView v, ExportArgs e) {
  __shared__ TilePlan sp[2];
  int64_t t = blockIdx.x;
  if (t >= e.ntiles) return;
  fetch_plan(&sp[0], &e.plan[t]);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  for (int it = 0; t < e.ntiles; t += gridDim.x, it ^= 1) {
    const TileHdr h = sp[it].h;
    const ExportPiece *P = sp[it].p;
    if (t + gridDim.x < e.ntiles) fetch_plan(&sp[it ^ 1], &e.plan[t + gridDim.x]);  // overlaps this tile
    const int64_t o = h.o;
    long long respmax = 0;
    if (h.np > 0 && (o & 3) == 0) {
      for (int k = 0; k < h.np; k++) export_runs(v, e, P[k], o, respmax);  // stores only
      int4 x[kExportSlots];
      uint32_t full = 0;  // slots inside one piece; the others straddle a piece boundary or the row end
#pragma unroll
      for (int j = 0; j < kExportSlots; j++) {
        const int32_t p = h.a + 4 * ((int)threadIdx.x + j * kExportNT);
        const ExportPiece &q = P[piece_at(P, h.np, p)];
        const bool ok = p + 4 <= q.pb;  // (q.pb <= h.b)
        full |= (uint32_t)ok << j;
        x[j] = ldg_stream_if(reinterpret_cast<const int4 *>(v.arena + q.vb + p), ok);
      }
      int4 *d4 = reinterpret_cast<int4 *>(e.tokens + o) + (h.a >> 2) + threadIdx.x;
#pragma unroll
      for (int j = 0; j < kExportSlots; j++) stg_if(d4 + j * kExportNT, x[j], (full >> j) & 1);
#pragma unroll 1
      for (int j = 0; j < kExportSlots; j++) {
        const int32_t p = h.a + 4 * ((int)threadIdx.x + j * kExportNT);
        if (!(full & (1u << j)) && p < h.b)
          for (int u = 0; u < 4 && p + u < h.b; u++)
            e.tokens[o + p + u] = v.arena[P[piece_at(P, h.np, p + u)].vb + p + u];
      }
    } else {
      export_tile_generic<kExportNT>(v, e, h, P, respmax);
    }
    if (e.resp && threadIdx.x == 0 && respmax > 0) atomicMax(&e.resp[h.row], (unsigned long long)respmax);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // next plan visible; this tile's plan no longer read
  }
}

// K3, TMA variant: token bodies never pass through registers.  Per tile one elected thread
// issues cp.async.bulk loads of every piece's 16-byte-aligned body from the arena into a
// 16 KB shared-memory tile (an mbarrier counts the bytes), the other threads put the <= 6
// edge words per piece into the tile and write the mask / version runs, then the tile
// leaves with ONE cp.async.bulk store (global <- shared).  Two tile buffers: a tile's
// store drains while the next tile loads.  Aligned rows only; the rest take
// export_tile_generic.
constexpr int kExportTmaNT = 128;
struct ExportTmaSmem {
  int4 buf[2][kExportTile / 4];
  TilePlan plan[2];
  uint64_t bar[2];
};

__global__ void __launch_bounds__(kExportTmaNT) k_export_tma(DevView v, ExportArgs e) {
  extern __shared__ __align__(128) char dyn[];
  ExportTmaSmem &sm = *reinterpret_cast<ExportTmaSmem *>(dyn);
  int64_t t = blockIdx.x;
  if (t >= e.ntiles) return;
  if (threadIdx.x == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // launched as a programmatic dependent of k_export_plan: the prologue above overlaps the
  // planner; everything it writes (plans, zeroed response starts) is read after this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  fetch_plan(&sm.plan[0], &e.plan[t]);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of stage s's barrier
  for (int it = 0; t < e.ntiles; t += gridDim.x, it ^= 1) {
    const TileHdr h = sm.plan[it].h;
    const ExportPiece *P = sm.plan[it].p;
    if (t + gridDim.x < e.ntiles) fetch_plan(&sm.plan[it ^ 1], &e.plan[t + gridDim.x]);
    const int64_t o = h.o;
    long long respmax = 0;
    if (h.np > 0 && (o & 3) == 0) {
      int32_t *B = reinterpret_cast<int32_t *>(sm.buf[it]);
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // store of tile t-2 read B
      __syncthreads();
      uint32_t bytes = 0;
      for (int k = 0; k < h.np; k++) {
        const int32_t ca = (P[k].pa + 3) & ~3, cb = P[k].pb & ~3;
        if (ca < cb) bytes += 4u * (uint32_t)(cb - ca);
      }
      if (threadIdx.x == 0 && bytes) {
        mbar_expect_tx(&sm.bar[it], bytes);
        for (int k = 0; k < h.np; k++) {
          const int32_t ca = (P[k].pa + 3) & ~3, cb = P[k].pb & ~3;
          if (ca < cb) bulk_g2s(B + (ca - h.a), v.arena + P[k].vb + ca, 4u * (uint32_t)(cb - ca), &sm.bar[it]);
        }
      }
      // edge words: thread 8k+w takes word w of piece k's head [pa, ca) / tail [cb, pb)
      if ((int)threadIdx.x < 8 * h.np) {
        const ExportPiece &q = P[threadIdx.x >> 3];
        const int w = threadIdx.x & 7;
        const int32_t ca = (q.pa + 3) & ~3, cb = q.pb & ~3;
        int32_t pos = -1;
        if (ca < cb) pos = w < 3 ? (q.pa + w < ca ? q.pa + w : -1) : (w < 6 && cb + (w - 3) < q.pb ? cb + (w - 3) : -1);
        else if (w < 7 && q.pa + w < q.pb) pos = q.pa + w;
        if (pos >= 0) B[pos - h.a] = v.arena[q.vb + pos];
      }
      for (int k = 0; k < h.np; k++) export_runs<kExportTmaNT>(v, e, P[k], o, respmax);  // stores only
      if (bytes) mbar_wait(&sm.bar[it], (phase >> it) & 1);
      if (bytes) phase ^= 1u << it;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // edge words -> visible to the bulk store
      __syncthreads();
      const int32_t body = (h.b & ~3) - h.a;  // whole int4s of the tile
      if (threadIdx.x == 0 && body > 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(e.tokens + o + h.a),
                     "r"(smem_u32(B)), "r"(4u * (uint32_t)body)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if ((int)threadIdx.x < h.b - (h.b & ~3)) e.tokens[o + (h.b & ~3) + threadIdx.x] = B[body + threadIdx.x];
    } else {
      export_tile_generic<kExportTmaNT>(v, e, h, P, respmax);
    }
    if (e.resp && threadIdx.x == 0 && respmax > 0) atomicMax(&e.resp[h.row], (unsigned long long)respmax);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // next plan visible; this tile's plan no longer read
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores done before smem goes away
}

// ----------------------------------------------------------------------------------
// NDJSON formatter (core.py:182-183 trajectory_to_line, byte-identical):
//   {"session_id":<json literal>,"tokens":[t,...],"loss_mask":[0|1,...],"versions":[v,...]}\n
// from packed rows.  Pass 1 (k_json_sums) sums the decimal widths of tokens and versions
// per 4096-position tile; the host turns them into byte offsets; pass 2 (k_json_write)
// prints every number at its offset (block scan of widths inside the tile).
constexpr int kJsonNT = 256;
constexpr int kJsonPer = 16;  // positions per thread: tile = 4096 = export tile
static_assert(kJsonNT * kJsonPer == kExportTile, "json tile == export tile");

__device__ __forceinline__ int dec_width(int32_t v) {
  uint32_t u = v < 0 ? (uint32_t)(-(int64_t)v) : (uint32_t)v;
  int d = 1;
  while (u >= 10) { u /= 10; d++; }
  return d + (v < 0);
}

__device__ __forceinline__ void dec_write(char *dst, int32_t v, int w) {
  uint32_t u = v < 0 ? (uint32_t)(-(int64_t)v) : (uint32_t)v;
  for (int i = w - 1; i >= (v < 0 ? 1 : 0); i--) { dst[i] = (char)('0' + u % 10); u /= 10; }
  if (v < 0) dst[0] = '-';
}

struct JsonArgs {
  int64_t n;                 // rows
  const int64_t *out_off;    // packed row offsets (n+1)
  const int64_t *tile_off;   // tiles per row prefix (n+1)
  int64_t ntiles;
  const int32_t *tokens;
  const uint8_t *mask;
  const int32_t *versions;
  long long *sums;           // pass 1: 2 per tile (token widths, version widths)
  const long long *toff;     // pass 2: 3 per tile (tokens, mask, versions byte offsets)
  const long long *roff;     // pass 2: 4 per row (row start, tokens start, mask start, versions start)
  const char *sid;           // session-id JSON literals, concatenated
  const int64_t *sid_off;    // n+1
  char *out;
};

__device__ __forceinline__ int64_t json_row_of(const JsonArgs &j, int64_t t) {
  int64_t lo = 0, hi = j.n;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (j.tile_off[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kJsonNT) k_json_sums(JsonArgs j) {
  __shared__ long long sm[2][kJsonNT / 32];
  for (int64_t t = blockIdx.x; t < j.ntiles; t += gridDim.x) {
    const int64_t i = json_row_of(j, t);
    const int64_t L = j.out_off[i + 1] - j.out_off[i];
    const int64_t a = (t - j.tile_off[i]) * kExportTile, b = min(a + (int64_t)kExportTile, L);
    const int64_t base = j.out_off[i];
    long long st = 0, sv = 0;
    for (int64_t p = a + threadIdx.x; p < b; p += kJsonNT) {
      st += dec_width(j.tokens[base + p]);
      sv += dec_width(j.versions[base + p]);
    }
    for (int d = 16; d > 0; d >>= 1) {
      st += __shfl_xor_sync(0xffffffffu, st, d);
      sv += __shfl_xor_sync(0xffffffffu, sv, d);
    }
    if ((threadIdx.x & 31) == 0) { sm[0][threadIdx.x >> 5] = st; sm[1][threadIdx.x >> 5] = sv; }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long a0 = 0, a1 = 0;
      for (int w = 0; w < kJsonNT / 32; w++) { a0 += sm[0][w]; a1 += sm[1][w]; }
      j.sums[2 * t] = a0;
      j.sums[2 * t + 1] = a1;
    }
    __syncthreads();
  }
}

// exclusive block scan of one value per thread
__device__ __forceinline__ long long block_excl_scan(long long x, long long *sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long y = x;
  for (int d = 1; d < 32; d <<= 1) {
    long long z = __shfl_up_sync(0xffffffffu, y, d);
    if (lane >= d) y += z;
  }
  if (lane == 31) sm[w] = y;
  __syncthreads();
  long long pre = 0;
  for (int k = 0; k < w; k++) pre += sm[k];
  __syncthreads();
  return pre + y - x;
}

__device__ __forceinline__ void put(char *dst, const char *s, int n) {
  for (int k = 0; k < n; k++) dst[k] = s[k];
}

// Copy `n` staged bytes from shared memory to out[base ...) with 4-byte aligned global
// stores (byte stores only for the unaligned head and tail): a warp writes 128
// contiguous bytes per instruction.
__device__ __forceinline__ void stage_out(char *__restrict__ out, long long base, const char *buf, int n) {
  const int head = (int)min((long long)n, (4 - (base & 3)) & 3);
  if ((int)threadIdx.x < head) out[base + threadIdx.x] = buf[threadIdx.x];
  const int nw = (n - head) >> 2;
  uint32_t *dst = reinterpret_cast<uint32_t *>(out + base + head);
  for (int w = threadIdx.x; w < nw; w += kJsonNT) {
    const char *s = buf + head + 4 * w;
    dst[w] = (uint32_t)(uint8_t)s[0] | ((uint32_t)(uint8_t)s[1] << 8) | ((uint32_t)(uint8_t)s[2] << 16) |
             ((uint32_t)(uint8_t)s[3] << 24);
  }
  const int t0 = head + 4 * nw;
  if ((int)threadIdx.x < n - t0) out[base + t0 + threadIdx.x] = buf[t0 + threadIdx.x];
}

__global__ void __launch_bounds__(kJsonNT) k_json_write(JsonArgs j) {
  constexpr int kHalf = kExportTile / 2;   // a tile is printed in two halves ...
  constexpr int kPer = kHalf / kJsonNT;    // ... of 8 positions per thread
  __shared__ long long sm[kJsonNT / 32];
  __shared__ int s_total;
  __shared__ char buf[kHalf * 12];         // widest half-section: 2048 x ("-2147483648,")
  for (int64_t t = blockIdx.x; t < j.ntiles; t += gridDim.x) {
    const int64_t i = json_row_of(j, t);
    const int64_t L = j.out_off[i + 1] - j.out_off[i];
    const int64_t a = (t - j.tile_off[i]) * kExportTile, b = min(a + (int64_t)kExportTile, L);
    const int64_t base = j.out_off[i];
    for (int sec = 0; sec < 2; sec++) {  // 0 tokens, 1 versions
      const int32_t *vals = sec ? j.versions : j.tokens;
      long long dst = j.toff[3 * t + (sec ? 2 : 0)];
      for (int64_t h0 = a; h0 < b; h0 += kHalf) {
        const int64_t pa = h0 + (int64_t)threadIdx.x * kPer, pb = min(pa + kPer, min(h0 + kHalf, b));
        long long mine = 0;
        for (int64_t p = pa; p < pb; p++) mine += dec_width(vals[base + p]) + (p + 1 < L ? 1 : 0);
        const long long excl = block_excl_scan(mine, sm);
        if ((int)threadIdx.x == kJsonNT - 1) s_total = (int)(excl + mine);
        int off = (int)excl;
        for (int64_t p = pa; p < pb; p++) {
          const int32_t v = vals[base + p];
          const int w = dec_width(v);
          dec_write(buf + off, v, w);
          if (p + 1 < L) buf[off + w] = ',';
          off += w + 1;
        }
        __syncthreads();
        const int n = s_total;
        stage_out(j.out, dst, buf, n);
        dst += n;
        __syncthreads();
      }
    }
    // loss mask: "d," per position (no comma after the row's last)
    for (int64_t h0 = a; h0 < b; h0 += kHalf) {
      const int64_t h1 = min(h0 + kHalf, b);
      for (int64_t p = h0 + threadIdx.x; p < h1; p += kJsonNT) {
        buf[2 * (p - h0)] = j.mask[base + p] ? '1' : '0';
        if (p + 1 < L) buf[2 * (p - h0) + 1] = ',';
      }
      __syncthreads();
      stage_out(j.out, j.toff[3 * t + 1] + 2 * (h0 - a), buf, (int)(2 * (h1 - h0) - (h1 == L ? 1 : 0)));
      __syncthreads();
    }
    if (t == j.tile_off[i] && threadIdx.x == 0) {  // fixed parts of the row
      const long long r0 = j.roff[4 * i], ts = j.roff[4 * i + 1], ms = j.roff[4 * i + 2], vs = j.roff[4 * i + 3];
      const int64_t s0 = j.sid_off[i], sl = j.sid_off[i + 1] - s0;
      put(j.out + r0, "{\"session_id\":", 14);
      put(j.out + r0 + 14, j.sid + s0, (int)sl);
      put(j.out + ts - 11, ",\"tokens\":[", 11);
      put(j.out + ms - 15, "],\"loss_mask\":[", 15);
      put(j.out + vs - 14, "],\"versions\":[", 14);
      put(j.out + j.roff[4 * (i + 1)] - 3, "]}\n", 3);
    }
  }
}

cudaError_t launch_json(const JsonArgsHost &h, int pass, int num_sms, cudaStream_t s) {
  JsonArgs j{h.n, h.out_off, h.tile_off, h.ntiles, h.tokens, h.mask, h.versions, (long long *)h.sums,
             (const long long *)h.toff, (const long long *)h.roff, h.sid, h.sid_off, h.out};
  int64_t grid = h.ntiles < (int64_t)num_sms * 8 ? h.ntiles : (int64_t)num_sms * 8;
  if (grid < 1) return cudaSuccess;
  if (pass == 1) k_json_sums<<<(int)grid, kJsonNT, 0, s>>>(j);
  else k_json_write<<<(int)grid, kJsonNT, 0, s>>>(j);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------
__global__ void k_rehash(DevView v, const uint64_t *ok0, const uint64_t *ok1, const int64_t *oval, int64_t ocap) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ocap; s += (int64_t)gridDim.x * blockDim.x) {
    if (ok0[s] != kEmpty) ht_insert(v, ok0[s], ok1[s], oval[s]);
  }
}

// Rebuild the branch index from the row table (snapshot restore): every row's key is
// (parent or ROOT|session, matched, its first own token), or the terminal key for rows
// that end where they branch off (prefix rows).  Row slots reserved by an entry that
// re-recorded an existing sequence are holes (row_len 0, written by k_record).
__global__ void k_rebuild_index(DevView v, int64_t nrows) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t L = v.row_len[r];
    if (L <= 0) continue;
    const int64_t m = v.row_m[r], par = v.row_parent[r];
    const int32_t sid = v.row_sess[r];
    const uint64_t owner = m > 0 ? (uint64_t)par : (kRootTag | (uint64_t)(uint32_t)sid);
    if (L > m) ht_insert(v, owner, dt_key(m, v.arena[v.row_vb[r] + m], false), r);
    else ht_insert(v, owner, dt_key(m, 0, true), r);
  }
}

__global__ void k_fill_u64(uint64_t *p, int64_t n, uint64_t val) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) p[s] = val;
}

// ----------------------------------------------------------------------------------
// launchers
constexpr int kWalkNT = 64;
constexpr int kWalkU = 8;

int64_t plan_items_ints(int64_t n) { return (int64_t)kPlanNB * n; }

cudaError_t launch_plan(const DevView &v, Batch &b, int64_t *root, int *items, cudaStream_t s) {
  b.bucket_items = items;
  b.root = root;
  const int grid = (int)((b.n + kPlanNT - 1) / kPlanNT);
  k_plan<<<grid, kPlanNT, 0, s>>>(v, b, root, b.sched->count, items);
  return cudaGetLastError();
}

template <int NT, int U>
static cudaError_t walk_variant(const DevView &v, const Batch &b, int num_sms, cudaStream_t s) {
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_walk<NT, U>, NT, 0);
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)num_sms * occ;
  if (grid > b.n) grid = b.n;
  if (grid < 1) grid = 1;
  k_walk<NT, U><<<(int)grid, NT, 0, s>>>(v, b);
  return cudaGetLastError();
}

// Default K1: the TMA-staged compare, 4 stages x 4 KB per stream (c4: 31.9 M q/s vs 30.7
// for the register-double-buffered "64x8").  The other shapes measured in round 1 are only
// compiled into tuning builds (make TUNING=1 -> -DTM_TUNING; TM_WALK_VARIANT selects).
cudaError_t launch_walk(const DevView &v, const Batch &b, int num_sms, cudaStream_t s) {
#ifdef TM_TUNING
  static int variant = -1;
  if (variant < 0) {
    static const char *names[] = {"tma", "256x2", "512x2", "128x4", "512x1", "128x2", "128x8", "64x8", "256x4",
                                  "64x4", "tma3", "tma8x128", "tma6x128", "tma2x512"};
    const char *e = getenv("TM_WALK_VARIANT");
    variant = 0;
    for (int i = 0; e && i < (int)(sizeof(names) / sizeof(names[0])); i++)
      if (!strcmp(e, names[i])) variant = i;
  }
  switch (variant) {
    case 1: return walk_variant<256, 2>(v, b, num_sms, s);
    case 2: return walk_variant<512, 2>(v, b, num_sms, s);
    case 3: return walk_variant<128, 4>(v, b, num_sms, s);
    case 4: return walk_variant<512, 1>(v, b, num_sms, s);
    case 5: return walk_variant<128, 2>(v, b, num_sms, s);
    case 6: return walk_variant<128, 8>(v, b, num_sms, s);
    case 7: return walk_variant<kWalkNT, kWalkU>(v, b, num_sms, s);
    case 8: return walk_variant<256, 4>(v, b, num_sms, s);
    case 9: return walk_variant<64, 4>(v, b, num_sms, s);
    case 10: return walk_tma_variant<3, 256>(v, b, num_sms, s);
    case 11: return walk_tma_variant<8, 128>(v, b, num_sms, s);
    case 12: return walk_tma_variant<6, 128>(v, b, num_sms, s);
    case 13: return walk_tma_variant<2, 512>(v, b, num_sms, s);
    default: break;
  }
#endif
  return walk_tma_variant<kTmaStages, kTmaChunk>(v, b, num_sms, s);
}

template <int S, int CHV, int MINB, int NT = 64, int NCW = 0>
static cudaError_t record_tma_variant(const DevView &v, const RecordArgs &a, int num_sms, cudaStream_t s,
                                      int *copy_warp) {
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_record_tma<NT, NCW, S, CHV, MINB>, NT + 32 * NCW, 0);
    if (occ < 1) occ = 1;
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * occ, a.nchains));
  k_record_tma<NT, NCW, S, CHV, MINB><<<(int)grid, NT + 32 * NCW, 0, s>>>(v, a);
  *copy_warp = NCW;
  return cudaGetLastError();
}

// K2 = k_record_tma, one launch per batch.  A chain's compare is TMA-staged (the stages
// live in shared memory, not registers).
//   <= 8 chains per SM (c2, 1,000 chains): 64 walk threads + 1 copy warp, 3 x 4 KB stages
//     per stream, every chain resident; the copies ride under the chains' latency-bound
//     walks
//   more chains (c3, 4,000 chains of 2 entries): one-warp CTAs, 32 per SM, 2 x 1 KB stages,
//     so up to 4,736 chains are resident at once (registers leave no room for copy warps);
//     each chain copies its own suffixes at its end, overlapping the walks of the others
// Tuning builds (-DTM_TUNING) select other shapes with TM_RECORD_VARIANT.
cudaError_t launch_record(const DevView &v, const RecordArgs &a, int num_sms, cudaStream_t s, int *copy_warp) {
  *copy_warp = 0;
#ifdef TM_TUNING
  static int variant = -1;
  if (variant < 0) {
    static const char *names[] = {"default", "tma3x256", "tma2x128", "tma4x256", "tma2x256", "tma4x128", "tma3x128",
                                  "t128x3x256", "t128x2x128", "t128x2x256", "t32x2x64", "t32x3x64", "t32x2x128",
                                  "ws64x3x256", "ws64x2x256", "ws32x2x64", "ws32x2x128", "ws64x2x128"};
    const char *e = getenv("TM_RECORD_VARIANT");
    variant = 0;
    for (int i = 0; e && i < (int)(sizeof(names) / sizeof(names[0])); i++)
      if (!strcmp(e, names[i])) variant = i;
  }
  switch (variant) {
    case 1: return record_tma_variant<3, 256, 8>(v, a, num_sms, s, copy_warp);
    case 2: return record_tma_variant<2, 128, 16>(v, a, num_sms, s, copy_warp);
    case 3: return record_tma_variant<4, 256, 6>(v, a, num_sms, s, copy_warp);
    case 4: return record_tma_variant<2, 256, 12>(v, a, num_sms, s, copy_warp);
    case 5: return record_tma_variant<4, 128, 12>(v, a, num_sms, s, copy_warp);
    case 6: return record_tma_variant<3, 128, 14>(v, a, num_sms, s, copy_warp);
    case 7: return record_tma_variant<3, 256, 8, 128>(v, a, num_sms, s, copy_warp);
    case 8: return record_tma_variant<2, 128, 12, 128>(v, a, num_sms, s, copy_warp);
    case 9: return record_tma_variant<2, 256, 8, 128>(v, a, num_sms, s, copy_warp);
    case 10: return record_tma_variant<2, 64, 32, 32>(v, a, num_sms, s, copy_warp);
    case 11: return record_tma_variant<3, 64, 28, 32>(v, a, num_sms, s, copy_warp);
    case 12: return record_tma_variant<2, 128, 24, 32>(v, a, num_sms, s, copy_warp);
    case 13: return record_tma_variant<3, 256, 8, 64, 1>(v, a, num_sms, s, copy_warp);
    case 14: return record_tma_variant<2, 256, 8, 64, 1>(v, a, num_sms, s, copy_warp);
    case 15: return record_tma_variant<2, 64, 16, 32, 1>(v, a, num_sms, s, copy_warp);
    case 16: return record_tma_variant<2, 128, 16, 32, 1>(v, a, num_sms, s, copy_warp);
    case 17: return record_tma_variant<2, 128, 12, 64, 1>(v, a, num_sms, s, copy_warp);
    default: break;
  }
#endif
  if (a.nchains <= (int64_t)num_sms * 8) return record_tma_variant<3, 256, 8, 64, 1>(v, a, num_sms, s, copy_warp);
  return record_tma_variant<2, 64, 32, 32>(v, a, num_sms, s, copy_warp);
}

cudaError_t launch_export(const DevView &v, const ExportArgsHost &h, int num_sms, cudaStream_t s) {
  if (h.ntiles < 1) return cudaSuccess;
  ExportArgs e{h.n, h.rows, h.out_off, h.tile_off, h.ntiles, h.tokens, h.mask, h.versions,
               (unsigned long long *)h.resp, reinterpret_cast<TilePlan *>(h.plan)};
  const int pgrid = (int)std::min<int64_t>((h.n * 32 + 255) / 256, (int64_t)num_sms * 8);  // a warp per row
  k_export_plan<<<pgrid, 256, 0, s>>>(v, e);
  // TM_EXPORT_VARIANT (tuning): "tma" (default: c2 0.271 ms = 6.3 TB/s, c3 0.073 ms) or
  // "regs" (register path: 0.295-0.310 / 0.089-0.093 ms)
  static int variant = -1;
  static int tma_ctas = 0;
  if (variant < 0) {
    const char *ev = getenv("TM_EXPORT_VARIANT");
    variant = (ev && !strcmp(ev, "regs")) ? 0 : 1;
    if (variant == 1) {
      cudaFuncSetAttribute(k_export_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ExportTmaSmem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tma_ctas, k_export_tma, kExportTmaNT, sizeof(ExportTmaSmem));
      if (tma_ctas < 1) tma_ctas = 1;
    }
  }
  if (variant == 1) {
    const int64_t grid = std::min<int64_t>(h.ntiles, (int64_t)num_sms * tma_ctas);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kExportTmaNT);
    cfg.dynamicSmemBytes = sizeof(ExportTmaSmem);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlaps the planner's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_export_tma, v, e);
  }
  const int64_t grid = std::min<int64_t>(h.ntiles, (int64_t)num_sms * kExportCtas);
  k_export<<<(int)grid, kExportNT, 0, s>>>(v, e);
  return cudaGetLastError();
}

// Rows that live on the host - open / paused requests (trajectory.py:329-340): the input
// span at the request's context version, then MODEL_OUTPUT runs by version.  One CTA per
// row (grid-stride): tokens move from the staged copy into the packed outputs, mask and
// versions are written from the row's few runs.
__global__ void __launch_bounds__(256) k_fill_host_rows(HostRowsArgs a) {
  for (int64_t k = blockIdx.x; k < a.n; k += gridDim.x) {
    const int64_t t0 = a.tok_off[k], L = a.tok_off[k + 1] - t0, o = a.out_off[k], ni = a.n_input[k];
    const int32_t cv = a.ctx_version[k];
    const int64_t r0 = a.run_off[k], r1 = a.run_off[k + 1];
    for (int64_t p = threadIdx.x; p < L; p += blockDim.x) {
      a.tokens[o + p] = a.src[t0 + p];
      a.mask[o + p] = p >= ni ? 1 : 0;
      int32_t ver = cv;
      if (p >= ni) {  // last run starting at or before p (runs ascend; a row has a handful)
        int64_t lo = r0, hi = r1;
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) >> 1;
          if (a.run_start[mid] <= p) lo = mid; else hi = mid;
        }
        ver = a.run_version[lo];
      }
      a.versions[o + p] = ver;
    }
    if (a.resp && threadIdx.x == 0) a.resp[k] = ni;  // 1 + the last AGENT_INPUT position
  }
}

cudaError_t launch_fill_host_rows(const HostRowsArgs &a, int num_sms, cudaStream_t s) {
  if (a.n < 1) return cudaSuccess;
  const int64_t grid = std::min<int64_t>(a.n, (int64_t)num_sms * 8);
  k_fill_host_rows<<<(int)grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

int64_t export_plan_bytes(int64_t ntiles) {
  return ntiles * (int64_t)sizeof(TilePlan);
}

// Packed host->device token copy (hostpack.h): one thread per 4 positions reads 8 B of
// the uint16 low plane and the aligned 4-byte word of the high plane that holds their
// 2-bit high parts, and stores one int4.
__global__ void k_unpack18(const uint16_t *__restrict__ lo, const uint8_t *__restrict__ hi, int32_t *__restrict__ out,
                           int64_t q0, int64_t q1) {
  for (int64_t q = q0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < q1; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = 4 * q;
    const uint2 l = *reinterpret_cast<const uint2 *>(lo + p);
    const int lane = (int)(p & 31);  // byte (lane & 7) + u of the group's 8 high-plane bytes
    const uint32_t h = *reinterpret_cast<const uint32_t *>(hi + (p >> 5) * 8 + (lane & 7)) >> (2 * (lane >> 3));
    int4 o;
    o.x = (int)((l.x & 0xFFFFu) | ((h & 3u) << 16));
    o.y = (int)((l.x >> 16) | (((h >> 8) & 3u) << 16));
    o.z = (int)((l.y & 0xFFFFu) | (((h >> 16) & 3u) << 16));
    o.w = (int)((l.y >> 16) | (((h >> 24) & 3u) << 16));
    reinterpret_cast<int4 *>(out)[q] = o;
  }
}

cudaError_t launch_unpack18(const uint16_t *lo, const uint8_t *hi, int32_t *out, int64_t p0, int64_t p1, int num_sms,
                            cudaStream_t s) {
  const int64_t nq = (p1 - p0) / 4;
  if (nq <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((nq + 255) / 256, (int64_t)num_sms * 8);
  k_unpack18<<<grid, 256, 0, s>>>(lo, hi, out, p0 / 4, p1 / 4);
  return cudaGetLastError();
}

cudaError_t launch_rehash(const DevView &v, const uint64_t *ok0, const uint64_t *ok1, const int64_t *oval,
                          int64_t ocap, cudaStream_t s) {
  k_rehash<<<1024, 256, 0, s>>>(v, ok0, ok1, oval, ocap);
  return cudaGetLastError();
}

cudaError_t launch_rebuild_index(const DevView &v, int64_t nrows, cudaStream_t s) {
  if (nrows > 0) k_rebuild_index<<<1024, 256, 0, s>>>(v, nrows);
  return cudaGetLastError();
}

// Per-block token hashes (the north star's "per-block prefix hashes", measured as an A/B
// against the exact walk): one warp per 128-word block, 32-bit multiply-add
// hashing per lane (cheap: the A/B must not blame the filter for an expensive hash), two
// xor-reduced words, finalised into 64 bits.  out[b] = hash of words [128 b, 128 b + 128).
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__global__ void __launch_bounds__(256) k_block_hash(const int32_t *__restrict__ tok, int64_t nblocks, uint64_t *out) {
  constexpr int U = 8;  // blocks per warp and round: 8 int4 loads in flight per lane
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * U; b0 < nblocks; b0 += warps * U) {
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      x[u] = ldg_stream_if(reinterpret_cast<const int4 *>(tok) + (b0 + u) * 32 + lane, b0 + u < nblocks);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t k = 2u * (uint32_t)lane + 1u;
      uint32_t a = fmix32(((uint32_t)x[u].x * 0x9e3779b1u + (uint32_t)x[u].y * 0x85ebca77u) ^ (k * 0x27d4eb2fu));
      uint32_t c = fmix32(((uint32_t)x[u].z * 0xc2b2ae3du + (uint32_t)x[u].w * 0x165667b1u) ^ (k * 0x9e3779b1u));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a ^= __shfl_xor_sync(0xffffffffu, a, o);
        c ^= __shfl_xor_sync(0xffffffffu, c, o);
      }
      if (lane == 0 && b0 + u < nblocks) out[b0 + u] = (uint64_t)fmix32(a ^ 0x5bd1e995u) << 32 | fmix32(c + a);
    }
  }
}

cudaError_t launch_block_hash(const int32_t *tok, int64_t nblocks, uint64_t *out, int num_sms, cudaStream_t s) {
  if (nblocks < 1) return cudaSuccess;
  const int64_t grid = std::min<int64_t>((nblocks * 32 / 8 + 255) / 256, (int64_t)num_sms * 8);
  k_block_hash<<<(int)std::max<int64_t>(grid, 1), 256, 0, s>>>(tok, nblocks, out);
  return cudaGetLastError();
}

cudaError_t launch_fill_u64(uint64_t *p, int64_t n, uint64_t val, cudaStream_t s) {
  k_fill_u64<<<1024, 256, 0, s>>>(p, n, val);
  return cudaGetLastError();
}

int export_tile_tokens() { return kExportTile; }

static int env_knob(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

cudaError_t launch_route_pack(char *region, int64_t n, const PushArgs &pa, cudaStream_t s) {
  if (n < 1) return cudaSuccess;
  // push routing measured best with 2 CTAs per SM (its P2P stores queue behind the walk's
  // traffic; N=2: 25.6 vs 24.6 M q/s at 8 per SM)
  static const int grid_pull = env_knob("TM_PACK_GRID", 148 * 8), grid_push = env_knob("TM_PACK_GRID", 148 * 2);
  k_route_pack<<<pa.stride ? grid_push : grid_pull, kPackNT, 0, s>>>(region, pa);
  return cudaGetLastError();
}

cudaError_t launch_route(char *region, const RouteHead &head, const PushArgs &pa, cudaStream_t s) {
  k_route<<<1, kRouteNT, 0, s>>>(region, head, pa);
  return cudaGetLastError();
}

cudaError_t launch_route_arrive(const RoutedArgs &a, cudaStream_t s) {
  k_route_arrive<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_route_wait_done(const DevView &v, const RoutedArgs &a, cudaStream_t s) {
  k_route_wait_done<<<1, 32, 0, s>>>(v, a);
  return cudaGetLastError();
}

// One rank (no peers): the register-path kernel (U = 8).  Peers: the packed TMA compare for
// every query whose requester packed its planes, the register path (U = 4: with the TMA
// compare inlined as well, U = 8 spills) for a requester with ids beyond 18 bits.
// With peers the walk is compiled for <= 128 registers (8 CTAs' worth) but launched with 6
// CTAs per SM: the registers left over hold one 256-thread k_route_pack CTA per SM, so the
// next batch's pack (match_pipelined) runs beside the walk instead of after it
// (N=2: 27.1 -> 28.8 M q/s; the walk itself is as fast as with 147 registers).
constexpr int kRoutedCtasPerSm = 6;
template <int U, bool PACKED, class RG = RoutedPackedRing, int MINB = 6>
static cudaError_t walk_routed_variant(const DevView &v, const RoutedArgs &a, int num_sms, cudaStream_t s) {
  static int occ[kMaxRanks + 1] = {0};
  const size_t smem = routed_smem_bytes<RG>(a.nranks, PACKED);
  auto kern = k_walk_routed<kWalkNT, U, PACKED, RG, MINB>;
  if (!occ[a.nranks]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[a.nranks], kern, kWalkNT, smem);
    if (occ[a.nranks] < 1) occ[a.nranks] = 1;
    static const int cap = env_knob(a.push_stride ? "TM_PUSH_WALK_OCC" : "TM_WALK_OCC", kRoutedCtasPerSm);
    if (PACKED) occ[a.nranks] = std::min(occ[a.nranks], cap);
  }
  kern<<<num_sms * occ[a.nranks], kWalkNT, smem, s>>>(v, a);
  return cudaGetLastError();
}

cudaError_t launch_walk_routed(const DevView &v, const RoutedArgs &a, int num_sms, cudaStream_t s) {
  if (a.nranks > 1) {
#ifdef TM_TUNING
    // remote-query ring (TM_ROUTED_RING = stages x positions per stage; tuning builds only)
    static const int ring = [] {
      const char *e = getenv("TM_ROUTED_RING");
      return e ? atoi(e) : 0;
    }();
    switch (ring) {
      case 1: return walk_routed_variant<4, true, PackedRing<8, 1024>>(v, a, num_sms, s);
      case 2: return walk_routed_variant<4, true, PackedRing<4, 2048>>(v, a, num_sms, s);
      case 3: return walk_routed_variant<4, true, PackedRing<6, 1024>>(v, a, num_sms, s);
      default: break;
    }
#endif
    return walk_routed_variant<4, true, RoutedPackedRing, 8>(v, a, num_sms, s);
  }
  // one rank: the register path with U = 8 (the TMA-staged int32 compare measured 6 % slower
  // here, 25.0-25.2 vs 26.7 M q/s on c5 at N=1; U = 4, which does not spill, 24.3 vs 26.6;
  // 4 CTAs per SM at 233 registers without spills 23.6 vs 26.3)
  return walk_routed_variant<kWalkU, false>(v, a, num_sms, s);
}
}  // namespace tms
