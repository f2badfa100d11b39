// tmstore host runtime + C ABI (include/tmstore.h).
//
// One store per GPU: device arena / row table / metadata runs / branch index /
// session counters, a host mirror of the row table (ids, lengths, parents, branch
// tokens) used for planning, lexicographic ordering and export sizing, pinned
// staging for host-memory calls, and one CUDA stream.  Every entry point locks the
// store mutex; ctypes callers release the GIL around the call.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/tmstore.h"
#include "hostpack.h"
#include "kernels.cuh"
#include "launch.h"

using tms::DevView;
using tms::Batch;

static thread_local std::string g_err;

namespace {

struct TmError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string &msg) { throw TmError{code, msg}; }

void ck(cudaError_t e, const char *what) {
  if (e != cudaSuccess) {
    fail(e == cudaErrorMemoryAllocation ? TM_ENOMEM : TM_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Grow a device array to new_n elements (at least need_n): try the doubled size first and
// fall back to exactly what is needed when HBM is tight (a 100 GB arena cannot double).
// Returns the capacity actually allocated.
template <class T>
int64_t dev_grow(T *&p, int64_t old_n, int64_t new_n, cudaStream_t s, int64_t need_n = -1) {
  T *q = nullptr;
  int64_t got = new_n;
  if (cudaMalloc((void **)&q, sizeof(T) * (size_t)std::max<int64_t>(new_n, 1)) != cudaSuccess) {
    cudaGetLastError();  // clear the allocation failure
    q = nullptr;
    if (need_n < 0 || need_n >= new_n) fail(TM_ENOMEM, "cudaMalloc(grow): out of device memory");
    ck(cudaMalloc((void **)&q, sizeof(T) * (size_t)std::max<int64_t>(need_n, 1)), "cudaMalloc(grow, exact)");
    got = need_n;
  }
  if (p && old_n > 0) ck(cudaMemcpyAsync(q, p, sizeof(T) * (size_t)old_n, cudaMemcpyDeviceToDevice, s), "grow copy");
  ck(cudaStreamSynchronize(s), "grow sync");
  if (p) cudaFree(p);
  p = q;
  return got;
}

// growable byte buffers (device scratch / pinned staging)
struct DevBytes {
  void *p = nullptr;
  size_t cap = 0;
  void *need(size_t n) {
    if (n > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      size_t c = std::max<size_t>(n, cap * 2);
      ck(cudaMalloc(&p, c), "cudaMalloc(scratch)");
      cap = c;
    }
    return p;
  }
  ~DevBytes() { if (p) cudaFree(p); }
};

// Pinned staging buffer.  Asynchronous calls return while a host->device copy out of the
// buffer may still be queued: mark() records the copy, and the next need() waits for it
// before the buffer is rewritten.
struct PinBytes {
  void *p = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
  void mark(cudaStream_t st) {
    if (!ev) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(ev, st), "cudaEventRecord(staging)");
    pending = true;
  }
  void *need(size_t n) {
    if (pending) {
      ck(cudaEventSynchronize(ev), "staging reuse");
      pending = false;
    }
    if (n > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      size_t c = std::max<size_t>(n, cap * 2);
      ck(cudaHostAlloc(&p, c, cudaHostAllocDefault), "cudaHostAlloc(staging)");
      cap = c;
    }
    return p;
  }
  ~PinBytes() {
    if (p) cudaFreeHost(p);
    if (ev) cudaEventDestroy(ev);
  }
};

// lay out several arrays in one buffer
struct Layout {
  size_t bytes = 0;
  size_t add(size_t n) {
    size_t o = bytes;
    bytes += (n + 255) / 256 * 256;
    return o;
  }
};

// A session's rows in insertion order.  Most sessions hold one or two rows: those stay
// inline (no heap allocation per new session - it dominated the host side of large
// record calls of fresh sessions).
struct RowList {
  int64_t n = 0;
  int64_t inl[2] = {0, 0};
  std::vector<int64_t> more;
  int64_t size() const { return n; }
  int64_t operator[](int64_t k) const { return k < 2 ? inl[k] : more[k - 2]; }
  void push_back(int64_t r) {
    if (n < 2) inl[n] = r;
    else more.push_back(r);
    n++;
  }
};

struct RowHost {
  int32_t sid, local;
  int64_t parent;
  int32_t m, len, depth;
  int32_t tnext, spar;
};

}  // namespace

struct tm_store {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t last = nullptr;
  cudaStream_t last_stream = (cudaStream_t)-1;  // stream `last` was recorded on (-1: none yet)
  std::mutex mu;
  DevView v{};
  int64_t arena_cap = 0, row_cap = 0, run_cap = 0, sess_cap = 0, ht_cap = 0;
  int64_t arena_used = 0, n_runs = 0, n_sess = 0;
  int64_t n_real_rows = 0;  // rows minus reserved-but-unused slots
  // row ids an entry reserved but did not use (it re-recorded an existing sequence): handed
  // out again before fresh ids, so the row table grows with distinct sequences, not calls
  std::vector<int64_t> free_rows;
  void *trace_buf = nullptr;  // TM_ROUTED_TRACE diagnostics
  // observability counters (tm_store_counters)
  int64_t c_record_calls = 0, c_records = 0, c_record_tokens = 0, c_match_calls = 0, c_queries = 0,
          c_export_calls = 0, c_export_rows = 0, c_export_tokens = 0;
  std::vector<uint64_t> chain_stamp;  // record: per-session batch stamp and chain slot
  std::vector<int32_t> chain_slot;
  uint64_t batch_stamp = 0;
  std::vector<RowHost> rows;
  std::vector<RowList> sess_rows;
  std::vector<int64_t> sess_stored, sess_naive;
  std::vector<int32_t> sess_maxdepth;  // deepest row per session (-1: none); sizes path-copy reservations
  int64_t max_depth = 0;
  DevBytes scratch, dtok;
  PinBytes pin, ptok, d2h_slot[2];
  // packed host->device token copies (hostpack.h): pinned + device 18-bit planes
  PinBytes plo, phi;
  DevBytes dlo, dhi;
  cudaEvent_t pack_ev = nullptr;  // last DMA out of the pinned planes
  int64_t *pin_ctr = nullptr;     // pinned copy of the device counters (arena, rows, runs, error)
  bool pack_pending = false;
  int64_t pack_min = int64_t(8) << 20;  // tokens per call below which the raw copy is used (TM_H2D_PACK_MIN; <0: off)
  bool pack_auto = true;                // TM_H2D_PACK_MIN unset: pack only as the node's sole GPU client
  double pack_frac = 0.9;               // share of a packed call's tokens that is packed (TM_H2D_PACK_FRAC)
  bool pack_frac_set = false;           // TM_H2D_PACK_FRAC given: split pageable sources too
  int local_world = 1;                  // LOCAL_WORLD_SIZE (torchrun) at creation
  int64_t c_pack_calls = 0, c_pack_tokens = 0, c_raw_calls = 0, c_raw_tokens = 0, c_pack_fallbacks = 0,
          c_h2d_bytes = 0;  // token bytes actually copied host->device
  // Device-memory match batches are read-only: they may overlap each other (a batch's
  // planner and grid ramp-up hide under the previous batch's tail) but not a mutation.
  // Each in-flight batch uses one slot (scratch + scheduler block + completion event).
  struct MatchSlot {
    cudaEvent_t done = nullptr;
    bool used = false;
    DevBytes scratch;
    tms::Sched *sched = nullptr;
  };
  static constexpr int kSlots = 4;
  MatchSlot slots[kSlots];
  int next_slot = 0;
  // optional per-kernel CUDA-event timing (tm_profile_*): pairs recorded around launches
  // batches at least this large get the longest-first planner.  Off by default: on the
  // c4 workload in-kernel root lookups are hidden by occupancy and the planner's ~10 us
  // costs more than the tail it removes (TM_PLAN_MIN at store creation overrides).
  int64_t plan_min = int64_t(1) << 62;
  int plan_roots = 0;           // planner also resolves root rows (TM_PLAN_ROOTS=1)
  tms::Sched *sched = nullptr;  // walk scheduler block (self-cleaning)
  bool profile = false;
  static constexpr int kProfKinds = 9;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kProfKinds];
  size_t ev_used[kProfKinds] = {};
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void ensure_rows(tm_store *s, int64_t need) {
  if (need <= s->row_cap) return;
  int64_t nc = std::max<int64_t>(need, s->row_cap * 2);
  int64_t n = (int64_t)s->rows.size();
  dev_grow(s->v.row_vb, n, nc, s->stream);
  dev_grow(s->v.row_m, n, nc, s->stream);
  dev_grow(s->v.row_len, n, nc, s->stream);
  dev_grow(s->v.row_parent, n, nc, s->stream);
  dev_grow(s->v.row_sess, n, nc, s->stream);
  dev_grow(s->v.row_local, n, nc, s->stream);
  dev_grow(s->v.row_depth, n, nc, s->stream);
  dev_grow(s->v.row_run0, n, nc, s->stream);
  dev_grow(s->v.row_nrun, n, nc, s->stream);
  dev_grow(s->v.row_ext, n, nc, s->stream);
  dev_grow(s->v.row_ext_tok, n, nc, s->stream);
  dev_grow(s->v.row_ext_len, n, nc, s->stream);
  dev_grow(s->v.row_ext_vb, n, nc, s->stream);
  dev_grow(s->v.row_jump, n, nc, s->stream);
  s->row_cap = nc;
  s->v.row_cap = nc;
  // the host mirror grows in place (no copy inside a record call), its new pages faulted in
  // here, once per doubling, instead of by every call that appends rows
  s->rows.reserve((size_t)nc);
  memset((void *)(s->rows.data() + s->rows.size()), 0, (s->rows.capacity() - s->rows.size()) * sizeof(RowHost));
}

void ensure_runs(tm_store *s, int64_t need) {
  if (need <= s->run_cap) return;
  int64_t nc = std::max<int64_t>(need, s->run_cap * 2);
  dev_grow(s->v.run_start, s->n_runs, nc, s->stream);
  dev_grow(s->v.run_version, s->n_runs, nc, s->stream);
  dev_grow(s->v.run_origin, s->n_runs, nc, s->stream);
  s->run_cap = nc;
  s->v.run_cap = nc;
}

void ensure_arena(tm_store *s, int64_t need) {
  if (need <= s->arena_cap) return;
  const int64_t exact = round_up(need, 1 << 20);
  const int64_t nc = dev_grow(s->v.arena, s->arena_used, std::max<int64_t>(exact, s->arena_cap * 2), s->stream, exact);
  s->arena_cap = nc;
  s->v.arena_cap = nc;
}

void ensure_sessions(tm_store *s, int64_t need) {
  if (need <= s->sess_cap) return;
  int64_t nc = std::max<int64_t>(need, s->sess_cap * 2);
  int64_t n = s->n_sess;
  dev_grow(s->v.s_nrows, n, nc, s->stream);
  dev_grow(s->v.s_stored, n, nc, s->stream);
  dev_grow(s->v.s_naive, n, nc, s->stream);
  ck(cudaMemsetAsync(s->v.s_nrows + n, 0, sizeof(int32_t) * (nc - n), s->stream), "memset");
  ck(cudaMemsetAsync(s->v.s_stored + n, 0, sizeof(int64_t) * (nc - n), s->stream), "memset");
  ck(cudaMemsetAsync(s->v.s_naive + n, 0, sizeof(int64_t) * (nc - n), s->stream), "memset");
  dev_grow(s->v.s_pc_row, n, nc, s->stream);
  dev_grow(s->v.s_pc_vb, n, nc, s->stream);
  dev_grow(s->v.s_pc_cap, n, nc, s->stream);
  ck(tms::launch_fill_u64((uint64_t *)(s->v.s_pc_row + n), nc - n, ~0ull, s->stream), "fill");  // -1: no copy
  ck(cudaMemsetAsync(s->v.s_pc_vb + n, 0, sizeof(int64_t) * (nc - n), s->stream), "memset");
  ck(cudaMemsetAsync(s->v.s_pc_cap + n, 0, sizeof(int64_t) * (nc - n), s->stream), "memset");
  s->sess_cap = nc;
}

void alloc_table(tm_store *s, int64_t cap) {
  ck(cudaMalloc((void **)&s->v.hk0, sizeof(uint64_t) * cap), "cudaMalloc(ht)");
  ck(cudaMalloc((void **)&s->v.hk1, sizeof(uint64_t) * cap), "cudaMalloc(ht)");
  ck(cudaMalloc((void **)&s->v.hval, sizeof(int64_t) * cap), "cudaMalloc(ht)");
  ck(tms::launch_fill_u64(s->v.hk0, cap, tms::kEmpty, s->stream), "ht fill");
  s->ht_cap = cap;
  s->v.ht_mask = (uint64_t)cap - 1;
}

// keep the branch index at load <= 1/2
void ensure_table(tm_store *s, int64_t entries) {
  if (entries * 2 <= s->ht_cap) return;
  int64_t nc = s->ht_cap;
  while (entries * 2 > nc) nc *= 2;
  uint64_t *o0 = s->v.hk0, *o1 = s->v.hk1;
  int64_t *ov = s->v.hval;
  int64_t oc = s->ht_cap;
  alloc_table(s, nc);
  ck(tms::launch_rehash(s->v, o0, o1, ov, oc, s->stream), "rehash");
  ck(cudaStreamSynchronize(s->stream), "rehash sync");
  cudaFree(o0);
  cudaFree(o1);
  cudaFree(ov);
}

// Bracket a launch with events when profiling (kind: 0 walk, 1 commit, 2 export, 3 plan,
// 4 route, 5 route pack, 6 routed wait).
struct ProfScope {
  tm_store *s;
  int kind;
  cudaStream_t st;
  ProfScope(tm_store *s_, int k, cudaStream_t st_) : s(s_), kind(k), st(st_) {
    if (!s->profile) return;
    auto &v = s->ev[kind];
    if (s->ev_used[kind] == v.size()) {
      cudaEvent_t a, b;
      ck(cudaEventCreate(&a), "event");
      ck(cudaEventCreate(&b), "event");
      v.push_back({a, b});
    }
    ck(cudaEventRecord(v[s->ev_used[kind]].first, st), "event");
  }
  ~ProfScope() {
    if (!s->profile) return;
    cudaEventRecord(s->ev[kind][s->ev_used[kind]].second, st);
    s->ev_used[kind]++;
  }
};

// exclusive operations (record, export, host-buffer match) wait for everything before them
// Device -> host copy of a large result.  A page-locked destination (DeviceStore's pinned
// export pool) is written by the copy engine directly.  For pageable memory the driver
// stages through a small bounce buffer (measured ~1.5-5 GB/s here), so pipeline 64 MB
// chunks through two pinned slots and spread the pinned->pageable memcpy over host threads.
void d2h_pageable(tm_store *s, void *dst, const void *src, int64_t bytes, cudaStream_t st) {
  static const int64_t CH = [] {  // TM_D2H_CHUNK_MB (tuning only)
    const char *e = getenv("TM_D2H_CHUNK_MB");
    return (e ? std::max(1, atoi(e)) : 64) * (int64_t(1) << 20);
  }();
  cudaPointerAttributes pa{};
  const bool pinned_dst = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  if (!pinned_dst) cudaGetLastError();  // clear the (harmless) error for unregistered memory
  if (bytes <= (8ll << 20) || pinned_dst) {  // page-locked destination: the copy engine writes it directly
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "D2H sync");
    return;
  }
  const int64_t nparts = 4 * (int64_t)tms::host_threads();
  const int64_t nch = (bytes + CH - 1) / CH;
  cudaEvent_t ev[2];
  for (auto &e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  auto issue = [&](int64_t c) {
    const int64_t off = c * CH, len = std::min(CH, bytes - off);
    char *slot = (char *)s->d2h_slot[c & 1].need(CH);
    ck(cudaMemcpyAsync(slot, (const char *)src + off, len, cudaMemcpyDeviceToHost, st), "D2H chunk");
    ck(cudaEventRecord(ev[c & 1], st), "event");
  };
  issue(0);
  for (int64_t c = 0; c < nch; c++) {
    ck(cudaEventSynchronize(ev[c & 1]), "D2H wait");
    if (c + 1 < nch) issue(c + 1);
    const int64_t off = c * CH, len = std::min(CH, bytes - off);
    const char *slot = (const char *)s->d2h_slot[c & 1].p;
    const int64_t part = (len + nparts - 1) / nparts;  // pool threads copy (and first-touch) the destination
    tms::parallel_for(nparts, [&](int64_t k) {
      const int64_t a = k * part, b = std::min(len, a + part);
      if (a < b) tms::copy_stream((char *)dst + off + a, slot + a, (size_t)(b - a));
    });
  }
  for (auto &e : ev) cudaEventDestroy(e);
}

// a device-side error code (kernels.cuh kErr*) becomes a loud host error
[[noreturn]] void raise_device_error(int64_t code) {
  static const char *names[] = {"", "branch index full", "arena bounds", "row bounds", "run bounds",
                                "peer rank timed out (routed match)"};
  fail(TM_ECUDA, std::string("device check failed: ") + (code > 0 && code < 6 ? names[code] : "unknown"));
}

void check_device_error(tm_store *s) {
  int64_t code = 0;
  ck(cudaMemcpy(&code, s->v.ctr + 3, sizeof(code), cudaMemcpyDeviceToHost), "D2H error flag");
  if (code) raise_device_error(code);
}

// host-memory calls: queue the counters' readback into pinned memory before the final
// sync (no extra round trip), then check the error word after it
void enqueue_ctr_readback(tm_store *s, cudaStream_t st) {
  ck(cudaMemcpyAsync(s->pin_ctr, s->v.ctr, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H counters");
}
void check_ctr_error(const tm_store *s) {
  if (s->pin_ctr[3]) raise_device_error(s->pin_ctr[3]);
}

bool valid_row(const tm_store *s, int64_t r) { return r >= 0 && r < (int64_t)s->rows.size() && s->rows[r].sid >= 0; }

void wait_prev(tm_store *s, cudaStream_t st) {
  if (s->last_stream != st) ck(cudaStreamWaitEvent(st, s->last, 0), "cudaStreamWaitEvent");  // same stream: ordered
  for (auto &sl : s->slots)
    if (sl.used) {
      ck(cudaStreamWaitEvent(st, sl.done, 0), "cudaStreamWaitEvent");
      sl.used = false;  // ordered behind this operation from now on (it records `last`)
    }
}

void mark_done(tm_store *s, cudaStream_t st) {
  ck(cudaEventRecord(s->last, st), "cudaEventRecord");
  s->last_stream = st;
}

// TM_TRACE_CALLS=1: per-phase host time of record calls on stderr (latency work only)
struct PhaseTrace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  char buf[512];
  int len = 0;
  PhaseTrace() {
    static const bool env = getenv("TM_TRACE_CALLS") != nullptr;
    on = env;
    if (on) t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char *name) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    len += snprintf(buf + len, sizeof(buf) - len, " %s=%.1f", name,
                    std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
  }
  ~PhaseTrace() {
    if (on) fprintf(stderr, "[tm trace]%s total=%.1f us\n", buf,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
};

// NVTX range around every C-ABI call (visible in nsys / ncu timelines)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
int guarded(tm_store *s, F &&f) {
  if (!s) {
    g_err = "null store";
    return TM_EINVAL;
  }
  try {
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard dg(s->device);
    f();
    return TM_OK;
  } catch (const TmError &e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc &) {
    g_err = "host allocation failed";
    return TM_ENOMEM;
  }
}

// Stage host sequences into the pinned buffer with 128-byte aligned starts and copy
// them to the device token scratch.  Returns device offsets (host vector).
// Packed copy (hostpack.h) of host tokens into dtok: pieces sorted by destination,
// disjoint, destinations multiples of 32.  One pool job packs every piece (threads take
// pieces in order); whenever a chunk of pieces is complete the calling thread - between
// its own pieces - enqueues that chunk's plane copies and its k_unpack18, so the copy
// engine streams chunk k while the pool packs chunk k+1.  false: a token is outside
// [0, 2^18) (the caller then does the raw copy on the same stream, which overwrites
// whatever the packed chunks wrote).
bool stage_packed(tm_store *s, const std::vector<tms::PackPiece> &pieces, int64_t end, int32_t *dtok, cudaStream_t st) {
  end = round_up(std::max<int64_t>(end, 32), 32);
  uint16_t *lo = (uint16_t *)s->plo.need(2 * (size_t)end);
  uint8_t *hi = (uint8_t *)s->phi.need((size_t)end / 4);
  uint16_t *dlo = (uint16_t *)s->dlo.need(2 * (size_t)end);
  uint8_t *dhi = (uint8_t *)s->dhi.need((size_t)end / 4);
  if (s->pack_pending) ck(cudaEventSynchronize(s->pack_ev), "pack staging free");
  s->pack_pending = false;
  int64_t total = 0;
  for (const auto &p : pieces) total += p.len;
  static const int64_t nsplit = [] {  // TM_H2D_CHUNKS (tuning): copies per call
    const char *e = getenv("TM_H2D_CHUNKS");
    return e ? std::max<int64_t>(1, atoll(e)) : 12;  // 24-core box: 12 -> 0.62-0.64, 24 -> 0.62, 48 -> 0.55 M q/s
  }();
  const int64_t chunk = std::max<int64_t>(int64_t(1) << 19, total / nsplit);
  std::vector<size_t> cbeg{0};  // chunk c = pieces [cbeg[c], cbeg[c+1])
  std::vector<int32_t> chunk_of(pieces.size());
  for (size_t i = 0, tok = 0; i < pieces.size(); i++) {
    if (tok >= (size_t)chunk) {
      cbeg.push_back(i);
      tok = 0;
    }
    chunk_of[i] = (int32_t)cbeg.size() - 1;
    tok += pieces[i].len;
  }
  const size_t nchunks = cbeg.size();
  cbeg.push_back(pieces.size());
  std::unique_ptr<std::atomic<int64_t>[]> left(new std::atomic<int64_t>[nchunks]);
  for (size_t c = 0; c < nchunks; c++) left[c].store((int64_t)(cbeg[c + 1] - cbeg[c]));
  std::atomic<bool> bad{false};
  size_t issued = 0;
  int64_t bytes = 0;
  cudaError_t err = cudaSuccess;
  const std::thread::id caller = std::this_thread::get_id();
  auto issue_ready = [&] {  // calling thread only
    while (issued < nchunks && err == cudaSuccess && !bad.load(std::memory_order_relaxed) &&
           left[issued].load(std::memory_order_acquire) == 0) {
      const tms::PackPiece &a = pieces[cbeg[issued]], &b = pieces[cbeg[issued + 1] - 1];
      const int64_t p0 = a.dst, p1 = round_up(b.dst + b.len, 32);
      err = cudaMemcpyAsync(dlo + p0, lo + p0, 2 * (size_t)(p1 - p0), cudaMemcpyHostToDevice, st);
      if (err == cudaSuccess) err = cudaMemcpyAsync(dhi + p0 / 4, hi + p0 / 4, (size_t)(p1 - p0) / 4, cudaMemcpyHostToDevice, st);
      if (err == cudaSuccess) err = tms::launch_unpack18(dlo, dhi, dtok, p0, p1, s->num_sms, st);
      bytes += (p1 - p0) * 9 / 4;
      issued++;
    }
  };
  tms::parallel_for((int64_t)pieces.size(), [&](int64_t i) {
    if (!tms::pack_piece(pieces[i], lo, hi)) bad.store(true, std::memory_order_relaxed);
    left[chunk_of[i]].fetch_sub(1, std::memory_order_acq_rel);
    if (std::this_thread::get_id() == caller) issue_ready();
  });
  issue_ready();  // the chunks finished by other threads after the caller's last piece
  ck(err, "packed H2D");
  ck(cudaEventRecord(s->pack_ev, st), "pack event");
  s->pack_pending = true;
  if (bad.load()) return false;
  s->c_h2d_bytes += bytes;
  return true;
}

void add_pieces(std::vector<tms::PackPiece> &out, const int32_t *src, int64_t dst, int64_t len) {
  for (int64_t o = 0; o < len; o += tms::kPackPieceMax)
    out.push_back({src + o, dst + o, std::min<int64_t>(tms::kPackPieceMax, len - o)});
}

std::atomic<int> g_live_stores{0};

// Packing halves the PCIe bytes but doubles the host-memory traffic (read 4 B, write
// 2.25 B, DMA-read 2.25 B per token instead of DMA-read 4 B).  It pays while PCIe is the
// bottleneck - one GPU client per node - and loses once several GPUs' copies share the
// host memory bandwidth, so by default it is used only when this
// is the node's sole GPU client (one rank, one live store).
bool use_packed(tm_store *s, int64_t tokens) {
  if (s->pack_min < 0 || tokens < s->pack_min || !tms::pack18_supported()) return false;
  return !s->pack_auto || (s->local_world == 1 && g_live_stores.load() == 1);
}

void stage_tokens(tm_store *s, int64_t n, const int32_t *tokens, const int64_t *tok_off, const int64_t *tok_len,
                  std::vector<int64_t> &doff, const std::vector<int64_t> *perm, cudaStream_t st) {
  doff.resize(n);
  // Fast path: every sequence already starts on a 128-byte boundary -> the device copy
  // keeps the caller's layout (one direct H2D of a pinned buffer goes at full PCIe rate).
  // Padding words after a sequence are never compared (positions >= len are masked).
  bool aligned = true;
  int64_t end = 0, ntok = 0;
  for (int64_t k = 0; k < n; k++) {
    aligned &= (tok_off[k] % tms::kAlignWords) == 0 && tok_off[k] >= 0;
    end = std::max<int64_t>(end, tok_off[k] + tok_len[k]);
    ntok += tok_len[k];
  }
  const bool packed = use_packed(s, ntok);
  if (aligned) {
    for (int64_t k = 0; k < n; k++) doff[k] = tok_off[perm ? (*perm)[k] : k];
    int32_t *d = (int32_t *)s->dtok.need(sizeof(int32_t) * (size_t)(round_up(std::max<int64_t>(end, 1), tms::kAlignWords) + tms::kAlignWords));
    if (packed) {
      // the sequences' own ranges, merged (sequences may share words of the caller's buffer)
      std::vector<std::pair<int64_t, int64_t>> iv;
      iv.reserve(n);
      for (int64_t k = 0; k < n; k++)
        if (tok_len[k] > 0) iv.push_back({tok_off[k], tok_off[k] + tok_len[k]});
      std::sort(iv.begin(), iv.end());
      std::vector<tms::PackPiece> pieces;
      for (size_t i = 0; i < iv.size();) {
        int64_t a = iv[i].first, b = iv[i].second;
        for (i++; i < iv.size() && iv[i].first < b; i++) b = std::max(b, iv[i].second);  // overlapping only
        add_pieces(pieces, tokens + a, a, b - a);
      }
      // Hybrid split: the tail of the range goes raw, straight from the caller's buffer,
      // and its DMA starts at once, while the host threads pack the head (TM_H2D_PACK_FRAC
      // of the tokens).  Packing alone leaves PCIe idle while the host packs; raw alone is
      // PCIe-bound - the split keeps both busy.
      size_t k = pieces.size();
      // (only from page-locked caller memory: a pageable source would be staged by the
      // driver on this thread before the packing starts)
      cudaPointerAttributes pa{};
      const bool pinned_src = cudaPointerGetAttributes(&pa, tokens) == cudaSuccess && pa.type == cudaMemoryTypeHost;
      cudaGetLastError();  // (a pageable pointer may leave an error on older drivers)
      if (s->pack_frac < 1.0 && !pieces.empty() && (pinned_src || s->pack_frac_set)) {
        int64_t tot = 0, acc = 0;
        for (const auto &pc : pieces) tot += pc.len;
        for (k = 0; k < pieces.size() && acc < (int64_t)(s->pack_frac * (double)tot); k++) acc += pieces[k].len;
      }
      int64_t raw_bytes = 0;
      if (k < pieces.size()) {
        const int64_t r0 = pieces[k].dst;  // a multiple of 32: no unpacked chunk writes past it
        raw_bytes = 4 * (end - r0);
        ck(cudaMemcpyAsync(d + r0, tokens + r0, (size_t)raw_bytes, cudaMemcpyHostToDevice, st), "H2D tokens (raw tail)");
        pieces.resize(k);
      }
      if (pieces.empty() || stage_packed(s, pieces, pieces.empty() ? 0 : pieces.back().dst + pieces.back().len, d, st)) {
        s->c_pack_calls++;
        s->c_pack_tokens += ntok;
        s->c_h2d_bytes += raw_bytes;
        return;
      }
      s->c_pack_fallbacks++;
    }
    s->c_raw_calls++;
    s->c_raw_tokens += ntok;
    s->c_h2d_bytes += 4 * end;
    if (end > 0) ck(cudaMemcpyAsync(d, tokens, sizeof(int32_t) * end, cudaMemcpyHostToDevice, st), "H2D tokens");
    return;
  }
  int64_t total = 0;
  for (int64_t k = 0; k < n; k++) {
    int64_t e = perm ? (*perm)[k] : k;
    doff[k] = total;
    total += round_up(std::max<int64_t>(tok_len[e], 1), tms::kAlignWords);
  }
  int32_t *d = (int32_t *)s->dtok.need(sizeof(int32_t) * (size_t)std::max<int64_t>(total, 32));
  if (packed) {
    std::vector<tms::PackPiece> pieces;
    for (int64_t k = 0; k < n; k++) {
      const int64_t e = perm ? (*perm)[k] : k;
      add_pieces(pieces, tokens + tok_off[e], doff[k], tok_len[e]);
    }
    if (stage_packed(s, pieces, total, d, st)) {
      s->c_pack_calls++;
      s->c_pack_tokens += ntok;
      return;
    }
    s->c_pack_fallbacks++;
  }
  s->c_raw_calls++;
  s->c_raw_tokens += ntok;
  s->c_h2d_bytes += 4 * total;
  int32_t *h = (int32_t *)s->ptok.need(sizeof(int32_t) * (size_t)std::max<int64_t>(total, 32));
  for (int64_t k = 0; k < n; k++) {
    int64_t e = perm ? (*perm)[k] : k;
    int64_t L = tok_len[e];
    memcpy(h + doff[k], tokens + tok_off[e], sizeof(int32_t) * (size_t)L);
    int64_t pad = round_up(std::max<int64_t>(L, 1), tms::kAlignWords) - L;
    memset(h + doff[k] + L, 0, sizeof(int32_t) * (size_t)pad);
  }
  if (total > 0) ck(cudaMemcpyAsync(d, h, sizeof(int32_t) * total, cudaMemcpyHostToDevice, st), "H2D tokens");
  s->ptok.mark(st);
}

// Lexicographic order of the subtree of row r.  kids[local] =
// children of that row sorted by (m, prefix-first, tnext).  For each branch depth d <
// len(r), ascending: [prefix row at d] + [subtrees of children whose token at d is below
// r's] ... then r itself, its extensions, and, deepest depth first, the subtrees of the
// children whose token at d is above r's.  Iterative (an explicit action stack): chains of
// thousands of turns must not exhaust the native stack.
void lex_emit(const tm_store *s, const std::vector<std::vector<int64_t>> &kids, int64_t root, std::vector<int64_t> &out) {
  struct Act {
    int64_t row;
    bool recurse;
  };
  std::vector<Act> stack{{root, true}};
  std::vector<Act> acts;
  std::vector<int64_t> hi_list;
  std::vector<size_t> hi_mark;
  while (!stack.empty()) {
    const Act act = stack.back();
    stack.pop_back();
    if (!act.recurse) {
      out.push_back(act.row);
      continue;
    }
    const int64_t r = act.row;
    const RowHost &R = s->rows[r];
    const auto &ch = kids[R.local];
    acts.clear();
    hi_list.clear();
    hi_mark.clear();
    size_t i = 0;
    while (i < ch.size() && s->rows[ch[i]].m < R.len) {
      const int32_t d = s->rows[ch[i]].m;
      hi_mark.push_back(hi_list.size());
      for (; i < ch.size() && s->rows[ch[i]].m == d; i++) {
        const RowHost &C = s->rows[ch[i]];
        if (C.len == C.m) acts.push_back({ch[i], false});
        else if (C.tnext < C.spar) acts.push_back({ch[i], true});
        else hi_list.push_back(ch[i]);
      }
    }
    acts.push_back({r, false});
    for (; i < ch.size(); i++) acts.push_back({ch[i], true});
    for (size_t g = hi_mark.size(); g-- > 0;) {
      const size_t a0 = hi_mark[g], b0 = (g + 1 < hi_mark.size()) ? hi_mark[g + 1] : hi_list.size();
      for (size_t k = a0; k < b0; k++) acts.push_back({hi_list[k], true});
    }
    for (size_t k = acts.size(); k-- > 0;) stack.push_back(acts[k]);
  }
}

}  // namespace

// ---- snapshot / restore -----------------------------------------------------------------
namespace {
constexpr char kMagic[8] = {'T', 'M', 'S', 'T', 'O', 'R', 'E', '3'};

struct FileW {
  FILE *f;
  void put(const void *p, size_t n) {
    if (n && fwrite(p, 1, n, f) != n) fail(TM_EINVAL, "snapshot write failed");
  }
  template <class T> void val(const T &x) { put(&x, sizeof(T)); }
};
struct FileR {
  FILE *f;
  void get(void *p, size_t n) {
    if (n && fread(p, 1, n, f) != n) fail(TM_EINVAL, "snapshot truncated");
  }
  template <class T> T val() { T x; get(&x, sizeof(T)); return x; }
};

template <class T>
void save_dev(tm_store *s, FileW &w, const T *d, int64_t n) {
  const int64_t bytes = (int64_t)sizeof(T) * n;
  constexpr int64_t CH = 64ll << 20;
  char *h = (char *)s->pin.need(CH);
  for (int64_t off = 0; off < bytes; off += CH) {
    const int64_t len = std::min(CH, bytes - off);
    ck(cudaMemcpy(h, (const char *)d + off, len, cudaMemcpyDeviceToHost), "snapshot D2H");
    w.put(h, len);
  }
}

template <class T>
void load_dev(tm_store *s, FileR &r, T *d, int64_t n) {
  const int64_t bytes = (int64_t)sizeof(T) * n;
  constexpr int64_t CH = 64ll << 20;
  char *h = (char *)s->pin.need(CH);
  for (int64_t off = 0; off < bytes; off += CH) {
    const int64_t len = std::min(CH, bytes - off);
    r.get(h, len);
    ck(cudaMemcpy((char *)d + off, h, len, cudaMemcpyHostToDevice), "restore H2D");
  }
}
}  // namespace

extern "C" {

const char *tm_last_error(void) { return g_err.c_str(); }
#ifdef TM_DEBUG
const char *tm_version(void) { return "tmstore 0.1.0 (sm_100a, debug checks)"; }
#else
const char *tm_version(void) { return "tmstore 0.1.0 (sm_100a)"; }
#endif

int tm_store_create(const tm_config *cfg, tm_store **out) {
  if (!out) {
    g_err = "null out";
    return TM_EINVAL;
  }
  tm_config c{0, 1 << 22, 1 << 12, 1 << 14, 1 << 10};
  if (cfg) c = *cfg;
  tm_store *s = new tm_store();
  s->device = c.device;
  if (const char *e = getenv("TM_PLAN_MIN")) s->plan_min = atoll(e);
  if (const char *e = getenv("TM_PLAN_ROOTS")) s->plan_roots = atoi(e);
  if (const char *e = getenv("TM_H2D_PACK_MIN")) {
    s->pack_min = atoll(e);
    s->pack_auto = false;
  }
  if (const char *e = getenv("TM_H2D_PACK_FRAC")) {
    s->pack_frac = std::min(1.0, std::max(0.0, atof(e)));
    s->pack_frac_set = true;
  }
  if (const char *e = getenv("LOCAL_WORLD_SIZE")) s->local_world = std::max(1, atoi(e));
  int rc = guarded(s, [&] {
    ck(cudaSetDevice(c.device), "cudaSetDevice");
    ck(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, c.device), "attr");
    ck(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&s->last, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&s->pack_ev, cudaEventDisableTiming), "event");
    ck(cudaHostAlloc((void **)&s->pin_ctr, 64, cudaHostAllocDefault), "pinned counters");
    ck(cudaMalloc((void **)&s->v.ctr, sizeof(int64_t) * 4), "ctr");
    ck(cudaMalloc((void **)&s->sched, sizeof(tms::Sched)), "sched");
    ck(cudaMemsetAsync(s->sched, 0, sizeof(tms::Sched), s->stream), "sched");
    for (auto &sl : s->slots) {
      ck(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming), "event");
      ck(cudaMalloc((void **)&sl.sched, sizeof(tms::Sched)), "sched");
      ck(cudaMemsetAsync(sl.sched, 0, sizeof(tms::Sched), s->stream), "sched");
    }
    ck(cudaMemsetAsync(s->v.ctr, 0, sizeof(int64_t) * 4, s->stream), "ctr");
    ensure_arena(s, std::max<int64_t>(c.arena_words, 1 << 16));
    ensure_rows(s, std::max<int64_t>(c.row_capacity, 64));
    ensure_runs(s, std::max<int64_t>(c.run_capacity, 64));
    ensure_sessions(s, std::max<int64_t>(c.session_capacity, 16));
    int64_t ht = 1024;
    while (ht < 2 * s->row_cap) ht *= 2;
    alloc_table(s, ht);
    mark_done(s, s->stream);
    ck(cudaStreamSynchronize(s->stream), "create sync");
  });
  if (rc) {
    delete s;
    return rc;
  }
  g_live_stores.fetch_add(1);
  *out = s;
  return TM_OK;
}

int tm_store_destroy(tm_store *s) {
  if (!s) return TM_OK;
  DeviceGuard dg(s->device);  // member destructors free device memory on the store's GPU
  cudaStreamSynchronize(s->stream);
  for (auto &sl : s->slots)
    if (sl.used) cudaEventSynchronize(sl.done);
  void *ptrs[] = {s->v.arena, s->v.row_vb, s->v.row_m, s->v.row_len, s->v.row_parent, s->v.row_sess,
                  s->v.row_local, s->v.row_depth, s->v.row_run0, s->v.row_nrun, s->v.row_ext,
                  s->v.row_ext_tok, s->v.row_ext_len, s->v.row_ext_vb, s->v.row_jump, s->v.run_start,
                  s->v.run_version, s->v.run_origin, s->v.hk0, s->v.hk1, s->v.hval, s->v.s_nrows,
                  s->v.s_stored, s->v.s_naive, s->v.s_pc_row, s->v.s_pc_vb, s->v.s_pc_cap, s->v.ctr, s->sched,
                  s->trace_buf};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  for (auto &sl : s->slots) {
    cudaEventDestroy(sl.done);
    if (sl.sched) cudaFree(sl.sched);
  }
  for (int k = 0; k < tm_store::kProfKinds; k++)
    for (auto &e : s->ev[k]) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  cudaEventDestroy(s->last);
  cudaEventDestroy(s->pack_ev);
  if (s->pin_ctr) cudaFreeHost(s->pin_ctr);
  cudaStreamDestroy(s->stream);
  g_live_stores.fetch_sub(1);
  delete s;  // DevBytes / PinBytes members release scratch and pinned staging
  return TM_OK;
}

int tm_session_create(tm_store *s, int32_t *out_sid) {
  return guarded(s, [&] {
    if (s->n_sess >= INT32_MAX) fail(TM_ENOMEM, "too many sessions");
    ensure_sessions(s, s->n_sess + 1);
    s->sess_rows.emplace_back();
    s->sess_stored.push_back(0);
    s->sess_naive.push_back(0);
    s->sess_maxdepth.push_back(-1);
    *out_sid = (int32_t)s->n_sess++;
    s->v.n_sess = s->n_sess;
  });
}

int tm_session_count(tm_store *s, int64_t *out_n) {
  return guarded(s, [&] { *out_n = s->n_sess; });
}

int tm_record_batch(tm_store *s, int64_t n, int32_t mem, const int32_t *sids, const int32_t *tokens,
                    const int64_t *tok_off, const int64_t *tok_len, const int64_t *run_off,
                    const int32_t *run_start, const uint8_t *run_origin, const int32_t *run_version,
                    int64_t *out_matched, int64_t *out_row, int32_t *out_local, int64_t *out_parent,
                    int32_t *out_parent_local, int64_t *out_added, void *stream) {
  NvtxRange nvtx_("tm_record_batch");
  PhaseTrace tr;
  return guarded(s, [&] {
    if (n < 0) fail(TM_EINVAL, "negative batch size");
    if (n == 0) return;
    if (mem != TM_MEM_HOST && mem != TM_MEM_DEVICE) fail(TM_EINVAL, "bad memory kind");
    // ---- validate (trie.py:128-131); group entries into per-session chains (batch order
    // inside a chain: sequential semantics), chains ordered longest first
    // session -> chain slot for this batch (stamped, so a 1-entry call on a store with
    // millions of sessions does not clear a million-entry table)
    if ((int64_t)s->chain_stamp.size() < s->n_sess) {
      s->chain_stamp.resize(s->n_sess, 0);
      s->chain_slot.resize(s->n_sess, -1);
    }
    const uint64_t stamp = ++s->batch_stamp;
    std::vector<int64_t> chain_tokens;
    std::vector<int32_t> chain_len;
    std::vector<int32_t> chain_idx(n);
    int64_t total_runs = 0, words_upper = 0;
    for (int64_t k = 0; k < n; k++) {
      int32_t sid = sids[k];
      if (sid < 0 || sid >= s->n_sess) fail(TM_ENOENT, "unknown session " + std::to_string(sid));
      int64_t L = tok_len[k];
      if (L <= 0) fail(TM_EINVAL, "cannot insert an empty sequence");
      if (L >= (int64_t)INT32_MAX - 64) fail(TM_EINVAL, "sequence too long");
      const int64_t r0 = run_off[k], r1 = run_off[k + 1];
      if (r1 <= r0) fail(TM_EINVAL, "tokens, origins, versions must be parallel");
      if (mem == TM_MEM_DEVICE && tok_off[k] % tms::kAlignWords)
        fail(TM_EINVAL, "device token offsets must be multiples of 32");
      int32_t c = s->chain_stamp[sid] == stamp ? s->chain_slot[sid] : -1;
      if (c < 0) {
        s->chain_stamp[sid] = stamp;
        c = s->chain_slot[sid] = (int32_t)chain_tokens.size();
        chain_tokens.push_back(0);
        chain_len.push_back(0);
      }
      chain_idx[k] = c;
      chain_tokens[c] += L;
      chain_len[c]++;
      total_runs += r1 - r0;
      words_upper += round_up(L, tms::kAlignWords) + tms::kAlignWords;
      // the entry's row may reach path-copy depth: room for a fresh copy with 2x headroom
      if (s->sess_maxdepth[sid] + chain_len[c] >= tms::kPathCopyDepth) words_upper += round_up(2 * L, tms::kAlignWords);
    }
    {  // the metadata runs of every entry (trie.py:128-131), over the host pool for large batches
      auto check_runs = [&](int64_t k0, int64_t k1) -> int {
        for (int64_t k = k0; k < k1; k++) {
          const int64_t L = tok_len[k], r0 = run_off[k], r1 = run_off[k + 1];
          if (run_start[r0] != 0) return 1;
          for (int64_t r = r0 + 1; r < r1; r++)
            if (run_start[r] <= run_start[r - 1] || run_start[r] >= L) return 1;
          for (int64_t r = r0; r < r1; r++)
            if (run_origin[r] > 1) return 2;
        }
        return 0;
      };
      int bad = 0;
      constexpr int64_t kCheckChunk = 4096;  // (a pool dispatch costs more than 16k entries' checks)
      if (n >= 16 * kCheckChunk) {
        std::atomic<int> worst{0};
        tms::parallel_for((n + kCheckChunk - 1) / kCheckChunk, [&](int64_t c) {
          const int r = check_runs(c * kCheckChunk, std::min(n, (c + 1) * kCheckChunk));
          if (r) worst.store(r);
        });
        bad = worst.load();
      } else {
        bad = check_runs(0, n);
      }
      if (bad == 1) fail(TM_EINVAL, "tokens, origins, versions must be parallel");
      if (bad == 2) fail(TM_EINVAL, "bad origin");
    }
    const int64_t nchains = (int64_t)chain_tokens.size();
    tr.mark("validate+chains");
    std::vector<int64_t> chain_beg(nchains + 1, 0);
    for (int64_t c = 0; c < nchains; c++) chain_beg[c + 1] = chain_beg[c] + chain_len[c];
    std::vector<int64_t> perm(n);  // position in chain order -> batch index
    {
      std::vector<int64_t> cur(chain_beg.begin(), chain_beg.end() - 1);
      for (int64_t k = 0; k < n; k++) perm[cur[chain_idx[k]]++] = k;
    }
    std::vector<int64_t> order(nchains);
    for (int64_t c = 0; c < nchains; c++) order[c] = c;
    bool ordered = true;  // already longest-first (e.g. equal chains): no sort
    for (int64_t c = 1; c < nchains && ordered; c++) ordered = chain_tokens[c - 1] >= chain_tokens[c];
    if (!ordered)
      std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return chain_tokens[x] > chain_tokens[y]; });
    // ---- capacity (upper bounds); every entry reserves a row id (batch order): holes left by
    // earlier re-recorded sequences first, then fresh ids
    const int64_t row_base = (int64_t)s->rows.size();
    std::vector<int64_t> reserved(n);
    const int64_t n_reuse = std::min<int64_t>(n, (int64_t)s->free_rows.size());
    for (int64_t e = 0; e < n_reuse; e++) reserved[e] = s->free_rows[s->free_rows.size() - 1 - e];
    s->free_rows.resize(s->free_rows.size() - n_reuse);
    for (int64_t e = n_reuse; e < n; e++) reserved[e] = row_base + (e - n_reuse);
    const int64_t n_fresh = n - n_reuse;
    ensure_arena(s, s->arena_used + words_upper);
    ensure_rows(s, row_base + n_fresh);
    ensure_runs(s, s->n_runs + total_runs);
    ensure_table(s, s->n_real_rows + n);
    tr.mark("validate+capacity");
    wait_prev(s, s->stream);
    if (mem == TM_MEM_DEVICE && stream && (cudaStream_t)stream != s->stream) {  // order after the producer
      cudaEvent_t ev;
      ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
      ck(cudaEventRecord(ev, (cudaStream_t)stream), "event");
      ck(cudaStreamWaitEvent(s->stream, ev, 0), "wait");
      cudaEventDestroy(ev);
    }
    // ---- stage tokens and per-entry arrays (chain order).  Small host batches (the per-request
    // lpm_insert path) carry their tokens inside the batch staging: one H2D for everything,
    // and a single-CTA copy kernel snapshots the counters next to the results: one D2H.
    std::vector<int64_t> doff;
    const int32_t *tok_base = nullptr;
    int64_t small_words = 0;
    if (mem == TM_MEM_HOST && n <= 256) {
      for (int64_t k = 0; k < n; k++) small_words += round_up(std::max<int64_t>(tok_len[k], 1), tms::kAlignWords);
      if (small_words > (int64_t(1) << 18) || use_packed(s, small_words)) small_words = 0;
    }
    const bool small = small_words > 0;
    if (mem == TM_MEM_DEVICE) {  // tokens already in HBM (e.g. produced by the engine)
      doff.resize(n);
      for (int64_t k = 0; k < n; k++) doff[k] = tok_off[perm[k]];
      tok_base = tokens;
    } else if (!small) {
      stage_tokens(s, n, tokens, tok_off, tok_len, doff, &perm, s->stream);
      tok_base = (const int32_t *)s->dtok.p;
    }
    Layout lay;
    size_t o_sid = lay.add(4 * n), o_off = lay.add(8 * n), o_len = lay.add(8 * n), o_roff = lay.add(8 * (n + 1)),
           o_rs = lay.add(4 * total_runs), o_ro = lay.add(total_runs), o_rv = lay.add(4 * total_runs),
           o_tok = lay.add(4 * (size_t)(small_words + tms::kAlignWords)),
           o_crow = lay.add(8 * n), o_chains = lay.add(24 * nchains), o_work = lay.add(16);
    size_t in_bytes = lay.bytes;
    size_t o_m = lay.add(8 * n), o_par = lay.add(8 * n), o_dup = lay.add(8 * n), o_tn = lay.add(4 * n),
           o_sp = lay.add(4 * n), o_cloc = lay.add(4 * n), o_ctr = lay.add(8 * 4);
    size_t out_end = lay.bytes;
    size_t o_cvb = lay.add(8 * n), o_cr0 = lay.add(8 * n), o_cfr = lay.add(4 * n);
    char *h = (char *)s->pin.need(lay.bytes);
    char *d = (char *)s->scratch.need(lay.bytes);
    if (small) {
      doff.resize(n);
      int32_t *ht = (int32_t *)(h + o_tok);
      int64_t w = 0;
      for (int64_t k = 0; k < n; k++) {
        const int64_t e = perm[k], L = tok_len[e], P = round_up(std::max<int64_t>(L, 1), tms::kAlignWords);
        doff[k] = w;
        memcpy(ht + w, tokens + tok_off[e], 4 * (size_t)L);
        memset(ht + w + L, 0, 4 * (size_t)(P - L));
        w += P;
      }
      tok_base = (const int32_t *)(d + o_tok);
      s->c_raw_calls++;
      s->c_raw_tokens += small_words;
      s->c_h2d_bytes += 4 * small_words;
    }
    int32_t *h_sid = (int32_t *)(h + o_sid);
    int64_t *h_off = (int64_t *)(h + o_off), *h_len = (int64_t *)(h + o_len), *h_roff = (int64_t *)(h + o_roff);
    int64_t *h_crow = (int64_t *)(h + o_crow);
    int32_t *h_rs = (int32_t *)(h + o_rs), *h_rv = (int32_t *)(h + o_rv);
    uint8_t *h_ro = (uint8_t *)(h + o_ro);
    // per-entry staging in chain order; the run offsets first (a prefix sum), then the
    // entries - spread over the host pool for large batches
    h_roff[0] = 0;
    for (int64_t k = 0; k < n; k++) h_roff[k + 1] = h_roff[k] + (run_off[perm[k] + 1] - run_off[perm[k]]);
    std::atomic<int64_t> qend_a{0};  // end of the query words (debug bounds of in-flight rows)
    auto stage_range = [&](int64_t k0, int64_t k1) {
      int64_t lq = 0;
      for (int64_t k = k0; k < k1; k++) {
        const int64_t e = perm[k], rr = h_roff[k];
        lq = std::max<int64_t>(lq, doff[k] + round_up(tok_len[e], 4));
        h_sid[k] = sids[e];
        h_off[k] = doff[k];
        h_len[k] = tok_len[e];
        h_crow[k] = reserved[e];  // reserved id (batch order)
        const int64_t r0 = run_off[e], r1 = run_off[e + 1];
        memcpy(h_rs + rr, run_start + r0, 4 * (r1 - r0));
        memcpy(h_ro + rr, run_origin + r0, (r1 - r0));
        memcpy(h_rv + rr, run_version + r0, 4 * (r1 - r0));
      }
      int64_t cur = qend_a.load(std::memory_order_relaxed);
      while (lq > cur && !qend_a.compare_exchange_weak(cur, lq)) {
      }
    };
    constexpr int64_t kStageChunk = 1024;
    if (n >= 4 * kStageChunk) {
      tms::parallel_for((n + kStageChunk - 1) / kStageChunk,
                        [&](int64_t c) { stage_range(c * kStageChunk, std::min(n, (c + 1) * kStageChunk)); });
    } else {
      stage_range(0, n);
    }
    memset(h + o_work, 0, 16);  // the launch's chain counter and CTAs-done counter start at zero
    {  // chains in processing order: first entry, end, session
      int64_t *hc = (int64_t *)(h + o_chains);
      for (int64_t it = 0; it < nchains; it++) {
        const int64_t c = order[it];
        hc[3 * it] = chain_beg[c];
        hc[3 * it + 1] = chain_beg[c + 1];
        hc[3 * it + 2] = sids[perm[chain_beg[c]]];
      }
    }
    tr.mark("stage");
    ck(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, s->stream), "H2D batch");
    tr.mark("h2d");
    bool direct_out = false;
    {
      tms::RecordArgs ra{};
      Batch &b = ra.b;
      b.n = n;
      b.sids = (const int32_t *)(d + o_sid);
      b.tok = tok_base;
      b.off = (const int64_t *)(d + o_off);
      b.len = (const int64_t *)(d + o_len);
      b.o_m = (int64_t *)(d + o_m);
      b.o_parent = (int64_t *)(d + o_par);
      b.o_dup = (int64_t *)(d + o_dup);
      b.o_tnext = (int32_t *)(d + o_tn);
      b.o_spar = (int32_t *)(d + o_sp);
      b.run_off = (const int64_t *)(d + o_roff);
      b.run_start = (const int32_t *)(d + o_rs);
      b.run_origin = (const uint8_t *)(d + o_ro);
      b.run_version = (const int32_t *)(d + o_rv);
      b.c_row = (int64_t *)(d + o_crow);
      b.c_vb = (int64_t *)(d + o_cvb);
      b.c_run0 = (int64_t *)(d + o_cr0);
      b.c_firstrun = (int32_t *)(d + o_cfr);
      b.c_local = (int32_t *)(d + o_cloc);
      ra.chains = (const int64_t *)(d + o_chains);
      ra.ctr_out = (int64_t *)(d + o_ctr);  // the last CTA out snapshots the counters beside the results
      ra.nchains = nchains;
      ra.work = (unsigned long long *)(d + o_work);
      ra.c0_e1 = -1;
      ra.out_dst = nullptr;
      if (small) {  // results come back through the kernel's own stores into the pinned staging
        void *hd = nullptr;
        if (cudaHostGetDevicePointer(&hd, h + o_crow, 0) == cudaSuccess && hd && (o_crow % 16) == 0 &&
            (out_end - o_crow) % 16 == 0) {
          ra.out_src = (const int4 *)(d + o_crow);
          ra.out_dst = (int4 *)hd;
          ra.out_len = (int64_t)(out_end - o_crow) / 16;
        }
        cudaGetLastError();
      }
      if (nchains == 1 && mem == TM_MEM_HOST) {  // one session (e.g. lpm_insert): chain 0 as parameters
        const int64_t e = perm[0];
        ra.c0_e1 = n;
        ra.c0_sid = sids[e];
        ra.c0_off = doff[0];
        ra.c0_len = (int32_t)tok_len[e];
        ra.c0_q0 = tokens[tok_off[e]];
      }
      tms::DevView dv = s->v;  // rows committed in the launch live in the query buffer until the copy
      const int64_t qend = qend_a.load();
      dv.qv_lo = (int64_t)(tok_base - s->v.arena);
      dv.qv_hi = dv.qv_lo + qend;
      direct_out = ra.out_dst != nullptr;
      int copy_warp = 0;
      ProfScope ps(s, 1, s->stream);
      ck(tms::launch_record(dv, ra, s->num_sms, s->stream, &copy_warp), "record");
      tr.mark("launch");
    }
    // ---- results back (chain order), into the host mirror in batch order
    if (!direct_out)
      ck(cudaMemcpyAsync(h + o_crow, d + o_crow, out_end - o_crow, cudaMemcpyDeviceToHost, s->stream), "D2H results");
    mark_done(s, s->stream);
    tr.mark("d2h+event");
    // the mirror's new slots are laid out while the GPU records
    s->rows.resize(row_base + n_fresh, RowHost{-1, -1, -1, 0, 0, 0, -1, -1});
    tr.mark("mirror-slots");
    ck(cudaStreamSynchronize(s->stream), "record sync");
    tr.mark("sync");
    const int64_t *ctr = (const int64_t *)(h + o_ctr);
    if (ctr[3]) raise_device_error(ctr[3]);
    const int64_t *r_m = (const int64_t *)(h + o_m), *r_par = (const int64_t *)(h + o_par),
                  *r_dup = (const int64_t *)(h + o_dup), *r_row = (const int64_t *)(h + o_crow);
    const int32_t *r_tn = (const int32_t *)(h + o_tn), *r_sp = (const int32_t *)(h + o_sp),
                  *r_loc = (const int32_t *)(h + o_cloc);
    // The host mirror, chain by chain (a chain is one session's entries in batch order).
    struct MirrorAcc {
      int64_t real = 0, maxd = 0;
      std::vector<int64_t> holes;
      bool bad_row = false, bad_ord = false;
    };
    auto mirror_chain = [&](int64_t c, MirrorAcc &acc) {
      for (int64_t k = chain_beg[c]; k < chain_beg[c + 1]; k++) {
        const int64_t e = perm[k];
        const int32_t sid = sids[e];
        const int64_t L = tok_len[e], m = r_m[k], row = r_row[k], par = r_par[k];
        if (r_dup[k] < 0) {
          if (row != reserved[e]) acc.bad_row = true;
          RowHost rh{sid, r_loc[k], par, (int32_t)m, (int32_t)L, 0, r_tn[k], r_sp[k]};
          rh.depth = par >= 0 ? s->rows[par].depth + 1 : 0;
          acc.maxd = std::max<int64_t>(acc.maxd, rh.depth);
          s->sess_maxdepth[sid] = std::max(s->sess_maxdepth[sid], rh.depth);
          s->rows[row] = rh;
          if (r_loc[k] != (int32_t)s->sess_rows[sid].size()) acc.bad_ord = true;
          s->sess_rows[sid].push_back(row);
          s->sess_stored[sid] += L - m;
          acc.real++;
        } else {
          acc.holes.push_back(reserved[e]);  // the reserved slot stayed empty: reuse it
        }
        s->sess_naive[sid] += L;
        if (out_matched) out_matched[e] = m;
        if (out_row) out_row[e] = row;
        if (out_local) out_local[e] = r_loc[k];
        if (out_parent) out_parent[e] = par;
        if (out_parent_local) out_parent_local[e] = par >= 0 ? s->rows[par].local : -1;
        if (out_added) out_added[e] = r_dup[k] < 0 ? L - m : 0;
      }
    };
    // chains touch disjoint sessions, rows and outputs: large batches spread over the host
    // pool (the row slots were faulted in ahead, see ensure_rows)
    constexpr int64_t kMirrorEntries = 1024;  // entries per pool work item (whole chains)
    std::vector<MirrorAcc> accs(1);
    if (n >= 4 * kMirrorEntries && nchains > 1) {
      std::vector<int64_t> cut{0};
      for (int64_t c = 0; c < nchains; c++)
        if (chain_beg[c + 1] - chain_beg[cut.back()] >= kMirrorEntries || c + 1 == nchains) cut.push_back(c + 1);
      const int64_t nck = (int64_t)cut.size() - 1;
      accs.resize((size_t)nck);
      tms::parallel_for(nck, [&](int64_t k) {
        for (int64_t c = cut[k]; c < cut[k + 1]; c++) mirror_chain(c, accs[k]);
      });
    } else {
      for (int64_t c = 0; c < nchains; c++) mirror_chain(c, accs[0]);
    }
    for (const MirrorAcc &acc : accs) {
      if (acc.bad_row) fail(TM_ECUDA, "row numbering out of sync");
      if (acc.bad_ord) fail(TM_ECUDA, "session ordinal out of sync");
      s->n_real_rows += acc.real;
      s->max_depth = std::max<int64_t>(s->max_depth, acc.maxd);
      s->free_rows.insert(s->free_rows.end(), acc.holes.begin(), acc.holes.end());
    }
    tr.mark("mirror");
    s->arena_used = ctr[0];
    s->n_runs = ctr[2];
    s->c_record_calls++;
    s->c_records += n;
    for (int64_t e = 0; e < n; e++) s->c_record_tokens += tok_len[e];
  });
}

int tm_record_one(tm_store *s, int32_t sid, const int32_t *tokens, int64_t ntok, const int32_t *run_start,
                  const uint8_t *run_origin, const int32_t *run_version, int64_t nruns, int64_t *out6) {
  const int64_t off = 0, run_off[2] = {0, nruns};
  int64_t m = 0, row = 0, par = 0, added = 0;
  int32_t local = 0, par_local = 0;
  const int rc = tm_record_batch(s, 1, TM_MEM_HOST, &sid, tokens, &off, &ntok, run_off, run_start, run_origin,
                                 run_version, &m, &row, &local, &par, &par_local, &added, nullptr);
  if (rc == TM_OK && out6) {
    const int64_t o[6] = {m, row, local, par, par_local, added};
    memcpy(out6, o, sizeof(o));
  }
  return rc;
}

int tm_match_batch(tm_store *s, int64_t n, int32_t mem, const int32_t *sids, const int32_t *tokens,
                   const int64_t *tok_off, const int64_t *tok_len, int64_t *out_matched, int64_t *out_parent,
                   int64_t *out_dup, void *stream) {
  NvtxRange nvtx_("tm_match_batch");
  return guarded(s, [&] {
    if (n < 0) fail(TM_EINVAL, "negative batch size");
    if (n == 0) return;
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    const bool dev = mem == TM_MEM_DEVICE;
    s->c_match_calls++;
    s->c_queries += n;
    tm_store::MatchSlot *slot = nullptr;
    if (dev) {  // read-only, device buffers: may overlap other device matches, not mutations
      slot = &s->slots[s->next_slot++ % tm_store::kSlots];
      ck(cudaStreamWaitEvent(st, s->last, 0), "cudaStreamWaitEvent");
      if (slot->used) ck(cudaStreamWaitEvent(st, slot->done, 0), "cudaStreamWaitEvent");
    } else {
      wait_prev(s, st);
    }
    Layout lay;
    size_t o_sid = lay.add(4 * n), o_off = lay.add(8 * n), o_len = lay.add(8 * n);
    size_t in_bytes = lay.bytes;
    size_t o_m = lay.add(8 * n), o_par = lay.add(8 * n), o_dup = lay.add(8 * n);
    size_t out_end = lay.bytes;
    size_t o_root = lay.add(8 * n), o_plan = lay.add(4 * (size_t)tms::plan_items_ints(n));
    char *d = (char *)(dev ? slot->scratch : s->scratch).need(lay.bytes);
    Batch b{};
    b.n = n;
    b.sched = dev ? slot->sched : s->sched;
    if (mem == TM_MEM_HOST) {
      for (int64_t k = 0; k < n; k++)
        if (sids[k] < 0 || sids[k] >= s->n_sess) fail(TM_ENOENT, "unknown session " + std::to_string(sids[k]));
      std::vector<int64_t> doff;
      stage_tokens(s, n, tokens, tok_off, tok_len, doff, nullptr, st);
      char *h = (char *)s->pin.need(lay.bytes);
      memcpy(h + o_sid, sids, 4 * n);
      memcpy(h + o_off, doff.data(), 8 * n);
      memcpy(h + o_len, tok_len, 8 * n);
      ck(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, st), "H2D batch");
      s->pin.mark(st);
      b.sids = (const int32_t *)(d + o_sid);
      b.tok = (const int32_t *)s->dtok.p;
      b.off = (const int64_t *)(d + o_off);
      b.len = (const int64_t *)(d + o_len);
      b.o_m = (int64_t *)(d + o_m);
      b.o_parent = (int64_t *)(d + o_par);
      b.o_dup = (int64_t *)(d + o_dup);
    } else if (mem == TM_MEM_DEVICE) {
      b.sids = sids;
      b.tok = tokens;
      b.off = tok_off;
      b.len = tok_len;
      b.o_m = out_matched;
      b.o_parent = out_parent;
      b.o_dup = out_dup;
    } else {
      fail(TM_EINVAL, "bad memory kind");
    }
    if (n >= s->plan_min) {
      ProfScope ps(s, 3, st);
      ck(tms::launch_plan(s->v, b, s->plan_roots ? (int64_t *)(d + o_root) : nullptr, (int *)(d + o_plan), st),
         "plan");
    }
    {
      ProfScope ps(s, 0, st);
      ck(tms::launch_walk(s->v, b, s->num_sms, st), "walk");
    }
    if (mem == TM_MEM_HOST) {
      char *h = (char *)s->pin.need(lay.bytes);
      ck(cudaMemcpyAsync(h + o_m, d + o_m, out_end - o_m, cudaMemcpyDeviceToHost, st), "D2H");
      enqueue_ctr_readback(s, st);
      mark_done(s, st);
      ck(cudaStreamSynchronize(st), "match sync");
      check_ctr_error(s);
      memcpy(out_matched, h + o_m, 8 * n);
      if (out_parent) memcpy(out_parent, h + o_par, 8 * n);
      if (out_dup) memcpy(out_dup, h + o_dup, 8 * n);
    } else {
      ck(cudaEventRecord(slot->done, st), "cudaEventRecord");
      slot->used = true;
    }
  });
}

int tm_rows_total(tm_store *s, int64_t n, const int64_t *rows, int64_t *out_total) {
  return guarded(s, [&] {
    int64_t t = 0;
    for (int64_t k = 0; k < n; k++) {
      if (!valid_row(s, rows[k])) fail(TM_ENOENT, "node " + std::to_string(rows[k]) + " not in store");
      t += s->rows[rows[k]].len;
    }
    *out_total = t;
  });
}

int tm_export_rows(tm_store *s, int64_t n, const int64_t *rows, int32_t mem_out, int64_t *out_offsets,
                   int32_t *out_tokens, uint8_t *out_mask, int32_t *out_versions, int64_t *out_resp_start,
                   void *stream) {
  NvtxRange nvtx_("tm_export_rows");
  return guarded(s, [&] {
    if (n < 0) fail(TM_EINVAL, "negative batch size");
    if (mem_out != TM_MEM_HOST && mem_out != TM_MEM_DEVICE) fail(TM_EINVAL, "bad memory kind");
    out_offsets[0] = 0;
    if (n == 0) return;
    const int64_t T = tms::export_tile_tokens();
    std::vector<int64_t> tile(n + 1);
    tile[0] = 0;
    for (int64_t k = 0; k < n; k++) {
      if (!valid_row(s, rows[k])) fail(TM_ENOENT, "node " + std::to_string(rows[k]) + " not in store");
      int64_t L = s->rows[rows[k]].len;
      out_offsets[k + 1] = out_offsets[k] + L;
      tile[k + 1] = tile[k] + (L + T - 1) / T;
    }
    const int64_t total = out_offsets[n];
    s->c_export_calls++;
    s->c_export_rows += n;
    s->c_export_tokens += total;
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    wait_prev(s, st);
    Layout lay;
    size_t o_rows = lay.add(8 * n), o_off = lay.add(8 * (n + 1)), o_tile = lay.add(8 * (n + 1));
    size_t in_bytes = lay.bytes;
    size_t o_tok = 0, o_msk = 0, o_ver = 0, o_resp = 0;
    const int64_t ntiles_all = tile[n];
    size_t o_plan = lay.add((size_t)tms::export_plan_bytes(ntiles_all));
    if (mem_out == TM_MEM_HOST) {
      o_tok = lay.add(4 * total);
      o_msk = lay.add(total);
      o_ver = lay.add(4 * total);
      o_resp = lay.add(8 * n);
    }
    // small host exports come back in ONE copy through the pinned staging (the outputs
    // are contiguous in the layout) and one sync; large ones stream through d2h_pageable
    const bool small_host = mem_out == TM_MEM_HOST && lay.bytes - o_tok <= (size_t(8) << 20);
    char *d = (char *)s->scratch.need(lay.bytes);
    char *h = (char *)s->pin.need(small_host ? lay.bytes : in_bytes);
    memcpy(h + o_rows, rows, 8 * n);
    memcpy(h + o_off, out_offsets, 8 * (n + 1));
    memcpy(h + o_tile, tile.data(), 8 * (n + 1));
    ck(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, st), "H2D export plan");
    s->pin.mark(st);
    tms::ExportArgsHost e{};
    e.n = n;
    e.rows = (const int64_t *)(d + o_rows);
    e.out_off = (const int64_t *)(d + o_off);
    e.tile_off = (const int64_t *)(d + o_tile);
    e.ntiles = tile[n];
    e.plan = d + o_plan;
    if (mem_out == TM_MEM_HOST) {
      e.tokens = (int32_t *)(d + o_tok);
      e.mask = (uint8_t *)(d + o_msk);
      e.versions = (int32_t *)(d + o_ver);
      e.resp = (int64_t *)(d + o_resp);
    } else {
      e.tokens = out_tokens;
      e.mask = out_mask;
      e.versions = out_versions;
      e.resp = out_resp_start;
    }
    // e.resp is zeroed by the export planner (no memset call)
    {
      ProfScope ps(s, 2, st);
      ck(tms::launch_export(s->v, e, s->num_sms, st), "export");
    }
    if (small_host) {
      ck(cudaMemcpyAsync(h + o_tok, d + o_tok, lay.bytes - o_tok, cudaMemcpyDeviceToHost, st), "D2H export");
      enqueue_ctr_readback(s, st);
      mark_done(s, st);
      ck(cudaStreamSynchronize(st), "export sync");
      check_ctr_error(s);
      if (out_tokens) memcpy(out_tokens, h + o_tok, 4 * (size_t)total);
      if (out_mask) memcpy(out_mask, h + o_msk, (size_t)total);
      if (out_versions) memcpy(out_versions, h + o_ver, 4 * (size_t)total);
      if (out_resp_start) memcpy(out_resp_start, h + o_resp, 8 * (size_t)n);
    } else if (mem_out == TM_MEM_HOST) {
      if (out_tokens) d2h_pageable(s, out_tokens, e.tokens, 4 * total, st);
      if (out_mask) d2h_pageable(s, out_mask, e.mask, total, st);
      if (out_versions) d2h_pageable(s, out_versions, e.versions, 4 * total, st);
      if (out_resp_start) ck(cudaMemcpyAsync(out_resp_start, e.resp, 8 * n, cudaMemcpyDeviceToHost, st), "D2H resp");
      enqueue_ctr_readback(s, st);
      mark_done(s, st);
      ck(cudaStreamSynchronize(st), "export sync");
      check_ctr_error(s);
    } else {
      mark_done(s, st);
    }
  });
}

int tm_export_host_rows(tm_store *s, int64_t n, const int32_t *tokens, const int64_t *tok_off,
                        const int64_t *n_input, const int32_t *ctx_version, const int64_t *run_off,
                        const int32_t *run_start, const int32_t *run_version, const int64_t *out_off,
                        int32_t *out_tokens, uint8_t *out_mask, int32_t *out_versions, int64_t *out_resp_start,
                        void *stream) {
  NvtxRange nvtx_("tm_export_host_rows");
  return guarded(s, [&] {
    if (n < 0) fail(TM_EINVAL, "negative batch size");
    if (n == 0) return;
    if (!out_tokens || !out_mask || !out_versions) fail(TM_EINVAL, "device output arrays required");
    const int64_t total = tok_off[n] - tok_off[0];
    for (int64_t k = 0; k < n; k++) {
      const int64_t L = tok_off[k + 1] - tok_off[k];
      if (L < 0 || n_input[k] < 0 || n_input[k] > L) fail(TM_EINVAL, "bad row extent");
      const int64_t r0 = run_off[k], r1 = run_off[k + 1];
      if (L > n_input[k] && (r1 <= r0 || run_start[r0] != n_input[k]))
        fail(TM_EINVAL, "tokens, origins, versions must be parallel");
      for (int64_t r = r0 + 1; r < r1; r++)
        if (run_start[r] <= run_start[r - 1] || run_start[r] >= L) fail(TM_EINVAL, "tokens, origins, versions must be parallel");
    }
    const int64_t nruns = run_off[n] - run_off[0];
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    wait_prev(s, st);
    Layout lay;
    size_t o_tok = lay.add(4 * (size_t)std::max<int64_t>(total, 1)), o_toff = lay.add(8 * (n + 1)),
           o_nin = lay.add(8 * n), o_cv = lay.add(4 * n), o_roff = lay.add(8 * (n + 1)),
           o_rs = lay.add(4 * (size_t)std::max<int64_t>(nruns, 1)), o_rv = lay.add(4 * (size_t)std::max<int64_t>(nruns, 1)),
           o_out = lay.add(8 * n);
    char *h = (char *)s->pin.need(lay.bytes);
    char *d = (char *)s->scratch.need(lay.bytes);
    memcpy(h + o_tok, tokens + tok_off[0], 4 * (size_t)total);
    int64_t *h_toff = (int64_t *)(h + o_toff), *h_roff = (int64_t *)(h + o_roff);
    for (int64_t k = 0; k <= n; k++) {
      h_toff[k] = tok_off[k] - tok_off[0];
      h_roff[k] = run_off[k] - run_off[0];
    }
    memcpy(h + o_nin, n_input, 8 * n);
    memcpy(h + o_cv, ctx_version, 4 * n);
    memcpy(h + o_rs, run_start + run_off[0], 4 * (size_t)nruns);
    memcpy(h + o_rv, run_version + run_off[0], 4 * (size_t)nruns);
    memcpy(h + o_out, out_off, 8 * n);
    ck(cudaMemcpyAsync(d, h, lay.bytes, cudaMemcpyHostToDevice, st), "H2D host rows");
    s->pin.mark(st);
    tms::HostRowsArgs a{};
    a.n = n;
    a.src = (const int32_t *)(d + o_tok);
    a.tok_off = (const int64_t *)(d + o_toff);
    a.n_input = (const int64_t *)(d + o_nin);
    a.ctx_version = (const int32_t *)(d + o_cv);
    a.run_off = (const int64_t *)(d + o_roff);
    a.run_start = (const int32_t *)(d + o_rs);
    a.run_version = (const int32_t *)(d + o_rv);
    a.out_off = (const int64_t *)(d + o_out);
    a.tokens = out_tokens;
    a.mask = out_mask;
    a.versions = out_versions;
    a.resp = out_resp_start;
    {
      ProfScope ps(s, 2, st);
      ck(tms::launch_fill_host_rows(a, s->num_sms, st), "fill host rows");
    }
    mark_done(s, st);
    s->c_export_calls++;
    s->c_export_rows += n;
    s->c_export_tokens += total;
  });
}

int tm_export_ndjson(tm_store *s, int64_t n, const int64_t *rows, const char *sid_json, const int64_t *sid_off,
                     int32_t mem_out, char *out, int64_t cap, int64_t *out_bytes, void *stream) {
  NvtxRange nvtx_("tm_export_ndjson");
  return guarded(s, [&] {
    if (n < 0) fail(TM_EINVAL, "negative batch size");
    if (mem_out != TM_MEM_HOST && mem_out != TM_MEM_DEVICE) fail(TM_EINVAL, "bad memory kind");
    *out_bytes = 0;
    if (n == 0) return;
    const int64_t T = tms::export_tile_tokens();
    std::vector<int64_t> off(n + 1), tile(n + 1);
    off[0] = tile[0] = 0;
    for (int64_t k = 0; k < n; k++) {
      if (!valid_row(s, rows[k])) fail(TM_ENOENT, "node " + std::to_string(rows[k]) + " not in store");
      const int64_t L = s->rows[rows[k]].len;
      off[k + 1] = off[k] + L;
      tile[k + 1] = tile[k] + (L + T - 1) / T;
    }
    const int64_t total = off[n], ntiles = tile[n];
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    wait_prev(s, st);
    Layout lay;
    size_t o_rows = lay.add(8 * n), o_off = lay.add(8 * (n + 1)), o_tile = lay.add(8 * (n + 1));
    size_t in_bytes = lay.bytes;
    size_t o_tok = lay.add(4 * total), o_msk = lay.add(total), o_ver = lay.add(4 * total), o_sums = lay.add(16 * ntiles),
           o_toff = lay.add(24 * ntiles), o_roff = lay.add(32 * (n + 1)), o_sidoff = lay.add(8 * (n + 1)),
           o_sid = lay.add((size_t)sid_off[n]), o_plan = lay.add((size_t)tms::export_plan_bytes(ntiles));
    char *d = (char *)s->scratch.need(lay.bytes);
    char *h = (char *)s->pin.need(std::max(in_bytes, (size_t)16 * ntiles));
    memcpy(h + o_rows, rows, 8 * n);
    memcpy(h + o_off, off.data(), 8 * (n + 1));
    memcpy(h + o_tile, tile.data(), 8 * (n + 1));
    ck(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, st), "H2D ndjson plan");
    s->pin.mark(st);
    tms::ExportArgsHost e{};
    e.n = n;
    e.rows = (const int64_t *)(d + o_rows);
    e.out_off = (const int64_t *)(d + o_off);
    e.tile_off = (const int64_t *)(d + o_tile);
    e.ntiles = ntiles;
    e.tokens = (int32_t *)(d + o_tok);
    e.mask = (uint8_t *)(d + o_msk);
    e.versions = (int32_t *)(d + o_ver);
    e.resp = nullptr;
    e.plan = d + o_plan;
    {
      ProfScope ps(s, 2, st);
      ck(tms::launch_export(s->v, e, s->num_sms, st), "export");
    }
    tms::JsonArgsHost j{};
    j.n = n;
    j.out_off = e.out_off;
    j.tile_off = e.tile_off;
    j.ntiles = ntiles;
    j.tokens = e.tokens;
    j.mask = e.mask;
    j.versions = e.versions;
    j.sums = (int64_t *)(d + o_sums);
    ck(tms::launch_json(j, 1, s->num_sms, st), "json pass 1");
    std::vector<int64_t> sums(2 * ntiles);
    ck(cudaMemcpyAsync(h, j.sums, 16 * ntiles, cudaMemcpyDeviceToHost, st), "D2H json sums");
    ck(cudaStreamSynchronize(st), "json sync");
    memcpy(sums.data(), h, 16 * ntiles);
    // byte layout of every row and tile
    std::vector<int64_t> toff(3 * ntiles), roff(4 * (n + 1));
    int64_t pos = 0;
    for (int64_t i = 0; i < n; i++) {
      const int64_t L = off[i + 1] - off[i], kl = sid_off[i + 1] - sid_off[i];
      int64_t ts_sum = 0, vs_sum = 0;
      for (int64_t t2 = tile[i]; t2 < tile[i + 1]; t2++) { ts_sum += sums[2 * t2]; vs_sum += sums[2 * t2 + 1]; }
      const int64_t r0 = pos, ts = r0 + 14 + kl + 11, ms = ts + ts_sum + L - 1 + 15, vs = ms + 2 * L - 1 + 14;
      roff[4 * i] = r0; roff[4 * i + 1] = ts; roff[4 * i + 2] = ms; roff[4 * i + 3] = vs;
      int64_t at = ts, av = vs;
      for (int64_t t2 = tile[i]; t2 < tile[i + 1]; t2++) {
        const int64_t a = (t2 - tile[i]) * T, cnt = std::min(T, L - a);
        toff[3 * t2] = at; toff[3 * t2 + 1] = ms + 2 * a; toff[3 * t2 + 2] = av;
        at += sums[2 * t2] + cnt;
        av += sums[2 * t2 + 1] + cnt;
      }
      pos = vs + vs_sum + L - 1 + 3;
    }
    roff[4 * n] = pos;
    *out_bytes = pos;
    if (!out || cap < pos) { mark_done(s, st); return; }  // size query
    char *h2 = (char *)s->pin.need(24 * ntiles + 32 * (n + 1) + 8 * (n + 1) + sid_off[n] + 1024);
    size_t a0 = 0, a1 = (24 * ntiles + 255) / 256 * 256, a2 = a1 + (32 * (n + 1) + 255) / 256 * 256,
           a3 = a2 + (8 * (n + 1) + 255) / 256 * 256;
    memcpy(h2 + a0, toff.data(), 24 * ntiles);
    memcpy(h2 + a1, roff.data(), 32 * (n + 1));
    memcpy(h2 + a2, sid_off, 8 * (n + 1));
    memcpy(h2 + a3, sid_json, sid_off[n]);
    ck(cudaMemcpyAsync(d + o_toff, h2 + a0, 24 * ntiles, cudaMemcpyHostToDevice, st), "H2D json");
    ck(cudaMemcpyAsync(d + o_roff, h2 + a1, 32 * (n + 1), cudaMemcpyHostToDevice, st), "H2D json");
    ck(cudaMemcpyAsync(d + o_sidoff, h2 + a2, 8 * (n + 1), cudaMemcpyHostToDevice, st), "H2D json");
    if (sid_off[n]) ck(cudaMemcpyAsync(d + o_sid, h2 + a3, sid_off[n], cudaMemcpyHostToDevice, st), "H2D json");
    char *text = (char *)s->dtok.need((size_t)pos);  // token staging doubles as the text buffer here
    j.toff = (const int64_t *)(d + o_toff);
    j.roff = (const int64_t *)(d + o_roff);
    j.sid = (const char *)(d + o_sid);
    j.sid_off = (const int64_t *)(d + o_sidoff);
    j.out = mem_out == TM_MEM_DEVICE ? out : text;
    ck(tms::launch_json(j, 2, s->num_sms, st), "json pass 2");
    if (mem_out == TM_MEM_HOST) d2h_pageable(s, out, text, pos, st);
    mark_done(s, st);
    ck(cudaStreamSynchronize(st), "json sync");
  });
}

int tm_session_stats(tm_store *s, int32_t sid, int64_t *stored, int64_t *naive, int64_t *nrows) {
  return guarded(s, [&] {
    if (sid < 0 || sid >= s->n_sess) fail(TM_ENOENT, "unknown session " + std::to_string(sid));
    if (stored) *stored = s->sess_stored[sid];
    if (naive) *naive = s->sess_naive[sid];
    if (nrows) *nrows = (int64_t)s->sess_rows[sid].size();
  });
}

int tm_session_rows(tm_store *s, int32_t sid, int32_t order, int64_t *out_rows, int64_t cap, int64_t *n_out) {
  return guarded(s, [&] {
    if (sid < 0 || sid >= s->n_sess) fail(TM_ENOENT, "unknown session " + std::to_string(sid));
    const auto &rs = s->sess_rows[sid];
    *n_out = (int64_t)rs.size();
    if (order == TM_ORDER_INSERT) {
      for (int64_t k = 0; k < (int64_t)rs.size() && k < cap; k++) out_rows[k] = rs[k];
      return;
    }
    if (order != TM_ORDER_LEX) fail(TM_EINVAL, "bad order");
    // children lists indexed by session-local ordinal; root rows hang off a virtual root
    const int64_t nr = (int64_t)rs.size();
    std::vector<std::vector<int64_t>> kids_local(nr);
    std::vector<int64_t> roots;
    for (int64_t k = 0; k < nr; k++) {
      const RowHost &R = s->rows[rs[k]];
      if (R.parent < 0) roots.push_back(rs[k]);
      else kids_local[s->rows[R.parent].local].push_back(rs[k]);
    }
    auto cmp = [&](int64_t a, int64_t b) {
      const RowHost &A = s->rows[a], &B = s->rows[b];
      if (A.m != B.m) return A.m < B.m;
      bool pa = A.len == A.m, pb = B.len == B.m;
      if (pa != pb) return pa;
      return A.tnext < B.tnext;
    };
    for (auto &v : kids_local) std::sort(v.begin(), v.end(), cmp);
    std::sort(roots.begin(), roots.end(), [&](int64_t a, int64_t b) { return s->rows[a].tnext < s->rows[b].tnext; });
    std::vector<int64_t> out;
    out.reserve(nr);
    for (int64_t r : roots) lex_emit(s, kids_local, r, out);
    for (int64_t k = 0; k < (int64_t)out.size() && k < cap; k++) out_rows[k] = out[k];
  });
}

int tm_row_info(tm_store *s, int64_t row, int32_t *sid, int32_t *local, int64_t *parent, int64_t *matched,
                int64_t *length) {
  return guarded(s, [&] {
    if (!valid_row(s, row)) fail(TM_ENOENT, "node " + std::to_string(row) + " not in store");
    const RowHost &R = s->rows[row];
    if (sid) *sid = R.sid;
    if (local) *local = R.local;
    if (parent) *parent = R.parent;
    if (matched) *matched = R.m;
    if (length) *length = R.len;
  });
}

int tm_store_stats(tm_store *s, int64_t *rows, int64_t *arena_used, int64_t *arena_cap, int64_t *max_depth) {
  return guarded(s, [&] {
    if (rows) *rows = s->n_real_rows;
    if (arena_used) *arena_used = s->arena_used;
    if (arena_cap) *arena_cap = s->arena_cap;
    if (max_depth) *max_depth = s->max_depth;
  });
}

int tm_store_h2d_stats(tm_store *s, int64_t *out6) {
  return guarded(s, [&] {
    const int64_t c[6] = {s->c_pack_calls, s->c_pack_tokens, s->c_raw_calls, s->c_raw_tokens, s->c_pack_fallbacks,
                          s->c_h2d_bytes};
    memcpy(out6, c, sizeof(c));
  });
}

int tm_store_counters(tm_store *s, int64_t *out8) {
  return guarded(s, [&] {
    const int64_t c[8] = {s->c_record_calls, s->c_records, s->c_record_tokens, s->c_match_calls,
                          s->c_queries, s->c_export_calls, s->c_export_rows, s->c_export_tokens};
    memcpy(out8, c, sizeof(c));
  });
}

int tm_store_stream(tm_store *s, void **out_stream) {
  return guarded(s, [&] { *out_stream = (void *)s->stream; });
}

int tm_shared_alloc(tm_store *s, int64_t bytes, void **out_ptr) {
  return guarded(s, [&] {
    if (bytes <= 0) fail(TM_EINVAL, "bad size");
    ck(cudaMalloc(out_ptr, (size_t)bytes), "cudaMalloc(shared)");  // a whole allocation: IPC-exportable
    ck(cudaMemset(*out_ptr, 0, (size_t)bytes), "memset(shared)");
  });
}

int tm_shared_free(tm_store *s, void *ptr) {
  return guarded(s, [&] { ck(cudaFree(ptr), "cudaFree(shared)"); });
}

int tm_ipc_handle(tm_store *s, void *ptr, void *out_handle) {
  return guarded(s, [&] {
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, ptr), "cudaIpcGetMemHandle");
    memcpy(out_handle, &h, sizeof(h));
  });
}

int tm_ipc_open(tm_store *s, const void *handle, void **out_ptr) {
  return guarded(s, [&] {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    ck(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int tm_ipc_close(tm_store *s, void *ptr) {
  return guarded(s, [&] { ck(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); });
}

int tm_route_desc_bytes(int64_t *out_bytes) {
  *out_bytes = (int64_t)sizeof(tms::RouteDesc);
  return TM_OK;
}

namespace {
int route_prepare(tm_store *s, void *region, int64_t n, const int64_t *offsets, int32_t nranks, int32_t rank,
                  const tms::PushArgs &pa, void *stream) {
  return guarded(s, [&] {
    if (nranks < 1 || nranks > tms::kMaxRanks || rank < 0 || rank >= nranks) fail(TM_EINVAL, "bad rank");
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    tms::RouteHead d{};  // counts are (re)written by k_route
    d.rank = rank;
    d.nranks = nranks;
    if (offsets[0] < (int64_t)sizeof(tms::RouteDesc)) fail(TM_EINVAL, "routing arrays overlap the RouteDesc header");
    d.n = n;
    d.sid_off = offsets[0];
    d.qoff_off = offsets[1];
    d.len_off = offsets[2];
    d.tok_off = offsets[3];
    d.idx_off = offsets[4];
    d.m_off = offsets[5];
    d.par_off = offsets[6];
    d.dup_off = offsets[7];
    // 18-bit planes for the owners to pull over NVLink (only with peers; TM_ROUTE_PACK=0 off)
    static const bool pack = [] {
      const char *e = getenv("TM_ROUTE_PACK");
      return !(e && !strcmp(e, "0"));
    }();
    const bool packed = pack && nranks > 1 && offsets[8] > 0 && offsets[9] > 0 && offsets[10] > 0;
    d.lo_off = packed ? offsets[8] : 0;
    d.hi_off = packed ? offsets[9] : 0;
    d.pkf_off = packed ? offsets[10] : 0;
    d.pk_bad = 0;
    // per-query records (gsid, offset, length, index, first token) at idx positions: own
    // queries' written by k_route, remote ones' with the pack; the walk starts an item
    // with one load
    // (with peers only when the pack runs: it writes the remote queries' records)
    d.rec_off = (offsets[11] > 0 && (packed || nranks == 1)) ? offsets[11] : 0;
    if (pa.stride && !packed) fail(TM_EINVAL, "push routing needs the plane and record offsets");
    {
      ProfScope ps(s, 4, st);
      ck(tms::launch_route((char *)region, d, pa, st), "route");
    }
    if (packed) {
      ProfScope ps(s, 5, st);
      ck(tms::launch_route_pack((char *)region, n, pa, st), "route pack");
    }
  });
}
}  // namespace

int tm_route_prepare(tm_store *s, void *region, int64_t n, const int64_t *offsets, int32_t nranks, int32_t rank,
                     void *stream) {
  NvtxRange nvtx_("tm_route_prepare");
  tms::PushArgs pa{};
  return route_prepare(s, region, n, offsets, nranks, rank, pa, stream);
}

int tm_route_prepare_push(tm_store *s, void *region, int64_t n, const int64_t *offsets, int32_t nranks,
                          int32_t rank, void *const *peer_regions, int64_t inbox_stride, void *stream) {
  NvtxRange nvtx_("tm_route_prepare_push");
  if (nranks < 1 || nranks > tms::kMaxRanks || inbox_stride <= 0 || !peer_regions) {
    g_err = "push routing: bad rank count, inbox stride or peer table";
    return TM_EINVAL;
  }
  tms::PushArgs pa{};
  for (int p = 0; p < nranks; p++) pa.peer[p] = (char *)peer_regions[p];
  pa.stride = inbox_stride;
  return route_prepare(s, region, n, offsets, nranks, rank, pa, stream);
}

int tm_route_counts(tm_store *s, const void *region, int32_t *out_counts, void *stream) {
  return guarded(s, [&] {
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    ck(cudaMemcpyAsync(out_counts, (const char *)region + offsetof(tms::RouteDesc, count), sizeof(int32_t) * tms::kMaxRanks,
                       cudaMemcpyDeviceToHost, st), "D2H route counts");
    ck(cudaStreamSynchronize(st), "route counts sync");
  });
}

namespace {
uint64_t peer_timeout_ns() {  // TM_PEER_TIMEOUT_MS (default 20 s)
  static const uint64_t ms = [] {
    const char *e = getenv("TM_PEER_TIMEOUT_MS");
    return e ? (uint64_t)std::max(1ll, atoll(e)) : 20000ull;
  }();
  return ms * 1000000ull;
}

int match_routed(tm_store *s, int32_t nranks, int32_t rank, void *const *peer_regions, const int32_t *g2l,
                 int64_t g2l_len, int64_t epoch, int64_t push_stride, void *stream, bool wait_done = true) {
  return guarded(s, [&] {
    if (nranks < 1 || nranks > tms::kMaxRanks || rank < 0 || rank >= nranks) fail(TM_EINVAL, "bad rank");
    if (g2l_len < 0 || (g2l_len > 0 && !g2l)) fail(TM_EINVAL, "bad g2l table");
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    tm_store::MatchSlot *slot = &s->slots[s->next_slot++ % tm_store::kSlots];
    ck(cudaStreamWaitEvent(st, s->last, 0), "cudaStreamWaitEvent");
    if (slot->used) ck(cudaStreamWaitEvent(st, slot->done, 0), "cudaStreamWaitEvent");
    tms::RoutedArgs a{};
    a.nranks = nranks;
    a.rank = rank;
    for (int p = 0; p < nranks; p++) a.peer[p] = (const char *)peer_regions[p];
    a.g2l = g2l;
    a.g2l_len = g2l_len;
    a.sched = slot->sched;
    a.push_stride = push_stride;
    a.epoch = epoch;
    a.timeout_ns = peer_timeout_ns();
    static const int tail_every = [] {  // TM_ROUTED_TAIL: 1 in N CTAs works from the short end (0: off)
      const char *e = getenv("TM_ROUTED_TAIL");
      return e ? std::max(0, atoi(e)) : 8;
    }();
    a.tail_every = tail_every;
    // diagnostics: TM_ROUTED_TRACE=<path> appends every routed call's per-item timeline
    // ({start ns, end ns, length | remote << 40 | matched << 41, CTA} per query) to
    // <path>.<rank> (synchronous; not for timing runs)
    static const char *trace_path = getenv("TM_ROUTED_TRACE");
    constexpr long long kTraceCap = 1 << 20;
    if (trace_path) {
      if (!s->trace_buf) ck(cudaMalloc(&s->trace_buf, 8 * (4 + 4 * kTraceCap)), "cudaMalloc(trace)");
      ck(cudaMemsetAsync(s->trace_buf, 0, 8 * (4 + 4 * kTraceCap), st), "memset(trace)");
      a.trace = (long long *)s->trace_buf;
      a.trace_cap = kTraceCap;
    }
    if (epoch > 0) ck(tms::launch_route_arrive(a, st), "route arrive");
    {
      ProfScope ps(s, 0, st);
      ck(tms::launch_walk_routed(s->v, a, s->num_sms, st), "walk_routed");
    }
    if (epoch > 0 && wait_done) {
      ProfScope ps(s, 6, st);
      ck(tms::launch_route_wait_done(s->v, a, st), "route wait");
    }
    if (trace_path) {
      long long cnt = 0;
      ck(cudaStreamSynchronize(st), "trace sync");
      ck(cudaMemcpy(&cnt, s->trace_buf, 8, cudaMemcpyDeviceToHost), "trace count");
      cnt = std::min(cnt, kTraceCap);
      std::vector<long long> buf(4 * (size_t)cnt);
      ck(cudaMemcpy(buf.data(), (char *)s->trace_buf + 32, 32 * (size_t)cnt, cudaMemcpyDeviceToHost), "trace D2H");
      const std::string fn = std::string(trace_path) + "." + std::to_string(rank);
      if (FILE *f = fopen(fn.c_str(), "ab")) {
        const long long hdr[2] = {cnt, (long long)epoch};
        fwrite(hdr, 8, 2, f);
        fwrite(buf.data(), 8, buf.size(), f);
        fclose(f);
      }
    }
    ck(cudaEventRecord(slot->done, st), "cudaEventRecord");
    slot->used = true;
  });
}
}  // namespace

int tm_match_routed(tm_store *s, int32_t nranks, int32_t rank, void *const *peer_regions, const int32_t *g2l,
                    int64_t g2l_len, void *stream) {
  NvtxRange nvtx_("tm_match_routed");
  return match_routed(s, nranks, rank, peer_regions, g2l, g2l_len, 0, 0, stream);
}

int tm_match_routed_sync(tm_store *s, int32_t nranks, int32_t rank, void *const *peer_regions, const int32_t *g2l,
                         int64_t g2l_len, int64_t epoch, void *stream) {
  NvtxRange nvtx_("tm_match_routed_sync");
  if (epoch <= 0) {
    g_err = "epoch must be positive and increase by one per routed call";
    return TM_EINVAL;
  }
  return match_routed(s, nranks, rank, peer_regions, g2l, g2l_len, epoch, 0, stream);
}

int tm_match_routed_nowait(tm_store *s, int32_t nranks, int32_t rank, void *const *peer_regions, const int32_t *g2l,
                           int64_t g2l_len, int64_t epoch, int64_t inbox_stride, void *stream) {
  NvtxRange nvtx_("tm_match_routed_nowait");
  if (epoch <= 0 || inbox_stride < 0) {
    g_err = "epoch must be positive, inbox stride non-negative";
    return TM_EINVAL;
  }
  return match_routed(s, nranks, rank, peer_regions, g2l, g2l_len, epoch, inbox_stride, stream, false);
}

int tm_route_wait_done(tm_store *s, int32_t nranks, int32_t rank, void *const *peer_regions, int64_t epoch,
                       void *stream) {
  NvtxRange nvtx_("tm_route_wait_done");
  return guarded(s, [&] {
    if (nranks < 1 || nranks > tms::kMaxRanks || rank < 0 || rank >= nranks || epoch <= 0)
      fail(TM_EINVAL, "bad rank or epoch");
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    tms::RoutedArgs a{};
    a.nranks = nranks;
    a.rank = rank;
    for (int p = 0; p < nranks; p++) a.peer[p] = (const char *)peer_regions[p];
    a.epoch = epoch;
    a.timeout_ns = peer_timeout_ns();
    ProfScope ps(s, 6, st);
    ck(tms::launch_route_wait_done(s->v, a, st), "route wait");
  });
}

int tm_match_routed_push(tm_store *s, int32_t nranks, int32_t rank, void *const *peer_regions, const int32_t *g2l,
                         int64_t g2l_len, int64_t epoch, int64_t inbox_stride, void *stream) {
  NvtxRange nvtx_("tm_match_routed_push");
  if (epoch <= 0 || inbox_stride <= 0) {
    g_err = "push routing: epoch and inbox stride must be positive";
    return TM_EINVAL;
  }
  return match_routed(s, nranks, rank, peer_regions, g2l, g2l_len, epoch, inbox_stride, stream);
}


int tm_store_save(tm_store *s, const char *path) {
  NvtxRange nvtx_("tm_store_save");
  return guarded(s, [&] {
    wait_prev(s, s->stream);
    ck(cudaStreamSynchronize(s->stream), "snapshot sync");
    FILE *f = fopen(path, "wb");
    if (!f) fail(TM_EINVAL, std::string("cannot open ") + path);
    FileW w{f};
    try {
      w.put(kMagic, 8);
      const int64_t nrows = (int64_t)s->rows.size();
      w.val(s->n_sess); w.val(nrows); w.val(s->n_real_rows); w.val(s->arena_used); w.val(s->n_runs); w.val(s->max_depth);
      w.put(s->rows.data(), sizeof(RowHost) * nrows);
      for (int64_t i = 0; i < s->n_sess; i++) {
        const int64_t k = (int64_t)s->sess_rows[i].size();
        w.val(s->sess_stored[i]); w.val(s->sess_naive[i]); w.val(k);
        for (int64_t j = 0; j < k; j++) w.val(s->sess_rows[i][j]);
      }
      save_dev(s, w, s->v.arena, s->arena_used);
      save_dev(s, w, s->v.row_vb, nrows); save_dev(s, w, s->v.row_m, nrows); save_dev(s, w, s->v.row_len, nrows);
      save_dev(s, w, s->v.row_parent, nrows); save_dev(s, w, s->v.row_sess, nrows);
      save_dev(s, w, s->v.row_local, nrows); save_dev(s, w, s->v.row_depth, nrows);
      save_dev(s, w, s->v.row_run0, nrows); save_dev(s, w, s->v.row_nrun, nrows);
      save_dev(s, w, s->v.row_ext, nrows); save_dev(s, w, s->v.row_ext_tok, nrows);
      save_dev(s, w, s->v.row_ext_len, nrows); save_dev(s, w, s->v.row_ext_vb, nrows);
      save_dev(s, w, s->v.row_jump, nrows);
      save_dev(s, w, s->v.run_start, s->n_runs); save_dev(s, w, s->v.run_version, s->n_runs);
      save_dev(s, w, s->v.run_origin, s->n_runs);
      save_dev(s, w, s->v.s_nrows, s->n_sess); save_dev(s, w, s->v.s_stored, s->n_sess);
      save_dev(s, w, s->v.s_naive, s->n_sess);
      save_dev(s, w, s->v.s_pc_row, s->n_sess);
      save_dev(s, w, s->v.s_pc_vb, s->n_sess);
      save_dev(s, w, s->v.s_pc_cap, s->n_sess);
      w.put(kMagic, 8);
    } catch (...) {
      fclose(f);
      throw;
    }
    if (fclose(f)) fail(TM_EINVAL, "snapshot close failed");
  });
}

int tm_store_load(tm_store *s, const char *path) {
  NvtxRange nvtx_("tm_store_load");
  return guarded(s, [&] {
    if (s->n_sess || !s->rows.empty()) fail(TM_EINVAL, "restore needs an empty store");
    FILE *f = fopen(path, "rb");
    if (!f) fail(TM_ENOENT, std::string("cannot open ") + path);
    FileR r{f};
    try {
      char m[8];
      r.get(m, 8);
      if (memcmp(m, kMagic, 8)) fail(TM_EINVAL, "not a tmstore snapshot");
      const int64_t nsess = r.val<int64_t>(), nrows = r.val<int64_t>(), nreal = r.val<int64_t>();
      const int64_t aused = r.val<int64_t>(), nruns = r.val<int64_t>(), maxd = r.val<int64_t>();
      ensure_sessions(s, nsess);
      ensure_rows(s, nrows);
      ensure_runs(s, nruns);
      ensure_arena(s, aused);
      ensure_table(s, nreal);
      s->rows.resize(nrows);
      r.get(s->rows.data(), sizeof(RowHost) * nrows);
      s->free_rows.clear();
      for (int64_t i = 0; i < nrows; i++)
        if (s->rows[i].sid < 0) s->free_rows.push_back(i);
      s->sess_rows.assign(nsess, {});
      s->sess_stored.assign(nsess, 0);
      s->sess_naive.assign(nsess, 0);
      s->sess_maxdepth.assign(nsess, -1);
      for (const RowHost &rh : s->rows)
        if (rh.sid >= 0) s->sess_maxdepth[rh.sid] = std::max(s->sess_maxdepth[rh.sid], rh.depth);
      for (int64_t i = 0; i < nsess; i++) {
        s->sess_stored[i] = r.val<int64_t>();
        s->sess_naive[i] = r.val<int64_t>();
        const int64_t k = r.val<int64_t>();
        for (int64_t j = 0; j < k; j++) s->sess_rows[i].push_back(r.val<int64_t>());
      }
      load_dev(s, r, s->v.arena, aused);
      load_dev(s, r, s->v.row_vb, nrows); load_dev(s, r, s->v.row_m, nrows); load_dev(s, r, s->v.row_len, nrows);
      load_dev(s, r, s->v.row_parent, nrows); load_dev(s, r, s->v.row_sess, nrows);
      load_dev(s, r, s->v.row_local, nrows); load_dev(s, r, s->v.row_depth, nrows);
      load_dev(s, r, s->v.row_run0, nrows); load_dev(s, r, s->v.row_nrun, nrows);
      load_dev(s, r, s->v.row_ext, nrows); load_dev(s, r, s->v.row_ext_tok, nrows);
      load_dev(s, r, s->v.row_ext_len, nrows); load_dev(s, r, s->v.row_ext_vb, nrows);
      load_dev(s, r, s->v.row_jump, nrows);
      load_dev(s, r, s->v.run_start, nruns); load_dev(s, r, s->v.run_version, nruns);
      load_dev(s, r, s->v.run_origin, nruns);
      load_dev(s, r, s->v.s_nrows, nsess); load_dev(s, r, s->v.s_stored, nsess);
      load_dev(s, r, s->v.s_naive, nsess);
      load_dev(s, r, s->v.s_pc_row, nsess);
      load_dev(s, r, s->v.s_pc_vb, nsess);
      load_dev(s, r, s->v.s_pc_cap, nsess);
      r.get(m, 8);
      if (memcmp(m, kMagic, 8)) fail(TM_EINVAL, "snapshot trailer missing");
      s->n_sess = nsess;
      s->v.n_sess = nsess;
      s->n_real_rows = nreal;
      s->arena_used = aused;
      s->n_runs = nruns;
      s->max_depth = maxd;
      const int64_t ctr[4] = {aused, nrows, nruns, 0};
      ck(cudaMemcpy(s->v.ctr, ctr, sizeof(ctr), cudaMemcpyHostToDevice), "ctr");
      // the branch index is derived state: rebuild it from the row table
      ck(tms::launch_rebuild_index(s->v, nrows, s->stream), "rebuild index");
      ck(cudaStreamSynchronize(s->stream), "restore sync");
    } catch (...) {
      fclose(f);
      throw;
    }
    fclose(f);
  });
}

int tm_block_hashes(tm_store *s, const int32_t *tokens, int64_t n_words, uint64_t *out, void *stream) {
  NvtxRange nvtx_("tm_block_hashes");
  return guarded(s, [&] {
    if (n_words < 0 || n_words % 128) fail(TM_EINVAL, "n_words must be a multiple of 128");
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    ProfScope ps(s, 8, st);
    ck(tms::launch_block_hash(tokens, n_words / 128, out, s->num_sms, st), "block hash");
  });
}

int tm_profile_reserve(tm_store *s, int64_t pairs) {
  return guarded(s, [&] {
    for (int k = 0; k < tm_store::kProfKinds; k++)
      while ((int64_t)s->ev[k].size() < pairs) {
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        s->ev[k].push_back({a, b});
      }
  });
}

int tm_profile_begin(tm_store *s) {
  return guarded(s, [&] {
    s->profile = true;
    for (int k = 0; k < tm_store::kProfKinds; k++) s->ev_used[k] = 0;
  });
}

int tm_profile_end(tm_store *s, int32_t kind, double *total_ms, int64_t *launches) {
  return guarded(s, [&] {
    if (kind < 0 || kind >= tm_store::kProfKinds) fail(TM_EINVAL, "bad kernel kind");
    double t = 0;
    for (size_t i = 0; i < s->ev_used[kind]; i++) {
      ck(cudaEventSynchronize(s->ev[kind][i].second), "event sync");
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, s->ev[kind][i].first, s->ev[kind][i].second), "elapsed");
      t += ms;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = (int64_t)s->ev_used[kind];
    s->profile = false;
  });
}

int tm_synchronize(tm_store *s) {
  return guarded(s, [&] {
    ck(cudaStreamSynchronize(s->stream), "sync");
    ck(cudaEventSynchronize(s->last), "sync");
    check_device_error(s);
    for (auto &sl : s->slots)
      if (sl.used) ck(cudaEventSynchronize(sl.done), "sync");
  });
}

}  // extern "C"
