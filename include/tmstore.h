/*
 * tmstore — B200-resident session-history store for the trajectory-manager hot path.
 *
 * C ABI (extern "C", plain pointers and sizes, no torch/CUDA types beyond an opaque
 * `void *stream` that is a cudaStream_t or NULL).  The reference has no FFI: its
 * boundary is the Python class SessionTrie (/root/reference/pkg/src/rolloutlab/trie.py)
 * called by TrajectoryManager (trajectory.py).  Each entry point below names the
 * reference interface it replaces; INTEGRATION.md shows the ctypes binding.
 *
 * Model: a store holds many sessions.  Every distinct recorded sequence of a session
 * is a ROW (global id int64; session-local ordinal int32 in order of first
 * appearance).  A row stores only its novel suffix [matched, len); its prefix is
 * inherited from its PARENT row = the earliest-inserted row whose longest common
 * prefix with it equals `matched` (-1 when matched == 0).  Shared prefixes keep the
 * metadata of their first writer (trie.py:9-11).
 *
 * Status codes: TM_OK, TM_EINVAL (reference: ValueError), TM_ENOENT (KeyError /
 * UnknownSessionError), TM_ENOMEM / TM_ECUDA (RuntimeError).  tm_last_error()
 * returns a thread-local message for the last failing call on this thread.
 *
 * Memory kinds: TM_MEM_HOST — every array argument is host memory (pageable or
 * pinned); the call is synchronous.  TM_MEM_DEVICE — token/offset/output arrays are
 * device pointers on the store's GPU; the call is asynchronous on `stream`.  Device
 * token buffers must start every sequence at a 128-byte aligned word offset
 * (tok_off[k] % 32 == 0) and be readable up to the next 128-byte boundary.
 *
 * Thread safety: every call locks the store; callers may use any thread.
 */
#ifndef TMSTORE_H
#define TMSTORE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tm_store tm_store;

enum { TM_OK = 0, TM_EINVAL = 1, TM_ENOENT = 2, TM_ENOMEM = 3, TM_ECUDA = 4 };
enum { TM_MEM_HOST = 0, TM_MEM_DEVICE = 1 };
enum { TM_ORDER_INSERT = 0, TM_ORDER_LEX = 1 };
enum { TM_ORIGIN_AGENT_INPUT = 0, TM_ORIGIN_MODEL_OUTPUT = 1 };

typedef struct {
  int32_t device;           /* CUDA device ordinal */
  int64_t arena_words;      /* initial token-arena capacity (int32 words); grows x2 */
  int64_t row_capacity;     /* initial row-table capacity; grows x2 */
  int64_t run_capacity;     /* initial metadata-run capacity; grows x2 */
  int64_t session_capacity; /* initial session capacity; grows x2 */
} tm_config;

/* Thread-local message describing the last error returned on this thread. */
const char *tm_last_error(void);
/* Library version string. */
const char *tm_version(void);

/* Create / destroy a store on one GPU.  cfg may be NULL (defaults).
 * Replaces: the per-session `SessionTrie(session_id)` objects held in
 * TrajectoryManager._sessions (trajectory.py:128, 137-145, trie.py:93-99). */
int tm_store_create(const tm_config *cfg, tm_store **out);
int tm_store_destroy(tm_store *store);

/* Open a new empty session; returns its dense id.
 * Replaces: `_Session(trie=SessionTrie(session_id))` (trajectory.py:143). */
int tm_session_create(tm_store *store, int32_t *out_sid);
int tm_session_count(tm_store *store, int64_t *out_n);

/* Record a batch of sequences: the batched `SessionTrie.lpm_insert` (trie.py:120-179)
 * with sequential semantics — entry k sees every earlier entry of the batch.
 *   sids[n]          session of each sequence
 *   tokens/tok_off/tok_len   sequence k = tokens[tok_off[k] : tok_off[k] + tok_len[k]]
 *   run_off[n+1]     metadata runs of sequence k = runs[run_off[k] : run_off[k+1]]
 *   run_start[]      run start relative to its sequence (first must be 0, ascending)
 *   run_origin[]     TM_ORIGIN_* ; run_version[] model version
 * Outputs (any may be NULL), one per entry:
 *   out_matched      matched_prefix_length           (InsertResult, trie.py:71-75)
 *   out_row          global row id of the sequence   (node_id)
 *   out_local        session-local row ordinal
 *   out_parent       global parent row (-1 if none)
 *   out_parent_local session-local parent ordinal (-1 if none)
 *   out_added        added_tokens (= len - matched, 0 for an existing sequence)
 * mem applies to `tokens` only (TM_MEM_DEVICE: a device buffer with 128-byte aligned
 * sequence starts, e.g. tokens produced on the GPU); every other array is host memory
 * and the call is synchronous, as lpm_insert is.  With TM_MEM_DEVICE the tokens are
 * read after all work already queued on `stream` (their producer; NULL = none).  Errors: empty sequence or non-parallel metadata
 * -> TM_EINVAL (trie.py:128-131); unknown session -> TM_ENOENT. */
int tm_record_batch(tm_store *store, int64_t n, int32_t mem, const int32_t *sids, const int32_t *tokens,
                    const int64_t *tok_off, const int64_t *tok_len, const int64_t *run_off,
                    const int32_t *run_start, const uint8_t *run_origin, const int32_t *run_version,
                    int64_t *out_matched, int64_t *out_row, int32_t *out_local, int64_t *out_parent,
                    int32_t *out_parent_local, int64_t *out_added, void *stream);

/* One record of host arrays (the per-request lpm_insert path, trie.py:120-179) without
 * building batch arrays: out6 = matched, row, local, parent, parent_local, added.
 * Same semantics and errors as tm_record_batch with n = 1. */
int tm_record_one(tm_store *store, int32_t sid, const int32_t *tokens, int64_t ntok, const int32_t *run_start,
                  const uint8_t *run_origin, const int32_t *run_version, int64_t nruns, int64_t *out6);

/* Read-only longest-prefix match of a batch of queries (no mutation): the LPM walk
 * of lpm_insert (trie.py:136-158) without the record step.
 *   out_matched[n]   LCP length with the best stored sequence of the session
 *   out_parent[n]    global row achieving it (earliest such), -1 if matched == 0
 *   out_dup[n]       global row equal to the query, -1 if none
 * TM_MEM_HOST: all arrays host, synchronous.  TM_MEM_DEVICE: all arrays device,
 * asynchronous on `stream` (NULL = the store's stream).  Unknown/empty -> matched 0. */
int tm_match_batch(tm_store *store, int64_t n, int32_t mem, const int32_t *sids, const int32_t *tokens,
                   const int64_t *tok_off, const int64_t *tok_len, int64_t *out_matched, int64_t *out_parent,
                   int64_t *out_dup, void *stream);

/* Total tokens of a list of rows (to size tm_export_rows outputs). */
int tm_rows_total(tm_store *store, int64_t n, const int64_t *rows, int64_t *out_total);

/* Reconstruct rows into packed token-id batches: path_trajectory / extract /
 * drain_batch assembly (trie.py:203-224, core.py:88-98, trajectory.py:342-363).
 *   rows[n]              global row ids (host array)
 *   out_offsets[n+1]     cu_seqlens-style row offsets (host array, always)
 *   out_tokens/mask/versions  packed arrays of out_offsets[n] entries; mask is
 *                        loss_mask (1 = MODEL_OUTPUT); memory kind `mem_out`
 *   out_resp_start[n]    1 + last position whose mask is 0 (0 if none): where the
 *                        trailing model response begins (kind `mem_out`, may be NULL)
 * TM_MEM_DEVICE outputs are written asynchronously on `stream`. */
int tm_export_rows(tm_store *store, int64_t n, const int64_t *rows, int32_t mem_out, int64_t *out_offsets,
                   int32_t *out_tokens, uint8_t *out_mask, int32_t *out_versions, int64_t *out_resp_start,
                   void *stream);

/* Rows that live on the host - open or paused requests exported with include_partials
 * (TrajectoryManager._partial_trajectory, trajectory.py:329-340) - written into a packed
 * DEVICE batch next to rows exported by tm_export_rows:
 *   row k = tokens[tok_off[k] : tok_off[k+1]] (host array): the first n_input[k] positions
 *   are AGENT_INPUT at ctx_version[k]; the rest MODEL_OUTPUT, versions given as runs
 *   run_start[run_off[k] : run_off[k+1]] (relative to the row; the first equals n_input[k])
 *   with run_version[...]
 *   out_off[k]   where row k starts in out_tokens / out_mask / out_versions (device)
 *   out_resp_start[k] (device, may be NULL) = n_input[k]
 * Asynchronous on `stream`.  Errors: non-parallel runs -> TM_EINVAL. */
int tm_export_host_rows(tm_store *store, int64_t n, const int32_t *tokens, const int64_t *tok_off,
                        const int64_t *n_input, const int32_t *ctx_version, const int64_t *run_off,
                        const int32_t *run_start, const int32_t *run_version, const int64_t *out_off,
                        int32_t *out_tokens, uint8_t *out_mask, int32_t *out_versions, int64_t *out_resp_start,
                        void *stream);

/* Canonical NDJSON of rows, formatted on the GPU and byte-identical to
 * "".join(trajectory_to_line(t) + "\n") (core.py:182-183; the /traj/export payload of
 * api.py:248-254).  sid_json/sid_off[n+1]: per row, the session id as a JSON string
 * literal exactly as json.dumps(session_id) prints it, concatenated.  With out == NULL
 * or cap too small only *out_bytes (the exact size) is set; otherwise the text is
 * written to `out` (host or device memory per mem_out). */
int tm_export_ndjson(tm_store *store, int64_t n, const int64_t *rows, const char *sid_json, const int64_t *sid_off,
                     int32_t mem_out, char *out, int64_t cap, int64_t *out_bytes, void *stream);

/* StorageStats of a session (trie.py:78-87, 184-185; trajectory.py:369-372). */
int tm_session_stats(tm_store *store, int32_t sid, int64_t *stored, int64_t *naive, int64_t *nrows);

/* Rows of a session (global ids) in insertion order or in lexicographic sequence
 * order — the order of SessionTrie.extract (trie.py:189-198, 210-216).
 * Writes min(cap, nrows) ids; *n_out = nrows. */
int tm_session_rows(tm_store *store, int32_t sid, int32_t order, int64_t *out_rows, int64_t cap,
                    int64_t *n_out);

/* Describe one global row. */
int tm_row_info(tm_store *store, int64_t row, int32_t *sid, int32_t *local, int64_t *parent,
                int64_t *matched, int64_t *length);

/* Store-wide counters: rows, arena words used, arena capacity, max row-tree depth. */
int tm_store_stats(tm_store *store, int64_t *rows, int64_t *arena_used, int64_t *arena_cap,
                   int64_t *max_depth);

/* Observability counters since creation: record calls, records, recorded tokens,
 * match calls, queries, export calls, exported rows, exported tokens (8 int64). */
int tm_store_counters(tm_store *store, int64_t *out8);

/* Host->device token copies of host-memory calls (6 int64): calls sent as packed 18-bit
 * planes, their tokens, calls sent as raw int32, their tokens, packed attempts that fell
 * back to raw (a token outside [0, 2^18)), token bytes actually copied.  Replaces nothing
 * in the reference (its trie is host-resident); TM_H2D_PACK_MIN (tokens per call,
 * default 8M, <0 off) selects. */
int tm_store_h2d_stats(tm_store *store, int64_t *out6);

/* The store's CUDA stream (cudaStream_t) for callers that want to order work after it. */
int tm_store_stream(tm_store *store, void **out_stream);

/* ---- Cross-GPU routing on one node (session-hash sharding, config 5) ----------------
 * Every rank publishes its query batch in a shared device region laid out as
 *   [RouteDesc header | int64 gsid[n] | int64 tok_off[n] | int64 len[n] | int32 tokens |
 *    int32 idx[n] | int64 out_matched[n] | int64 out_parent[n] | int64 out_dup[n] |
 *    uint16 low plane[tokens + 128] | uint8 high plane[(tokens + 128) / 4] | int32 pk[n + 1] |
 *    32-byte query records[n]]
 * (offsets[12] = byte offsets of those arrays: sid, qoff, len, tok, idx, m, par, dup, lo,
 * hi, pk, rec; lo = hi = pk = rec = 0: no planes.  The pack writes each remote query's
 * record - gsid, offset, length, index, first token - at its idx position, so an owner
 * starts it with one load instead of three dependent ones).  tm_route_prepare writes the header, buckets the batch by
 * owner rank (owner = splitmix64(gsid) mod nranks) and, with peers, packs the tokens of the
 * queries owned by OTHER ranks (this is `rank`) into the 18-bit planes (hostpack.h layout;
 * TM_ROUTE_PACK=0 disables) so remote owners move 2.25 B per compared position over NVLink
 * instead of 4.  Then either tm_match_routed_sync
 * (device-side barriers) or a cross-rank barrier + tm_match_routed + a second barrier:
 * every owner's kernel reads its queries directly from the requesters' regions over
 * NVLink and writes the results back into them (P2P).
 * Regions come from tm_shared_alloc (whole cudaMalloc allocations, IPC-exportable);
 * peers map them with tm_ipc_handle (64-byte cudaIpcMemHandle) / tm_ipc_open. */
int tm_route_desc_bytes(int64_t *out_bytes); /* size of the RouteDesc header */
int tm_shared_alloc(tm_store *store, int64_t bytes, void **out_ptr);
int tm_shared_free(tm_store *store, void *ptr);
int tm_ipc_handle(tm_store *store, void *ptr, void *out_handle64);
int tm_ipc_open(tm_store *store, const void *handle64, void **out_ptr);
int tm_ipc_close(tm_store *store, void *ptr);
int tm_route_prepare(tm_store *store, void *region, int64_t n, const int64_t *offsets, int32_t nranks,
                     int32_t rank, void *stream);
/* Per-owner query counts of a prepared region (kMaxRanks = 16 int32; synchronous). */
int tm_route_counts(tm_store *store, const void *region, int32_t *out_counts16, void *stream);
/* g2l: device int32[g2l_len] global session id -> this store's session id (-1 if not
 * owned); a query whose global id is outside [0, g2l_len) or maps to -1 gets matched = -1.
 * peer_regions: host array of nranks device pointers (this rank's own region at [rank]). */
int tm_match_routed(tm_store *store, int32_t nranks, int32_t rank, void *const *peer_regions, const int32_t *g2l,
                    int64_t g2l_len, void *stream);

/* tm_match_routed with the two cross-rank barriers done on the device instead of by the
 * caller: a 32-thread kernel writes this rank's `arrive` epoch into every peer's region
 * header (NVLink store, release), the owners' match kernel waits for all arrivals
 * (acquire), its last CTA writes `done` into every requester's header, and a wait
 * kernel on this rank's stream holds later work until every owner is done.  `epoch`:
 * the same value on every rank, one larger per routed call (1, 2, ...).  A peer that
 * never signals becomes a device error after 20 s (TM_PEER_TIMEOUT_MS; tm_synchronize reports it). */
int tm_match_routed_sync(tm_store *store, int32_t nranks, int32_t rank, void *const *peer_regions,
                         const int32_t *g2l, int64_t g2l_len, int64_t epoch, void *stream);

/* tm_match_routed_sync (inbox_stride 0) or tm_match_routed_push without its last step: the
 * wait for every owner's `done` flag is left to tm_route_wait_done, which the caller
 * enqueues on another stream (ordered after this call), so the next batch's walk does not
 * queue behind the peers' tails.  Results are visible to work ordered after that wait. */
int tm_match_routed_nowait(tm_store *store, int32_t nranks, int32_t rank, void *const *peer_regions,
                           const int32_t *g2l, int64_t g2l_len, int64_t epoch, int64_t inbox_stride, void *stream);
int tm_route_wait_done(tm_store *store, int32_t nranks, int32_t rank, void *const *peer_regions, int64_t epoch,
                       void *stream);

/* Push routing: the same exchange with the plane traffic turned around.  Each region
 * also holds an inbox of nranks slices at `inbox_stride` bytes apart (slice p = the
 * lo / hi / rec arrays of source rank p at offsets[8], [9], [11] + p * inbox_stride);
 * tm_route_prepare_push packs every remote query's planes and record straight into its
 * owner's inbox slice for this rank (P2P stores over NVLink, overlapping the previous
 * batch's walk when pipelined), and tm_match_routed_push (device barriers as in
 * tm_match_routed_sync) has each owner read them from its own HBM.  A region's inbox
 * may be rewritten once every owner has finished the batch that last used it (the
 * done wait of that batch).  Same results as tm_match_routed_sync. */
int tm_route_prepare_push(tm_store *store, void *region, int64_t n, const int64_t *offsets, int32_t nranks,
                          int32_t rank, void *const *peer_regions, int64_t inbox_stride, void *stream);
int tm_match_routed_push(tm_store *store, int32_t nranks, int32_t rank, void *const *peer_regions,
                         const int32_t *g2l, int64_t g2l_len, int64_t epoch, int64_t inbox_stride, void *stream);

/* Snapshot / restore (the reference store is in-memory only, trajectory.py:128): write
 * the arena, row table, metadata runs, session counters and the host row mirror to a
 * file; load them into an EMPTY store (any GPU), rebuilding the branch index. */
int tm_store_save(tm_store *store, const char *path);
int tm_store_load(tm_store *store, const char *path);

/* Per-block token hashes of a device buffer: out[b] = hash of words [128 b, 128 b + 128)
 * (n_words a multiple of 128; device pointers; asynchronous on `stream`).  The building
 * block of the north star's hash-first candidate filter, kept to measure it against the
 * exact walk (hashing the query costs a full extra read of it, and an equal
 * hash never proves a match, so the filter cannot remove bytes from an exact LPM). */
int tm_block_hashes(tm_store *store, const int32_t *tokens, int64_t n_words, uint64_t *out, void *stream);

/* Per-kernel CUDA-event timing for benchmarks.  tm_profile_begin starts recording an
 * event pair around every launch; tm_profile_end(kind) waits for them and returns the
 * summed device time and launch count of one kernel kind (TM_KERNEL_*), then stops. */
enum {
  TM_KERNEL_WALK = 0, TM_KERNEL_COMMIT = 1, TM_KERNEL_EXPORT = 2, TM_KERNEL_PLAN = 3,
  TM_KERNEL_ROUTE = 4, TM_KERNEL_ROUTE_PACK = 5, TM_KERNEL_ROUTE_WAIT = 6,
  TM_KERNEL_RECORD_COPY = 7, /* (no longer launched: K2 copies inside its one launch; always 0) */
  TM_KERNEL_BLOCK_HASH = 8
};
int tm_profile_begin(tm_store *store);
/* Create the event pairs of `pairs` launches per kernel kind up front (so a timed region
 * never calls cudaEventCreate). */
int tm_profile_reserve(tm_store *store, int64_t pairs);
int tm_profile_end(tm_store *store, int32_t kind, double *total_ms, int64_t *launches);

/* Block until all work queued on the store's stream is done. */
int tm_synchronize(tm_store *store);

#ifdef __cplusplus
}
#endif
#endif
