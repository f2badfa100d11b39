// Host-visible launchers for the tmstore kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tms {
struct DevView;
struct Batch;
struct RoutedArgs;

struct ExportArgsHost {
  int64_t n;
  const int64_t *rows;
  const int64_t *out_off;
  const int64_t *tile_off;
  int64_t ntiles;
  int32_t *tokens;
  uint8_t *mask;
  int32_t *versions;
  int64_t *resp;
  char *plan;  // planner scratch: export_plan_bytes(ntiles), 16-byte aligned
};
int64_t export_plan_bytes(int64_t ntiles);

// rows that live on the host (open / paused requests): tokens already in device memory
struct HostRowsArgs {
  int64_t n;
  const int32_t *src;        // tokens, row k at src[tok_off[k] .. tok_off[k+1])
  const int64_t *tok_off;    // n + 1
  const int64_t *n_input;    // n: AGENT_INPUT prefix length
  const int32_t *ctx_version;// n: version of the input prefix
  const int64_t *run_off;    // n + 1: version runs of the MODEL_OUTPUT part
  const int32_t *run_start;  // relative to the row
  const int32_t *run_version;
  const int64_t *out_off;    // n: where row k starts in the outputs
  int32_t *tokens;
  uint8_t *mask;
  int32_t *versions;
  int64_t *resp;             // n, may be null
};
cudaError_t launch_fill_host_rows(const HostRowsArgs &a, int num_sms, cudaStream_t s);

// expand 18-bit split planes (hostpack.h) into int32 tokens for positions [p0, p1)
// (multiples of 32)
cudaError_t launch_unpack18(const uint16_t *lo, const uint8_t *hi, int32_t *out, int64_t p0, int64_t p1, int num_sms,
                            cudaStream_t s);

// fills b.root (if root != null) and b.bucket_items (plan_items_ints(n) ints); counts go to b.sched
struct JsonArgsHost {
  int64_t n;
  const int64_t *out_off, *tile_off;
  int64_t ntiles;
  const int32_t *tokens;
  const uint8_t *mask;
  const int32_t *versions;
  int64_t *sums;
  const int64_t *toff, *roff;
  const char *sid;
  const int64_t *sid_off;
  char *out;
};
cudaError_t launch_json(const JsonArgsHost &h, int pass, int num_sms, cudaStream_t s);

cudaError_t launch_plan(const DevView &v, Batch &b, int64_t *root, int *items, cudaStream_t s);
int64_t plan_items_ints(int64_t n);
cudaError_t launch_walk(const DevView &v, const Batch &b, int num_sms, cudaStream_t s);
struct RecordArgs;
// K2: records the whole batch in one launch (chains walked and committed, suffixes copied
// into the arena, rows switched to it); *copy_warp = 1 when the chain CTAs carried a copy warp
cudaError_t launch_record(const DevView &v, const RecordArgs &a, int num_sms, cudaStream_t s, int *copy_warp);
cudaError_t launch_export(const DevView &v, const ExportArgsHost &e, int num_sms, cudaStream_t s);
cudaError_t launch_rehash(const DevView &v, const uint64_t *ok0, const uint64_t *ok1, const int64_t *oval,
                          int64_t ocap, cudaStream_t s);
cudaError_t launch_rebuild_index(const DevView &v, int64_t nrows, cudaStream_t s);
cudaError_t launch_fill_u64(uint64_t *p, int64_t n, uint64_t val, cudaStream_t s);
cudaError_t launch_block_hash(const int32_t *tok, int64_t nblocks, uint64_t *out, int num_sms, cudaStream_t s);
int export_tile_tokens();
cudaError_t launch_route(char *region, const RouteHead &head, const PushArgs &pa, cudaStream_t s);
// pack the region's query tokens into its 18-bit planes (RouteDesc::lo_off / hi_off)
cudaError_t launch_route_pack(char *region, int64_t n, const PushArgs &pa, cudaStream_t s);
// device-side barriers of the routed match (RoutedArgs::epoch > 0)
cudaError_t launch_route_arrive(const RoutedArgs &a, cudaStream_t s);
cudaError_t launch_route_wait_done(const DevView &v, const RoutedArgs &a, cudaStream_t s);
cudaError_t launch_walk_routed(const DevView &v, const RoutedArgs &a, int num_sms, cudaStream_t s);
}  // namespace tms
