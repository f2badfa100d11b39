// NVLink all-to-all probe (tuning tool): every GPU moves an equal share of a buffer to or
// from every peer at once, the pattern of config 5's cross-shard exchange.  Modes:
//   read-ldg   SM loads (LDG.128) of peer HBM (the routed walk's plane pulls)
//   read-bulk  TMA 1-D bulk copies peer HBM -> shared memory
//   write-st   SM stores (STG.128) of local HBM data into peer HBM
//   write-bulk TMA 1-D bulk copies shared memory -> peer HBM (cp.async.bulk.global.shared::cta)
//   ce         copy engine (cudaMemcpyPeerAsync), one copy per peer
// Per GPU GB/s = bytes the GPU sent (writes) or received (reads) / slowest GPU's time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/a2a_probe tools/a2a_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kMax = 8;
struct Peers { char *p[kMax]; int n; int self; };

// CTA b works on peer (b % (n-1)) shifted past self, a contiguous share of that peer's slice
__device__ __forceinline__ int peer_of(int b, const Peers &P) { int q = b % (P.n - 1); return q < P.self ? q : q + 1; }

__global__ void k_read_ldg(Peers P, int64_t slice, int *out) {
  const int peer = peer_of(blockIdx.x, P);
  const int per_peer = gridDim.x / (P.n - 1), k = blockIdx.x / (P.n - 1);
  const int64_t share = slice / per_peer / 16 * 16;
  const int4 *src = reinterpret_cast<const int4 *>(P.p[peer] + (int64_t)P.self * slice + k * share);
  const int64_t n = share / 16;
  int acc = 0;
  for (int64_t i = threadIdx.x; i < n; i += 4 * blockDim.x) {
    int4 a = src[i];
    int4 b = i + blockDim.x < n ? src[i + blockDim.x] : make_int4(0, 0, 0, 0);
    int4 c = i + 2 * blockDim.x < n ? src[i + 2 * blockDim.x] : make_int4(0, 0, 0, 0);
    int4 d = i + 3 * blockDim.x < n ? src[i + 3 * blockDim.x] : make_int4(0, 0, 0, 0);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

__device__ __forceinline__ void bar_init(uint64_t *b) {
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)));
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t ph) {
  asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(
      (uint32_t)__cvta_generic_to_shared(b)), "r"(ph));
}

template <int CH, int ST>
__global__ void k_read_bulk(Peers P, int64_t slice, int *out) {
  __shared__ __align__(128) char buf[ST][CH];
  __shared__ __align__(8) uint64_t bar[ST];
  const int peer = peer_of(blockIdx.x, P);
  const int per_peer = gridDim.x / (P.n - 1), k = blockIdx.x / (P.n - 1);
  const int64_t share = slice / per_peer / CH * CH;
  const char *src = P.p[peer] + (int64_t)P.self * slice + k * share;
  const int nch = (int)(share / CH);
  if (threadIdx.x == 0) for (int s = 0; s < ST; s++) bar_init(&bar[s]);
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % ST;
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(buf[s])), "l"(src + (int64_t)c * CH), "r"(CH), "r"(a) : "memory");
  };
  if (threadIdx.x == 0) for (int c = 0; c < ST && c < nch; c++) issue(c);
  int acc = 0;
  for (int c = 0; c < nch; c++) {
    bar_wait(&bar[c % ST], (c / ST) & 1);
    acc ^= reinterpret_cast<int *>(buf[c % ST])[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + ST < nch) issue(c + ST);
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

// local source slice for peer q -> peer q's receive slice for self
__global__ void k_write_st(Peers P, const char *local, int64_t slice) {
  const int peer = peer_of(blockIdx.x, P);
  const int per_peer = gridDim.x / (P.n - 1), k = blockIdx.x / (P.n - 1);
  const int64_t share = slice / per_peer / 16 * 16;
  const int4 *src = reinterpret_cast<const int4 *>(local + (int64_t)peer * slice + k * share);
  int4 *dst = reinterpret_cast<int4 *>(P.p[peer] + (int64_t)P.self * slice + k * share);
  const int64_t n = share / 16;
  for (int64_t i = threadIdx.x; i < n; i += 4 * blockDim.x) {
    int4 a = src[i];
    int4 b = i + blockDim.x < n ? src[i + blockDim.x] : make_int4(0, 0, 0, 0);
    int4 c = i + 2 * blockDim.x < n ? src[i + 2 * blockDim.x] : make_int4(0, 0, 0, 0);
    int4 d = i + 3 * blockDim.x < n ? src[i + 3 * blockDim.x] : make_int4(0, 0, 0, 0);
    dst[i] = a;
    if (i + blockDim.x < n) dst[i + blockDim.x] = b;
    if (i + 2 * blockDim.x < n) dst[i + 2 * blockDim.x] = c;
    if (i + 3 * blockDim.x < n) dst[i + 3 * blockDim.x] = d;
  }
}

// TMA bulk: local HBM -> smem (load ring), smem -> peer HBM (bulk store, bulk_group waits)
template <int CH, int ST>
__global__ void k_write_bulk(Peers P, const char *local, int64_t slice) {
  __shared__ __align__(128) char buf[ST][CH];
  __shared__ __align__(8) uint64_t bar[ST];
  const int peer = peer_of(blockIdx.x, P);
  const int per_peer = gridDim.x / (P.n - 1), k = blockIdx.x / (P.n - 1);
  const int64_t share = slice / per_peer / CH * CH;
  const char *src = local + (int64_t)peer * slice + k * share;
  char *dst = P.p[peer] + (int64_t)P.self * slice + k * share;
  const int nch = (int)(share / CH);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ST; s++) bar_init(&bar[s]);
  asm volatile("fence.proxy.async.shared::cta;");
  auto issue = [&](int c) {
    const int s = c % ST;
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(buf[s])), "l"(src + (int64_t)c * CH), "r"(CH), "r"(a) : "memory");
  };
  for (int c = 0; c < ST / 2 && c < nch; c++) issue(c);
  for (int c = 0; c < nch; c++) {
    bar_wait(&bar[c % ST], (c / ST) & 1);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (int64_t)c * CH), "r"(
                     (uint32_t)__cvta_generic_to_shared(buf[c % ST])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    // the stage refilled next (c + ST/2) was stored ST/2 groups ago: allow ST/2 - 1 pending
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(ST / 2 - 1) : "memory");
    if (c + ST / 2 < nch) issue(c + ST / 2);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
  int n;
  CK(cudaGetDeviceCount(&n));
  if (argc > 1) n = atoi(argv[1]) < n ? atoi(argv[1]) : n;
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const int64_t slice = 256ll << 20;  // bytes per (GPU, peer) pair
  char *recv[kMax], *send[kMax];
  int *out[kMax];
  cudaStream_t st[kMax][kMax];
  cudaEvent_t e0[kMax], e1[kMax];
  for (int d = 0; d < n; d++) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < n; p++) if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&recv[d], slice * n));
    CK(cudaMalloc(&send[d], slice * n));
    CK(cudaMemset(recv[d], d + 1, slice * n));
    CK(cudaMemset(send[d], d + 7, slice * n));
    CK(cudaMalloc(&out[d], 64));
    for (int p = 0; p < n; p++) CK(cudaStreamCreateWithFlags(&st[d][p], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  const int64_t moved = slice * (n - 1);  // per GPU
  auto run = [&](const char *name, int mode, int ctas_per_sm) {
    float best = 1e9;
    for (int rep = 0; rep < 5; rep++) {
      for (int d = 0; d < n; d++) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < n; d++) {
        CK(cudaSetDevice(d));
        Peers P;
        P.n = n;
        P.self = d;
        for (int p = 0; p < n; p++) P.p[p] = (mode == 0 || mode == 1) ? send[p] : recv[p];
        const int grid = 148 * ctas_per_sm / (n - 1) * (n - 1);
        cudaStream_t s = st[d][0];
        CK(cudaEventRecord(e0[d], s));
        switch (mode) {
          case 0: k_read_ldg<<<grid, 256, 0, s>>>(P, slice, out[d]); break;
          case 1: k_read_bulk<8192, 4><<<grid, 128, 0, s>>>(P, slice, out[d]); break;
          case 2: k_write_st<<<grid, 256, 0, s>>>(P, send[d], slice); break;
          case 3: k_write_bulk<4096, 8><<<grid, 32, 0, s>>>(P, send[d], slice); break;
          case 4:
            for (int p = 0; p < n; p++) {
              if (p == d) continue;
              if (p != 0) { CK(cudaEventRecord(e1[d], s)); CK(cudaStreamWaitEvent(st[d][p], e1[d], 0)); }
            }
            for (int p = 0; p < n; p++) {
              if (p == d) continue;
              cudaStream_t sp = p == 0 ? s : st[d][p];
              CK(cudaMemcpyPeerAsync(recv[p] + (int64_t)d * slice, p, send[d] + (int64_t)p * slice, d, slice, sp));
            }
            for (int p = 1; p < n; p++) {
              if (p == d) continue;
              cudaEvent_t ev;
              CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
              CK(cudaEventRecord(ev, st[d][p]));
              CK(cudaStreamWaitEvent(s, ev, 0));
              CK(cudaEventDestroy(ev));
            }
            break;
        }
        CK(cudaEventRecord(e1[d], s));
      }
      float worst = 0;
      for (int d = 0; d < n; d++) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      if (rep > 0 && worst < best) best = worst;
    }
    printf("N=%d %-34s %8.1f GB/s per GPU\n", n, name, moved / best / 1e6);
  };
  run("read-ldg (8 CTA/SM)", 0, 8);
  run("read-bulk (4 CTA/SM)", 1, 4);
  run("read-bulk (8 CTA/SM)", 1, 8);
  run("write-st (4 CTA/SM)", 2, 4);
  run("write-st (8 CTA/SM)", 2, 8);
  run("write-bulk (4 CTA/SM)", 3, 4);
  run("write-bulk (8 CTA/SM)", 3, 8);
  run("ce", 4, 1);
  return 0;
}
