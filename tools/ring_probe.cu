// Routed-walk access-pattern probe (tuning tool): a CTA streams "queries" through a ring of
// TMA stages the way k_walk_routed does for a remote query - per stage a low-plane bulk
// copy (2 B/position) and a high-plane bulk copy (0.25 B/position) from the PEER GPU plus
// the history chunk (4 B/position) from local HBM - with both GPUs doing it at once.
// Reports peer-plane GB/s per GPU for ring shapes, CTAs per SM, and whether the high plane
// travels as its own request or is fused with the low plane (one request per stage).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ring_probe tools/ring_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(bar)) : "memory");
}

// each CTA streams `per` positions of the peer planes (and local history) from its own
// contiguous range; query boundaries every QLEN positions add a stage-drain (like a new
// query's ring restart)
template <int S, int CH, bool FUSED, bool LOCAL>
__global__ void k_ring(const char *peer_planes, const int *local_hist, int64_t per, int qlen, int *out) {
  extern __shared__ __align__(16) char sm[];
  constexpr int LO = 2 * CH, HI = CH / 4, A = 4 * CH;
  char *lo = sm;                    // S x LO (FUSED: S x (LO + HI))
  char *hi = lo + S * (LO + HI);    // unused when fused
  char *a = hi + S * HI;            // S x A
  uint64_t *bar = reinterpret_cast<uint64_t *>(a + S * A);
  const int64_t base = (int64_t)blockIdx.x * per;
  if (threadIdx.x == 0)
    for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  int acc = 0;
  uint32_t ch = 0;
  for (int64_t q0 = 0; q0 + qlen <= per; q0 += qlen) {
    const int nch = qlen / CH;
    auto issue = [&](int c) {
      const int s = (int)((ch + c) % S);
      const int64_t p = base + q0 + (int64_t)c * CH;
      const uint32_t bytes = (FUSED ? LO + HI : LO + HI) + (LOCAL ? A : 0);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(bytes) : "memory");
      if (FUSED) {
        g2s(lo + s * (LO + HI), peer_planes + p / CH * (LO + HI), LO + HI, &bar[s]);
      } else {
        g2s(lo + s * LO, peer_planes + 2 * p, LO, &bar[s]);
        g2s(hi + s * HI, peer_planes + (int64_t)2 * (1ll << 30) + p / 4, HI, &bar[s]);
      }
      if (LOCAL) g2s(a + s * A, local_hist + p % ((1ll << 28) - CH), A, &bar[s]);
    };
    if (threadIdx.x == 0)
      for (int c = 0; c < S && c < nch; c++) issue(c);
    for (int c = 0; c < nch; c++) {
      const int s = (int)((ch + c) % S);
      const uint32_t ph = ((ch + c) / S) & 1;
      asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(sa(&bar[s])),
                   "r"(ph) : "memory");
      acc ^= reinterpret_cast<const int *>(lo + s * LO)[threadIdx.x];
      if (LOCAL) acc ^= reinterpret_cast<const int *>(a + s * A)[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0 && c + S < nch) issue(c + S);
    }
    ch += nch;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

int main() {
  int n;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const int64_t pbytes = 3ll << 30;  // planes: lo [0, 2 GB), hi [2 GB, 2.5 GB)
  char *planes[2];
  int *hist[2], *out[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; d++) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&planes[d], pbytes));
    CK(cudaMemset(planes[d], d + 1, pbytes));
    CK(cudaMalloc(&hist[d], 4ll << 28));
    CK(cudaMemset(hist[d], 0, 4ll << 28));
    CK(cudaMalloc(&out[d], 64));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  auto run = [&](const char *name, auto kern, int S, int CH, bool fused, bool local, int ctas_per_sm, int qlen) {
    const size_t smem = (size_t)S * (2 * CH + 2 * (CH / 4) + 4 * CH) + 8 * S + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = 148 * ctas_per_sm;
    const int64_t total = 512ll << 20;  // positions per GPU
    const int64_t per = total / grid / qlen * qlen;
    float best = 1e9;
    for (int rep = 0; rep < 4; rep++) {
      for (int d = 0; d < 2; d++) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        kern<<<grid, 64, smem, st[d]>>>(planes[1 - d], hist[d], per, qlen, out[d]);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[d], st[d]));
      }
      float worst = 0;
      for (int d = 0; d < 2; d++) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      if (rep > 0 && worst < best) best = worst;
    }
    const double pos = (double)per * grid;
    printf("%-44s S=%d CH=%5d %s %s %d CTA/SM qlen=%6d: planes %6.1f GB/s per GPU (local %6.1f GB/s)\n", name, S, CH,
           fused ? "fused" : "split", local ? "+hist" : "     ", ctas_per_sm, qlen, pos * 2.25 / best / 1e6,
           local ? pos * 4 / best / 1e6 : 0.0);
  };
  run("walk-like", k_ring<4, 1024, false, true>, 4, 1024, false, true, 6, 32768);
  run("walk-like, planes only", k_ring<4, 1024, false, false>, 4, 1024, false, false, 6, 32768);
  run("fused request", k_ring<4, 1024, true, true>, 4, 1024, true, true, 6, 32768);
  for (int ql : {16384, 4096, 2048, 1024}) {
    run("walk-like", k_ring<4, 1024, false, true>, 4, 1024, false, true, 6, ql);
    run("fused request", k_ring<4, 1024, true, true>, 4, 1024, true, true, 6, ql);
  }
  return 0;
}
