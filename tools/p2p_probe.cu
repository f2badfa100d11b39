// NVLink read-path probe (tuning tool): bandwidth of reading a peer GPU's HBM with
// (a) LDG.128 from SMs, (b) cp.async.bulk (TMA 1-D bulk) into shared memory,
// (c) the copy engine (cudaMemcpyPeerAsync), and local HBM reads for reference;
// one direction and both directions at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe tools/p2p_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ldg(const int4 *__restrict__ p, int64_t n, int *out) {
  int acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x * 4) {
    int4 a = p[i];
    int4 b = i + (int64_t)gridDim.x * blockDim.x < n ? p[i + (int64_t)gridDim.x * blockDim.x] : make_int4(0,0,0,0);
    int4 c = i + 2 * (int64_t)gridDim.x * blockDim.x < n ? p[i + 2 * (int64_t)gridDim.x * blockDim.x] : make_int4(0,0,0,0);
    int4 d = i + 3 * (int64_t)gridDim.x * blockDim.x < n ? p[i + 3 * (int64_t)gridDim.x * blockDim.x] : make_int4(0,0,0,0);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

// each CTA streams its contiguous share with a 4-stage ring of 16 KB bulk copies
__global__ void k_bulk(const char *p, int64_t bytes, int *out) {
  constexpr int STAGES = 4, CH = 8192;
  __shared__ __align__(128) char buf[STAGES][CH];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const int64_t per = (bytes / gridDim.x) / CH * CH;
  const char *base = p + blockIdx.x * per;
  const int nch = (int)(per / CH);
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; s++) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
    }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  int acc = 0;
  auto issue = [&](int c) {
    int s = c % STAGES;
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(base + (int64_t)c * CH), "r"(CH), "r"(a) : "memory");
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < STAGES && c < nch; c++) issue(c);
  for (int c = 0; c < nch; c++) {
    int s = c % STAGES;
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t phase = (c / STAGES) & 1;
    asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(a), "r"(phase));
    acc ^= reinterpret_cast<int *>(buf[s])[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + STAGES < nch) issue(c + STAGES);
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

int main() {
  int n;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const int64_t bytes = 1ll << 30;
  char *buf[2];
  int *out[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; d++) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d], bytes));
    CK(cudaMemset(buf[d], d + 1, bytes));
    CK(cudaMalloc(&out[d], 64));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  char *tmp[2];
  for (int d = 0; d < 2; d++) { CK(cudaSetDevice(d)); CK(cudaMalloc(&tmp[d], bytes)); }
  auto run = [&](const char *name, int mode, bool both, bool remote, int grid_mult) -> int {
    float best = 1e9;
    for (int rep = 0; rep < 4; rep++) {
      int ndev = both ? 2 : 1;
      for (int d = 0; d < ndev; d++) {
        CK(cudaSetDevice(d));
        const char *src = remote ? buf[1 - d] : buf[d];
        CK(cudaEventRecord(e0[d], st[d]));
        if (mode == 0) k_ldg<<<148 * grid_mult, 256, 0, st[d]>>>((const int4 *)src, bytes / 16, out[d]);
        else if (mode == 1) k_bulk<<<148 * grid_mult, 128, 0, st[d]>>>(src, bytes, out[d]);
        else CK(cudaMemcpyPeerAsync(tmp[d], d, src, remote ? 1 - d : d, bytes, st[d]));
        CK(cudaEventRecord(e1[d], st[d]));
      }
      float worst = 0;
      for (int d = 0; d < ndev; d++) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      if (rep > 0 && worst < best) best = worst;
    }
    printf("%-40s %8.1f GB/s per GPU\n", name, bytes / best / 1e6);
    return 0;
  };
  run("local LDG.128 read", 0, false, false, 8);
  run("local bulk read", 1, false, false, 4);
  run("peer LDG.128 read, one direction", 0, false, true, 8);
  run("peer LDG.128 read, one dir, 16x grid", 0, false, true, 16);
  run("peer bulk read, one direction", 1, false, true, 4);
  run("peer bulk read, one dir, 8x grid", 1, false, true, 8);
  run("peer copy engine, one direction", 2, false, true, 1);
  run("peer LDG.128 read, both directions", 0, true, true, 8);
  run("peer bulk read, both directions", 1, true, true, 4);
  run("peer copy engine, both directions", 2, true, true, 1);
  return 0;
}
