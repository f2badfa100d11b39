// Per-call latency floor probe (tuning tool): what one small synchronous GPU round trip
// costs on this box, for the drop-in's per-request path (lpm_insert -> tm_record_one).
//   a  empty kernel + cudaStreamSynchronize
//   b  H2D 1 KB + kernel + D2H 1 KB + sync (today's tm_record_one shape)
//   c  kernel reading its input from and writing its output to mapped pinned host memory + sync
//   d  (b) as a CUDA graph (one cudaGraphLaunch) + sync
//   e  persistent kernel polling a pinned mailbox; host writes a request, spins on the reply
//   f  as (c) with a spin-wait on a host flag instead of cudaStreamSynchronize
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency_probe tools/latency_probe.cu
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_empty() {}
__global__ void k_touch(const int *in, int *out, int n) {
  int i = threadIdx.x;
  if (i < n) out[i] = in[i] + 1;
}
__global__ void k_touch_flag(const int *in, int *out, int n, volatile int *flag, int seq) {
  int i = threadIdx.x;
  if (i < n) out[i] = in[i] + 1;
  __syncthreads();
  if (i == 0) { __threadfence_system(); *flag = seq; }
}
// mailbox: req[0] = sequence number written last by the host; reply[0] = sequence when done
__global__ void k_worker(volatile int *req, const int *in, int *out, volatile int *reply, int n) {
  int seen = 0;
  for (;;) {
    __shared__ int s;
    if (threadIdx.x == 0) {
      int v;
      do { v = req[0]; } while (v == seen);
      s = v;
    }
    __syncthreads();
    const int v = s;
    if (v < 0) return;
    if ((int)threadIdx.x < n) out[threadIdx.x] = ((volatile const int *)in)[threadIdx.x] + v;
    __syncthreads();
    if (threadIdx.x == 0) { __threadfence_system(); reply[0] = v; }
    seen = v;
    __syncthreads();
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaSetDeviceFlags(cudaDeviceMapHost));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int n = 256, bytes = n * 4;
  int *h_in, *h_out, *d_in, *d_out;
  CK(cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d_in, bytes));
  CK(cudaMalloc(&d_out, bytes));
  int *m_in, *m_out;
  CK(cudaHostGetDevicePointer(&m_in, h_in, 0));
  CK(cudaHostGetDevicePointer(&m_out, h_out, 0));
  for (int i = 0; i < n; i++) h_in[i] = i;
  const int R = 2000;
  auto report = [&](const char *name, std::vector<double> &t) {
    std::sort(t.begin(), t.end());
    printf("%-62s p50 %6.2f us  p10 %6.2f  p90 %6.2f\n", name, t[t.size() / 2], t[t.size() / 10], t[t.size() * 9 / 10]);
  };
  std::vector<double> t(R);
  for (int r = 0; r < R; r++) {
    double t0 = now_us();
    k_empty<<<1, 32, 0, st>>>();
    cudaStreamSynchronize(st);
    t[r] = now_us() - t0;
  }
  report("a empty kernel + sync", t);
  for (int r = 0; r < R; r++) {
    double t0 = now_us();
    cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, st);
    k_touch<<<1, 256, 0, st>>>(d_in, d_out, n);
    cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    t[r] = now_us() - t0;
  }
  report("b H2D + kernel + D2H + sync", t);
  for (int r = 0; r < R; r++) {
    double t0 = now_us();
    k_touch<<<1, 256, 0, st>>>(m_in, m_out, n);
    cudaStreamSynchronize(st);
    t[r] = now_us() - t0;
  }
  report("c kernel on mapped pinned in/out + sync", t);
  {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, st);
    k_touch<<<1, 256, 0, st>>>(d_in, d_out, n);
    cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, st);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int r = 0; r < R; r++) {
      double t0 = now_us();
      cudaGraphLaunch(ge, st);
      cudaStreamSynchronize(st);
      t[r] = now_us() - t0;
    }
    report("d graph(H2D + kernel + D2H) + sync", t);
  }
  {
    int *h_flag, *m_flag;
    CK(cudaHostAlloc(&h_flag, 64, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&m_flag, h_flag, 0));
    *(volatile int *)h_flag = 0;
    for (int r = 0; r < R; r++) {
      double t0 = now_us();
      k_touch_flag<<<1, 256, 0, st>>>(m_in, m_out, n, m_flag, r + 1);
      while (*(volatile int *)h_flag != r + 1) {}
      t[r] = now_us() - t0;
    }
    cudaStreamSynchronize(st);
    report("f kernel on mapped pinned + host spin on a flag", t);
  }
  {
    int *h_req, *h_rep, *m_req, *m_rep;
    CK(cudaHostAlloc(&h_req, 64, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h_rep, 64, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&m_req, h_req, 0));
    CK(cudaHostGetDevicePointer(&m_rep, h_rep, 0));
    *(volatile int *)h_req = 0;
    *(volatile int *)h_rep = 0;
    cudaStream_t ws;
    CK(cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking));
    k_worker<<<1, 256, 0, ws>>>(m_req, m_in, d_out, m_rep, n);
    for (int r = 0; r < R; r++) {
      double t0 = now_us();
      h_in[0] = r;
      __atomic_store_n(h_req, r + 1, __ATOMIC_RELEASE);
      while (*(volatile int *)h_rep != r + 1) {}
      t[r] = now_us() - t0;
    }
    __atomic_store_n(h_req, -1, __ATOMIC_RELEASE);
    CK(cudaStreamSynchronize(ws));
    report("e persistent worker, pinned mailbox round trip", t);
  }
  return 0;
}
