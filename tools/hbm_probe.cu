// Single-GPU HBM ceilings for the roofline discussion (tuning tool): pure LDG.128 read,
// pure STG.128 write, and an int4 copy over 4 GiB, best of 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_probe tools/hbm_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const int4 *__restrict__ p, long long n, int *out) {
  int acc = 0;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += 4 * st) {
    int4 a = p[i];
    int4 b = i + st < n ? p[i + st] : make_int4(0, 0, 0, 0);
    int4 c = i + 2 * st < n ? p[i + 2 * st] : make_int4(0, 0, 0, 0);
    int4 d = i + 3 * st < n ? p[i + 3 * st] : make_int4(0, 0, 0, 0);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

__global__ void k_write(int4 *__restrict__ p, long long n) {
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += st) p[i] = make_int4(i, 1, 2, 3);
}

__global__ void k_copy(const int4 *__restrict__ s, int4 *__restrict__ d, long long n) {
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += st) d[i] = s[i];
}

int main() {
  const long long bytes = 4ll << 30, n = bytes / 16;
  int4 *a, *b;
  int *o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&o, 64);
  cudaMemset(a, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, int which, double moved) {
    float best = 1e9;
    for (int r = 0; r < 6; r++) {
      cudaEventRecord(e0);
      if (which == 0) k_read<<<148 * 8, 256>>>(a, n, o);
      else if (which == 1) k_write<<<148 * 8, 256>>>(b, n);
      else k_copy<<<148 * 8, 256>>>(a, b, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    printf("%-28s %8.1f GB/s\n", name, moved / best / 1e6);
  };
  run("read  (LDG.128)", 0, (double)bytes);
  run("write (STG.128)", 1, (double)bytes);
  run("copy  (read+write bytes)", 2, 2.0 * bytes);
  return 0;
}
