// Host->device token path probe (tuning tool): can host-side packing of int32 token ids
// into 18-bit split planes (uint16 low plane + 2-bit high plane) beat the raw PCIe copy?
// Measures (1) raw pinned H2D, (2) AVX2 pack throughput with T threads, (3) the pipelined
// pack -> H2D -> unpack path end to end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -mavx2,-fopenmp -o tools/pcie_pack_probe tools/pcie_pack_probe.cu
#include <immintrin.h>
#include <omp.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// 32 tokens -> 64 B low plane + 8 B high plane (byte j: tokens j, j+8, j+16, j+24 at bits 0,2,4,6)
template <bool NT = true>
static inline bool pack32(const int32_t *src, uint16_t *lo, uint8_t *hi) {
  const __m256i m16 = _mm256_set1_epi32(0xFFFF);
  __m256i a = _mm256_loadu_si256((const __m256i *)src), b = _mm256_loadu_si256((const __m256i *)(src + 8));
  __m256i c = _mm256_loadu_si256((const __m256i *)(src + 16)), d = _mm256_loadu_si256((const __m256i *)(src + 24));
  __m256i bad = _mm256_or_si256(_mm256_or_si256(_mm256_srli_epi32(a, 18), _mm256_srli_epi32(b, 18)),
                                _mm256_or_si256(_mm256_srli_epi32(c, 18), _mm256_srli_epi32(d, 18)));
  __m256i l0 = _mm256_permute4x64_epi64(_mm256_packus_epi32(_mm256_and_si256(a, m16), _mm256_and_si256(b, m16)), 0xD8);
  __m256i l1 = _mm256_permute4x64_epi64(_mm256_packus_epi32(_mm256_and_si256(c, m16), _mm256_and_si256(d, m16)), 0xD8);
  if (NT) {
    _mm256_stream_si256((__m256i *)lo, l0);  // non-temporal: no read-for-ownership of the pinned buffer
    _mm256_stream_si256((__m256i *)(lo + 16), l1);
  } else {
    _mm256_store_si256((__m256i *)lo, l0);
    _mm256_store_si256((__m256i *)(lo + 16), l1);
  }
  __m256i h = _mm256_or_si256(_mm256_or_si256(_mm256_srli_epi32(a, 16), _mm256_slli_epi32(_mm256_srli_epi32(b, 16), 2)),
                              _mm256_or_si256(_mm256_slli_epi32(_mm256_srli_epi32(c, 16), 4), _mm256_slli_epi32(_mm256_srli_epi32(d, 16), 6)));
  h = _mm256_and_si256(h, _mm256_set1_epi32(0xFF));
  __m256i h16 = _mm256_packus_epi32(h, h);      // lanes: [h0..h3 h0..h3 | h4..h7 h4..h7] as u16
  __m256i h8 = _mm256_packus_epi16(h16, h16);   // bytes
  uint32_t x0 = (uint32_t)_mm256_extract_epi32(h8, 0), x1 = (uint32_t)_mm256_extract_epi32(h8, 4);
  uint64_t hv = (uint64_t)x0 | ((uint64_t)x1 << 32);
  if (NT) _mm_stream_si64((long long *)hi, (long long)hv);
  else memcpy(hi, &hv, 8);
  return _mm256_testz_si256(bad, bad);
}

__global__ void k_unpack(const uint16_t *lo, const uint8_t *hi, int32_t *out, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = p >> 5;
    const int l = (int)(p & 31);
    const uint32_t h = (hi[g * 8 + (l & 7)] >> (2 * (l >> 3))) & 3;
    out[p] = (int32_t)(lo[p] | (h << 16));
  }
}

int main(int argc, char **argv) {
  const int64_t n = 120LL << 20;  // 125.8 M tokens = 503 MB
  const int64_t chunk = argc > 1 ? atoll(argv[1]) << 20 : 4LL << 20;
  int32_t *src;
  uint16_t *lo;
  uint8_t *hi;
  CK(cudaHostAlloc(&src, n * 4, 0));
  CK(cudaHostAlloc(&lo, n * 2, 0));
  CK(cudaHostAlloc(&hi, n / 4, 0));
  {
    std::mt19937 rng(1);
    #pragma omp parallel for
    for (int64_t i = 0; i < n; i++) src[i] = (int32_t)((uint64_t)(i * 2654435761ULL) % 151936);
  }
  int32_t *d_tok;
  uint16_t *d_lo;
  uint8_t *d_hi;
  CK(cudaMalloc(&d_tok, n * 4));
  CK(cudaMalloc(&d_lo, n * 2));
  CK(cudaMalloc(&d_hi, n / 4));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // (1) raw H2D
  for (int r = 0; r < 3; r++) {
    double t0 = now();
    CK(cudaMemcpyAsync(d_tok, src, n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    double dt = now() - t0;
    printf("raw H2D: %.2f ms  %.1f GB/s  %.2f Gtok/s\n", dt * 1e3, n * 4 / dt / 1e9, n / dt / 1e9);
  }
  // (2) pack alone
  int maxt = (int)std::thread::hardware_concurrency();
  printf("hardware threads: %d\n", maxt);
  for (int T : {1, 4, 8, 16, maxt}) {
    if (T > maxt) continue;
    omp_set_num_threads(T);
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      double t0 = now();
      int okall = 1;
      #pragma omp parallel for schedule(static) reduction(& : okall)
      for (int64_t g = 0; g < n / 32; g++) okall &= pack32(src + g * 32, lo + g * 32, hi + g * 8);
      double dt = now() - t0;
      if (dt < best) best = dt;
      if (!okall) printf("bad!\n");
    }
    printf("pack T=%d: %.2f ms  %.2f Gtok/s  (read %.1f GB/s)\n", T, best * 1e3, n / best / 1e9, n * 4 / best / 1e9);
  }
  // (3) pipelined: pack chunk k+1 on T threads while chunk k is copied; unpack on device
  for (int T : {8, 16, maxt}) {
    if (T > maxt) continue;
    omp_set_num_threads(T);
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      CK(cudaDeviceSynchronize());
      double t0 = now();
      std::vector<cudaEvent_t> ev;
      for (int64_t c0 = 0; c0 < n; c0 += chunk) {
        const int64_t c1 = std::min(n, c0 + chunk);
        #pragma omp parallel for schedule(static)
        for (int64_t g = c0 / 32; g < c1 / 32; g++) pack32(src + g * 32, lo + g * 32, hi + g * 8);
        _mm_sfence();
        CK(cudaMemcpyAsync(d_lo + c0, lo + c0, (c1 - c0) * 2, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_hi + c0 / 4, hi + c0 / 4, (c1 - c0) / 4, cudaMemcpyHostToDevice, s));
        k_unpack<<<1184, 256, 0, s>>>(d_lo + c0, d_hi + c0 / 4, d_tok + c0, c1 - c0);
      }
      CK(cudaStreamSynchronize(s));
      double dt = now() - t0;
      if (dt < best) best = dt;
    }
    printf("pipelined pack+H2D+unpack T=%d chunk=%lld: %.2f ms  %.2f Gtok/s\n", T, (long long)chunk, best * 1e3, n / best / 1e9);
  }
  // (4) ring of small pinned slots reused while hot in the LLC (regular stores): the DMA may
  // read the packed planes from cache instead of DRAM
  for (int nt = 0; nt < 2; nt++)
  for (int64_t slot_tok : {int64_t(1) << 19, int64_t(1) << 20, int64_t(2) << 20}) {
    const int nslot = 6;
    omp_set_num_threads(maxt);
    uint16_t *rlo; uint8_t *rhi;
    CK(cudaHostAlloc(&rlo, 2 * slot_tok * nslot, 0));
    CK(cudaHostAlloc(&rhi, slot_tok / 4 * nslot, 0));
    cudaEvent_t evs[nslot];
    for (auto &ev_ : evs) CK(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      CK(cudaDeviceSynchronize());
      double t0 = now();
      int64_t c = 0;
      for (int64_t c0 = 0; c0 < n; c0 += slot_tok, c++) {
        const int64_t c1 = std::min(n, c0 + slot_tok);
        const int sl = (int)(c % nslot);
        if (c >= nslot) CK(cudaEventSynchronize(evs[sl]));
        uint16_t *lo_s = rlo + sl * slot_tok; uint8_t *hi_s = rhi + sl * (slot_tok / 4);
        if (nt) {
          #pragma omp parallel for schedule(static)
          for (int64_t g = c0 / 32; g < c1 / 32; g++) pack32<true>(src + g * 32, lo_s + (g * 32 - c0), hi_s + (g * 8 - c0 / 4));
          _mm_sfence();
        } else {
          #pragma omp parallel for schedule(static)
          for (int64_t g = c0 / 32; g < c1 / 32; g++) pack32<false>(src + g * 32, lo_s + (g * 32 - c0), hi_s + (g * 8 - c0 / 4));
        }
        CK(cudaMemcpyAsync(d_lo + c0, lo_s, (c1 - c0) * 2, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_hi + c0 / 4, hi_s, (c1 - c0) / 4, cudaMemcpyHostToDevice, s));
        k_unpack<<<1184, 256, 0, s>>>(d_lo + c0, d_hi + c0 / 4, d_tok + c0, c1 - c0);
        CK(cudaEventRecord(evs[sl], s));
      }
      CK(cudaStreamSynchronize(s));
      double dt = now() - t0;
      if (dt < best) best = dt;
    }
    printf("ring %s stores slot=%lldK x %d: %.2f ms  %.2f Gtok/s\n", nt ? "NT" : "regular", (long long)(slot_tok >> 10), nslot,
           best * 1e3, n / best / 1e9);
  }
  // check
  std::vector<int32_t> back(1 << 20);
  CK(cudaMemcpy(back.data(), d_tok + n - (1 << 20), 4 << 20, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < (1 << 20); i++) bad += back[i] != src[n - (1 << 20) + i];
  printf("mismatches: %d\n", bad);
  return 0;
}
