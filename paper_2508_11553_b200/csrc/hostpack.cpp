// Host thread pool + 18-bit split-plane token packing (see hostpack.h).
#include "hostpack.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace tms {
namespace {

class Pool {
 public:
  explicit Pool(int nthreads) {
    for (int i = 1; i < nthreads; i++) th_.emplace_back([this] { worker(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_.store(true);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }

  // A job is fanned out to every worker; workers that finish keep polling for the next job
  // for a short while before they sleep, so the several parallel steps of one call (e.g. a
  // record batch's checks, staging and mirror) do not each pay a futex wake-up per thread.
  void run(int64_t n, const std::function<void(int64_t)> &fn) {
    std::lock_guard<std::mutex> one_job(call_mu_);
    if (th_.empty() || n <= 1) {
      for (int64_t i = 0; i < n; i++) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> l(mu_);
      job_ = &fn;
      n_ = n;
      next_.store(0);
      active_.store((int)th_.size(), std::memory_order_relaxed);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    drain();  // the calling thread works too
    for (int spin = 0; active_.load(std::memory_order_acquire) != 0; spin++) {
      if (spin < kSpin) {
        _mm_pause();
        continue;
      }
      std::unique_lock<std::mutex> l(mu_);
      done_cv_.wait(l, [&] { return active_.load(std::memory_order_acquire) == 0; });
    }
    job_ = nullptr;
  }

 private:
  static constexpr int kSpin = 1 << 14;  // ~50 us of polling before sleeping
  void drain() {
    for (int64_t i; (i = next_.fetch_add(1)) < n_;) (*job_)(i);
  }
  void worker() {
    uint64_t seen = 0;
    for (;;) {
      int spin = 0;
      while (gen_.load(std::memory_order_acquire) == seen && spin < kSpin) {
        _mm_pause();
        spin++;
      }
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_.load(std::memory_order_acquire) != seen; });
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      drain();
      if (active_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
        std::lock_guard<std::mutex> l(mu_);
        done_cv_.notify_all();
      }
    }
  }

  std::vector<std::thread> th_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)> *job_ = nullptr;
  std::atomic<int64_t> next_{0};
  int64_t n_ = 0;
  std::atomic<int> active_{0};
  std::atomic<uint64_t> gen_{0};
  std::atomic<bool> stop_{false};
};

Pool &pool() {
  static Pool p(host_threads());
  return p;
}

// 32 tokens -> 64 B of the low plane + 8 B of the high plane.  Returns a nonzero mask
// if any token is outside [0, 2^18).
__attribute__((target("avx2"))) inline __m256i pack32(const int32_t *src, uint16_t *lo, uint8_t *hi) {
  const __m256i m16 = _mm256_set1_epi32(0xFFFF);
  const __m256i a = _mm256_loadu_si256((const __m256i *)src), b = _mm256_loadu_si256((const __m256i *)(src + 8));
  const __m256i c = _mm256_loadu_si256((const __m256i *)(src + 16)), d = _mm256_loadu_si256((const __m256i *)(src + 24));
  const __m256i bad = _mm256_or_si256(_mm256_or_si256(_mm256_srli_epi32(a, 18), _mm256_srli_epi32(b, 18)),
                                      _mm256_or_si256(_mm256_srli_epi32(c, 18), _mm256_srli_epi32(d, 18)));
  // packus works per 128-bit lane; the qword permute restores position order
  const __m256i l0 = _mm256_permute4x64_epi64(_mm256_packus_epi32(_mm256_and_si256(a, m16), _mm256_and_si256(b, m16)), 0xD8);
  const __m256i l1 = _mm256_permute4x64_epi64(_mm256_packus_epi32(_mm256_and_si256(c, m16), _mm256_and_si256(d, m16)), 0xD8);
  _mm256_stream_si256((__m256i *)lo, l0);  // non-temporal: no read-for-ownership of the pinned plane
  _mm256_stream_si256((__m256i *)(lo + 16), l1);
  __m256i h = _mm256_or_si256(
      _mm256_or_si256(_mm256_srli_epi32(a, 16), _mm256_slli_epi32(_mm256_srli_epi32(b, 16), 2)),
      _mm256_or_si256(_mm256_slli_epi32(_mm256_srli_epi32(c, 16), 4), _mm256_slli_epi32(_mm256_srli_epi32(d, 16), 6)));
  h = _mm256_and_si256(h, _mm256_set1_epi32(0xFF));
  const __m256i h8 = _mm256_packus_epi16(_mm256_packus_epi32(h, h), _mm256_packus_epi32(h, h));
  const uint64_t hv = (uint64_t)(uint32_t)_mm256_extract_epi32(h8, 0) | ((uint64_t)(uint32_t)_mm256_extract_epi32(h8, 4) << 32);
  _mm_stream_si64((long long *)hi, (long long)hv);
  return bad;
}

// a partial last group (n < 32 tokens; the rest of the group is zero)
bool pack_tail(const int32_t *src, int64_t n, uint16_t *lo, uint8_t *hi) {
  uint32_t bad = 0;
  uint8_t hb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int l = 0; l < 32; l++) {
    const uint32_t t = l < n ? (uint32_t)src[l] : 0u;
    bad |= t >> 18;
    lo[l] = (uint16_t)t;
    hb[l & 7] |= (uint8_t)(((t >> 16) & 3) << (2 * (l >> 3)));
  }
  memcpy(hi, hb, 8);
  return bad == 0;
}

}  // namespace

__attribute__((target("avx2"))) bool pack_piece(const PackPiece &p, uint16_t *lo, uint8_t *hi) {
  const int64_t full = p.len / 32;
  __m256i bad = _mm256_setzero_si256();
  const int64_t g0 = p.dst / 32;
  for (int64_t g = 0; g < full; g++) bad = _mm256_or_si256(bad, pack32(p.src + 32 * g, lo + 32 * (g0 + g), hi + 8 * (g0 + g)));
  bool ok = _mm256_testz_si256(bad, bad);
  if (p.len % 32) ok &= pack_tail(p.src + 32 * full, p.len % 32, lo + 32 * (g0 + full), hi + 8 * (g0 + full));
  _mm_sfence();  // this thread's non-temporal stores land before it reports the piece done
  return ok;
}

__attribute__((target("avx2"))) static void copy_stream_avx2(char *dst, const char *src, size_t n) {
  size_t head = (32 - ((uintptr_t)dst & 31)) & 31;
  if (head > n) head = n;
  memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256((const __m256i *)(src + i)), b = _mm256_loadu_si256((const __m256i *)(src + i + 32));
    const __m256i c = _mm256_loadu_si256((const __m256i *)(src + i + 64)), d = _mm256_loadu_si256((const __m256i *)(src + i + 96));
    _mm256_stream_si256((__m256i *)(dst + i), a);
    _mm256_stream_si256((__m256i *)(dst + i + 32), b);
    _mm256_stream_si256((__m256i *)(dst + i + 64), c);
    _mm256_stream_si256((__m256i *)(dst + i + 96), d);
  }
  memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

void copy_stream(void *dst, const void *src, size_t n) {
  if (pack18_supported()) copy_stream_avx2((char *)dst, (const char *)src, n);
  else memcpy(dst, src, n);
}

bool pack18_supported() {
  static const bool ok = __builtin_cpu_supports("avx2");
  return ok;
}

int host_threads() {
  static const int n = [] {
    const char *e = getenv("TM_HOST_THREADS");
    // default: all cores up to 16 - packing is host-memory-bound, and more threads only
    // crowd the copy engine's reads (24-core box, c4 e2e: 0.57 M q/s at 24 threads, 0.60-0.61 at 16)
    int v = e ? atoi(e) : std::min(16, (int)std::thread::hardware_concurrency());
    return std::max(1, std::min(v, 64));
  }();
  return n;
}

void parallel_for(int64_t n, const std::function<void(int64_t)> &fn) { pool().run(n, fn); }

}  // namespace tms
