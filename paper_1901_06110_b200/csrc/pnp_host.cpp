// Host-side float casts of the numpy drop-in path (the reference's call shape
// is float64 numpy in, float64 numpy out; the device computes in fp32).
//
// The casts are host-memory-bandwidth bound and sit on the critical path of a
// synchronous call: the result's f32 -> f64 cast runs after the device has
// finished (band by band as the download lands).  Plain stores of the f64
// result read every destination line before writing it (read for ownership),
// 1.5x the bytes; these loops use AVX2 conversions with non-temporal stores
// and a small persistent worker pool, so a band costs the bytes it moves.
// Rounding is the hardware's round-to-nearest-even, i.e. bit-identical to a
// C cast / torch's copy_.
#include <immintrin.h>
#include <stdint.h>
#include <unistd.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "pnp_b200.h"

namespace {

class Pool {
 public:
  explicit Pool(int n) : pid_(getpid()) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return (int)workers_.size() + 1; }
  // run fn(part) for part in [0, parts) on the caller + workers; returns when all are done
  void run(int parts, const std::function<void(int)>& fn) {
    if (getpid() != pid_) {  // a forked child has no workers: run inline
      for (int p = 0; p < parts; ++p) fn(p);
      return;
    }
    std::unique_lock<std::mutex> call(call_m_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(m_);
      fn_ = &fn;
      parts_ = parts;
      pending_ = std::min(parts, size()) - 1;
      ++gen_;
    }
    cv_.notify_all();
    for (int p = 0; p < parts; p += size()) fn(p);
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* fn;
      int parts;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        fn = fn_;
        parts = parts_;
      }
      if (id >= parts) continue;  // not part of this job
      for (int p = id; p < parts; p += size()) (*fn)(p);
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  const pid_t pid_;
  std::vector<std::thread> workers_;
  std::mutex m_, call_m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int parts_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool p(std::max(0, std::min(63, (int)std::thread::hardware_concurrency() - 1)));
  return p;
}

__attribute__((target("avx2"))) void f32_to_f64_avx2(const float* s, double* d, int64_t n) {
  int64_t i = 0;
  // scalar head until the destination is 32-byte aligned (stream stores)
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
  for (; i + 8 <= n; i += 8) {
    const __m256 v = _mm256_loadu_ps(s + i);
    _mm256_stream_pd(d + i, _mm256_cvtps_pd(_mm256_castps256_ps128(v)));
    _mm256_stream_pd(d + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)));
  }
  for (; i < n; ++i) d[i] = s[i];
  _mm_sfence();
}

__attribute__((target("avx2"))) void f64_to_f32_avx2(const double* s, float* d, int64_t n) {
  int64_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = (float)s[i];
  for (; i + 8 <= n; i += 8) {
    const __m128 lo = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i));
    const __m128 hi = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i + 4));
    _mm256_stream_ps(d + i, _mm256_set_m128(hi, lo));
  }
  for (; i < n; ++i) d[i] = (float)s[i];
  _mm_sfence();
}

template <class S, class D>
void cast_scalar(const S* s, D* d, int64_t n) {
  for (int64_t i = 0; i < n; ++i) d[i] = (D)s[i];
}

template <class S, class D>
int cast(const S* s, D* d, int64_t n, int nthreads, void (*vec)(const S*, D*, int64_t)) {
  if (n < 0 || (n && (!s || !d))) return PNP_EINVAL;
  if (n == 0) return PNP_OK;
  static const bool avx2 = __builtin_cpu_supports("avx2");
  Pool& p = pool();
  int parts = nthreads > 0 ? nthreads : p.size();
  // at least 256 K elements per part: small bands are not worth a wake-up
  parts = (int)std::max<int64_t>(1, std::min<int64_t>(parts, n >> 18));
  const int64_t per = ((n + parts - 1) / parts + 7) & ~int64_t(7);
  p.run(parts, [&](int k) {
    const int64_t a = std::min(n, k * per), b = std::min(n, a + per);
    if (b <= a) return;
    if (avx2) vec(s + a, d + a, b - a);
    else cast_scalar(s + a, d + a, b - a);
  });
  return PNP_OK;
}

__attribute__((target("avx2"))) void zero_avx2(const double*, double* d, int64_t n) {
  int64_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = 0.0;
  const __m256d z = _mm256_setzero_pd();
  for (; i + 4 <= n; i += 4) _mm256_stream_pd(d + i, z);
  for (; i < n; ++i) d[i] = 0.0;
  _mm_sfence();
}

void zero_scalar(const double*, double* d, int64_t n) {
  for (int64_t i = 0; i < n; ++i) d[i] = 0.0;
}

}  // namespace

extern "C" int pnp_host_zero_f64(double* dst, int64_t n, int nthreads) {
  if (n < 0 || (n && !dst)) return PNP_EINVAL;
  if (n == 0) return PNP_OK;
  static const bool avx2 = __builtin_cpu_supports("avx2");
  Pool& p = pool();
  int parts = nthreads > 0 ? nthreads : p.size();
  parts = (int)std::max<int64_t>(1, std::min<int64_t>(parts, n >> 18));
  const int64_t per = ((n + parts - 1) / parts + 7) & ~int64_t(7);
  p.run(parts, [&](int k) {
    const int64_t a = std::min(n, k * per), b = std::min(n, a + per);
    if (b > a) (avx2 ? zero_avx2 : zero_scalar)(nullptr, dst + a, b - a);
  });
  return PNP_OK;
}

extern "C" int pnp_host_cast_f32_f64(const float* src, double* dst, int64_t n, int nthreads) {
  return cast<float, double>(src, dst, n, nthreads, f32_to_f64_avx2);
}

extern "C" int pnp_host_cast_f64_f32(const double* src, float* dst, int64_t n, int nthreads) {
  return cast<double, float>(src, dst, n, nthreads, f64_to_f32_avx2);
}
