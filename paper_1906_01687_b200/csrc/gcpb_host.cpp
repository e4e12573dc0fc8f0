// gcpb_host.cpp — host-side halves of the narrowed model transfer.
//
// An fp32 engine rounds the host's fp64 model (the reference's KruskalModel is
// double, kruskal.hpp:16) to fp32 on arrival and widens it on the way out.  For
// models of hundreds of megabytes the PCIe copy is the whole cost of a
// host-buffer step (gcpb_step_host), so the rounding is done on the host, by
// several threads, chunk by chunk while the DMA of the previous chunks runs:
// half the bytes cross the bus.  The rounding is the device's own
// (round-to-nearest-even, cvtpd2ps under the default MXCSR = __double2float_rn),
// so the result is bit-identical to converting on the device.
#include <cstddef>
#include <cstdint>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace gcpb {

#if defined(__x86_64__)
__attribute__((target("avx2"))) static void narrow_avx2(const double* src, float* dst, size_t n) {
  size_t i = 0;
  // non-temporal stores need a 32-byte aligned destination
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u)) {
    dst[i] = static_cast<float>(src[i]);
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m128 lo = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i));
    const __m128 hi = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i + 4));
    _mm256_stream_ps(dst + i, _mm256_set_m128(hi, lo));
  }
  for (; i < n; ++i) dst[i] = static_cast<float>(src[i]);
  _mm_sfence();
}

__attribute__((target("avx2"))) static void widen_avx2(const float* src, double* dst, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u)) {
    dst[i] = static_cast<double>(src[i]);
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m256 v = _mm256_loadu_ps(src + i);
    _mm256_stream_pd(dst + i, _mm256_cvtps_pd(_mm256_castps256_ps128(v)));
    _mm256_stream_pd(dst + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)));
  }
  for (; i < n; ++i) dst[i] = static_cast<double>(src[i]);
  _mm_sfence();
}

static bool have_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}
#endif

// dst[i] = (float)src[i], round-to-nearest-even.
void narrow_f64_f32(const double* src, float* dst, size_t n) {
#if defined(__x86_64__)
  if (have_avx2()) {
    narrow_avx2(src, dst, n);
    return;
  }
#endif
  for (size_t i = 0; i < n; ++i) dst[i] = static_cast<float>(src[i]);
}

// dst[i] = (double)src[i] (exact).
void widen_f32_f64(const float* src, double* dst, size_t n) {
#if defined(__x86_64__)
  if (have_avx2()) {
    widen_avx2(src, dst, n);
    return;
  }
#endif
  for (size_t i = 0; i < n; ++i) dst[i] = static_cast<double>(src[i]);
}

}  // namespace gcpb
