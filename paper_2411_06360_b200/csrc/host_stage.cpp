// Host-side staging of a session vector: copy v into the pinned staging buffer and classify it
// in the same pass (csrc/host.cu).  Plain loops written for the compiler's AVX2 vectoriser
// (built with -O3 -march=x86-64-v3, like the oracle): the int32 pass is a copy plus an int64
// sum of |v|; the float64 pass converts to int32 and checks integrality on the way.
//
// Classes (see rsr_host_session_multiply in include/rsr_b200.h):
//   kStageI32   integer-valued, sum |v| <= 2^31 - 1: staged as int32, exact on the int32 kernel
//   kStageWide  integer-valued, |v| < 2^63 otherwise: staged as int64 for the wide multiply
//   kStageF32   float32, staged as is
//   kStageF64   float64 with a non-integer (or beyond-int64) entry, staged as is
//   kStageNonFinite   a NaN / inf entry (core.py:115 raises "vector entries must be finite")
#include "host_stage.h"

#include <immintrin.h>

#include <cmath>
#include <cstring>

namespace rsr {
namespace {

constexpr int64_t kI32Max = 2147483647;
constexpr double kTwo63 = 9223372036854775808.0;

uint64_t uabs64(int64_t x) { return x < 0 ? 0 - (uint64_t)x : (uint64_t)x; }

StageInfo stage_i32(const int32_t* __restrict__ src, int64_t n, void* dst, bool force_i32) {
  // pass 1: copy and max |v| (3 vector ops per 8 entries); max |v| * n <= 2^31 - 1 bounds the sum
  int32_t* __restrict__ d = static_cast<int32_t*>(dst);
  uint32_t mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t x = src[i];
    d[i] = x;
    const uint32_t a = x < 0 ? 0u - (uint32_t)x : (uint32_t)x;
    mx = a > mx ? a : mx;
  }
  if (force_i32 || (uint64_t)mx * (uint64_t)n <= (uint64_t)kI32Max) return {kStageI32, mx};
  int64_t sum = 0;  // pass 2 (large activations only): the exact bound
  for (int64_t i = 0; i < n; ++i) sum += src[i] < 0 ? -(int64_t)src[i] : (int64_t)src[i];
  if (sum <= kI32Max) return {kStageI32, mx};
  int64_t* __restrict__ w = static_cast<int64_t*>(dst);
  for (int64_t i = n - 1; i >= 0; --i) w[i] = src[i];  // widen (src is the caller's buffer)
  return {kStageWide, mx};
}

StageInfo stage_i64(const int64_t* __restrict__ src, int64_t n, void* dst) {
  uint64_t sum = 0, mx = 0;
  bool sat = false;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t a = uabs64(src[i]);
    mx = a > mx ? a : mx;
    const uint64_t t = sum + a;
    sat |= t < sum;
    sum = t;
  }
  if (!sat && sum <= (uint64_t)kI32Max) {
    int32_t* __restrict__ d = static_cast<int32_t*>(dst);
    for (int64_t i = 0; i < n; ++i) d[i] = (int32_t)src[i];
    return {kStageI32, mx};
  }
  std::memcpy(dst, src, (size_t)n * 8);
  return {kStageWide, mx};
}

StageInfo stage_f64(const double* __restrict__ src, int64_t n, void* dst) {
  // pass 1 (vectorised): clamp to the int32 range, truncate, and check that the round trip
  // gives x back (NaN / inf and non-integers fail it); sum of |int32 value| in int64
  int32_t* __restrict__ d = static_cast<int32_t*>(dst);
  int64_t i = 0;
  const __m256d lo = _mm256_set1_pd(-2147483647.0), hi = _mm256_set1_pd(2147483647.0);
  __m256d okv = _mm256_castsi256_pd(_mm256_set1_epi64x(-1));
  __m256i sumv = _mm256_setzero_si256();
  for (; i + 4 <= n; i += 4) {  // explicit AVX2: the compiler leaves this loop scalar
    const __m256d x = _mm256_loadu_pd(src + i);
    const __m128i ci = _mm256_cvttpd_epi32(_mm256_min_pd(_mm256_max_pd(x, lo), hi));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i), ci);
    okv = _mm256_and_pd(okv, _mm256_cmp_pd(_mm256_cvtepi32_pd(ci), x, _CMP_EQ_OQ));  // NaN: false
    sumv = _mm256_add_epi64(sumv, _mm256_cvtepu32_epi64(_mm_abs_epi32(ci)));
  }
  int ok = _mm256_movemask_pd(okv) == 0xf;
  alignas(32) int64_t part[4];
  _mm256_store_si256(reinterpret_cast<__m256i*>(part), sumv);
  int64_t sum = part[0] + part[1] + part[2] + part[3];
  for (; i < n; ++i) {
    const double x = src[i];
    double c = x < -2147483647.0 ? -2147483647.0 : x;
    c = c > 2147483647.0 ? 2147483647.0 : c;
    const int32_t ci = (int32_t)c;
    d[i] = ci;
    ok &= (double)ci == x;
    sum += ci < 0 ? -(int64_t)ci : (int64_t)ci;
  }
  if (ok && sum <= kI32Max) return {kStageI32, 0};
  // pass 2 (rare): finiteness, integrality in the int64 range, max |v|
  bool integral = true;
  uint64_t mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = src[i];
    if (!std::isfinite(x)) return {kStageNonFinite, 0};
    if (!(std::fabs(x) < kTwo63) || x != std::trunc(x)) {
      integral = false;
    } else {
      const uint64_t a = uabs64((int64_t)x);
      mx = a > mx ? a : mx;
    }
  }
  if (integral) {
    int64_t* __restrict__ w = static_cast<int64_t*>(dst);
    for (int64_t i = 0; i < n; ++i) w[i] = (int64_t)src[i];
    return {kStageWide, mx};
  }
  std::memcpy(dst, src, (size_t)n * 8);
  return {kStageF64, 0};
}

StageInfo stage_f32(const float* __restrict__ src, int64_t n, void* dst) {
  float* __restrict__ d = static_cast<float*>(dst);
  int finite = 1;
  for (int64_t i = 0; i < n; ++i) {
    const float x = src[i];
    d[i] = x;
    finite &= std::fabs(x) <= 3.402823466e38f;  // false for NaN and inf
  }
  return {finite ? kStageF32 : kStageNonFinite, 0};
}

}  // namespace

StageInfo stage_vector(const void* src, rsr_dtype t, int64_t n, void* dst, bool force_i32) {
  switch (t) {
    case RSR_I32: return stage_i32(static_cast<const int32_t*>(src), n, dst, force_i32);
    case RSR_I64: return stage_i64(static_cast<const int64_t*>(src), n, dst);
    case RSR_F64: return stage_f64(static_cast<const double*>(src), n, dst);
    case RSR_F32: return stage_f32(static_cast<const float*>(src), n, dst);
  }
  return {kStageNonFinite, 0};
}

}  // namespace rsr
