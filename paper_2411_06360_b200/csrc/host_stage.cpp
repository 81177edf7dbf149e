// Host-side staging of a session vector: copy v into the pinned staging buffer and classify it
// in the same pass (csrc/host.cu).  Plain loops written for the compiler's AVX2 vectoriser
// (built with -O3 -march=x86-64-v3, like the oracle): the int32 pass is a copy plus an int64
// sum of |v|; the float64 pass converts to int32 and checks integrality on the way.
//
// Classes (see rsr_host_session_multiply in include/rsr_b200.h):
//   kStageI32   integer-valued, sum |v| <= 2^31 - 1: staged as int32, exact on the int32 kernel
//   kStageWide  integer-valued, |v| < 2^63 otherwise: staged as int64 for the wide multiply
//   kStageF32   float32, staged as is
//   kStageFixed float64 with a non-integer entry, >= 8192 rows and max / min nonzero |v| <= 2^21: staged as the
//               int64 fixed point round(v * 2^e), |v_q| < 2^62 (exact integer product, rounded once)
//   kStageF64   other float64 (wider dynamic range, or beyond-int64 integers), staged as is
//   kStageNonFinite   a NaN / inf entry (core.py:115 raises "vector entries must be finite")
#include "host_stage.h"

#include <immintrin.h>

#include <cmath>
#include <algorithm>
#include <cstring>

namespace rsr {
namespace {

constexpr int64_t kI32Max = 2147483647;
constexpr double kTwo63 = 9223372036854775808.0;
constexpr int64_t kFixedMinRows = 8192;  // fixed point vs fp64 gather: 16384^2 156 vs 324 us, 4096^2 58 vs 51 us (e2e)

uint64_t uabs64(int64_t x) { return x < 0 ? 0 - (uint64_t)x : (uint64_t)x; }

StageInfo stage_i32(const int32_t* __restrict__ src, int64_t n, void* dst, bool force_i32) {
  // pass 1 (explicit AVX2, two accumulators): copy and max |v|; max |v| * n <= 2^31 - 1 bounds
  // the sum (|INT32_MIN| reads as 2^31 unsigned, so it never passes)
  int32_t* __restrict__ d = static_cast<int32_t*>(dst);
  int64_t i = 0;
  __m256i m0 = _mm256_setzero_si256(), m1 = m0;
  for (; i + 16 <= n; i += 16) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 8));
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(d + i + 8), b);
    m0 = _mm256_max_epu32(m0, _mm256_abs_epi32(a));
    m1 = _mm256_max_epu32(m1, _mm256_abs_epi32(b));
  }
  alignas(32) uint32_t mm[8];
  _mm256_store_si256(reinterpret_cast<__m256i*>(mm), _mm256_max_epu32(m0, m1));
  uint32_t mx = 0;
  for (int e = 0; e < 8; ++e) mx = mm[e] > mx ? mm[e] : mx;
  for (; i < n; ++i) {
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
  // pass 1 (explicit AVX2, two accumulators; the compiler leaves this loop scalar): truncate to
  // int32 and check that the round trip gives x back — NaN, inf, non-integers and values outside
  // the int32 range (truncated to INT32_MIN) fail it, except x = -2^31 itself, whose |v| reads as
  // 2^31 below; max |int32 value| bounds the sum
  int32_t* __restrict__ d = static_cast<int32_t*>(dst);
  int64_t i = 0;
  __m256d ok0 = _mm256_castsi256_pd(_mm256_set1_epi64x(-1)), ok1 = ok0;
  __m128i mx0 = _mm_setzero_si128(), mx1 = mx0;
  for (; i + 8 <= n; i += 8) {
    const __m256d x0 = _mm256_loadu_pd(src + i), x1 = _mm256_loadu_pd(src + i + 4);
    const __m128i c0 = _mm256_cvttpd_epi32(x0), c1 = _mm256_cvttpd_epi32(x1);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(d + i), _mm256_set_m128i(c1, c0));
    ok0 = _mm256_and_pd(ok0, _mm256_cmp_pd(_mm256_cvtepi32_pd(c0), x0, _CMP_EQ_OQ));  // NaN: false
    ok1 = _mm256_and_pd(ok1, _mm256_cmp_pd(_mm256_cvtepi32_pd(c1), x1, _CMP_EQ_OQ));
    mx0 = _mm_max_epu32(mx0, _mm_abs_epi32(c0));
    mx1 = _mm_max_epu32(mx1, _mm_abs_epi32(c1));
  }
  int ok = _mm256_movemask_pd(_mm256_and_pd(ok0, ok1)) == 0xf;
  alignas(16) uint32_t mm[4];
  _mm_store_si128(reinterpret_cast<__m128i*>(mm), _mm_max_epu32(mx0, mx1));
  uint32_t mx = 0;
  for (int e = 0; e < 4; ++e) mx = mm[e] > mx ? mm[e] : mx;
  for (; i < n; ++i) {
    const double x = src[i];
    const int32_t ci = _mm_cvttsd_si32(_mm_set_sd(x));  // INT32_MIN out of range, like cvttpd
    d[i] = ci;
    ok &= (double)ci == x;
    const uint32_t a = ci < 0 ? 0u - (uint32_t)ci : (uint32_t)ci;
    mx = a > mx ? a : mx;
  }
  if (ok) {
    if ((uint64_t)mx * (uint64_t)n <= (uint64_t)kI32Max) return {kStageI32, mx};
    int64_t sum = 0;  // large activations: the exact bound over the staged int32 values
    for (int64_t j = 0; j < n; ++j) sum += d[j] < 0 ? -(int64_t)d[j] : (int64_t)d[j];
    if (sum <= kI32Max) return {kStageI32, mx};
  }
  // pass 2 (non-integer or large values; explicit AVX2, branch-free): finiteness, max |v|, the
  // smallest nonzero |v|, integrality in the int64 range
  const __m256d absmask = _mm256_castsi256_pd(_mm256_set1_epi64x(0x7fffffffffffffffLL));
  const __m256d inf = _mm256_set1_pd(HUGE_VAL), two63 = _mm256_set1_pd(kTwo63), zero = _mm256_setzero_pd();
  __m256d vmax = zero, vmin = inf, fin = _mm256_castsi256_pd(_mm256_set1_epi64x(-1)), integ = fin;
  int64_t j = 0;
  for (; j + 4 <= n; j += 4) {
    const __m256d x = _mm256_loadu_pd(src + j);
    const __m256d a = _mm256_and_pd(x, absmask);
    fin = _mm256_and_pd(fin, _mm256_cmp_pd(a, inf, _CMP_LT_OQ));  // NaN, inf: false
    vmax = _mm256_max_pd(vmax, a);
    vmin = _mm256_min_pd(vmin, _mm256_blendv_pd(inf, a, _mm256_cmp_pd(a, zero, _CMP_GT_OQ)));
    integ = _mm256_and_pd(integ, _mm256_and_pd(_mm256_cmp_pd(_mm256_round_pd(x, _MM_FROUND_TO_ZERO | _MM_FROUND_NO_EXC), x,
                                                             _CMP_EQ_OQ),
                                               _mm256_cmp_pd(a, two63, _CMP_LT_OQ)));
  }
  alignas(32) double mx4[4], mn4[4];
  _mm256_store_pd(mx4, vmax);
  _mm256_store_pd(mn4, vmin);
  bool finite = _mm256_movemask_pd(fin) == 0xf, integral = _mm256_movemask_pd(integ) == 0xf;
  double amax = std::max(std::max(mx4[0], mx4[1]), std::max(mx4[2], mx4[3]));
  double amin = std::min(std::min(mn4[0], mn4[1]), std::min(mn4[2], mn4[3]));
  for (; j < n; ++j) {
    const double x = src[j], a = std::fabs(x);
    finite &= a < HUGE_VAL;
    amax = a > amax ? a : amax;
    if (a > 0 && a < amin) amin = a;
    integral &= a < kTwo63 && x == std::trunc(x);
  }
  if (!finite) return {kStageNonFinite, 0};
  if (integral) {
    int64_t* __restrict__ w = static_cast<int64_t*>(dst);
    for (int64_t i = 0; i < n; ++i) w[i] = (int64_t)src[i];
    return {kStageWide, (uint64_t)amax};  // exact: an integer below 2^63
  }
  // fixed point: v_q = round(v * 2^e) with |v_q| < 2^62 when max / min nonzero |v| <= 2^21, so
  // every nonzero entry keeps >= 40 significant bits (relative error <= 2^-41 per entry); the
  // product is then exact in integers (rsr_multiply_fixed) and rounded once
  // (>= 8192 rows: below that the fp64 gather kernel is faster than the 4 limb launches)
  if (n >= kFixedMinRows && amax > 0 && amax <= amin * 2097152.0) {
    const int e = 61 - std::ilogb(amax);  // amax * 2^e < 2^62
    // y = x * 2^e as two exact power-of-two multiplies (2^e alone may overflow a double); the
    // int64 round-to-nearest-even of y as hi * 2^32 + lo (AVX2 has no double -> int64):
    // hi = floor(y / 2^32) (|hi| < 2^30), lo = y - hi * 2^32 in [0, 2^32) exactly, rounded
    const int e1 = e / 2, e2 = e - e1;
    const double s1 = std::ldexp(1.0, e1), s2 = std::ldexp(1.0, e2);
    const __m256d vs1 = _mm256_set1_pd(s1), vs2 = _mm256_set1_pd(s2);
    const __m256d t32 = _mm256_set1_pd(4294967296.0), it32 = _mm256_set1_pd(1.0 / 4294967296.0),
                  t31 = _mm256_set1_pd(2147483648.0), one = _mm256_set1_pd(1.0);
    const __m256i t31i = _mm256_set1_epi64x(2147483648LL);
    int64_t* __restrict__ w = static_cast<int64_t*>(dst);
    int64_t i = 0;
    for (; i + 4 <= n; i += 4) {
      const __m256d y = _mm256_mul_pd(_mm256_mul_pd(_mm256_loadu_pd(src + i), vs1), vs2);
      __m256d hi = _mm256_floor_pd(_mm256_mul_pd(y, it32));
      __m256d lo = _mm256_round_pd(_mm256_sub_pd(y, _mm256_mul_pd(hi, t32)), _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
      const __m256d carry = _mm256_cmp_pd(lo, t32, _CMP_EQ_OQ);  // lo rounded up to 2^32
      hi = _mm256_add_pd(hi, _mm256_and_pd(carry, one));
      lo = _mm256_andnot_pd(carry, lo);
      const __m256i hi64 = _mm256_slli_epi64(_mm256_cvtepi32_epi64(_mm256_cvtpd_epi32(hi)), 32);
      const __m256i lo64 = _mm256_add_epi64(_mm256_cvtepi32_epi64(_mm256_cvtpd_epi32(_mm256_sub_pd(lo, t31))), t31i);
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(w + i), _mm256_add_epi64(hi64, lo64));
    }
    for (; i < n; ++i) w[i] = _mm_cvtsd_si64(_mm_set_sd(src[i] * s1 * s2));  // round-to-nearest-even
    StageInfo r{kStageFixed, (uint64_t)_mm_cvtsd_si64(_mm_set_sd(amax * s1 * s2))};  // max |v_q| (monotone rounding)
    r.exp2 = e;
    return r;
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
