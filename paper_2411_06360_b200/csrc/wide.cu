// Exact wide-integer multiply: int64 activations whose column sums may exceed int32.
//
// The reference computes in fp64 (core.py:110-117 casts every vector), so it is exact for any
// integer vector whose partial sums stay below 2^53 (SPEC.md:276 promises |v| <= 2^20 at up to
// 2^20 rows).  The scatter kernel accumulates in int32, exact modulo 2^32: the result of a
// column is right whenever sum_r |v_r| <= 2^31 - 1 (every column result is bounded by it, and
// intermediate wraparound cancels in modular arithmetic).  Beyond that bound the product is
// linear in v, so v is split into L balanced base-2^s digit vectors (limbs)
//     v = sum_l d_l * 2^(s*l),   |d_l| <= 2^(s-1),   rows * 2^(s-1) <= 2^31 - 1,
// each limb runs through the int32 scatter kernel (exact: every limb's column sums fit), and
// the limb results recombine exactly in 128-bit integers:  out = sum_l r_l * 2^(s*l).
// fp64 results are the exact integer rounded once, so they equal the reference's whenever the
// reference itself is exact (every partial sum below 2^53).
// Fixed-point use (exp2 != 0): non-integer fp64 vectors staged as v_q = round(v * 2^exp2) (host
// staging picks exp2 so every nonzero |v| keeps >= 41 significant bits, csrc/host_stage.cpp);
// the result is the exact product of v_q rounded once and scaled by 2^-exp2.
#include <type_traits>

#include "common.cuh"

namespace rsr {

rsr_status multiply(const rsr_index_desc& d, const void* v, rsr_dtype vt, void* out, rsr_dtype ot, rsr_variant var,
                    rsr_form form, int b0, int b1, cudaStream_t s, const Publish* pub, bool* published,
                    bool independent);

namespace {

__global__ void limb_split_kernel(const int64_t* __restrict__ v, int64_t rows, int L, int s,
                                  int32_t* __restrict__ limbs) {
  const int64_t half = (int64_t)1 << (s - 1);
  const uint64_t mask = ((uint64_t)1 << s) - 1;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = v[r];
    for (int l = 0; l + 1 < L; ++l) {
      const int64_t dgt = (int64_t)(((uint64_t)x + (uint64_t)half) & mask) - half;  // balanced digit
      limbs[(int64_t)l * rows + r] = (int32_t)dgt;
      x = (int64_t)((uint64_t)x - (uint64_t)dgt) >> s;  // exact: x - dgt is a multiple of 2^s
    }
    limbs[(int64_t)(L - 1) * rows + r] = (int32_t)x;  // remainder, |x| <= 2^(s-1) by the host's L
  }
}

template <typename OutT>
__global__ void limb_combine_kernel(const int32_t* __restrict__ r, int64_t cols, int L, int s, int64_t c0, int64_t c1,
                                    double scale, OutT* __restrict__ out) {
  for (int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < c1; c += (int64_t)gridDim.x * blockDim.x) {
    __int128 acc = 0;
    for (int l = L - 1; l >= 0; --l) acc = acc * ((__int128)1 << s) + (__int128)r[(int64_t)l * cols + c];
    if constexpr (std::is_same<OutT, int64_t>::value) {  // int64: wraps like torch int64
      out[c] = (OutT)(int64_t)(uint64_t)acc;
    } else {
      const int64_t lo = (int64_t)acc;
      // one correctly rounded conversion, then the exact power-of-two scale (fixed-point inputs)
      if ((__int128)lo == acc) {
        out[c] = (OutT)((double)lo * scale);
      } else {  // beyond int64 (the reference is inexact there too)
        const int64_t hi = (int64_t)(acc >> 64);
        out[c] = (OutT)(((double)hi * 18446744073709551616.0 + (double)(uint64_t)acc) * scale);
      }
    }
  }
}

}  // namespace

// Digit width s: rows * 2^(s-1) <= 2^31 - 1.
int wide_digit_bits(int64_t rows) {
  int s = 1;
  while (s < 31 && (rows << s) <= (int64_t)INT32_MAX) ++s;  // rows * 2^(s) still fits -> s + 1 ok
  return s;
}

// Limbs needed for |v| <= max_abs (0: the whole int64 range).
int wide_limb_count(int64_t rows, uint64_t max_abs) {
  const int s = wide_digit_bits(rows);
  const uint64_t half = (uint64_t)1 << (s - 1);
  uint64_t b = max_abs ? max_abs : ((uint64_t)1 << 63);
  int L = 1;
  while (b > half) {  // remainder after one more balanced digit: |x'| <= |x| / 2^s + 1
    b = (b >> s) + 1;
    ++L;
  }
  return L;
}

size_t wide_workspace_bytes(const rsr_index_desc& d, uint64_t max_abs) {
  const int L = wide_limb_count(d.rows, max_abs);
  const size_t lb = ((size_t)L * d.rows * 4 + 255) & ~(size_t)255;
  return lb + (size_t)L * d.cols * 4;
}

rsr_status multiply_wide(const rsr_index_desc& d, const int64_t* v, uint64_t max_abs, void* out, rsr_dtype ot,
                         rsr_variant var, int b0, int b1, void* ws, size_t ws_bytes, cudaStream_t s, int exp2) {
  if (ot != RSR_I64 && ot != RSR_F64) return fail(RSR_ERR_INVALID, "int64 activations produce int64 or float64");
  if (exp2 != 0 && ot != RSR_F64) return fail(RSR_ERR_INVALID, "scaled (fixed-point) activations produce float64");
  if (exp2 < -1000 || exp2 > 1000) return fail(RSR_ERR_INVALID, "fixed-point exponent out of range");
  if (d.rows > ((int64_t)1 << 29)) return fail(RSR_ERR_UNSUPPORTED, "wide multiply supports at most 2^29 rows");
  if (b0 >= b1) return RSR_OK;
  if (!ws || ws_bytes < wide_workspace_bytes(d, max_abs)) return fail(RSR_ERR_INVALID, "wide multiply: workspace too small");
  const int sb = wide_digit_bits(d.rows);
  const int L = wide_limb_count(d.rows, max_abs);
  int32_t* limbs = reinterpret_cast<int32_t*>(ws);
  int32_t* res = reinterpret_cast<int32_t*>((char*)ws + (((size_t)L * d.rows * 4 + 255) & ~(size_t)255));
  const int sms = device_sm_count();
  limb_split_kernel<<<std::max<int64_t>(1, std::min<int64_t>(4 * sms, (d.rows + 255) / 256)), 256, 0, s>>>(v, d.rows, L,
                                                                                                        sb, limbs);
  rsr_status st = cuda_check(cudaGetLastError(), "limb_split_kernel launch");
  for (int l = 0; l < L && st == RSR_OK; ++l)
    st = multiply(d, limbs + (int64_t)l * d.rows, RSR_I32, res + (int64_t)l * d.cols, RSR_I32, var, RSR_FORM_AUTO, b0,
                  b1, s, nullptr, nullptr, false);
  if (st != RSR_OK) return st;
  const int64_t c0 = (int64_t)b0 * d.k, c1 = std::min<int64_t>(d.cols, (int64_t)b1 * d.k);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * sms, (c1 - c0 + 255) / 256));
  const double scale = exp2 == 0 ? 1.0 : ldexp(1.0, -exp2);
  if (ot == RSR_I64) limb_combine_kernel<int64_t><<<grid, 256, 0, s>>>(res, d.cols, L, sb, c0, c1, 1.0, (int64_t*)out);
  else limb_combine_kernel<double><<<grid, 256, 0, s>>>(res, d.cols, L, sb, c0, c1, scale, (double*)out);
  return cuda_check(cudaGetLastError(), "limb_combine_kernel launch");
}

}  // namespace rsr
