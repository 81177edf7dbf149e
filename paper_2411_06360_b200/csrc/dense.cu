// Dense ternary GEMV on B200 — the paper's "standard" multiply (core.py:135-169 naive_multiply,
// PAPER.md:679-699) as an honest GPU comparator for the RSR++ path.
//
// The matrix is stored as two bit-planes (2 bits per entry, 1/4 of int8): P[w][j] and N[w][j]
// hold bit i of rows 32w + i of column j being +1 / -1.  Layout [rows/32][cols]: the 32
// lanes of a warp own 32 consecutive output columns and read one coalesced 128-byte word row
// per 32 matrix rows.  y_j = sum_i v_i (P_ij - N_ij): every lane walks the 32 rows of a word
// against v staged in shared memory (broadcast reads), so the kernel is bound by the ~4
// integer instructions per matrix entry, not by the 2-bit bytes.  Rows are split across CTAs
// (partial column sums combined with exact int32 / fp32 atomics into a zeroed output).
#include "common.cuh"

namespace rsr {

namespace {

constexpr int kDenseThreads = 256;   // 8 warps = 256 columns per CTA
constexpr int kDenseRowChunk = 512;  // rows per CTA (16 words)

__global__ void dense_pack_kernel(const int8_t* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                  uint32_t* __restrict__ P, uint32_t* __restrict__ N, int32_t* bad) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t w = blockIdx.y;
  if (j >= cols) return;
  uint32_t p = 0, n = 0;
  int badc = 0;
  for (int i = 0; i < 32; ++i) {
    const int64_t r = w * 32 + i;
    if (r >= rows) break;
    const int8_t a = A[r * lda + j];
    p |= (uint32_t)(a == 1) << i;
    n |= (uint32_t)(a == -1) << i;
    badc += (a < -1 || a > 1);
  }
  P[w * cols + j] = p;
  N[w * cols + j] = n;
  if (badc) atomicAdd(bad, badc);
}

template <typename T>
__device__ __forceinline__ T from_u32(uint32_t x) {
  if constexpr (sizeof(T) == 4 && T(0.5) != T(0)) return __uint_as_float(x);
  else return (T)(int32_t)x;
}

// acc + (bits & mask ? x : 0) as one bit-test predicate and one predicated add
__device__ __forceinline__ int32_t pred_add(int32_t acc, int32_t x, uint32_t bits, uint32_t mask) {
  asm("{\n\t.reg .pred q;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.u32 q, t, 0;\n\t@q add.s32 %0, %0, %1;\n\t}"
      : "+r"(acc) : "r"(x), "r"(bits), "r"(mask));
  return acc;
}
__device__ __forceinline__ float pred_add(float acc, float x, uint32_t bits, uint32_t mask) {
  asm("{\n\t.reg .pred q;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.u32 q, t, 0;\n\t@q add.f32 %0, %0, %1;\n\t}"
      : "+f"(acc) : "f"(x), "r"(bits), "r"(mask));
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(kDenseThreads) dense_gemv_kernel(const uint32_t* __restrict__ P,
                                                                   const uint32_t* __restrict__ N, int64_t rows,
                                                                   int64_t cols, const T* __restrict__ v,
                                                                   T* __restrict__ out) {
  __shared__ __align__(16) T vs[kDenseRowChunk];
  const int64_t r0 = (int64_t)blockIdx.y * kDenseRowChunk;
  const int nr = (int)((rows - r0) < kDenseRowChunk ? (rows - r0) : kDenseRowChunk);
  for (int i = threadIdx.x; i < kDenseRowChunk; i += blockDim.x) vs[i] = i < nr ? v[r0 + i] : T(0);
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const int nw = (nr + 31) / 32;
  const int64_t w0 = r0 / 32;
  T accp = T(0), accn = T(0);
  const uint32_t* pp = P + w0 * cols + j;
  const uint32_t* np_ = N + w0 * cols + j;
  uint32_t p = __ldg(pp), n = __ldg(np_);
  for (int w = 0; w < nw; ++w) {
    // next word's planes a word ahead
    const uint32_t pn = w + 1 < nw ? __ldg(pp + (int64_t)(w + 1) * cols) : 0u;
    const uint32_t nn = w + 1 < nw ? __ldg(np_ + (int64_t)(w + 1) * cols) : 0u;
    const uint4* v4 = reinterpret_cast<const uint4*>(vs + w * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 x4 = v4[q];  // 4 activations, broadcast (16-byte shared load)
      const T xs[4] = {from_u32<T>(x4.x), from_u32<T>(x4.y), from_u32<T>(x4.z), from_u32<T>(x4.w)};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * q + e;
        accp = pred_add(accp, xs[e], p, 1u << i);  // bit test -> predicate -> predicated add
        accn = pred_add(accn, xs[e], n, 1u << i);
      }
    }
    p = pn;
    n = nn;
  }
  const T acc = accp - accn;
  if (gridDim.y == 1) out[j] = acc;
  else atomicAdd(out + j, acc);
}

}  // namespace

size_t dense_plane_words(int64_t rows, int64_t cols) { return (size_t)((rows + 31) / 32) * (size_t)cols; }

rsr_status dense_pack_ternary(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* P, uint32_t* N,
                              int32_t* bad, cudaStream_t s) {
  if (!A || !P || !N || !bad || rows < 1 || cols < 1 || lda < cols) return fail(RSR_ERR_INVALID, "bad dense pack arguments");
  dim3 grid((unsigned)((cols + 255) / 256), (unsigned)((rows + 31) / 32));
  dense_pack_kernel<<<grid, 256, 0, s>>>(A, lda, rows, cols, P, N, bad);
  return cuda_check(cudaGetLastError(), "dense_pack_kernel launch");
}

rsr_status dense_multiply(const uint32_t* P, const uint32_t* N, int64_t rows, int64_t cols, const void* v,
                          rsr_dtype dt, void* out, cudaStream_t s) {
  if (!P || !N || !v || !out || rows < 1 || cols < 1) return fail(RSR_ERR_INVALID, "bad dense multiply arguments");
  dim3 grid((unsigned)((cols + kDenseThreads - 1) / kDenseThreads), (unsigned)((rows + kDenseRowChunk - 1) / kDenseRowChunk));
  const size_t osz = dt == RSR_F32 ? 4 : 4;
  if (grid.y > 1) {
    rsr_status st = cuda_check(cudaMemsetAsync(out, 0, cols * osz, s), "memset dense out");
    if (st != RSR_OK) return st;
  }
  if (dt == RSR_I32)
    dense_gemv_kernel<int32_t><<<grid, kDenseThreads, 0, s>>>(P, N, rows, cols, (const int32_t*)v, (int32_t*)out);
  else if (dt == RSR_F32)
    dense_gemv_kernel<float><<<grid, kDenseThreads, 0, s>>>(P, N, rows, cols, (const float*)v, (float*)out);
  else
    return fail(RSR_ERR_UNSUPPORTED, "dense multiply takes int32 or fp32 activations");
  return cuda_check(cudaGetLastError(), "dense_gemv_kernel launch");
}

}  // namespace rsr
