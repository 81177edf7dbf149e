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

// ---------------------------------------------------------------------------------------------
// int8-activation form (IDP4A): the comparator at HBM speed for the reference's own activation
// range (integers in [-100, 100], bench.py:85).  Q [ceil(rows / 16)][cols] u32: entry (row
// 16 r + 4 t + k, column j) is the 2-bit field t of byte k of Q[r][j], 01 = +1, 11 = -1, 00 = 0.
// Shifted to the top of its byte and masked, (Q << (6 - 2t)) & 0xC0C0C0C0 holds the four
// entries of rows 4t .. 4t + 3 as signed bytes 64 * a, so with those rows' int8 activations as
// one int8x4 word x_t,   acc += dp4a((Q << (6 - 2t)) & 0xC0C0C0C0, x_t)   over t and row groups
// gives 64 * sum a v exactly: one shift, one mask and one IDP4A per four matrix entries.
constexpr int kI8Threads = 128;
constexpr int kI8RowGroups = 32;  // 16-row groups per CTA (512 rows)

__global__ void dense_pack_i8_kernel(const int8_t* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                     uint32_t* __restrict__ Q, int32_t* bad) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = blockIdx.y;
  if (j >= cols) return;
  uint32_t q = 0;
  int badc = 0;
  for (int i = 0; i < 16; ++i) {
    const int64_t r = g * 16 + i;
    if (r >= rows) break;
    const int8_t a = A[r * lda + j];
    const int t = i >> 2, k = i & 3;
    q |= (uint32_t)(a != 0) << (8 * k + 2 * t);       // field t of byte k: 01 = +1, 11 = -1
    q |= (uint32_t)(a == -1) << (8 * k + 2 * t + 1);
    badc += (a < -1 || a > 1);
  }
  Q[g * cols + j] = q;
  if (badc) atomicAdd(bad, badc);
}

// Each thread owns 4 adjacent columns (one 16-byte load per 16-row group: a warp streams 512
// contiguous bytes), so one broadcast of the group's 16 activations (a 16-byte shared load, which
// costs a full data-pipe pass) serves 64 matrix entries.
__global__ void __launch_bounds__(kI8Threads) dense_gemv_i8_kernel(const uint32_t* __restrict__ Q, int64_t rows,
                                                                   int64_t cols, const int8_t* __restrict__ v,
                                                                   int32_t* __restrict__ out) {
  __shared__ __align__(16) uint32_t vs[kI8RowGroups * 4];  // int8x4 words, zero past the rows
  const int64_t g0 = (int64_t)blockIdx.y * kI8RowGroups;
  const int64_t ngroups = (rows + 15) / 16;
  const int ng = (int)((ngroups - g0) < kI8RowGroups ? (ngroups - g0) : kI8RowGroups);
  for (int i = threadIdx.x; i < kI8RowGroups * 4; i += blockDim.x) {
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t r = g0 * 16 + 4 * (int64_t)i + b;
      if (r < rows) w |= (uint32_t)(uint8_t)v[r] << (8 * b);
    }
    vs[i] = w;
  }
  __syncthreads();
  const int64_t j0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (j0 >= cols) return;
  const bool vec = (cols & 3) == 0 && j0 + 4 <= cols;  // 16-byte aligned rows of Q
  const uint32_t* qp = Q + g0 * cols + j0;
  int32_t acc[4] = {0, 0, 0, 0};  // 64 * partial sum per column
  constexpr int U = 4;  // 16-row groups in flight per thread
  for (int r0 = 0; r0 < ng; r0 += U) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t* p = qp + (int64_t)(r0 + u) * cols;
      if (r0 + u >= ng) q[u] = make_uint4(0, 0, 0, 0);
      else if (vec) q[u] = __ldg(reinterpret_cast<const uint4*>(p));
      else q[u] = make_uint4(__ldg(p), j0 + 1 < cols ? __ldg(p + 1) : 0u, j0 + 2 < cols ? __ldg(p + 2) : 0u,
                             j0 + 3 < cols ? __ldg(p + 3) : 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4 x = reinterpret_cast<const uint4*>(vs)[r0 + u];  // broadcast: the group's 16 activations
      const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
      const uint32_t qc[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[c] = __dp4a((int)((qc[c] << (6 - 2 * t)) & 0xC0C0C0C0u), (int)xs[t], acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (j0 + c >= cols) break;
    const int32_t y = acc[c] >> 6;  // exact: a multiple of 64
    if (gridDim.y == 1) out[j0 + c] = y;
    else atomicAdd(out + j0 + c, y);
  }
}

}  // namespace

size_t dense_i8_words(int64_t rows, int64_t cols) { return (size_t)((rows + 15) / 16) * (size_t)cols; }

rsr_status dense_pack_i8(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* Q, int32_t* bad,
                         cudaStream_t s) {
  if (!A || !Q || !bad || rows < 1 || cols < 1 || lda < cols) return fail(RSR_ERR_INVALID, "bad dense pack arguments");
  dim3 grid((unsigned)((cols + 255) / 256), (unsigned)((rows + 15) / 16));
  dense_pack_i8_kernel<<<grid, 256, 0, s>>>(A, lda, rows, cols, Q, bad);
  return cuda_check(cudaGetLastError(), "dense_pack_i8_kernel launch");
}

rsr_status dense_multiply_i8(const uint32_t* Q, int64_t rows, int64_t cols, const int8_t* v, int32_t* out,
                             cudaStream_t s) {
  if (!Q || !v || !out || rows < 1 || cols < 1) return fail(RSR_ERR_INVALID, "bad dense multiply arguments");
  dim3 grid((unsigned)((cols + 4 * kI8Threads - 1) / (4 * kI8Threads)),
            (unsigned)(((rows + 15) / 16 + kI8RowGroups - 1) / kI8RowGroups));
  if (grid.y > 1) {
    rsr_status st = cuda_check(cudaMemsetAsync(out, 0, cols * 4, s), "memset dense out");
    if (st != RSR_OK) return st;
  }
  dense_gemv_i8_kernel<<<grid, kI8Threads, 0, s>>>(Q, rows, cols, v, out);
  return cuda_check(cudaGetLastError(), "dense_gemv_i8_kernel launch");
}

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
