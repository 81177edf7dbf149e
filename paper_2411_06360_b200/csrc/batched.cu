// Batched multiply: B activation vectors against ONE index (BASELINE config "ternary
// 16384x16384, batch of 64 activation vectors (index-read amortisation)").
//
// Gather form of the reference's per-vector hot loop (`_segment_sums` + `_product_fold`,
// kernels.py:50-91, driven per vector by `multiply_ternary`, kernels.py:196-206), turned
// inside out so that every index byte is read once per batch instead of once per vector:
//
//  * V [B][rows] is transposed once into VT [rows][ld] (ld = B padded to the slice width),
//    a few MB that stay resident in the 126 MB L2.
//  * One CTA per (column block, slice of 32*VW vectors); its 8 warps split the block's 2^w
//    buckets.  A warp walks its buckets' sorted positions (u16/u32 perm, coalesced), and for
//    each position every lane adds VW values of the row VT[perm[p]] — one 32*VW*4-byte row
//    gather per position serves the whole slice, so the index is read once per slice.
//  * The RSR++ fold (Alg. 3, kernels.py:74-91) is applied on the fly to the running prefix
//    sum S: when bucket j ends, the bits that turn off between j and j+1 add S to their
//    output column and the bit that turns on subtracts it (telescoping of sum_j u_j bit_c(j),
//    about two adds per bucket); variant "rsr" instead adds each finished bucket sum u_j to
//    every column whose bit is set (the dense product, kernels.py:63-71).
//  * Both halves of a ternary index run in the same warp (the negative half subtracts), the
//    8 warps' partial columns are summed in a fixed order through shared memory, and each
//    output element is written exactly once: deterministic, no atomics.
// Bound: the L2 -> SM row gathers (2 halves x rows x 32*VW*4 bytes per block and slice);
// tools/microbench/l2_rows.cu measures 13-14 TB/s for 256-byte rows on B200.
#include <type_traits>

#include "common.cuh"

namespace rsr {

namespace {

constexpr int kBatchWarps = 8;
constexpr int kBatchChunk = 16;  // row gathers in flight per warp
constexpr int kMaxW = 16;

template <typename T, int VW>
struct Lanes {
  T x[VW];
};

template <typename T>
__device__ __forceinline__ T from_bits(int x) {
  if constexpr (std::is_same<T, float>::value) return __int_as_float(x);
  else return x;
}

template <typename T, int VW>
__device__ __forceinline__ Lanes<T, VW> load_lanes(const T* p) {
  Lanes<T, VW> r;
  if constexpr (VW == 1) {
    r.x[0] = __ldg(p);
  } else if constexpr (VW == 2) {
    const int2 q = __ldg(reinterpret_cast<const int2*>(p));
    r.x[0] = from_bits<T>(q.x);
    r.x[1] = from_bits<T>(q.y);
  } else {
    const int4 q = __ldg(reinterpret_cast<const int4*>(p));
    r.x[0] = from_bits<T>(q.x);
    r.x[1] = from_bits<T>(q.y);
    r.x[2] = from_bits<T>(q.z);
    r.x[3] = from_bits<T>(q.w);
  }
  return r;
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ V, int64_t rows, int64_t batch, T* __restrict__ VT, int64_t ld) {
  __shared__ T tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, b0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t b = b0 + i, r = r0 + threadIdx.x;
    tile[i][threadIdx.x] = (b < batch && r < rows) ? V[b * rows + r] : T(0);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, b = b0 + threadIdx.x;
    if (r < rows && b < ld) VT[r * ld + b] = tile[threadIdx.x][i];
  }
}

struct BatchParams {
  const void* perm[2];
  const uint32_t* seg[2];
  const void* vt;
  void* out;
  int64_t rows, cols, row_stride, seg_stride, ld, batch;
  int k, halves;
  int b_begin;  // first column block of the launch (grid.x covers [b_begin, b_begin + grid.x))
};

template <typename T, int VW, bool FOLDPP, bool PERM16>
__global__ void __launch_bounds__(kBatchWarps * 32) batched_kernel(const BatchParams p) {
  using PermT = typename std::conditional<PERM16, uint16_t, uint32_t>::type;
  extern __shared__ __align__(16) unsigned char bsm[];
  const int b = p.b_begin + (int)blockIdx.x, slice = blockIdx.y;
  const int w = block_width(p.cols, p.k, b);
  const int nbk = 1 << w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* seg_s = reinterpret_cast<uint32_t*>(bsm);  // [halves][nbk + 1]
  const uint32_t* seg0 = p.seg[0];  // (no dynamic indexing of the parameter arrays)
  const uint32_t* seg1 = p.seg[1];
  const void* perm0 = p.perm[0];
  const void* perm1 = p.perm[1];
  for (int j = threadIdx.x; j <= nbk; j += blockDim.x) {
    seg_s[j] = seg0[(int64_t)b * p.seg_stride + j];
    if (p.halves == 2) seg_s[nbk + 1 + j] = seg1[(int64_t)b * p.seg_stride + j];
  }
  __syncthreads();

  // warp w takes positions [q0, q1) of each half: an even split of the rows (bucket sizes
  // are skewed: with P(bit) = 1/3 the first eighth of the buckets holds ~30% of the rows)
  // Work split: each half's positions are cut into kPieces * 8 equal pieces and warp w takes
  // pieces w, w + 8, ...: bucket density varies along the sorted order (dense low keys,
  // sparse high keys with a boundary every ~2 positions), interleaving evens it out.
  constexpr int kPieces = 4;
  const T* vt = reinterpret_cast<const T*>(p.vt) + (int64_t)slice * 32 * VW + lane * VW;
  T R[kMaxW][VW];  // R[bit][.]: bit b of the bucket index <-> output column w - 1 - b
#pragma unroll
  for (int c = 0; c < kMaxW; ++c)
#pragma unroll
    for (int e = 0; e < VW; ++e) R[c][e] = T(0);

  const uint32_t ld = (uint32_t)p.ld;  // host guarantees rows * ld < 2^32
  for (int hp = 0; hp < p.halves * kPieces; ++hp) {
    const int h = hp / kPieces, piece = (hp % kPieces) * kBatchWarps + warp;
    const int64_t q0 = p.rows * piece / (kPieces * kBatchWarps);
    const int64_t q1 = p.rows * (piece + 1) / (kPieces * kBatchWarps);
    if (q0 >= q1) continue;
    const uint32_t sg_base = smem_u32(seg_s) + (uint32_t)(h * (nbk + 1)) * 4u;
    auto sg = [&](int jj) -> uint32_t {  // shared-space load (no generic address math)
      uint32_t x;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(sg_base + (uint32_t)jj * 4u));
      return x;
    };
    const PermT* pm = reinterpret_cast<const PermT*>(h ? perm1 : perm0) + (int64_t)b * p.row_stride;
    const bool neg = h == 1;
    // bucket holding position q0: sg[j] <= q0 < sg[j + 1]
    int j = 0;
    {
      int hi = nbk;
      while (hi - j > 1) {
        const int mid = (j + hi) >> 1;
        if (sg(mid) <= (uint32_t)q0) j = mid;
        else hi = mid;
      }
    }
    uint32_t nbnd = sg(j + 1);  // end position of bucket j
    T S[VW], S0[VW];  // running prefix of this warp's positions; prefix at the bucket start
#pragma unroll
    for (int e = 0; e < VW; ++e) S[e] = S0[e] = T(0);
    // A bucket ends at position q with the prefix Sb: move from bucket j to the bucket j2
    // holding q (the buckets in between are empty).  RSR++: the run of every bit set in j
    // but not j2 closes (+Sb), every bit set in j2 but not j opens (-Sb); the bits of a warp's
    // first bucket open at S = 0 and its last bucket closes all its bits, so runs split
    // across warps (or halves of a bucket) add up exactly.  RSR: the finished bucket sum
    // u_j = Sb - S0 is added to the column of every set bit.
    auto advance = [&](uint32_t q, const T (&Sb)[VW]) {
      int j2 = j + 1;
      while (sg(j2 + 1) <= q) ++j2;  // skip empty buckets (uniform)
      if constexpr (FOLDPP) {
        const uint32_t off = (uint32_t)j & ~(uint32_t)j2, on = (uint32_t)j2 & ~(uint32_t)j;
        const uint32_t any = off | on;
#pragma unroll
        for (int c = 0; c < kMaxW; ++c) {
          if ((any >> c) == 0u) break;
          if ((any >> c) & 1u)
#pragma unroll
            for (int e = 0; e < VW; ++e) R[c][e] += ((off >> c) & 1u) ? Sb[e] : -Sb[e];
        }
      } else {
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          const T u = Sb[e] - S0[e];
          S0[e] = Sb[e];
#pragma unroll
          for (int c = 0; c < kMaxW; ++c)
            if (((uint32_t)j >> c) & 1u) R[c][e] += u;
        }
      }
      j = j2;
      nbnd = sg(j2 + 1);
    };
    for (int64_t base = q0; base < q1; base += 32) {
      const int cnt = (int)(q1 - base < 32 ? q1 - base : 32);
      const uint32_t myp = lane < cnt ? (uint32_t)pm[base + lane] : 0u;  // padding: row 0
#pragma unroll 1
      for (int c0 = 0; c0 < cnt; c0 += kBatchChunk) {
        Lanes<T, VW> L[kBatchChunk];
#pragma unroll
        for (int i = 0; i < kBatchChunk; ++i) {
          const uint32_t r = __shfl_sync(0xffffffffu, myp, c0 + i);
          L[i] = load_lanes<T, VW>(vt + (size_t)(r * ld));
        }
        const int valid = cnt - c0 < kBatchChunk ? cnt - c0 : kBatchChunk;
        if (valid < kBatchChunk)  // the warp's last chunk: drop the padding rows
#pragma unroll
          for (int i = 0; i < kBatchChunk; ++i)
            if (i >= valid)
#pragma unroll
              for (int e = 0; e < VW; ++e) L[i].x[e] = T(0);
        // chunk prefix sums in place: L[i] = x_0 + ... + x_i (signed by the half)
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          if (neg) L[0].x[e] = -L[0].x[e];
#pragma unroll
          for (int i = 1; i < kBatchChunk; ++i) L[i].x[e] = neg ? L[i - 1].x[e] - L[i].x[e] : L[i - 1].x[e] + L[i].x[e];
        }
        // buckets ending inside the chunk (position nbnd starts the next one): one compact
        // handler, the prefix at the boundary picked with a 4-level select tree
        const uint32_t qb = (uint32_t)(base + c0);
        while (nbnd < qb + (uint32_t)valid) {
          const int o = (int)(nbnd - qb);  // chunk positions [0, o) belong to bucket j
          T Sb[VW];
#pragma unroll
          for (int e = 0; e < VW; ++e) {
            const int id = o - 1;
            T a[8], c4[4], c2[2];
#pragma unroll
            for (int t = 0; t < 8; ++t) a[t] = (id & 1) ? L[2 * t + 1].x[e] : L[2 * t].x[e];
#pragma unroll
            for (int t = 0; t < 4; ++t) c4[t] = (id & 2) ? a[2 * t + 1] : a[2 * t];
#pragma unroll
            for (int t = 0; t < 2; ++t) c2[t] = (id & 4) ? c4[2 * t + 1] : c4[2 * t];
            const T pref = (id & 8) ? c2[1] : c2[0];
            Sb[e] = o > 0 ? S[e] + pref : S[e];
          }
          advance(nbnd, Sb);
        }
#pragma unroll
        for (int e = 0; e < VW; ++e) S[e] += L[kBatchChunk - 1].x[e];
      }
    }
    // close the bucket holding the warp's last position
    if constexpr (FOLDPP) {
#pragma unroll
      for (int c = 0; c < kMaxW; ++c)
        if (((uint32_t)j >> c) & 1u)
#pragma unroll
          for (int e = 0; e < VW; ++e) R[c][e] += S[e];
    } else {
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        const T u = S[e] - S0[e];
#pragma unroll
        for (int c = 0; c < kMaxW; ++c)
          if (((uint32_t)j >> c) & 1u) R[c][e] += u;
      }
    }
  }
  // fixed-order reduction of the 8 warps' partial columns, one write per output element
  __syncthreads();
  T* red = reinterpret_cast<T*>(bsm);  // [kBatchWarps][w][32 * VW]
#pragma unroll
  for (int c = 0; c < kMaxW; ++c)
    if (c < w)
#pragma unroll
      for (int e = 0; e < VW; ++e) red[(warp * w + c) * 32 * VW + lane * VW + e] = R[c][e];
  __syncthreads();
  T* out = reinterpret_cast<T*>(p.out);
  for (int i = threadIdx.x; i < w * 32 * VW; i += blockDim.x) {
    const int c = i / (32 * VW), v = i % (32 * VW);
    const int64_t vec = (int64_t)slice * 32 * VW + v;
    if (vec >= p.batch) continue;
    T s = T(0);
#pragma unroll
    for (int ww = 0; ww < kBatchWarps; ++ww) s += red[((int64_t)ww * w + c) * 32 * VW + v];
    out[vec * p.cols + (int64_t)b * p.k + (w - 1 - c)] = s;
  }
}

template <typename T>
rsr_status launch_batched_t(const rsr_index_desc& d, const void* V, int64_t batch, void* out, bool pp, void* ws,
                            cudaStream_t s, int b0, int b1) {
  const int vw = batch <= 32 ? 1 : batch <= 64 ? 2 : 4;
  const int64_t sw = 32 * vw;                      // vectors per slice
  const int64_t ld = (batch + sw - 1) / sw * sw;   // padded batch
  T* vt = reinterpret_cast<T*>(ws);
  dim3 tg((unsigned)((d.rows + 31) / 32), (unsigned)(ld / 32));
  transpose_kernel<T><<<tg, dim3(32, 8), 0, s>>>(reinterpret_cast<const T*>(V), d.rows, batch, vt, ld);
  rsr_status st = cuda_check(cudaGetLastError(), "transpose_kernel launch");
  if (st != RSR_OK) return st;
  BatchParams p{};
  for (int h = 0; h < d.halves; ++h) {
    p.perm[h] = d.half[h].perm;
    p.seg[h] = d.half[h].seg;
  }
  p.vt = vt;
  p.out = out;
  p.rows = d.rows;
  p.cols = d.cols;
  p.row_stride = d.row_stride;
  p.seg_stride = d.seg_stride;
  p.ld = ld;
  p.batch = batch;
  p.k = d.k;
  p.halves = d.halves;
  p.b_begin = b0;
  const size_t seg_bytes = (size_t)d.halves * (((size_t)1 << d.k) + 1) * 4;
  const size_t red_bytes = (size_t)kBatchWarps * d.k * sw * sizeof(T);
  const size_t smem = std::max(seg_bytes, red_bytes);
  if (smem > device_max_smem_optin()) return fail(RSR_ERR_UNSUPPORTED, "batched multiply: k too large for shared memory");
  if ((uint64_t)d.rows * (uint64_t)ld >= (1ull << 32))
    return fail(RSR_ERR_UNSUPPORTED, "batched multiply: rows * padded batch must be < 2^32");
  dim3 grid((unsigned)(b1 - b0), (unsigned)(ld / sw));
  auto go = [&](auto kern) -> rsr_status {
    if (smem > 48 * 1024) {
      rsr_status a = set_max_smem((const void*)kern, smem);
      if (a != RSR_OK) return a;
    }
    kern<<<grid, kBatchWarps * 32, smem, s>>>(p);
    return cuda_check(cudaGetLastError(), "batched_kernel launch");
  };
  const bool p16 = d.perm_bytes == 2;
#define RSR_BATCH_GO(VW_)                                                                                    \
  return pp ? (p16 ? go(batched_kernel<T, VW_, true, true>) : go(batched_kernel<T, VW_, true, false>))      \
            : (p16 ? go(batched_kernel<T, VW_, false, true>) : go(batched_kernel<T, VW_, false, false>));
  if (vw == 1) { RSR_BATCH_GO(1) }
  if (vw == 2) { RSR_BATCH_GO(2) }
  RSR_BATCH_GO(4)
#undef RSR_BATCH_GO
}

}  // namespace

size_t batched_workspace_bytes(const rsr_index_desc& d, int64_t batch, rsr_dtype dt) {
  if (batch <= 0 || dt == RSR_F64) return 0;
  const int64_t sw = batch <= 32 ? 32 : batch <= 64 ? 64 : 128;
  return (size_t)d.rows * (size_t)((batch + sw - 1) / sw * sw) * 4;
}

// Short last block of an int32 batch (capi.cu packed-pair path): its few key bits make buckets
// heavy, so it is computed densely.  tail_keys_kernel: key of every row from perm + seg (the
// bucket holding sorted position p is the largest j with seg[j] <= p, indexer.py:176-186);
// tail_dense_kernel: grid (vector, row split), out[c] += sum_r v[r] * (bit_c(key+[r]) - bit_c(key-[r]))
// over the split's rows, int32 reductions (exact modulo 2^32 like every int32 path; out zeroed).
__global__ void tail_keys_kernel(const rsr_index_desc d, int b, uint16_t* keys) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int h = blockIdx.y;
  if (p >= d.rows) return;
  const int w = block_width(d.cols, d.k, b);
  const uint32_t* seg = (h ? d.half[1].seg : d.half[0].seg) + (int64_t)b * d.seg_stride;
  int lo = 0, hi = (1 << w) - 1;  // largest j in [0, 2^w) with seg[j] <= p (seg[0] = 0)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)__ldg(seg + mid) <= p) lo = mid;
    else hi = mid - 1;
  }
  const int64_t off = (int64_t)b * d.row_stride + p;
  const void* perm = h ? d.half[1].perm : d.half[0].perm;
  const int64_t row = d.perm_bytes == 2 ? (int64_t)__ldg(reinterpret_cast<const uint16_t*>(perm) + off)
                                        : (int64_t)__ldg(reinterpret_cast<const uint32_t*>(perm) + off);
  keys[h * d.rows + row] = (uint16_t)lo;
}

__global__ void __launch_bounds__(256) tail_dense_kernel(const rsr_index_desc d, int b, const uint16_t* __restrict__ keys,
                                                         const int32_t* __restrict__ V, int32_t* __restrict__ out) {
  const int64_t vec = blockIdx.x;
  const int w = block_width(d.cols, d.k, b);
  const int32_t* v = V + vec * d.rows;
  int32_t acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0;
  const int64_t chunk = (d.rows + gridDim.y - 1) / gridDim.y;
  const int64_t r1 = std::min<int64_t>(d.rows, (blockIdx.y + 1) * chunk);
  for (int64_t r = blockIdx.y * chunk + threadIdx.x; r < r1; r += blockDim.x) {
    const int32_t x = __ldg(v + r);
    const uint32_t kp = __ldg(keys + r);
    const uint32_t kn = d.halves == 2 ? __ldg(keys + d.rows + r) : 0u;
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] += (int32_t)(((kp >> c) & 1u) - ((kn >> c) & 1u)) * x;
  }
  __shared__ int32_t part[8][16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int32_t s = __reduce_add_sync(0xffffffffu, acc[c]);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5][c] = s;
  }
  __syncthreads();
  if (threadIdx.x < w) {  // column c of the block = key bit w - 1 - c (MSB-first)
    const int bit = w - 1 - threadIdx.x;
    int32_t s = 0;
    for (int i = 0; i < 8; ++i) s += part[i][bit];
    if (s != 0) atomicAdd(out + vec * d.cols + (int64_t)b * d.k + threadIdx.x, s);
  }
}

rsr_status multiply_batched_tail(const rsr_index_desc& d, int b, const int32_t* V, int64_t batch, int32_t* out, void* ws,
                                 cudaStream_t s) {
  uint16_t* keys = reinterpret_cast<uint16_t*>(ws);
  tail_keys_kernel<<<dim3((unsigned)((d.rows + 255) / 256), (unsigned)d.halves), 256, 0, s>>>(d, b, keys);
  rsr_status st = cuda_check(cudaGetLastError(), "tail_keys_kernel launch");
  if (st != RSR_OK) return st;
  const int w = block_width(d.cols, d.k, b);
  st = cuda_check(cudaMemset2DAsync(out + (int64_t)b * d.k, d.cols * 4, 0, w * 4, batch, s), "memset tail");
  if (st != RSR_OK) return st;
  const unsigned splits = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (d.rows + 1023) / 1024));
  tail_dense_kernel<<<dim3((unsigned)batch, splits), 256, 0, s>>>(d, b, keys, V, out);
  return cuda_check(cudaGetLastError(), "tail_dense_kernel launch");
}

rsr_status multiply_batched(const rsr_index_desc& d, const void* V, rsr_dtype vt, int64_t batch, void* out,
                            rsr_dtype ot, rsr_variant var, void* ws, size_t ws_bytes, cudaStream_t s, int b0, int b1) {
  if (b1 < 0) b1 = d.nblocks;
  if (batch == 0 || b0 >= b1) return RSR_OK;
  if (vt != ot) return fail(RSR_ERR_INVALID, "batched multiply writes the activation dtype");
  if (vt == RSR_F64) return fail(RSR_ERR_UNSUPPORTED, "batched kernel takes int32 or fp32 activations");
  if (d.k > kMaxW) return fail(RSR_ERR_UNSUPPORTED, "batched multiply supports k <= 16");
  if (!ws || ws_bytes < batched_workspace_bytes(d, batch, vt))
    return fail(RSR_ERR_INVALID, "batched multiply: workspace too small (rsr_multiply_batched_workspace_bytes)");
  const bool pp = var == RSR_VARIANT_RSRPP;
  if (vt == RSR_I32) return launch_batched_t<int32_t>(d, V, batch, out, pp, ws, s, b0, b1);
  return launch_batched_t<float>(d, V, batch, out, pp, ws, s, b0, b1);
}

}  // namespace rsr
