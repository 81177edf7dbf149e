// Microbenchmark for a single-vector RSR scatter where the 32 lanes of a warp span 32 COLUMN
// BLOCKS of 8 columns (k = 8, u8 keys) instead of 32 rows: lane l owns row r = r0 + l (its v in a
// register) and, in step j, block (l + j) mod 32 of a 32-block set.  The histogram of a set is
// [256 bins][32 blocks] int32 (32 KB), so the 32 lanes of a reduction always hit 32 distinct banks
// (bank = block), whatever the keys.  Keys live in a [row][block] u8 matrix (the bit-packed binary
// half itself, MSB-first per 8 columns), stored set-major [set][row][32] so a unit's keys are one
// contiguous run, each row's 32-byte slice rotated by row mod 32 so that step j reads byte j of
// the lane's registers (static).  The next unit's keys are bulk-prefetched into L2.
//   units = (block set, 1024-row range); 16 warps x 64 rows; both halves (+v, -v)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_s(uint32_t a, int v) { asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int ROWS = 16384, NB = 2048, SETS = NB / 32, RRANGE = 1024, WARPS = 16;

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) kern(const uint4* __restrict__ kp, const uint4* __restrict__ kn,
                                                       const int* __restrict__ v, int* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  int* hist = reinterpret_cast<int*>(smem);  // [256][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const uint32_t hs = su32(hist);
  const int nunits = SETS * (ROWS / RRANGE);
  auto prefetch = [&](int u) {  // this warp's rows of unit u, both halves (64 rows x 32 B each)
    const int set = u % SETS, q = u / SETS;
    const size_t off = ((size_t)set * ROWS + q * RRANGE + warp * (RRANGE / WARPS)) * 32;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)kp + off), "r"(RRANGE / WARPS * 32) : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)kn + off), "r"(RRANGE / WARPS * 32) : "memory");
  };
  if (lane == 0 && MODE != 2) prefetch(blockIdx.x);
  if (MODE == 3) {  // software-pipelined: the next chunk's keys (and v) load while this chunk reduces
    constexpr int CH = RRANGE / WARPS / 32;  // chunks per warp per unit
    auto addr = [&](int u, int c, const uint4* base) {
      const int set = u % SETS, q = u / SETS;
      const int row = q * RRANGE + warp * (RRANGE / WARPS) + c * 32 + lane;
      return base + ((size_t)set * ROWS + row) * 2;
    };
    auto vrow = [&](int u, int c) { return (u / SETS) * RRANGE + warp * (RRANGE / WARPS) + c * 32 + lane; };
    int u = blockIdx.x, c = 0;
    uint4 a0 = __ldg(addr(u, c, kp)), a1 = __ldg(addr(u, c, kp) + 1), b0 = __ldg(addr(u, c, kn)), b1 = __ldg(addr(u, c, kn) + 1);
    int x = v[vrow(u, c)];
    while (u < nunits) {
      int un = u, cn = c + 1;
      if (cn == CH) { cn = 0; un = u + gridDim.x; if (lane == 0 && un + (int)gridDim.x < nunits) prefetch(un + gridDim.x); }
      const bool more = un < nunits;
      uint4 na0, na1, nb0, nb1;
      int nxv = 0;
      if (more) {
        na0 = __ldg(addr(un, cn, kp)); na1 = __ldg(addr(un, cn, kp) + 1);
        nb0 = __ldg(addr(un, cn, kn)); nb1 = __ldg(addr(un, cn, kn) + 1);
        nxv = v[vrow(un, cn)];
      }
      const uint32_t wp[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const uint32_t wn[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      const int nx = -x;
      uint32_t bank4 = (uint32_t)lane * 4u;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int sh = 8 * (j & 3);
        red_s(hs + ((((wp[j >> 2] >> sh) & 0xffu) << 7) | bank4), x);
        red_s(hs + ((((wn[j >> 2] >> sh) & 0xffu) << 7) | bank4), nx);
        bank4 = (bank4 + 4u) & 124u;
      }
      if (!more) break;
      a0 = na0; a1 = na1; b0 = nb0; b1 = nb1; x = nxv;
      u = un; c = cn;
    }
  }
  for (int u = blockIdx.x; u < nunits && MODE != 3; u += gridDim.x) {
    const int set = u % SETS, q = u / SETS;
    if (lane == 0 && MODE != 2 && u + (int)gridDim.x < nunits) prefetch(u + gridDim.x);
#pragma unroll 1
    for (int c = 0; c < RRANGE / WARPS / 32; ++c) {
      const int row = q * RRANGE + warp * (RRANGE / WARPS) + c * 32 + lane;
      const int x = v[row], nx = -x;
      // this row's 32 keys of the set (rotated by row % 32 in memory): 2 x 16 B per half
      const uint4* pp = kp + ((size_t)set * ROWS + row) * 2;
      const uint4* pn = kn + ((size_t)set * ROWS + row) * 2;
      const uint4 a0 = __ldg(pp), a1 = __ldg(pp + 1), b0 = __ldg(pn), b1 = __ldg(pn + 1);
      const uint32_t wp[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const uint32_t wn[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      uint32_t bank4 = (uint32_t)lane * 4u;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int sh = 8 * (j & 3);
        // (key << 7) | bank4: bin row of 128 bytes, the block's word
        const uint32_t ap = (((wp[j >> 2] >> sh) & 0xffu) << 7) | bank4;
        const uint32_t an = (((wn[j >> 2] >> sh) & 0xffu) << 7) | bank4;
        if (MODE != 1) {
          red_s(hs + ap, x);
          red_s(hs + an, nx);
        } else {
          red_s(hs + ap, x);
        }
        bank4 = (bank4 + 4u) & 124u;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = hist[lane];
}

int main() {
  const size_t nkeys = (size_t)ROWS * NB;
  std::vector<uint8_t> hk(nkeys);
  uint32_t s = 7;
  for (size_t i = 0; i < nkeys; ++i) { s = s * 1664525u + 1013904223u; hk[i] = (uint8_t)(s >> 24); }
  std::vector<int> hv(ROWS);
  for (int i = 0; i < ROWS; ++i) hv[i] = (i * 37) % 201 - 100;
  const int copies = 4;  // rotate copies: 4 x 2 x 32 MB > L2
  std::vector<uint8_t*> dk(2 * copies);
  for (auto& p : dk) { cudaMalloc(&p, nkeys); cudaMemcpy(p, hk.data(), nkeys, cudaMemcpyHostToDevice); }
  int *dv, *sink;
  cudaMalloc(&dv, ROWS * 4);
  cudaMemcpy(dv, hv.data(), ROWS * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 4096);
  const size_t smem = 256 * 32 * 4;
  auto run = [&](auto kfn, const char* name) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 3; ++i)
      kfn<<<148, WARPS * 32, smem>>>((const uint4*)dk[0], (const uint4*)dk[1], dv, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 40;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) {
      const int c = i % copies;
      kfn<<<148, WARPS * 32, smem>>>((const uint4*)dk[2 * c], (const uint4*)dk[2 * c + 1], dv, sink);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %7.2f us per 16384 x 16384 matvec scatter (keys 2 x %.0f MB, rotating %d copies) err=%s\n", name,
           ms * 1e3 / reps, nkeys / 1e6, copies, cudaGetErrorString(cudaGetLastError()));
  };
  run(kern<0>, "both halves (+v, -v), k = 8, lanes span blocks");
  run(kern<1>, "positive half only (binary)");
  run(kern<2>, "both halves, no L2 prefetch");
  run(kern<3>, "both halves, pipelined one chunk ahead");
  return 0;
}
