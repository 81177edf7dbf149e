// Microbenchmark (truly random addresses via a hash): shared-memory gather (LDS) and
// int32 atomic (ATOMS.ADD) cost per warp instruction on B200, plus conflict-free baselines.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE, int WORDS>
__global__ void __launch_bounds__(1024) bench(int iters, int* out) {
  extern __shared__ int smem[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) smem[i] = i;
  __syncthreads();
  const uint32_t seed = (blockIdx.x * 1024 + threadIdx.x) * 0x9E3779B9u;
  const int lane = threadIdx.x & 31;
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = mix(seed + i);
  int acc = 0;
  for (int it0 = 0; it0 < iters; it0 += 16) {
    const uint32_t c = mix(it0);  // same for all lanes: XOR keeps the conflict pattern random
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    uint32_t a = (r[i] ^ c) & (WORDS - 1);
    if (MODE == 0) acc += smem[a];                                       // random LDS
    if (MODE == 1) atomicAdd(&smem[a], (int)(a & 7));                    // random ATOMS
    if (MODE == 2) acc += smem[(a & ~31u) | lane];                       // conflict-free LDS
    if (MODE == 3) atomicAdd(&smem[(a & ~31u) | lane], (int)(a & 7));    // conflict-free ATOMS
    if (MODE == 4) acc += (int)a;                                        // ALU only
  }
  }
  if (acc == 0x7fffffff) out[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] += smem[blockIdx.x & (WORDS - 1)];
}

template <int MODE, int WORDS>
void run(const char* name) {
  int* out; cudaMalloc(&out, 4096 * 4); cudaMemset(out, 0, 4096 * 4);
  cudaFuncSetAttribute(bench<MODE, WORDS>, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
  const int iters = 4096, grid = 148, thr = 1024;
  for (int w = 0; w < 2; ++w) bench<MODE, WORDS><<<grid, thr, WORDS * 4>>>(iters, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) bench<MODE, WORDS><<<grid, thr, WORDS * 4>>>(iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double warp_instr_per_sm = double(thr / 32) * iters * 5;
  double cycles = ms * 1e-3 * 1.92e9;  // ~sustained SM clock under this load
  printf("%-22s words=%5d  %.3f ms  %.2f cycles per warp-instruction per SM\n", name, WORDS, ms / 5,
         cycles / warp_instr_per_sm);
}

int main() {
  run<4, 2048>("ALU hash only");
  run<0, 16384>("LDS random");
  run<0, 2048>("LDS random");
  run<2, 16384>("LDS conflict-free");
  run<1, 2048>("ATOMS random");
  run<1, 16384>("ATOMS random");
  run<3, 2048>("ATOMS conflict-free");
  return 0;
}
