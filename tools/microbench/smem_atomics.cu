// Microbenchmark: shared-memory random gather / atomic throughput on B200.
// Decides the multiply kernel's formulation (gather vs scatter histogram).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int WORDS>
__global__ void __launch_bounds__(1024) bench(int iters, int* out) {
  extern __shared__ int smem[];
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) smem[i] = i;
  __syncthreads();
  uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 97u + 1u;
  int lane = threadIdx.x & 31;
  int acc = 0;
  float facc = 0.f;
  constexpr int SH = 32 - __builtin_ctz(WORDS);
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t a = s >> SH;
    if (MODE == 0) acc += smem[a];                                   // random LDS gather
    else if (MODE == 1) atomicAdd(&smem[a], int(s & 7u));                      // random ATOMS int
    else if (MODE == 2) atomicAdd(reinterpret_cast<float*>(&smem[a]), 1.f);  // random RED f32
    else if (MODE == 3) acc += smem[(a & ~31u) | lane];              // bank-distinct LDS
    else if (MODE == 4) atomicAdd(&smem[(a & ~31u) | lane], int(s & 7u));      // bank-distinct ATOMS
    else if (MODE == 5) atomicAdd(reinterpret_cast<float*>(&smem[(a & ~31u) | lane]), 1.f);
    else if (MODE == 6) { int x = smem[(a & ~31u) | lane]; smem[(a & ~31u) | lane] = x + 1; }  // LDS+STS distinct
    else if (MODE == 8) { float val = 1.f; unsigned addr = (unsigned)__cvta_generic_to_shared(&smem[a]);
      asm volatile("red.shared.add.f32 [%0], %1;" :: "r"(addr), "f"(val) : "memory"); }
    else if (MODE == 9) atomicAdd(reinterpret_cast<unsigned long long*>(smem) + (a >> 1), (unsigned long long)(s & 7u));
    else if (MODE == 10) atomicAdd(reinterpret_cast<unsigned long long*>(smem) + ((a >> 1) & ~31u) + lane, (unsigned long long)(s & 7u));
    else if (MODE == 7) { acc += smem[a & (WORDS-1)]; atomicAdd(&smem[(a*7u) & (WORDS - 1)], int(s & 7u)); }
  }
  __syncthreads();
  if (acc == 0x7fffffff || facc == 1.2345f) out[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] += smem[blockIdx.x & (WORDS - 1)];
}

template <int MODE, int WORDS>
void run(const char* name, int threads, int ctas_per_sm) {
  int* out; cudaMalloc(&out, 4096 * 4); cudaMemset(out, 0, 4096 * 4);
  int smem = WORDS * 4;
  cudaFuncSetAttribute(bench<MODE, WORDS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int grid = 148 * ctas_per_sm;
  int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) bench<MODE, WORDS><<<grid, threads, smem>>>(iters, out);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) bench<MODE, WORDS><<<grid, threads, smem>>>(iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  double ops = double(grid) * threads * iters * reps;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_sm_per_ns = ops / 148.0 / (ms * 1e6);
  printf("%-28s words=%6d thr=%4d cta/sm=%d  %8.3f ms  %7.2f Gop/s/SM  %6.2f lanes/clk@1.9GHz  warp-cyc/instr=%5.2f %s\n",
         name, WORDS, threads, ctas_per_sm, ms / reps, per_sm_per_ns, per_sm_per_ns / 1.9,
         32.0 / (per_sm_per_ns / 1.9), err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
}

int main() {
  run<0, 16384>("LDS random gather", 1024, 1);
  run<0, 4096>("LDS random gather", 1024, 1);
  run<3, 16384>("LDS bank-distinct", 1024, 1);
  run<1, 2048>("ATOMS int random", 1024, 1);
  run<1, 8192>("ATOMS int random", 1024, 1);
  run<2, 2048>("RED f32 random", 1024, 1);
  run<4, 2048>("ATOMS int bank-distinct", 1024, 1);
  run<5, 2048>("RED f32 bank-distinct", 1024, 1);
  run<6, 2048>("LDS+STS bank-distinct", 1024, 1);
  run<7, 2048>("LDS+ATOMS random", 1024, 1);
  run<8, 2048>("red.shared.add.f32 ptx", 1024, 1);
  run<9, 4096>("ATOMS u64 random 2048", 1024, 1);
  run<10, 4096>("ATOMS u64 lane-distinct", 1024, 1);
  run<0, 16384>("LDS random gather", 512, 2);
  run<1, 2048>("ATOMS int random", 512, 2);
  return 0;
}
