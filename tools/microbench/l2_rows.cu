// Microbenchmark: aggregate L2 -> SM bandwidth of random whole-row gathers from an
// L2-resident table (the batched gather-form multiply reads one v^T row per index position).
// Each warp loads rows of ROWB bytes (lanes cover the row with 4/8/16-byte vectors).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <typename V, int UNROLL>
__global__ void __launch_bounds__(512) gather_rows(const V* __restrict__ tab, int nrows_mask, int iters, int* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t s = mix(gw * 0x9E3779B9u + 17);
  int acc = 0;
  for (int it = 0; it < iters; it += UNROLL) {
    V x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      s = mix(s + u);
      const uint32_t row = s & nrows_mask;  // warp-uniform
      x[u] = __ldg(tab + (size_t)row * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int* p = reinterpret_cast<const int*>(&x[u]);
#pragma unroll
      for (int i = 0; i < (int)(sizeof(V) / 4); ++i) acc += p[i];
    }
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

template <typename V, int UNROLL>
void run(const char* name, int threads, int ctas_per_sm) {
  const int nrows = 16384;
  V* tab;
  int* out;
  cudaMalloc(&tab, (size_t)nrows * 32 * sizeof(V));
  cudaMemset(tab, 1, (size_t)nrows * 32 * sizeof(V));
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm, iters = 4096;
  gather_rows<V, UNROLL><<<grid, threads>>>(tab, nrows - 1, iters, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather_rows<V, UNROLL><<<grid, threads>>>(tab, nrows - 1, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 5.0 * grid * (threads / 32) * (double)iters * 32 * sizeof(V);
  printf("%-28s threads %4d x %d/SM unroll %2d: %7.2f TB/s  (%.2f B/clk/SM @1.92GHz)\n", name, threads,
         ctas_per_sm, UNROLL, bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / sms / 1.92e9);
  cudaFree(tab);
  cudaFree(out);
}

int main() {
  run<int, 8>("row 128B (int/lane)", 512, 2);
  run<int2, 8>("row 256B (int2/lane)", 512, 2);
  run<int4, 8>("row 512B (int4/lane)", 512, 2);
  run<int2, 16>("row 256B (int2/lane)", 512, 2);
  run<int2, 8>("row 256B (int2/lane)", 256, 4);
  run<int4, 4>("row 512B (int4/lane)", 512, 2);
  run<int, 16>("row 128B (int/lane)", 512, 2);
  return 0;
}
