// Microbenchmark: does streaming the key bytes compete with shared-memory REDs?
// 16 warps/CTA, 1 CTA/SM; each lane issues random red.shared.add.s32 into an 8 KB histogram
// at the scatter kernel's ratio of one 16-byte key load per 8 REDs.
//   mode 0: REDs only (keys synthesized in registers)
//   mode 1: + keys streamed from HBM with ld.global.nc.L1::no_allocate.v4 (registers only)
//   mode 2: + keys streamed with 1-D TMA bulk copies into smem and read back with LDS.128
//   mode 3: streaming only (mode 1 without REDs)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void red_s(uint32_t a, int v) { asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int WARPS = 16, STEPS = 8;  // STEPS x 16 B per lane per unit
template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) kern(const uint4* __restrict__ keys, size_t unit_stride, int units, int* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  int* hist = reinterpret_cast<int*>(smem);           // 2048 ints
  uint4* ring = reinterpret_cast<uint4*>(smem + 8192);  // [WARPS][2][32*STEPS] uint4
  __shared__ uint64_t bar[WARPS][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) hist[i] = 0;
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t hs = su32(hist);
  // this warp's key stream: unit u covers 32*STEPS uint4 contiguous
  const uint4* base = keys + (size_t)(blockIdx.x * WARPS + warp) * 32 * STEPS;
  uint4* myring = ring + warp * 2 * 32 * STEPS;
  const uint32_t bytes = 32 * STEPS * 16;
  auto issue = [&](int u) {
    if (lane == 0) {
      const int s = u & 1;
      const uint32_t b = su32(&bar[warp][s]);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(myring + s * 32 * STEPS)), "l"(base + (size_t)u * unit_stride), "r"(bytes), "r"(b) : "memory");
    }
  };
  if (MODE == 2) { issue(0); issue(1); }
  uint32_t salt = mix(blockIdx.x * 977 + threadIdx.x);
  uint32_t acc = 0;
  uint4 qn[STEPS];
  if (MODE == 4) {
#pragma unroll
    for (int i = 0; i < STEPS; ++i) qn[i] = ldg_stream(base + i * 32 + lane);
  }
  for (int u = 0; u < units; ++u) {
    uint4 q[STEPS];
    if (MODE == 4) {
#pragma unroll
      for (int i = 0; i < STEPS; ++i) q[i] = qn[i];
      const int un = u + 1 < units ? u + 1 : u;
#pragma unroll
      for (int i = 0; i < STEPS; ++i) qn[i] = ldg_stream(base + (size_t)un * unit_stride + i * 32 + lane);
    } else if (MODE == 1 || MODE == 3) {
#pragma unroll
      for (int i = 0; i < STEPS; ++i) q[i] = ldg_stream(base + (size_t)u * unit_stride + i * 32 + lane);
    } else if (MODE == 2) {
      const int s = u & 1;
      const uint32_t b = su32(&bar[warp][s]);
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }"
                   ::"r"(b), "r"((u >> 1) & 1) : "memory");
#pragma unroll
      for (int i = 0; i < STEPS; ++i) q[i] = myring[s * 32 * STEPS + i * 32 + lane];
      __syncwarp();
      if (u + 2 < units) issue(u + 2);
    } else {
#pragma unroll
      for (int i = 0; i < STEPS; ++i) q[i] = make_uint4(mix(salt + i), mix(salt + 7 * i), mix(salt ^ i), mix(salt + 3 * i));
      salt = mix(salt);
    }
    if (MODE != 3) {
#pragma unroll
      for (int i = 0; i < STEPS; ++i) {
        const uint32_t w[4] = {q[i].x ^ salt, q[i].y ^ salt, q[i].z ^ salt, q[i].w ^ salt};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          red_s(hs + ((w[e] & 2047u) << 2), 1);
          red_s(hs + (((w[e] >> 16) & 2047u) << 2), 1);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < STEPS; ++i) acc += q[i].x + q[i].y + q[i].z + q[i].w;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = hist[blockIdx.x & 2047] + (int)acc;
}

template <int MODE>
void run(const char* name, const uint4* keys, size_t stride, int units, int* out, int sms) {
  const size_t smem = 8192 + WARPS * 2 * 32 * STEPS * 16;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<MODE><<<sms, WARPS * 32, smem>>>(keys, stride, units, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<MODE><<<sms, WARPS * 32, smem>>>(keys, stride, units, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  const double reds = (double)sms * WARPS * 32 * units * STEPS * 8;
  const double bytes = (double)sms * WARPS * 32 * units * STEPS * 16;
  printf("%-44s %8.1f us  REDs %.2f/clk/SM  stream %.2f TB/s  err=%s\n", name, ms * 1e3,
         reds / (ms * 1e-3) / sms / 1.92e9, bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int units = 64;
  const size_t stride = (size_t)sms * WARPS * 32 * STEPS;  // uint4 per unit across the grid
  const size_t total = stride * units;                     // 148*16*32*8*16 B * 64 = 1.24 GB... scaled below
  uint4* keys;
  int* out;
  if (cudaMalloc(&keys, total * 16) != cudaSuccess) { printf("alloc fail\n"); return 1; }
  cudaMemset(keys, 0x5a, total * 16);
  cudaMalloc(&out, sms * 4);
  printf("key stream %.1f MB\n", total * 16 / 1e6);
  run<0>("mode0 REDs only", keys, stride, units, out, sms);
  run<1>("mode1 REDs + LDG.nc.no_allocate stream", keys, stride, units, out, sms);
  run<2>("mode2 REDs + TMA->smem + LDS.128 stream", keys, stride, units, out, sms);
  run<3>("mode3 LDG stream only", keys, stride, units, out, sms);
  run<4>("mode4 REDs + LDG stream, 1-unit prefetch", keys, stride, units, out, sms);
  run<0>("mode0 REDs only (again)", keys, stride, units, out, sms);
  return 0;
}
