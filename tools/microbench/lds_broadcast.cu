// Cost of warp-uniform (broadcast) shared-memory loads on the LSU data pipe: 16 warps per SM each
// issue N loads where all 32 lanes read the same address, for 4-, 8- and 16-byte loads, against a
// shuffle of a 32-bit word (the batch kernel's code hand-out).  Prints cycles per warp instruction
// per SM (the data pipe issues one wavefront per cycle per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 lds_broadcast.cu -o lds_broadcast
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(int* sink, long long* cycles) {
  __shared__ __align__(16) uint4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned acc = 0;
  const long long t0 = clock64();
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    const int idx = (it * 7 + warp) & 1023;  // warp-uniform address
    if (MODE == 0) acc += reinterpret_cast<const unsigned*>(buf)[idx * 4];
    if (MODE == 1) { const uint2 q = reinterpret_cast<const uint2*>(buf)[idx * 2]; acc += q.x ^ q.y; }
    if (MODE == 2) { const uint4 q = buf[idx]; acc += q.x ^ q.y ^ q.z ^ q.w; }
    if (MODE == 3) acc += __shfl_sync(0xffffffffu, (unsigned)(it * 3 + lane), (it + warp) & 31);  // independent
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  (void)lane;
}

int main() {
  int* sink;
  long long* cyc;
  cudaMalloc(&sink, 4096);
  cudaMalloc(&cyc, 148 * 8);
  auto run = [&](auto k, const char* name) {
    k<<<148, 512>>>(sink, cyc);
    k<<<148, 512>>>(sink, cyc);
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    // 16 warps x kIters instructions per SM
    printf("%-40s %.3f cycles per warp instruction per SM\n", name, (double)c[0] / (16.0 * kIters));
  };
  run(kern<0>, "LDS.32 broadcast");
  run(kern<1>, "LDS.64 broadcast");
  run(kern<2>, "LDS.128 broadcast");
  run(kern<3>, "SHFL.IDX");
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
