// Latencies behind the session pull (csrc/multiply.cu pull_payload), per CTA with %globaltimer:
//   (1) one 16-byte .nc load of mapped host memory, one thread of one CTA
//   (2) 148 CTAs, each loading its own 448-byte chunk (28 threads x 16 B) at once
//   (3) (2) + storing the chunk to global + __threadfence
//   (4) a 64-bit atomicAdd round trip to L2 (148 CTAs on one word)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 pcie_latency.cu -o pcie_latency
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE>
__global__ void probe(const uint4* host, uint4* dst, unsigned long long* ctr, unsigned long long* out) {
  __shared__ unsigned long long t0s;
  if (threadIdx.x == 0) t0s = gt();
  __syncthreads();
  const int t = threadIdx.x;
  if (MODE == 1) {
    if (blockIdx.x == 0 && t == 0) {
      uint4 q;
      asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(host));
      dst[0] = q;  // dependent store: the load has returned
    }
  } else if (MODE == 2 || MODE == 3) {
    if (t < 28) {
      uint4 q;
      asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                   : "l"(host + blockIdx.x * 28 + t));
      dst[blockIdx.x * 28 + t] = q;
      if (MODE == 3) __threadfence();
    }
  } else if (MODE == 5 || MODE == 6 || MODE == 7) {  // one 4-byte sysmem read: relaxed.sys / volatile / cv
    if (blockIdx.x == 0 && t == 0) {
      unsigned x;
      if (MODE == 5) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(host) : "memory");
      if (MODE == 6) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(x) : "l"(host) : "memory");
      if (MODE == 7) asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(x) : "l"(host) : "memory");
      dst[0].x = x;
    }
  } else if (MODE == 4) {
    if (t == 0) {
      unsigned long long o = atomicAdd(ctr, 1ull);
      dst[blockIdx.x].x = (unsigned)o;
    }
  }
  __syncthreads();
  if (t == 0) out[blockIdx.x] = gt() - t0s;
}

int main() {
  uint4 *h, *hd, *dst;
  cudaHostAlloc((void**)&h, 1 << 20, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  cudaMalloc(&dst, 1 << 20);
  unsigned long long *ctr, *out;
  cudaMalloc(&ctr, 8);
  cudaMalloc(&out, 148 * 8);
  auto run = [&](auto kern, int grid, const char* name) {
    std::vector<double> med, mx;
    std::vector<unsigned long long> o(148);
    for (int it = 0; it < 50; ++it) {
      kern<<<grid, 640>>>(hd, dst, ctr, out);
      cudaMemcpy(o.data(), out, grid * 8, cudaMemcpyDeviceToHost);
      std::vector<unsigned long long> s(o.begin(), o.begin() + grid);
      std::sort(s.begin(), s.end());
      if (it >= 5) {
        med.push_back(s[grid / 2] / 1e3);
        mx.push_back(s[grid - 1] / 1e3);
      }
    }
    std::sort(med.begin(), med.end());
    std::sort(mx.begin(), mx.end());
    printf("%-52s per-CTA median %5.2f us, slowest CTA %5.2f us\n", name, med[med.size() / 2], mx[mx.size() / 2]);
  };
  run(probe<1>, 1, "(1) one 16-byte sysmem load (1 CTA)");
  run(probe<2>, 148, "(2) 148 CTAs x 448-byte chunk from sysmem");
  run(probe<3>, 148, "(3) (2) + store + __threadfence");
  run(probe<4>, 148, "(4) 64-bit atomicAdd round trip (148 CTAs, 1 word)");
  run(probe<5>, 1, "(5) one 4-byte ld.relaxed.sys of sysmem");
  run(probe<6>, 1, "(6) one 4-byte ld.volatile of sysmem");
  run(probe<7>, 1, "(7) one 4-byte ld.cv of sysmem");
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
