// Reading a host-written vector straight from MAPPED pinned memory in every CTA (148 CTAs x
// 64 KB each): time per launch and staleness across launches (the host rewrites the vector
// before every launch), for plain (.ca), .cg, .cv and .nc loads.  Answers: does the GPU merge the
// CTAs' sysmem reads in L2 (one PCIe transfer) and is a line cached by launch i ever seen by
// launch i + 1?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 pull_probe.cu -o pull_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

template <int MODE>
__device__ __forceinline__ int4 load(const int4* p) {
  int4 r;
  if (MODE == 0) asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 1) asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 2) asm volatile("ld.global.cv.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 3) asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// every CTA reads the whole vector (n16 int4) and counts entries != expected pattern
template <int MODE>
__global__ void __launch_bounds__(640) read_all(const int4* hv, int n16, int expect, unsigned* bad,
                                                unsigned long long* span) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int nb = 0;
  for (int i = threadIdx.x; i < n16; i += blockDim.x) {
    const int4 q = load<MODE>(hv + i);
    nb += (q.x != expect + 4 * i) + (q.y != expect + 4 * i + 1) + (q.z != expect + 4 * i + 2) + (q.w != expect + 4 * i + 3);
  }
  __syncthreads();
  if (nb) atomicAdd(bad, (unsigned)nb);
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) atomicMax(span, t1 - t0);
}

int main() {
  const int n = 16384, n16 = n / 4;
  int *h, *hd;
  cudaHostAlloc((void**)&h, 4 * n, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  unsigned* bad;
  unsigned long long* span;
  cudaMalloc(&bad, 4);
  cudaMalloc(&span, 8);
  auto run = [&](auto kern, const char* name) {
    std::vector<float> ms;
    std::vector<unsigned long long> spans;
    unsigned tot_bad = 0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < 60; ++it) {
      const int expect = it * 100000;
      for (int i = 0; i < n; ++i) h[i] = expect + i;  // rewritten before every launch
      cudaMemset(bad, 0, 4);
      cudaMemset(span, 0, 8);
      cudaEventRecord(a);
      kern<<<148, 640>>>(reinterpret_cast<const int4*>(hd), n16, expect, bad, span);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float t;
      cudaEventElapsedTime(&t, a, b);
      unsigned nb;
      unsigned long long sp;
      cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(&sp, span, 8, cudaMemcpyDeviceToHost);
      if (it >= 10) {
        ms.push_back(t);
        spans.push_back(sp);
      }
      tot_bad += nb;
    }
    std::sort(ms.begin(), ms.end());
    std::sort(spans.begin(), spans.end());
    printf("%-12s launch median %6.2f us, longest CTA median %6.2f us, stale/wrong entries over 60 launches: %u\n", name,
           ms[ms.size() / 2] * 1e3, spans[spans.size() / 2] / 1e3, tot_bad);
  };
  run(read_all<0>, "ld (.ca)");
  run(read_all<1>, "ld.cg");
  run(read_all<2>, "ld.cv");
  run(read_all<3>, "ld.nc");
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
