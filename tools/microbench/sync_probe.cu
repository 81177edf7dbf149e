// Host round-trip floors for the host-buffer (e2e) multiply: launch + completion notification,
// pinned copies, and the alternatives to cudaStreamSynchronize (event polling, a mapped host
// flag written by the last kernel).  nvcc -gencode arch=compute_100a,code=sm_100a -O2 sync_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cstring>
#include <cstdint>

__global__ void empty_kernel() {}
__global__ void flag_kernel(volatile unsigned* flag, unsigned val) {
  __threadfence_system();
  *flag = val;
}
// a ~20 us kernel: spin on the clock
__global__ void spin_kernel(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}
__global__ void spin_flag_kernel(long long cycles, volatile unsigned* flag, unsigned val) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    __threadfence_system();
    *flag = val;
  }
}

__global__ void publish_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int64_t n32,
                               uint32_t* counter, uint32_t* flag, uint32_t seq) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t n4 = n32 >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n4; i += stride)
    reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      __threadfence_system();
      *counter = 0;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
    }
  }
}

// a ~20 us kernel ending like the fused publish: every CTA stores its slice of the result into
// mapped host memory, fences, arrives on a counter; the last CTA raises the flag
__global__ void spin_publish_kernel(long long cycles, const uint32_t* src, uint32_t* dst, int per_cta, uint32_t* counter,
                                    uint32_t* flag, uint32_t seq, int smem_touch) {
  extern __shared__ uint32_t sm[];
  if (smem_touch) sm[threadIdx.x] = threadIdx.x;
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  for (int i = threadIdx.x; i < per_cta; i += blockDim.x) dst[blockIdx.x * per_cta + i] = __ldcg(src + blockIdx.x * per_cta + i);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      __threadfence_system();
      *counter = 0;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
    }
  }
}

// the last CTA (device-scope counter) copies the whole result to the host, one system fence
__global__ void spin_lastcopy_kernel(long long cycles, const uint32_t* src, uint32_t* dst, int n, uint32_t* counter,
                                     uint32_t* flag, uint32_t seq) {
  __shared__ uint32_t last;
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < n / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = __ldcg(reinterpret_cast<const uint4*>(src) + i);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    *counter = 0;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
  }
}

// every CTA reads the whole vector from mapped host memory (zero copy), then spins, then its
// slice of the result goes straight to mapped host memory (no fence: kernel completion flushes)
__global__ void zc_kernel(long long cycles, const int4* __restrict__ vhost, int n16, uint32_t* dst, int per_cta,
                          int* sink) {
  int acc = 0;
  for (int i = threadIdx.x; i < n16; i += blockDim.x) {
    int4 q = __ldg(vhost + i);
    acc += q.x + q.y + q.z + q.w;
  }
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  for (int i = threadIdx.x; i < per_cta; i += blockDim.x) dst[blockIdx.x * per_cta + i] = i;
  if (acc == 0x7fffffff) *sink = acc;
}

using clk = std::chrono::steady_clock;
template <typename F>
double med_us(F f, int reps = 400) {
  std::vector<double> t;
  for (int i = 0; i < reps + 50; ++i) {
    auto a = clk::now();
    f();
    auto b = clk::now();
    if (i >= 50) t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main(int argc, char** argv) {
  unsigned flags = 0;
  if (argc > 1 && argv[1][0] == 's') flags = cudaDeviceScheduleSpin;
  if (argc > 1 && argv[1][0] == 'y') flags = cudaDeviceScheduleYield;
  if (argc > 1 && argv[1][0] == 'b') flags = cudaDeviceScheduleBlockingSync;
  if (flags) cudaSetDeviceFlags(flags | cudaDeviceMapHost);
  cudaFree(0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void *dv, *dout, *hv, *hout;
  cudaMalloc(&dv, 1 << 20);
  cudaMalloc(&dout, 1 << 20);
  cudaHostAlloc(&hv, 1 << 20, cudaHostAllocDefault);
  cudaHostAlloc(&hout, 1 << 20, cudaHostAllocDefault);
  unsigned* hflag;
  cudaHostAlloc((void**)&hflag, 64, cudaHostAllocMapped);
  unsigned* dflag;
  cudaHostGetDevicePointer((void**)&dflag, hflag, 0);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const long long cyc20 = (long long)clk_khz * 20 / 1000;  // ~20 us at the rated clock
  printf("flags=%s\n", argc > 1 ? argv[1] : "default");
  printf("empty kernel + StreamSync           %7.2f us\n", med_us([&] { empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }));
  printf("empty kernel + EventQuery spin      %7.2f us\n", med_us([&] {
           empty_kernel<<<1, 32, 0, s>>>();
           cudaEventRecord(ev, s);
           while (cudaEventQuery(ev) != cudaSuccess) {
           }
         }));
  unsigned seq = 0;
  printf("flag kernel + host spin             %7.2f us\n", med_us([&] {
           ++seq;
           flag_kernel<<<1, 32, 0, s>>>(dflag, seq);
           while (*(volatile unsigned*)hflag != seq) {
           }
         }));
  printf("launch call only (empty)            %7.2f us\n", med_us([&] { empty_kernel<<<1, 32, 0, s>>>(); }));
  cudaStreamSynchronize(s);
  printf("H2D 64KB + sync                     %7.2f us\n", med_us([&] { cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); }));
  printf("D2H 128KB + sync                    %7.2f us\n", med_us([&] { cudaMemcpyAsync(hout, dout, 131072, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }));
  printf("D2H 64KB + sync                     %7.2f us\n", med_us([&] { cudaMemcpyAsync(hout, dout, 65536, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }));
  printf("spin20 + sync                       %7.2f us\n", med_us([&] { spin_kernel<<<148, 128, 0, s>>>(cyc20); cudaStreamSynchronize(s); }));
  printf("H2D64K + spin20 + D2H128K + sync    %7.2f us\n", med_us([&] {
           cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
           spin_kernel<<<148, 128, 0, s>>>(cyc20);
           cudaMemcpyAsync(hout, dout, 131072, cudaMemcpyDeviceToHost, s);
           cudaStreamSynchronize(s);
         }));
  printf("H2D64K + spin20 + D2H128K + evspin  %7.2f us\n", med_us([&] {
           cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
           spin_kernel<<<148, 128, 0, s>>>(cyc20);
           cudaMemcpyAsync(hout, dout, 131072, cudaMemcpyDeviceToHost, s);
           cudaEventRecord(ev, s);
           while (cudaEventQuery(ev) != cudaSuccess) {
           }
         }));
  printf("H2D64K + spin20 + D2H64K + sync     %7.2f us\n", med_us([&] {
           cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
           spin_kernel<<<148, 128, 0, s>>>(cyc20);
           cudaMemcpyAsync(hout, dout, 65536, cudaMemcpyDeviceToHost, s);
           cudaStreamSynchronize(s);
         }));
  printf("H2D64K + spin20flag(mapped) + spin  %7.2f us\n", med_us([&] {
           ++seq;
           cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
           spin_flag_kernel<<<1, 128, 0, s>>>(cyc20, dflag, seq);
           while (*(volatile unsigned*)hflag != seq) {
           }
         }));
  // CUDA graph of H2D + kernel + D2H
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
  spin_kernel<<<148, 128, 0, s>>>(cyc20);
  cudaMemcpyAsync(hout, dout, 131072, cudaMemcpyDeviceToHost, s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  printf("graph(H2D+spin20+D2H128K) + sync    %7.2f us\n", med_us([&] { cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); }));
  printf("graph(...) + evspin                 %7.2f us\n", med_us([&] {
           cudaGraphLaunch(ge, s);
           cudaEventRecord(ev, s);
           while (cudaEventQuery(ev) != cudaSuccess) {
           }
         }));
  // stream write value after the graph (driver API), host spin on it
  CUdeviceptr dflag_cu = (CUdeviceptr)dflag;
  printf("graph(...) + WriteValue32 + spin    %7.2f us\n", med_us([&] {
           ++seq;
           cudaGraphLaunch(ge, s);
           cuStreamWriteValue32((CUstream)s, dflag_cu, seq, 0);
           while (*(volatile unsigned*)hflag != seq) {
           }
         }));
  printf("H2D+spin20+D2H + WriteValue32 + spin %7.2f us\n", med_us([&] {
           ++seq;
           cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
           spin_kernel<<<148, 128, 0, s>>>(cyc20);
           cudaMemcpyAsync(hout, dout, 131072, cudaMemcpyDeviceToHost, s);
           cuStreamWriteValue32((CUstream)s, dflag_cu, seq, 0);
           while (*(volatile unsigned*)hflag != seq) {
           }
         }));
  {
    void* hres;
    cudaHostAlloc(&hres, 1 << 20, cudaHostAllocMapped);
    void* hres_dev;
    cudaHostGetDevicePointer(&hres_dev, hres, 0);
    uint32_t* counter;
    cudaMalloc(&counter, 64);
    cudaMemset(counter, 0, 64);
    for (int ctas : {1, 4, 8, 32}) {
      for (int pdl : {0, 1}) {
        printf("H2D+spin20+publish64K ctas=%2d pdl=%d %7.2f us\n", ctas, pdl, med_us([&] {
                 ++seq;
                 cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
                 spin_kernel<<<148, 128, 0, s>>>(cyc20);
                 cudaLaunchConfig_t cfg = {};
                 cfg.gridDim = dim3(ctas);
                 cfg.blockDim = dim3(256);
                 cfg.stream = s;
                 cudaLaunchAttribute attr[1];
                 attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                 attr[0].val.programmaticStreamSerializationAllowed = pdl;
                 cfg.attrs = attr;
                 cfg.numAttrs = 1;
                 cudaLaunchKernelEx(&cfg, publish_kernel, (const uint32_t*)dout, (uint32_t*)hres_dev, (int64_t)16384,
                                    counter, dflag, seq);
                 while (*(volatile unsigned*)hflag != seq) {
                 }
               }));
      }
    }
    cudaFuncSetAttribute(spin_publish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int threads : {128, 640}) {
      for (int smem : {0, 100 * 1024, 200 * 1024}) {
        for (int per : {1, 111}) {
          printf("H2D+spinpub threads=%d smem=%6d per_cta=%3d %7.2f us\n", threads, smem, per, med_us([&] {
                   ++seq;
                   cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
                   spin_publish_kernel<<<148, threads, smem, s>>>(cyc20, (const uint32_t*)dout, (uint32_t*)hres_dev, per,
                                                                 counter, dflag, seq, smem > 0);
                   while (*(volatile unsigned*)hflag != seq) {
                   }
                 }));
        }
      }
    }
    for (int threads : {128, 640}) {
      for (int nw : {16, 16384, 32768}) {
        printf("H2D+spin lastcopy threads=%d words=%5d   %7.2f us\n", threads, nw, med_us([&] {
                 ++seq;
                 cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
                 spin_lastcopy_kernel<<<148, threads, 0, s>>>(cyc20, (const uint32_t*)dout, (uint32_t*)hres_dev, nw, counter,
                                                              dflag, seq);
                 while (*(volatile unsigned*)hflag != seq) {
                 }
               }));
      }
    }
    void* hvm;
    cudaHostAlloc(&hvm, 1 << 20, cudaHostAllocMapped);
    void* hvm_dev;
    cudaHostGetDevicePointer(&hvm_dev, hvm, 0);
    int* sink;
    cudaMalloc(&sink, 64);
    for (long long cyc : {0LL, cyc20}) {
      printf("zc read64K (148 CTAs) + spin%lld + write + sync %7.2f us\n", cyc ? 20LL : 0LL, med_us([&] {
               zc_kernel<<<148, 640, 0, s>>>(cyc, (const int4*)hvm_dev, 4096, (uint32_t*)hres_dev, 111, sink);
               cudaStreamSynchronize(s);
             }));
      printf("zc no-read + spin%lld + write + sync          %7.2f us\n", cyc ? 20LL : 0LL, med_us([&] {
               zc_kernel<<<148, 640, 0, s>>>(cyc, (const int4*)hvm_dev, 0, (uint32_t*)hres_dev, 111, sink);
               cudaStreamSynchronize(s);
             }));
      printf("H2D + zc(dev v) + spin%lld + write + sync     %7.2f us\n", cyc ? 20LL : 0LL, med_us([&] {
               cudaMemcpyAsync(dv, hv, 65536, cudaMemcpyHostToDevice, s);
               zc_kernel<<<148, 640, 0, s>>>(cyc, (const int4*)dv, 4096, (uint32_t*)hres_dev, 111, sink);
               cudaStreamSynchronize(s);
             }));
    }
    std::vector<double> out(16384);
    printf("convert 16K int32 mapped->f64       %7.2f us\n", med_us([&] {
             const int* src = (const int*)hres;
             for (int i = 0; i < 16384; ++i) out[i] = src[i];
           }));
    std::vector<int> src2(16384);
    printf("memcpy 64KB pageable->pinned        %7.2f us\n", med_us([&] { memcpy(hv, src2.data(), 65536); }));
  }
  printf("spin20 alone (events)               ");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 100; ++i) spin_kernel<<<148, 128, 0, s>>>(cyc20);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%7.2f us\n", ms * 10);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
