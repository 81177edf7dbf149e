// Host-observed round trips of the pieces of a host-buffer call (one B200, idle GPU):
//   (a) launch a 148-CTA kernel that raises a mapped flag           -> host sees the flag
//   (b) H2D of 64 KB (pinned) + the same kernel, direct stream calls
//   (c) (b) captured as one graph
//   (d) the kernel pulls the 64 KB from MAPPED host memory itself (each CTA a slice -> global,
//       grid barrier), then raises the flag: no copy node
//   (e) (a) with a system-scope fence before the flag
//   (f) the host reading + converting 64 KB of int32 results (mapped, written by the GPU) to fp64
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 launch_latency.cu -o launch_latency
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void flag_kernel(volatile unsigned* flag, unsigned seq, int fence) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (fence) __threadfence_system();
    *flag = seq;
  }
}

// each CTA copies its slice of the mapped vector to global, then a grid barrier, then CTA 0 flags
__global__ void pull_kernel(const int4* __restrict__ hv, int4* dv, int n16, unsigned* bar, volatile unsigned* flag,
                            unsigned call, int* sink) {
  const int per = (n16 + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * per, hi = min(n16, lo + per);
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) dv[i] = hv[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (atomicAdd(bar, 0u) < call * gridDim.x) {
    }
  }
  __syncthreads();
  // every CTA now reads the whole vector from L2 (what the scatter prologue does)
  int acc = 0;
  for (int i = threadIdx.x; i < n16; i += blockDim.x) acc += __ldcg(dv + i).x;
  if (acc == 0x7fffffff) sink[0] = acc;
  if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 0x80000000u | call;
}

int main() {
  const int n = 16384, bytes = 4 * n, reps = 300;
  unsigned *h_flag, *d_flag;
  cudaHostAlloc((void**)&h_flag, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&d_flag, h_flag, 0);
  int *h_v, *d_v, *h_vm, *d_vm, *sink;
  unsigned* bar;
  cudaHostAlloc((void**)&h_v, bytes, cudaHostAllocDefault);
  cudaHostAlloc((void**)&h_vm, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&d_vm, h_vm, 0);
  cudaMalloc(&d_v, bytes);
  cudaMalloc(&sink, 64);
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  for (int i = 0; i < n; ++i) h_v[i] = h_vm[i] = i % 201 - 100;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned seq = 0;
  auto wait = [&](unsigned q) {
    while (*(volatile unsigned*)h_flag != q) {
    }
  };
  auto run = [&](const char* name, auto&& fn) {
    std::vector<double> t;
    for (int i = 0; i < reps; ++i) {
      const double t0 = now_us();
      fn();
      t.push_back(now_us() - t0);
    }
    cudaStreamSynchronize(s);
    std::sort(t.begin() + 0, t.end());
    printf("%-58s median %6.2f us  p10 %6.2f  p90 %6.2f\n", name, t[reps / 2], t[reps / 10], t[reps * 9 / 10]);
  };
  run("(a) launch 148x640 kernel -> flag", [&] {
    flag_kernel<<<148, 640, 0, s>>>(h_flag ? d_flag : nullptr, ++seq, 0);
    wait(seq);
  });
  run("(e) (a) + __threadfence_system before the flag", [&] {
    flag_kernel<<<148, 640, 0, s>>>(d_flag, ++seq, 1);
    wait(seq);
  });
  run("(b) H2D 64 KB + kernel -> flag (direct)", [&] {
    cudaMemcpyAsync(d_v, h_v, bytes, cudaMemcpyHostToDevice, s);
    flag_kernel<<<148, 640, 0, s>>>(d_flag, ++seq, 0);
    wait(seq);
  });
  // (c) graph: the seq word travels inside the copied payload, the kernel reads it
  {
    cudaGraph_t g;
    cudaGraphExec_t ex;
    cudaStream_t cap;
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    unsigned* h_seqsrc = reinterpret_cast<unsigned*>(h_v);  // first word of the payload = seq
    cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    cudaMemcpyAsync(d_v, h_v, bytes, cudaMemcpyHostToDevice, cap);
    flag_kernel<<<148, 640, 0, cap>>>(d_flag, 0, 0);  // flag value patched below: use kernel reading d_v
    cudaStreamEndCapture(cap, &g);
    cudaGraphInstantiate(&ex, g, 0);
    run("(c) graph [H2D 64 KB -> kernel] -> flag (seq 0 written)", [&] {
      *h_flag = 1;
      h_seqsrc[0] = ++seq;
      cudaGraphLaunch(ex, s);
      wait(0);
    });
  }
  unsigned call = 0;  // the barrier counter counts 148 arrivals per call
  run("(d) kernel pulls 64 KB from mapped memory, grid barrier -> flag", [&] {
    ++call;
    pull_kernel<<<148, 640, 0, s>>>(reinterpret_cast<const int4*>(d_vm), reinterpret_cast<int4*>(d_v), n / 4, bar,
                                    d_flag, call, sink);
    wait(0x80000000u | call);
  });
  // (g) graph of the flag kernel alone; (i) direct H2D + kernel
  // launched with cudaLaunchKernelEx and the programmatic-serialization attribute (as multiply.cu)
  {
    cudaStream_t cap;
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    unsigned* d_seq;
    cudaMalloc(&d_seq, 4);
    cudaGraph_t g;
    cudaGraphExec_t ex;
    cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    flag_kernel<<<148, 640, 0, cap>>>(d_flag, 0, 0);
    cudaStreamEndCapture(cap, &g);
    cudaGraphInstantiate(&ex, g, 0);
    run("(g) graph [kernel] -> flag", [&] {
      *h_flag = 1;
      cudaGraphLaunch(ex, s);
      wait(0);
    });
    run("(i) direct H2D 64 KB + cudaLaunchKernelEx(PDL attr) -> flag", [&] {
      cudaMemcpyAsync(d_v, h_v, bytes, cudaMemcpyHostToDevice, s);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(640);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      ++seq;
      cudaLaunchKernelEx(&cfg, flag_kernel, (volatile unsigned*)d_flag, seq, 0);
      wait(seq);
    });
  }
  // (f) host read + convert of 64 KB of GPU-written mapped results
  {
    int* h_res;
    int* d_res;
    cudaHostAlloc((void**)&h_res, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void**)&d_res, h_res, 0);
    std::vector<double> out(n);
    std::vector<double> t;
    for (int i = 0; i < 100; ++i) {
      cudaMemcpyAsync(d_res, d_v, bytes, cudaMemcpyDeviceToDevice, s);  // GPU writes the mapped buffer
      cudaStreamSynchronize(s);
      const double t0 = now_us();
      for (int j = 0; j < n; ++j) out[j] = (double)h_res[j];
      t.push_back(now_us() - t0);
    }
    std::sort(t.begin(), t.end());
    printf("%-58s median %6.2f us\n", "(f) host converts 64 KB of GPU-written mapped int32 -> fp64", t[50]);
    std::vector<double> fresh_t;
    for (int i = 0; i < 100; ++i) {
      const double t0 = now_us();
      double* o = (double*)malloc(8 * n);
      for (int j = 0; j < n; ++j) o[j] = (double)h_res[j];
      fresh_t.push_back(now_us() - t0);
      asm volatile("" ::"r"(o) : "memory");
      free(o);
    }
    std::sort(fresh_t.begin(), fresh_t.end());
    printf("%-58s median %6.2f us\n", "(f') same into a fresh malloc(128 KB) each call", fresh_t[50]);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
