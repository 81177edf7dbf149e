// Host cost of enqueueing one multiply (rsr_multiply, int32, 16384^2 ternary) vs an empty
// kernel launch, no synchronization inside the measured loop (200 calls, queue never full).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "rsr_b200.h"

__global__ void empty_kernel() {}

int main() {
  const int64_t n = 16384, m = 16384;
  rsr_index_desc d{};
  size_t pb, sb, bb;
  rsr_index_layout(n, m, 11, 2, &d, &pb, &sb, &bb);
  for (int h = 0; h < 2; ++h) {
    cudaMalloc(&d.half[h].perm, pb);
    cudaMalloc((void**)&d.half[h].seg, sb);
    cudaMalloc((void**)&d.half[h].bucket, bb);
  }
  std::vector<int8_t> A(n * m);
  std::mt19937 rng(1);
  for (auto& a : A) a = (int8_t)((int)(rng() % 3) - 1);
  int8_t* dA;
  cudaMalloc(&dA, n * m);
  cudaMemcpy(dA, A.data(), n * m, cudaMemcpyHostToDevice);
  size_t wsb = rsr_preprocess_workspace_bytes(&d);
  void* ws;
  cudaMalloc(&ws, wsb);
  int32_t* bad;
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  rsr_preprocess_ternary(dA, m, &d, bad, ws, wsb, s);
  cudaStreamSynchronize(s);
  int32_t *dv, *dout;
  cudaMalloc(&dv, n * 4);
  cudaMalloc(&dout, m * 4);
  cudaMemset(dv, 0, n * 4);
  auto run = [&](const char* name, auto f) {
    for (int i = 0; i < 20; ++i) f();
    cudaStreamSynchronize(s);
    double best = 1e30;
    for (int rep = 0; rep < 5; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < 200; ++i) f();
      auto t1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(s);
      best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / 200);
    }
    printf("%-34s %6.2f us per enqueue\n", name, best);
  };
  run("empty kernel <<<>>>", [&] { empty_kernel<<<1, 32, 0, s>>>(); });
  run("cudaMemcpyAsync H2D 64KB (device)", [&] { cudaMemcpyAsync(dv, dout, n * 4, cudaMemcpyDeviceToDevice, s); });
  run("rsr_multiply (int32 scatter)", [&] {
    rsr_multiply(&d, dv, RSR_I32, dout, RSR_I32, RSR_VARIANT_RSRPP, RSR_FORM_AUTO, 0, d.nblocks, s);
  });
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
