// Host + device timeline of one host-buffer session call (16384^2 ternary, int32), against the
// diagnostic trace build (make trace): host phase stamps vs the scatter kernel's per-CTA
// globaltimer stamps, aligned by a calibration kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../include session_timeline.cu \
//        -L../../paper_2411_06360_b200/lib/trace -lrsr_b200_trace -Xlinker -rpath,... -o session_timeline
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "rsr_b200.h"

extern "C" int rsr_debug_trace_copy(unsigned long long* host, size_t n);

__global__ void stamp_kernel(volatile unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  *dst = t;
}

static double host_ns() {
  return (double)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

#define CK(x)                                                          \
  do {                                                                 \
    int _e = (int)(x);                                                 \
    if (_e) {                                                          \
      printf("fail %s: %d %s\n", #x, _e, rsr_b200_last_error());       \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main() {
  const int64_t n = 16384, m = 16384;
  const int k = 11;
  const int ncopies = getenv("COPIES") ? atoi(getenv("COPIES")) : 1;  // > 1: cold index (rotating copies)
  std::vector<rsr_index_desc> ds(ncopies);
  size_t pb, sb, bb;
  for (auto& d : ds) {
    CK(rsr_index_layout(n, m, k, 2, &d, &pb, &sb, &bb));
    for (int h = 0; h < 2; ++h) {
      CK(cudaMalloc(&d.half[h].perm, pb));
      CK(cudaMalloc((void**)&d.half[h].seg, sb));
      CK(cudaMalloc((void**)&d.half[h].bucket, bb));
    }
  }
  std::vector<int8_t> A(n * m);
  std::mt19937 rng(1);
  for (auto& a : A) a = (int8_t)((int)(rng() % 3) - 1);
  int8_t* dA;
  CK(cudaMalloc(&dA, n * m));
  CK(cudaMemcpy(dA, A.data(), n * m, cudaMemcpyHostToDevice));
  size_t wsb = rsr_preprocess_workspace_bytes(&ds[0]);
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  int32_t* bad;
  CK(cudaMalloc(&bad, 4));
  CK(cudaMemset(bad, 0, 4));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<rsr_host_session*> sess(ncopies);
  for (int c = 0; c < ncopies; ++c) {
    CK(rsr_preprocess_ternary(dA, m, &ds[c], bad, ws, wsb, s));
    CK(cudaStreamSynchronize(s));
    CK(rsr_host_session_create(&ds[c], &sess[c]));
  }
  std::vector<int32_t> v(n);
  for (auto& x : v) x = (int32_t)(rng() % 201) - 100;
  std::vector<double> out(m);
  // calibration: device globaltimer -> host steady clock (offset includes the flag latency)
  unsigned long long* hs;
  CK(cudaHostAlloc((void**)&hs, 64, cudaHostAllocMapped));
  unsigned long long* hs_dev;
  CK(cudaHostGetDevicePointer((void**)&hs_dev, hs, 0));
  double off = 1e300;
  for (int i = 0; i < 50; ++i) {
    *(volatile unsigned long long*)hs = 0;
    stamp_kernel<<<1, 1, 0, s>>>(hs_dev);
    while (*(volatile unsigned long long*)hs == 0) {
    }
    const double h = host_ns();
    off = std::min(off, h - (double)*hs);  // host = gt + off (upper bound on device->host latency)
  }
  cudaStreamSynchronize(s);
  std::vector<unsigned long long> tr(148 * 512);
  long steals = 0;
  std::vector<double> rows[12];
  for (int it = 0; it < 400; ++it) {
    const double t0 = host_ns();
    CK(rsr_host_session_multiply(sess[it % ncopies], v.data(), RSR_I32, n * 4, out.data(), RSR_F64, m * 8,
                                 RSR_VARIANT_RSRPP, s));
    const double t1 = host_ns();
    CK(rsr_debug_trace_copy(tr.data(), tr.size()));
    double cs = 1e300, ce = 0, fe = 0, pe = 0, p0 = 0, p1 = 0, p2 = 0, p3 = 0, p4 = 0, p5 = 0;
    for (int c = 0; c < 148; ++c) {
      cs = std::min(cs, (double)tr[c * 512 + 0]);
      pe = std::max(pe, (double)tr[c * 512 + 1]);
      ce = std::max(ce, (double)tr[c * 512 + 7]);
      fe = std::max(fe, (double)tr[c * 512 + 6]);
      p0 = std::max(p0, (double)tr[c * 512 + 4]);  // PDL wait passed (the pull starts)
      p1 = std::max(p1, (double)tr[c * 512 + 502]);  // chunk copied + fenced
      p2 = std::max(p2, (double)tr[c * 512 + 503]);  // all chunks seen
      p3 = std::max(p3, (double)tr[c * 512 + 505]);  // arrived
      p4 = std::max(p4, (double)tr[c * 512 + 506]);  // the seq reader saw the call's seq
      p5 = std::max(p5, (double)tr[c * 512 + 507]);  // past the seq wait (speculative) / start of the copy
      if (tr[c * 512 + 504] > tr[c * 512 + 503]) ++steals;
    }
    const double flag_seen = t1 - t0;  // upper bound (includes the host conversion)
    (void)flag_seen;
    if (it >= 40) {
      rows[0].push_back((t1 - t0) / 1e3);
      rows[1].push_back((cs + off - t0) / 1e3);
      rows[2].push_back((pe + off - t0) / 1e3);
      rows[3].push_back((ce + off - t0) / 1e3);
      rows[4].push_back((fe + off - t0) / 1e3);
      rows[5].push_back((fe - cs) / 1e3);
      rows[6].push_back((p0 + off - t0) / 1e3);
      rows[7].push_back((p1 + off - t0) / 1e3);
      rows[8].push_back((p2 + off - t0) / 1e3);
      rows[9].push_back((p3 + off - t0) / 1e3);
      rows[10].push_back((p4 + off - t0) / 1e3);
      rows[11].push_back((p5 + off - t0) / 1e3);
    }
  }
  const char* names[12] = {"call total", "first CTA start", "last prologue end (v pulled, in registers)",
                          "last scatter end", "last fold end", "kernel span", "last CTA at the pull",
                          "last chunk copied", "last CTA past the wait", "last arrival", "seq seen by the reader",
                          "last CTA starting its copy"};
  for (int i = 0; i < 12; ++i) {
    std::sort(rows[i].begin(), rows[i].end());
    printf("%-24s median %7.2f us  (p10 %7.2f  p90 %7.2f)\n", names[i], rows[i][rows[i].size() / 2],
           rows[i][rows[i].size() / 10], rows[i][rows[i].size() * 9 / 10]);
  }
  printf("CTA-calls that stole the payload: %ld\n", steals);
  printf("(device stamps are shifted by the calibration latency, an upper bound of ~1-2 us)\n");
  return 0;
}
