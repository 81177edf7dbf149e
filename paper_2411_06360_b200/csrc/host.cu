// Host-buffer sessions: the end-to-end call a reference-side binding makes
// (`multiply_ternary(numpy v, idx)`, kernels.py:196-206 — host vector in, fresh host result out).
//
// A session owns, for one index and one vector type, pinned staging for v, a device copy of v
// and of the result, a MAPPED pinned result buffer and a mapped completion flag, allocated once
// and reused every call.  A call is: memcpy v -> pinned staging, H2D(v), the multiply, and the
// conversion into the caller's buffer.  A single-split scatter multiply (int32 / fp32
// activations, rows <= 16384) publishes its results itself (csrc/multiply.cu, Publish: every
// CTA stores its columns into the mapped buffer, the last one raises the flag), and the host
// polls the flag — no D2H copy and no stream synchronize between the kernel and the caller
// (tools/microbench/sync_probe.cu, session_timeline.cu measured the completion schemes on the
// B200 box).  Other forms are followed by a D2H copy and a stream synchronize.
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace rsr {
namespace {
size_t dsize(rsr_dtype t) { return t == RSR_F64 ? 8 : 4; }
}  // namespace
}  // namespace rsr

struct rsr_host_session {
  rsr_index_desc desc;
  rsr_dtype v_dtype;        // host vector type = device result type (int32 -> int32, fp32 -> fp32, fp64 -> fp64)
  void* h_v = nullptr;      // pinned staging [rows]
  void* h_res = nullptr;    // pinned, mapped [cols] of v_dtype (published results)
  void* h_res_dev = nullptr;
  void* h_copy = nullptr;   // pinned [cols] of v_dtype (D2H path)
  uint32_t* h_flag = nullptr;  // pinned, mapped
  uint32_t* h_flag_dev = nullptr;
  void* d_v = nullptr;
  void* d_out = nullptr;
  uint32_t* d_counter = nullptr;
  uint32_t seq = 0;
};

using rsr::cuda_check;
using rsr::fail;

namespace {
void session_free(rsr_host_session* h) {
  if (!h) return;
  if (h->h_v) cudaFreeHost(h->h_v);
  if (h->h_res) cudaFreeHost(h->h_res);
  if (h->h_copy) cudaFreeHost(h->h_copy);
  if (h->h_flag) cudaFreeHost(h->h_flag);
  if (h->d_counter) cudaFree(h->d_counter);
  if (h->d_v) cudaFree(h->d_v);
  if (h->d_out) cudaFree(h->d_out);
  delete h;
}

template <typename S, typename D>
void convert(const S* __restrict__ s, D* __restrict__ d, int64_t n) {
  for (int64_t i = 0; i < n; ++i) d[i] = (D)s[i];
}

// Diagnostics only (RSR_B200_SESSION_TRACE=1): median host time of each phase, printed at exit.
struct PhaseTrace {
  bool on = getenv("RSR_B200_SESSION_TRACE") != nullptr;
  std::vector<double> v[4];
  ~PhaseTrace() {
    if (!on || v[0].empty()) return;
    const char* names[4] = {"memcpy", "enqueue", "wait", "convert"};
    fprintf(stderr, "session phases, median us:");
    for (int i = 0; i < 4; ++i) {
      std::sort(v[i].begin(), v[i].end());
      fprintf(stderr, "  %s %.2f", names[i], v[i][v[i].size() / 2]);
    }
    fprintf(stderr, "  calls %zu\n", v[0].size());
  }
};
PhaseTrace g_trace;
inline double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

rsr_status rsr_host_session_create(const rsr_index_desc* desc, rsr_dtype v_dtype, rsr_host_session** out) {
  if (!desc || !out) return fail(RSR_ERR_INVALID, "null argument");
  if (desc->rows < 1 || desc->cols < 1 || (desc->halves != 1 && desc->halves != 2))
    return fail(RSR_ERR_INVALID, "bad index descriptor");
  if (v_dtype != RSR_I32 && v_dtype != RSR_F32 && v_dtype != RSR_F64) return fail(RSR_ERR_INVALID, "unknown dtype");
  auto* h = new rsr_host_session();
  h->desc = *desc;
  h->v_dtype = v_dtype;
  const size_t vb = rsr::dsize(v_dtype) * (size_t)desc->rows;
  const size_t ob = rsr::dsize(v_dtype) * (size_t)desc->cols;
  rsr_status st = cuda_check(cudaHostAlloc(&h->h_v, vb, cudaHostAllocDefault), "session pinned v");
  if (st == RSR_OK) st = cuda_check(cudaHostAlloc(&h->h_res, ob, cudaHostAllocMapped), "session mapped result");
  if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer(&h->h_res_dev, h->h_res, 0), "session result mapping");
  if (st == RSR_OK) st = cuda_check(cudaHostAlloc(&h->h_copy, ob, cudaHostAllocDefault), "session pinned result");
  if (st == RSR_OK) st = cuda_check(cudaHostAlloc((void**)&h->h_flag, 64, cudaHostAllocMapped), "session flag");
  if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer((void**)&h->h_flag_dev, h->h_flag, 0), "session flag mapping");
  if (st == RSR_OK) st = cuda_check(cudaMalloc((void**)&h->d_counter, 64), "session counter");
  if (st == RSR_OK) st = cuda_check(cudaMemset(h->d_counter, 0, 64), "session counter init");
  if (st == RSR_OK) st = cuda_check(cudaMalloc(&h->d_v, vb), "session device v");
  if (st == RSR_OK) st = cuda_check(cudaMalloc(&h->d_out, ob), "session device result");
  if (st != RSR_OK) {
    session_free(h);
    return st;
  }
  *h->h_flag = 0;
  *out = h;
  return RSR_OK;
}

void rsr_host_session_destroy(rsr_host_session* h) { session_free(h); }

rsr_status rsr_host_session_multiply(rsr_host_session* h, const void* v_host, size_t v_bytes, void* out_host,
                                     size_t out_bytes, rsr_dtype out_dtype, rsr_variant variant, void* stream) {
  if (!h || !v_host || !out_host) return fail(RSR_ERR_INVALID, "null argument");
  const rsr_index_desc& d = h->desc;
  if (v_bytes != rsr::dsize(h->v_dtype) * (size_t)d.rows)
    return fail(RSR_ERR_INVALID, "vector length does not match " + std::to_string(d.rows) + " rows");
  if (out_dtype != RSR_F64 && out_dtype != h->v_dtype)
    return fail(RSR_ERR_INVALID, "result type must be float64 or the vector type");
  if (out_bytes != rsr::dsize(out_dtype) * (size_t)d.cols) return fail(RSR_ERR_INVALID, "result buffer size does not match");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP) return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  cudaStream_t s = (cudaStream_t)stream;
  const bool tr = g_trace.on;
  double t0 = tr ? now_us() : 0, t1 = 0;
  const size_t vb = rsr::dsize(h->v_dtype) * (size_t)d.rows, ob = rsr::dsize(h->v_dtype) * (size_t)d.cols;
  std::memcpy(h->h_v, v_host, vb);
  if (tr) { t1 = now_us(); g_trace.v[0].push_back(t1 - t0); t0 = t1; }
  rsr_status st = cuda_check(cudaMemcpyAsync(h->d_v, h->h_v, vb, cudaMemcpyHostToDevice, s), "H2D v");
  if (st != RSR_OK) return st;
  const uint32_t seq = ++h->seq == 0 ? ++h->seq : h->seq;  // never 0 (the flag's initial value)
  const rsr::Publish pub{h->h_res_dev, h->d_counter, h->h_flag_dev, seq};
  bool published = false;
  st = rsr::multiply(d, h->d_v, h->v_dtype, h->d_out, h->v_dtype, variant, RSR_FORM_AUTO, 0, d.nblocks, s, &pub,
                     &published);
  if (st != RSR_OK) return st;
  if (!published && (st = cuda_check(cudaMemcpyAsync(h->h_copy, h->d_out, ob, cudaMemcpyDeviceToHost, s), "D2H out")) != RSR_OK)
    return st;
  if (tr) { t1 = now_us(); g_trace.v[1].push_back(t1 - t0); t0 = t1; }
  if (published) {
    // poll the flag; every few thousand polls ask the stream whether it failed
    volatile uint32_t* flag = h->h_flag;
    for (uint32_t spins = 1; *flag != seq; ++spins) {
      _mm_pause();
      if ((spins & 1023u) == 0) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) {
          if (*flag != seq) return fail(RSR_ERR_CUDA, "host session: the multiply completed without publishing");
          break;
        }
        if (e != cudaErrorNotReady) return cuda_check(e, "host session multiply");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  } else if ((st = cuda_check(cudaStreamSynchronize(s), "stream sync")) != RSR_OK) {
    return st;
  }
  if (tr) { t1 = now_us(); g_trace.v[2].push_back(t1 - t0); t0 = t1; }
  const void* res = published ? h->h_res : h->h_copy;
  if (out_dtype == h->v_dtype) std::memcpy(out_host, res, ob);
  else if (h->v_dtype == RSR_I32) convert((const int32_t*)res, (double*)out_host, d.cols);
  else convert((const float*)res, (double*)out_host, d.cols);
  if (tr) g_trace.v[3].push_back(now_us() - t0);
  return RSR_OK;
}

}  // extern "C"
