// Host-buffer sessions: the end-to-end call a reference-side binding makes
// (`multiply_ternary(numpy v, idx)`, kernels.py:196-206 — host vector in, fresh host result out).
//
// A session owns, for one index, mapped pinned staging for v, a device copy of v and of the
// result, and mapped pinned result memory, allocated once and reused every call.  A call copies
// v into the staging while classifying it (host_stage.cpp: integer-valued vectors run on the
// exact int32 kernel when sum |v| fits int32, on the exact wide multiply otherwise).  A
// single-split scatter multiply (int32 / fp32 activations, rows <= 16384) is then ONE kernel
// launch (a captured one-node graph after the first call): the kernel pulls the staged v from
// mapped memory itself and streams each folded block's results into mapped memory as seq-tagged
// 64-bit words (csrc/common.cuh Publish), which the host converts into the caller's buffer while
// later blocks still run — no copy node, no D2H, no stream synchronize
// (tools/microbench/launch_latency.cu, session_timeline.cu measured the alternatives on the B200
// box).  Other forms are H2D, the multiply, a D2H copy and a stream synchronize.
#include <emmintrin.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "host_stage.h"

namespace rsr {
size_t wide_workspace_bytes(const rsr_index_desc& d, uint64_t max_abs);
rsr_status multiply_wide(const rsr_index_desc& d, const int64_t* v, uint64_t max_abs, void* out, rsr_dtype ot,
                         rsr_variant var, int b0, int b1, void* ws, size_t ws_bytes, cudaStream_t s, int exp2 = 0);
namespace {
size_t dsize(rsr_dtype t) { return (t == RSR_F64 || t == RSR_I64) ? 8 : 4; }
}  // namespace
}  // namespace rsr

struct rsr_host_session {
  rsr_index_desc desc;
  void* h_v = nullptr;                      // pinned, mapped staging [rows], 8 bytes per row (+ the seq word)
  void* h_v_dev = nullptr;                  // its device address (the kernel's pull source)
  unsigned long long* h_tag = nullptr;      // pinned, mapped [cols] tagged results (seq << 32 | value)
  unsigned long long* h_tag_dev = nullptr;
  uint32_t* d_sync = nullptr;               // device pull arrival counters (Publish::sync), int32 and fp32 kinds
  void* h_copy = nullptr;   // pinned [cols], 8 bytes per column (D2H path)
  void* d_v = nullptr;      // [rows], 8 bytes per row
  void* d_out = nullptr;    // [cols], 8 bytes per column
  void* d_wide = nullptr;   // wide-multiply workspace (whole int64 range), allocated on first use
  size_t wide_bytes = 0;
  uint32_t seq = 0;
  // Publishing calls replay a captured one-node graph (the pulling, publishing multiply):
  // [kind: int32, fp32][variant]
  cudaGraphExec_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int direct_calls[2][2] = {{0, 0}, {0, 0}};
  cudaStream_t cap = nullptr;
  size_t seq_off = 0;       // byte offset of the seq word in h_v / d_v (after a 4-byte-element v)
};

using rsr::cuda_check;
using rsr::fail;

namespace {
void session_free(rsr_host_session* h) {
  if (!h) return;
  if (h->h_v) cudaFreeHost(h->h_v);
  if (h->h_tag) cudaFreeHost(h->h_tag);
  if (h->d_sync) cudaFree(h->d_sync);
  if (h->h_copy) cudaFreeHost(h->h_copy);
  if (h->d_v) cudaFree(h->d_v);
  if (h->d_out) cudaFree(h->d_out);
  if (h->d_wide) cudaFree(h->d_wide);
  for (auto& gk : h->graph)
    for (auto& g : gk)
      if (g) cudaGraphExecDestroy(g);
  if (h->cap) cudaStreamDestroy(h->cap);
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
    const char* names[4] = {"stage", "enqueue", "wait", "convert"};
    fprintf(stderr, "session phases, median us:");
    for (int i = 0; i < 4; ++i) {
      if (v[i].empty()) continue;
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

// Published (tagged) int32 / fp32 results -> out_host (float64, or the 4-byte vector type).
rsr_status read_published(rsr_host_session* h, uint32_t seq, rsr_dtype vt, void* out_host, rsr_dtype out_dtype,
                          cudaStream_t s) {
  const rsr_index_desc& d = h->desc;
  rsr_status st = RSR_OK;
  // tagged: every word is accepted once its tag is this call's seq (an aligned 16-byte load sees
  // two whole 64-bit stores); two words per step, SSE2: the tag check, the int32 / fp32 -> fp64
  // conversion and the store.  While a pair is not ready, spin (asking the stream every few
  // thousand polls whether the launch failed).
  const int64_t m = d.cols;
  const unsigned long long* res = h->h_tag;
  const __m128i want = _mm_set1_epi32((int)seq);
  const bool f64 = out_dtype == RSR_F64, i32 = vt == RSR_I32;
  auto wait_ready = [&](int64_t i, int64_t n) -> rsr_status {  // words [i, i + n) tagged
    for (uint32_t spins = 1;; ++spins) {
      asm volatile("" ::: "memory");
      bool ok = true;
      for (int64_t j = i; j < i + n; ++j) ok &= (uint32_t)(((const volatile unsigned long long*)res)[j] >> 32) == seq;
      if (ok) return RSR_OK;
      _mm_pause();
      if ((spins & 1023u) == 0) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) {
          asm volatile("" ::: "memory");
          bool done = true;
          for (int64_t j = i; j < i + n; ++j) done &= (uint32_t)(((const volatile unsigned long long*)res)[j] >> 32) == seq;
          if (!done) return fail(RSR_ERR_CUDA, "host session: the multiply completed without publishing");
        } else if (e != cudaErrorNotReady) {
          return cuda_check(e, "host session multiply");
        }
      }
    }
  };
  int64_t i = 0;
  while (i + 2 <= m) {
    asm volatile("" ::: "memory");
    const __m128i x = _mm_load_si128(reinterpret_cast<const __m128i*>(res + i));
    const __m128i tags = _mm_shuffle_epi32(x, _MM_SHUFFLE(3, 1, 3, 1));
    if ((_mm_movemask_epi8(_mm_cmpeq_epi32(tags, want)) & 0xff) != 0xff) {
      if ((st = wait_ready(i, 2)) != RSR_OK) return st;
      continue;  // reload the pair
    }
    const __m128i vals = _mm_shuffle_epi32(x, _MM_SHUFFLE(2, 0, 2, 0));
    if (f64) _mm_storeu_pd((double*)out_host + i, i32 ? _mm_cvtepi32_pd(vals) : _mm_cvtps_pd(_mm_castsi128_ps(vals)));
    else _mm_storel_epi64(reinterpret_cast<__m128i*>((uint32_t*)out_host + i), vals);
    i += 2;
  }
  if (i < m) {
    if ((st = wait_ready(i, 1)) != RSR_OK) return st;
    const uint32_t bits = (uint32_t)((const volatile unsigned long long*)res)[i];
    if (f64) ((double*)out_host)[i] = i32 ? (double)(int32_t)bits : (double)__builtin_bit_cast(float, bits);
    else ((uint32_t*)out_host)[i] = bits;
  }
  return RSR_OK;
}
}  // namespace

extern "C" {

rsr_status rsr_host_session_create(const rsr_index_desc* desc, rsr_host_session** out) {
  if (!desc || !out) return fail(RSR_ERR_INVALID, "null argument");
  if (desc->rows < 1 || desc->cols < 1 || (desc->halves != 1 && desc->halves != 2))
    return fail(RSR_ERR_INVALID, "bad index descriptor");
  auto* h = new rsr_host_session();
  h->desc = *desc;
  h->seq_off = (4 * (size_t)desc->rows + 15) & ~(size_t)15;  // after a 4-byte-element v
  const size_t vb = std::max(8 * (size_t)desc->rows, h->seq_off + 16);
  const size_t ob = 8 * (size_t)desc->cols;
  rsr_status st = cuda_check(cudaHostAlloc(&h->h_v, vb, cudaHostAllocMapped), "session pinned v");
  if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer(&h->h_v_dev, h->h_v, 0), "session staging mapping");
  if (st == RSR_OK) st = cuda_check(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking), "session capture stream");
  if (st == RSR_OK)
    st = cuda_check(cudaHostAlloc((void**)&h->h_tag, 8 * (size_t)desc->cols, cudaHostAllocMapped), "session mapped result");
  if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer((void**)&h->h_tag_dev, h->h_tag, 0), "session result mapping");
  if (st == RSR_OK) std::memset(h->h_tag, 0, 8 * (size_t)desc->cols);  // tag 0: no call's result
  if (st == RSR_OK) st = cuda_check(cudaMalloc((void**)&h->d_sync, 64), "session pull counter");
  if (st == RSR_OK) st = cuda_check(cudaMemset(h->d_sync, 0, 64), "session pull counter init");
  if (st == RSR_OK) st = cuda_check(cudaHostAlloc(&h->h_copy, ob, cudaHostAllocDefault), "session pinned result");
  if (st == RSR_OK) st = cuda_check(cudaMalloc(&h->d_v, vb), "session device v");
  if (st == RSR_OK) st = cuda_check(cudaMalloc(&h->d_out, ob), "session device result");
  if (st != RSR_OK) {
    session_free(h);
    return st;
  }
  *out = h;
  return RSR_OK;
}

void rsr_host_session_destroy(rsr_host_session* h) { session_free(h); }

rsr_status rsr_host_session_multiply(rsr_host_session* h, const void* v_host, rsr_dtype v_dtype, size_t v_bytes,
                                     void* out_host, rsr_dtype out_dtype, size_t out_bytes, rsr_variant variant,
                                     void* stream) {
  if (!h || !v_host || !out_host) return fail(RSR_ERR_INVALID, "null argument");
  const rsr_index_desc& d = h->desc;
  if (v_dtype != RSR_I32 && v_dtype != RSR_I64 && v_dtype != RSR_F32 && v_dtype != RSR_F64)
    return fail(RSR_ERR_INVALID, "unknown dtype");
  if (v_bytes != rsr::dsize(v_dtype) * (size_t)d.rows)
    return fail(RSR_ERR_INVALID, "vector length " + std::to_string(v_bytes / rsr::dsize(v_dtype)) + " does not match " +
                                     std::to_string(d.rows) + " rows");
  if (out_dtype != RSR_F64 && out_dtype != v_dtype)
    return fail(RSR_ERR_INVALID, "result type must be float64 or the vector type");
  if (out_bytes != rsr::dsize(out_dtype) * (size_t)d.cols) return fail(RSR_ERR_INVALID, "result buffer size does not match");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP) return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  cudaStream_t s = (cudaStream_t)stream;
  const bool tr = g_trace.on;
  double t0 = tr ? now_us() : 0, t1 = 0;
  // stage + classify (one pass for the common case)
  const rsr::StageInfo cls = rsr::stage_vector(v_host, v_dtype, d.rows, h->h_v, out_dtype == RSR_I32);
  if (cls.kind == rsr::kStageNonFinite) return fail(RSR_ERR_INVALID, "vector entries must be finite");
  if (tr) { t1 = now_us(); g_trace.v[0].push_back(t1 - t0); t0 = t1; }
  const rsr_dtype kt = cls.kind == rsr::kStageI32 ? RSR_I32
                       : (cls.kind == rsr::kStageWide || cls.kind == rsr::kStageFixed) ? RSR_I64
                       : cls.kind == rsr::kStageF32 ? RSR_F32 : RSR_F64;  // computed (and staged) type
  const size_t vb = rsr::dsize(kt) * (size_t)d.rows;
  rsr_status st = RSR_OK;
  rsr_dtype rt = kt;  // device result type
  if (rsr::publishes(d, kt)) {
    // one launch: the kernel pulls the staging (v, then the seq word) and streams tagged results
    const uint32_t seq = ++h->seq == 0 ? ++h->seq : h->seq;  // never 0 (the buffer's initial tag)
    const int gk = kt == RSR_I32 ? 0 : 1, gv = variant == RSR_VARIANT_RSRPP ? 1 : 0;
    *reinterpret_cast<volatile uint32_t*>((char*)h->h_v + h->seq_off) = seq;
    // (one arrival counter per kind: the int32 and fp32 launches may differ in grid)
    // RSR_B200_PULL_STEAL_NS (tests): the chunk wait after which a CTA copies the payload itself
    static const uint32_t steal_ns = getenv("RSR_B200_PULL_STEAL_NS") ? (uint32_t)atol(getenv("RSR_B200_PULL_STEAL_NS")) : 20000u;
    const rsr::Publish pub{h->h_tag_dev, h->h_v_dev, (uint32_t)(h->seq_off + 16), (uint32_t)h->seq_off, h->d_sync + 8 * gk, 0,
                           steal_ns};
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const bool can_graph = cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
    bool published = false;
    if (h->graph[gk][gv] == nullptr && can_graph && h->direct_calls[gk][gv] >= 1) {
      // capture once (after one direct call, which set the kernel's attributes)
      cudaGraph_t g = nullptr;
      bool gpublished = false;
      if (cuda_check(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal), "session capture") == RSR_OK) {
        const rsr_status a = rsr::multiply(d, h->d_v, kt, h->d_out, kt, variant, RSR_FORM_AUTO, 0, d.nblocks, h->cap,
                                           &pub, &gpublished);
        const cudaError_t e = cudaStreamEndCapture(h->cap, &g);
        if (a == RSR_OK && e == cudaSuccess && gpublished) {
          cudaGraphExec_t ex = nullptr;
          if (cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) h->graph[gk][gv] = ex;
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // a failed capture only means no graph: the direct path stays
      }
    }
    if (can_graph && h->graph[gk][gv]) {
      st = cuda_check(cudaGraphLaunch(h->graph[gk][gv], s), "session graph launch");
      published = true;
    } else {
      ++h->direct_calls[gk][gv];
      st = rsr::multiply(d, h->d_v, kt, h->d_out, kt, variant, RSR_FORM_AUTO, 0, d.nblocks, s, &pub, &published);
    }
    if (st == RSR_OK && !published) st = fail(RSR_ERR_CUDA, "host session: the multiply did not publish");
    if (st != RSR_OK) return st;
    if (tr) { t1 = now_us(); g_trace.v[1].push_back(t1 - t0); t0 = t1; }
    // int32 / int64 vectors staged as int32 deliver int32 results
    const rsr_dtype od = out_dtype == RSR_F64 ? RSR_F64 : kt;
    if (out_dtype == RSR_I64) {  // int64 vector whose sum fit int32: widen the int32 results
      st = read_published(h, seq, kt, h->h_copy, RSR_I32, s);
      if (st == RSR_OK) convert((const int32_t*)h->h_copy, (int64_t*)out_host, d.cols);
    } else {
      st = read_published(h, seq, kt, out_host, od, s);
    }
    if (tr) g_trace.v[3].push_back(now_us() - t0);
    return st;
  }
  st = cuda_check(cudaMemcpyAsync(h->d_v, h->h_v, vb, cudaMemcpyHostToDevice, s), "H2D v");
  if (st != RSR_OK) return st;
  if (kt == RSR_I64) {
    rt = (out_dtype == RSR_I64 && cls.kind != rsr::kStageFixed) ? RSR_I64 : RSR_F64;
    const size_t need = rsr::wide_workspace_bytes(d, 0);
    if (h->wide_bytes < need) {
      if (h->d_wide) cudaFree(h->d_wide);
      h->d_wide = nullptr;
      h->wide_bytes = 0;
      if ((st = cuda_check(cudaMalloc(&h->d_wide, need), "session wide workspace")) != RSR_OK) return st;
      h->wide_bytes = need;
    }
    st = rsr::multiply_wide(d, (const int64_t*)h->d_v, cls.max_abs, h->d_out, rt, variant, 0, d.nblocks, h->d_wide,
                            h->wide_bytes, s, cls.kind == rsr::kStageFixed ? cls.exp2 : 0);
  } else {
    st = rsr::multiply(d, h->d_v, kt, h->d_out, kt, variant, RSR_FORM_AUTO, 0, d.nblocks, s);
  }
  if (st != RSR_OK) return st;
  const size_t ob = rsr::dsize(rt) * (size_t)d.cols;
  if ((st = cuda_check(cudaMemcpyAsync(h->h_copy, h->d_out, ob, cudaMemcpyDeviceToHost, s), "D2H out")) != RSR_OK)
    return st;
  if (tr) { t1 = now_us(); g_trace.v[1].push_back(t1 - t0); t0 = t1; }
  if ((st = cuda_check(cudaStreamSynchronize(s), "stream sync")) != RSR_OK) return st;
  if (tr) { t1 = now_us(); g_trace.v[2].push_back(t1 - t0); t0 = t1; }
  if (rt == out_dtype) std::memcpy(out_host, h->h_copy, ob);
  else if (rt == RSR_I32 && out_dtype == RSR_F64) convert((const int32_t*)h->h_copy, (double*)out_host, d.cols);
  else if (rt == RSR_I32 && out_dtype == RSR_I64) convert((const int32_t*)h->h_copy, (int64_t*)out_host, d.cols);
  else if (rt == RSR_F32) convert((const float*)h->h_copy, (double*)out_host, d.cols);
  else return fail(RSR_ERR_INVALID, "unsupported result conversion");
  if (tr) g_trace.v[3].push_back(now_us() - t0);
  return RSR_OK;
}

}  // extern "C"
