// Host-buffer sessions: the end-to-end call a reference-side binding makes
// (`multiply_ternary(numpy v, idx)`, kernels.py:196-206 — host vector in, fresh host result out).
//
// A session owns, for one index, pinned staging for v, a device copy of v and of the result,
// and mapped pinned result memory, allocated once and reused every call.  A call is: copy v
// into the pinned staging while classifying it (host_stage.cpp: integer-valued vectors run on
// the exact int32 kernel when sum |v| fits int32, on the exact wide multiply otherwise), H2D(v),
// the multiply, and the conversion into the caller's buffer.  A single-split scatter multiply
// (int32 / fp32 activations, rows <= 16384)
// publishes its results into the mapped memory itself (csrc/common.cuh Publish: seq-tagged
// 64-bit words up to 8 K columns, 4-byte results + a fenced completion flag beyond), so no D2H
// copy and no stream synchronize sit between the kernel and the caller
// (tools/microbench/sync_probe.cu, session_timeline.cu measured the alternatives on the B200
// box).  Other forms are followed by a D2H copy and a stream synchronize.
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
                         rsr_variant var, int b0, int b1, void* ws, size_t ws_bytes, cudaStream_t s);
namespace {
size_t dsize(rsr_dtype t) { return (t == RSR_F64 || t == RSR_I64) ? 8 : 4; }
}  // namespace
}  // namespace rsr

struct rsr_host_session {
  rsr_index_desc desc;
  void* h_v = nullptr;      // pinned staging [rows], 8 bytes per row
  bool tagged = false;                      // publish mode (see rsr::Publish)
  unsigned long long* h_tag = nullptr;      // pinned, mapped [cols] tagged results (seq << 32 | value)
  unsigned long long* h_tag_dev = nullptr;
  void* h_res = nullptr;                    // pinned, mapped [cols] 4-byte results (flagged)
  void* h_res_dev = nullptr;
  uint32_t* h_flag = nullptr;               // pinned, mapped (flagged)
  uint32_t* h_flag_dev = nullptr;
  uint32_t* d_counter = nullptr;
  void* h_copy = nullptr;   // pinned [cols], 8 bytes per column (D2H path)
  void* d_v = nullptr;      // [rows], 8 bytes per row
  void* d_out = nullptr;    // [cols], 8 bytes per column
  void* d_wide = nullptr;   // wide-multiply workspace (whole int64 range), allocated on first use
  size_t wide_bytes = 0;
  uint32_t seq = 0;
  // Publishing calls (int32 / fp32 scatter) replay a captured graph: H2D of v plus the call's
  // seq word (staged right after v) -> the publishing multiply, one cudaGraphLaunch instead of a
  // memcpy and a kernel launch (~4 us of host time); [kind: int32, fp32][variant]
  cudaGraphExec_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int direct_calls[2][2] = {{0, 0}, {0, 0}};
  cudaStream_t cap = nullptr;
  size_t seq_off = 0;       // byte offset of the seq word in h_v / d_v
};

using rsr::cuda_check;
using rsr::fail;

namespace {
void session_free(rsr_host_session* h) {
  if (!h) return;
  if (h->h_v) cudaFreeHost(h->h_v);
  if (h->h_tag) cudaFreeHost(h->h_tag);
  if (h->h_res) cudaFreeHost(h->h_res);
  if (h->h_flag) cudaFreeHost(h->h_flag);
  if (h->d_counter) cudaFree(h->d_counter);
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

// Published int32 / fp32 results -> out_host (float64, or the 4-byte vector type).
rsr_status read_published(rsr_host_session* h, uint32_t seq, rsr_dtype vt, void* out_host, rsr_dtype out_dtype,
                          cudaStream_t s) {
  const rsr_index_desc& d = h->desc;
  rsr_status st = RSR_OK;
  if (!h->tagged) {
    // flagged: poll the flag; every few thousand polls ask the stream whether it failed
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
    if (out_dtype == vt) std::memcpy(out_host, h->h_res, 4 * (size_t)d.cols);
    else if (vt == RSR_I32) convert((const int32_t*)h->h_res, (double*)out_host, d.cols);
    else convert((const float*)h->h_res, (double*)out_host, d.cols);
    return RSR_OK;
  }
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
  rsr_status st = cuda_check(cudaHostAlloc(&h->h_v, vb, cudaHostAllocDefault), "session pinned v");
  if (st == RSR_OK) st = cuda_check(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking), "session capture stream");
  // tagged words up to 8 K columns, the fenced flag beyond (the host reads 8 vs 4 bytes per
  // result against a ~4 us fence + arrival; session_timeline.cu / e2e probes)
  h->tagged = desc->cols <= 8192;
  if (h->tagged) {
    if (st == RSR_OK)
      st = cuda_check(cudaHostAlloc((void**)&h->h_tag, 8 * (size_t)desc->cols, cudaHostAllocMapped), "session mapped result");
    if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer((void**)&h->h_tag_dev, h->h_tag, 0), "session result mapping");
    if (st == RSR_OK) std::memset(h->h_tag, 0, 8 * (size_t)desc->cols);  // tag 0: no call's result
  } else {
    if (st == RSR_OK) st = cuda_check(cudaHostAlloc(&h->h_res, 4 * (size_t)desc->cols, cudaHostAllocMapped), "session mapped result");
    if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer(&h->h_res_dev, h->h_res, 0), "session result mapping");
    if (st == RSR_OK) st = cuda_check(cudaHostAlloc((void**)&h->h_flag, 64, cudaHostAllocMapped), "session flag");
    if (st == RSR_OK) st = cuda_check(cudaHostGetDevicePointer((void**)&h->h_flag_dev, h->h_flag, 0), "session flag mapping");
    if (st == RSR_OK) st = cuda_check(cudaMalloc((void**)&h->d_counter, 64), "session counter");
    if (st == RSR_OK) st = cuda_check(cudaMemset(h->d_counter, 0, 64), "session counter init");
    if (st == RSR_OK) *h->h_flag = 0;
  }
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
  const rsr_dtype kt = cls.kind == rsr::kStageI32 ? RSR_I32 : cls.kind == rsr::kStageWide ? RSR_I64
                       : cls.kind == rsr::kStageF32 ? RSR_F32 : RSR_F64;  // computed (and staged) type
  const size_t vb = rsr::dsize(kt) * (size_t)d.rows;
  const bool graph_kind = kt == RSR_I32 || kt == RSR_F32;  // publishing kinds: the H2D is part of the graph
  rsr_status st = RSR_OK;
  if (!graph_kind || !h->graph[kt == RSR_I32 ? 0 : 1][variant == RSR_VARIANT_RSRPP ? 1 : 0])
    st = cuda_check(cudaMemcpyAsync(h->d_v, h->h_v, graph_kind ? h->seq_off + 16 : vb, cudaMemcpyHostToDevice, s),
                    "H2D v");
  if (st != RSR_OK) return st;
  bool published = false;
  rsr_dtype rt = kt;  // device result type
  if (kt == RSR_I64) {
    rt = out_dtype == RSR_I64 ? RSR_I64 : RSR_F64;
    const size_t need = rsr::wide_workspace_bytes(d, 0);
    if (h->wide_bytes < need) {
      if (h->d_wide) cudaFree(h->d_wide);
      h->d_wide = nullptr;
      h->wide_bytes = 0;
      if ((st = cuda_check(cudaMalloc(&h->d_wide, need), "session wide workspace")) != RSR_OK) return st;
      h->wide_bytes = need;
    }
    st = rsr::multiply_wide(d, (const int64_t*)h->d_v, cls.max_abs, h->d_out, rt, variant, 0, d.nblocks, h->d_wide,
                            h->wide_bytes, s);
  } else {
    const uint32_t seq = ++h->seq == 0 ? ++h->seq : h->seq;  // never 0 (the buffer's initial tag)
    const int gk = kt == RSR_I32 ? 0 : 1, gv = variant == RSR_VARIANT_RSRPP ? 1 : 0;
    const uint32_t* seq_dev = reinterpret_cast<const uint32_t*>((char*)h->d_v + h->seq_off);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    // graphs for the 4-byte kinds only (the seq word sits right after a 4-byte-element v)
    const bool can_graph = graph_kind && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
    if (graph_kind) *reinterpret_cast<uint32_t*>((char*)h->h_v + h->seq_off) = seq;
    if (h->graph[gk][gv] == nullptr && can_graph && h->direct_calls[gk][gv] >= 1) {
      // capture once (after one direct call, which set the kernels' attributes): H2D(v + seq), multiply
      const rsr::Publish gpub = h->tagged ? rsr::Publish{h->h_tag_dev, nullptr, nullptr, nullptr, 0, seq_dev}
                                          : rsr::Publish{nullptr, h->h_res_dev, h->d_counter, h->h_flag_dev, 0, seq_dev};
      cudaGraph_t g = nullptr;
      bool gpublished = false;
      rsr_status cst = cuda_check(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal), "session capture");
      if (cst == RSR_OK) {
        rsr_status a = cuda_check(cudaMemcpyAsync(h->d_v, h->h_v, h->seq_off + 16, cudaMemcpyHostToDevice, h->cap), "H2D v");
        if (a == RSR_OK)
          a = rsr::multiply(d, h->d_v, kt, h->d_out, kt, variant, RSR_FORM_AUTO, 0, d.nblocks, h->cap, &gpub, &gpublished);
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
      if (graph_kind) ++h->direct_calls[gk][gv];
      const rsr::Publish pub = h->tagged ? rsr::Publish{h->h_tag_dev, nullptr, nullptr, nullptr, seq, nullptr}
                                         : rsr::Publish{nullptr, h->h_res_dev, h->d_counter, h->h_flag_dev, seq, nullptr};
      st = rsr::multiply(d, h->d_v, kt, h->d_out, kt, variant, RSR_FORM_AUTO, 0, d.nblocks, s, &pub, &published);
    }
    if (st == RSR_OK && published) {
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
