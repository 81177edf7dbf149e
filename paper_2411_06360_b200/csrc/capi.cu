// extern "C" entry points of librsr_b200.so (declared in include/rsr_b200.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace rsr {

// implemented in preprocess.cu / multiply.cu
size_t preprocess_workspace_bytes(const rsr_index_desc* d);
rsr_status preprocess_ternary(const int8_t* A, int64_t lda, const rsr_index_desc* d, int32_t* bad, void* ws,
                              size_t ws_bytes, cudaStream_t s);
rsr_status preprocess_binary(const uint8_t* bits, int64_t ldb, const rsr_index_desc* d, void* ws, size_t ws_bytes,
                             cudaStream_t s);
rsr_status segmented_sum(const rsr_index_desc& d, int half, int block, const void* v, rsr_dtype dt, void* u,
                         cudaStream_t s);
rsr_status naive_ternary(const int8_t* A, int64_t rows, int64_t cols, int64_t lda, const void* v, rsr_dtype dt,
                         void* out, cudaStream_t s);
rsr_status block_product(const double* u, int w, int use_fold, double* buf, double* out, cudaStream_t s);
size_t batched_workspace_bytes(const rsr_index_desc& d, int64_t batch, rsr_dtype dt);
size_t index_import_workspace_bytes(const rsr_index_desc* d);
size_t wide_workspace_bytes(const rsr_index_desc& d, uint64_t max_abs);
rsr_status batch_plan_layout(const rsr_index_desc& d, rsr_batch_plan* pl, size_t* code_bytes, size_t* map_bytes,
                             size_t* ws_bytes);
rsr_status batch_plan_build(const rsr_index_desc& d, rsr_batch_plan* pl, void* ws, size_t ws_bytes, cudaStream_t s);
size_t batched_plan_workspace_bytes(const rsr_batch_plan& pl, int64_t batch);
rsr_status multiply_batched_plan(const rsr_index_desc& d, const rsr_batch_plan& pl, const int32_t* V, int64_t batch,
                                 int32_t* out, rsr_variant var, void* ws, size_t ws_bytes, cudaStream_t s);
rsr_status multiply_wide(const rsr_index_desc& d, const int64_t* v, uint64_t max_abs, void* out, rsr_dtype ot,
                         rsr_variant var, int b0, int b1, void* ws, size_t ws_bytes, cudaStream_t s, int exp2 = 0);
size_t dense_plane_words(int64_t rows, int64_t cols);
size_t dense_i8_words(int64_t rows, int64_t cols);
rsr_status dense_pack_i8(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* Q, int32_t* bad,
                         cudaStream_t s);
rsr_status dense_multiply_i8(const uint32_t* Q, int64_t rows, int64_t cols, const int8_t* v, int32_t* out,
                             cudaStream_t s);
rsr_status dense_pack_ternary(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* P, uint32_t* N,
                              int32_t* bad, cudaStream_t s);
rsr_status dense_multiply(const uint32_t* P, const uint32_t* N, int64_t rows, int64_t cols, const void* v,
                          rsr_dtype dt, void* out, cudaStream_t s);
rsr_status index_import(const rsr_index_desc* d, const uint32_t* perm0, const uint32_t* seg0, const uint32_t* perm1,
                        const uint32_t* seg1, int64_t seg_in_stride, void* ws, size_t ws_bytes, int32_t* err,
                        cudaStream_t s);

rsr_status multiply_batched(const rsr_index_desc& d, const void* V, rsr_dtype vt, int64_t batch, void* out,
                            rsr_dtype ot, rsr_variant var, void* ws, size_t ws_bytes, cudaStream_t s, int b0 = 0,
                            int b1 = -1);
rsr_status multiply_batched_tail(const rsr_index_desc& d, int b, const int32_t* V, int64_t batch, int32_t* out, void* ws,
                                 cudaStream_t s);

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

rsr_status fail(rsr_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

rsr_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RSR_OK;
  return fail(RSR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Per-device attribute cache (queried once; safe to call while a stream is capturing).
namespace {
constexpr int kMaxDevices = 64;
int g_sm_count[kMaxDevices];
int g_smem_optin[kMaxDevices];
int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}
}  // namespace

int device_sm_count() {
  const int dev = current_device();
  if (!g_sm_count[dev]) {
    int n = kSmSlots;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sm_count[dev] = n;
  }
  return g_sm_count[dev];
}

size_t device_max_smem_optin() {
  const int dev = current_device();
  if (!g_smem_optin[dev]) {
    int n = 227 * 1024;
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    g_smem_optin[dev] = n;
  }
  return (size_t)g_smem_optin[dev];
}

rsr_status set_max_smem(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, kernel}];
  if (have >= smem) return RSR_OK;
  rsr_status st = cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                             "max dynamic smem attribute");
  if (st == RSR_OK) have = smem;
  return st;
}

static rsr_status check_k(int64_t rows, int32_t k) {
  // indexer.py:19-23 `_check_k` (same messages)
  if (k < 1 || k > 30) return fail(RSR_ERR_INVALID, "k must be in [1, 30], got " + std::to_string(k));
  int64_t maxk = 1;
  for (int64_t r = rows; r > 1; r >>= 1) ++maxk;
  maxk = std::max<int64_t>(1, std::min<int64_t>(30, maxk - 1));
  if (k > maxk)
    return fail(RSR_ERR_INVALID,
                "k=" + std::to_string(k) + " exceeds max " + std::to_string(maxk) + " for " + std::to_string(rows) + " rows");
  if (k > kMaxDeviceK) return fail(RSR_ERR_UNSUPPORTED, "k=" + std::to_string(k) + " exceeds the device limit of 16");
  return RSR_OK;
}

static rsr_status check_range(const rsr_index_desc* d, int32_t b0, int32_t b1) {
  if (!d) return fail(RSR_ERR_INVALID, "null index descriptor");
  if (b0 < 0 || b1 > d->nblocks || b0 > b1) return fail(RSR_ERR_INVALID, "block range out of bounds");
  if (d->halves != 1 && d->halves != 2) return fail(RSR_ERR_INVALID, "halves must be 1 or 2");
  return RSR_OK;
}

}  // namespace rsr

using namespace rsr;

namespace rsr {
namespace {
// Stream-ordered wait of a rank for its gathered vector (see common.cuh Gather): one thread polls
// the rank's signal word at system scope until every rank's launch of this call has arrived.  A
// peer that never arrives traps after 4 s instead of hanging the stream.
__global__ void allgather_wait_kernel(const unsigned long long* sig, unsigned long long target) {
  if (threadIdx.x != 0) return;
  unsigned long long t0, t1, c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(c) : "l"(sig) : "memory");
    if (c >= target) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 4000000000ull) __trap();
    __nanosleep(100);
  }
}
}  // namespace
}  // namespace rsr

extern "C" {

int rsr_b200_abi_version(void) { return RSR_B200_ABI_VERSION; }

const char* rsr_b200_last_error(void) { return g_last_error.c_str(); }

rsr_status rsr_index_layout(int64_t rows, int64_t cols, int32_t k, int32_t halves, rsr_index_desc* desc,
                            size_t* perm_bytes, size_t* seg_bytes, size_t* bucket_bytes) {
  if (rows < 1 || cols < 1) return fail(RSR_ERR_INVALID, "index dimensions must be at least 1x1");
  if (halves != 1 && halves != 2) return fail(RSR_ERR_INVALID, "halves must be 1 or 2");
  rsr_status st = check_k(rows, k);
  if (st != RSR_OK) return st;
  if (!desc) return fail(RSR_ERR_INVALID, "null index descriptor");
  std::memset(desc, 0, sizeof(*desc));
  desc->rows = rows;
  desc->cols = cols;
  desc->k = k;
  desc->nblocks = (int32_t)((cols + k - 1) / k);
  desc->perm_bytes = rows <= 65536 ? 2 : 4;
  desc->halves = halves;
  desc->row_stride = (rows + 7) / 8 * 8;
  desc->seg_stride = ((int64_t)1 << k) + 1;
  const size_t nb = (size_t)desc->nblocks;
  if (perm_bytes) *perm_bytes = nb * desc->row_stride * desc->perm_bytes;
  if (seg_bytes) *seg_bytes = nb * desc->seg_stride * sizeof(uint32_t);
  if (bucket_bytes) *bucket_bytes = nb * desc->row_stride * sizeof(uint16_t);
  return RSR_OK;
}

size_t rsr_preprocess_workspace_bytes(const rsr_index_desc* desc) {
  return desc ? preprocess_workspace_bytes(desc) : 0;
}

rsr_status rsr_preprocess_ternary(const int8_t* A, int64_t lda, const rsr_index_desc* desc, int32_t* d_bad_entries,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  return preprocess_ternary(A, lda, desc, d_bad_entries, workspace, workspace_bytes, (cudaStream_t)stream);
}

rsr_status rsr_preprocess_binary(const uint8_t* bits, int64_t ldb, const rsr_index_desc* desc, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  return preprocess_binary(bits, ldb, desc, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t rsr_index_import_workspace_bytes(const rsr_index_desc* desc) { return index_import_workspace_bytes(desc); }

rsr_status rsr_index_import(const rsr_index_desc* desc, const uint32_t* d_perm0, const uint32_t* d_seg0,
                            const uint32_t* d_perm1, const uint32_t* d_seg1, int64_t seg_stride, void* workspace,
                            size_t workspace_bytes, int32_t* d_error, void* stream) {
  return index_import(desc, d_perm0, d_seg0, d_perm1, d_seg1, seg_stride, workspace, workspace_bytes, d_error,
                      (cudaStream_t)stream);
}

rsr_status rsr_multiply_ex(const rsr_index_desc* desc, const void* v, rsr_dtype v_dtype, void* out,
                           rsr_dtype out_dtype, rsr_variant variant, rsr_form form, int32_t block_begin,
                           int32_t block_end, uint32_t flags, void* stream) {
  rsr_status st = check_range(desc, block_begin, block_end);
  if (st != RSR_OK) return st;
  if (!v || !out) return fail(RSR_ERR_INVALID, "null vector or output");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  if (v_dtype == RSR_I64) return fail(RSR_ERR_INVALID, "int64 activations go through rsr_multiply_wide");
  if (flags & ~RSR_MULTIPLY_INDEPENDENT) return fail(RSR_ERR_INVALID, "unknown multiply flags");
  return multiply(*desc, v, v_dtype, out, out_dtype, variant, form, block_begin, block_end, (cudaStream_t)stream,
                  nullptr, nullptr, (flags & RSR_MULTIPLY_INDEPENDENT) != 0);
}

rsr_status rsr_multiply(const rsr_index_desc* desc, const void* v, rsr_dtype v_dtype, void* out, rsr_dtype out_dtype,
                        rsr_variant variant, rsr_form form, int32_t block_begin, int32_t block_end, void* stream) {
  return rsr_multiply_ex(desc, v, v_dtype, out, out_dtype, variant, form, block_begin, block_end, 0u, stream);
}

size_t rsr_multiply_wide_workspace_bytes(const rsr_index_desc* desc, uint64_t max_abs) {
  return desc ? wide_workspace_bytes(*desc, max_abs) : 0;
}

rsr_status rsr_multiply_wide(const rsr_index_desc* desc, const int64_t* v, uint64_t max_abs, void* out,
                             rsr_dtype out_dtype, rsr_variant variant, int32_t block_begin, int32_t block_end,
                             void* workspace, size_t workspace_bytes, void* stream) {
  rsr_status st = check_range(desc, block_begin, block_end);
  if (st != RSR_OK) return st;
  if (!v || !out) return fail(RSR_ERR_INVALID, "null vector or output");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  return multiply_wide(*desc, v, max_abs, out, out_dtype, variant, block_begin, block_end, workspace, workspace_bytes,
                       (cudaStream_t)stream);
}

rsr_status rsr_multiply_fixed(const rsr_index_desc* desc, const int64_t* v_q, uint64_t max_abs, int32_t exp2,
                              double* out, rsr_variant variant, int32_t block_begin, int32_t block_end, void* workspace,
                              size_t workspace_bytes, void* stream) {
  rsr_status st = check_range(desc, block_begin, block_end);
  if (st != RSR_OK) return st;
  if (!v_q || !out) return fail(RSR_ERR_INVALID, "null vector or output");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  return multiply_wide(*desc, v_q, max_abs, out, RSR_F64, variant, block_begin, block_end, workspace, workspace_bytes,
                       (cudaStream_t)stream, exp2);
}

rsr_status rsr_multiply_allgather(const rsr_index_desc* desc, const int32_t* v, int32_t* out, rsr_variant variant,
                                  int32_t* const* peer_out, unsigned long long* const* peer_sig, int32_t npeers,
                                  int64_t col_base, unsigned long long* done, void* stream) {
  if (!desc || !v || !out || !peer_out || !peer_sig || !done) return fail(RSR_ERR_INVALID, "null argument");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  if (npeers < 1 || npeers > kMaxPeers) return fail(RSR_ERR_INVALID, "all-gather: 1 to 8 ranks");
  if (col_base < 0) return fail(RSR_ERR_INVALID, "negative column base");
  Gather g{};
  for (int r = 0; r < npeers; ++r) {
    if (!peer_out[r] || !peer_sig[r]) return fail(RSR_ERR_INVALID, "null peer pointer");
    g.out[r] = peer_out[r];
    g.sig[r] = peer_sig[r];
  }
  g.done = done;
  g.npeers = npeers;
  g.col_base = col_base;
  return multiply_allgather(*desc, v, out, variant, g, (cudaStream_t)stream);
}

rsr_status rsr_allgather_wait(const unsigned long long* sig, unsigned long long target, void* stream) {
  if (!sig) return fail(RSR_ERR_INVALID, "null signal");
  allgather_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(sig, target);
  return cuda_check(cudaGetLastError(), "allgather_wait_kernel launch");
}

rsr_status rsr_batch_plan_layout(const rsr_index_desc* desc, rsr_batch_plan* plan, size_t* code_bytes,
                                 size_t* map_bytes, size_t* workspace_bytes) {
  rsr_status st = check_range(desc, 0, desc ? desc->nblocks : 0);
  if (st != RSR_OK) return st;
  if (!plan) return fail(RSR_ERR_INVALID, "null plan");
  return batch_plan_layout(*desc, plan, code_bytes, map_bytes, workspace_bytes);
}

rsr_status rsr_batch_plan_build(const rsr_index_desc* desc, rsr_batch_plan* plan, void* workspace,
                                size_t workspace_bytes, void* stream) {
  rsr_status st = check_range(desc, 0, desc ? desc->nblocks : 0);
  if (st != RSR_OK) return st;
  if (!plan) return fail(RSR_ERR_INVALID, "null plan");
  return batch_plan_build(*desc, plan, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t rsr_multiply_batched_plan_workspace_bytes(const rsr_batch_plan* plan, int64_t batch) {
  return plan ? batched_plan_workspace_bytes(*plan, batch) : 0;
}

rsr_status rsr_multiply_batched_plan(const rsr_index_desc* desc, const rsr_batch_plan* plan, const int32_t* V,
                                     int64_t batch, int32_t* OUT, rsr_variant variant, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  rsr_status st = check_range(desc, 0, desc ? desc->nblocks : 0);
  if (st != RSR_OK) return st;
  if (!plan) return fail(RSR_ERR_INVALID, "null plan");
  if (batch < 0) return fail(RSR_ERR_INVALID, "batch must be non-negative");
  if (batch > 0 && (!V || !OUT)) return fail(RSR_ERR_INVALID, "null vector or output");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  return multiply_batched_plan(*desc, *plan, V, batch, OUT, variant, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t rsr_multiply_batched_workspace_bytes(const rsr_index_desc* desc, int64_t batch, rsr_dtype v_dtype) {
  return desc ? batched_workspace_bytes(*desc, batch, v_dtype) : 0;
}

rsr_status rsr_multiply_batched(const rsr_index_desc* desc, const void* V, rsr_dtype v_dtype, int64_t batch, void* OUT,
                                rsr_dtype out_dtype, rsr_variant variant, void* workspace, size_t workspace_bytes,
                                void* stream) {
  rsr_status st = check_range(desc, 0, desc ? desc->nblocks : 0);
  if (st != RSR_OK) return st;
  if (batch < 0) return fail(RSR_ERR_INVALID, "batch must be non-negative");
  if (batch > 0 && (!V || !OUT)) return fail(RSR_ERR_INVALID, "null vector or output");
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  // int32 / fp32: the batched gather kernel reads the index once per slice of vectors; the
  // per-vector scatter kernel re-reads it per vector but runs ~1.3x faster per vector while
  // the index is L2-resident.  RSR_B200_BATCH_FORM=loop|gather overrides (diagnostics).
  bool loop = v_dtype == RSR_F64;
  if (!loop) {
    const size_t index_bytes = (size_t)desc->halves * desc->nblocks * desc->row_stride * 2;
    // (only where the per-vector AUTO path is the scatter kernel: int32, or fp32 within the
    // fixed-point limits)
    const bool scatter = desc->k <= 14 && (v_dtype == RSR_I32 || desc->rows <= 16384);
    loop = index_bytes <= ((size_t)96 << 20) && scatter && out_dtype == v_dtype;
    static const char* env_form = getenv("RSR_B200_BATCH_FORM");  // diagnostics, read once
    if (env_form) loop = env_form[0] == 'l';
  }
  if (loop) {  // one multiply per vector
    const size_t vsz = v_dtype == RSR_F64 ? 8 : 4, osz = out_dtype == RSR_F64 ? 8 : 4;
    int64_t i = 0;
    // int32 pairs: one scatter launch per two vectors (v + v' * 2^16 in every reduction) when the
    // guard proves every bucket sum fits in int16; the guard costs one host sync, so not while
    // the stream is being captured.  RSR_B200_PACK=0 disables it (diagnostics).
    static const bool env_nopack = getenv("RSR_B200_PACK") && getenv("RSR_B200_PACK")[0] == '0';
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    // Pairs cover the full-width blocks; a short last block (few key bits, so heavy buckets) goes
    // to the batched gather kernel for all vectors at once.
    const int nfull = desc->cols % desc->k == 0 ? desc->nblocks : desc->nblocks - 1;
    if (v_dtype == RSR_I32 && out_dtype == RSR_I32 && batch >= 2 && nfull > 0 && !env_nopack && workspace &&
        workspace_bytes >= batched_workspace_bytes(*desc, batch, v_dtype) &&
        (uint64_t)desc->rows * (uint64_t)((batch + 127) / 128 * 128) < (1ull << 32) &&
        cudaStreamIsCapturing((cudaStream_t)stream, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
      uint32_t* res = reinterpret_cast<uint32_t*>(workspace);
      uint32_t h[2] = {0, 0};
      st = cuda_check(cudaMemsetAsync(res, 0, 8, (cudaStream_t)stream), "memset guard");
      if (st == RSR_OK) st = rsr::pack_guard(*desc, nfull, (const int32_t*)V, batch * desc->rows, res, (cudaStream_t)stream);
      if (st == RSR_OK) st = cuda_check(cudaMemcpyAsync(h, res, 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream), "guard copy");
      if (st == RSR_OK) st = cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "guard sync");
      if (st != RSR_OK) return st;
      if ((uint64_t)h[0] * h[1] <= 32767u) {
        for (; i + 2 <= batch; i += 2) {
          const int32_t* va = (const int32_t*)V + i * desc->rows;
          int32_t* oa = (int32_t*)OUT + i * desc->cols;
          st = rsr::multiply_pair(*desc, nfull, va, va + desc->rows, oa, oa + desc->cols, variant, (cudaStream_t)stream,
                                  i > 0);
          if (st != RSR_OK) return st;
        }
        if (nfull < desc->nblocks) {  // every vector's short last block (unpaired one included)
          st = multiply_batched_tail(*desc, nfull, (const int32_t*)V, batch, (int32_t*)OUT, workspace,
                                     (cudaStream_t)stream);
          if (st != RSR_OK) return st;
        }
        for (; i < batch; ++i) {  // the unpaired vector: its full-width blocks
          st = multiply(*desc, (const char*)V + i * desc->rows * vsz, v_dtype, (char*)OUT + i * desc->cols * osz,
                        out_dtype, variant, RSR_FORM_AUTO, 0, nfull, (cudaStream_t)stream, nullptr, nullptr, false);
          if (st != RSR_OK) return st;
        }
        return RSR_OK;
      }
    }
    for (; i < batch; ++i) {
      // vector i > 0 depends only on what vector 0's launch already waited for: its launch
      // overlaps the previous vector's tail (distinct V row and OUT row)
      st = multiply(*desc, (const char*)V + i * desc->rows * vsz, v_dtype, (char*)OUT + i * desc->cols * osz, out_dtype,
                    variant, RSR_FORM_AUTO, 0, desc->nblocks, (cudaStream_t)stream, nullptr, nullptr, i > 0);
      if (st != RSR_OK) return st;
    }
    return RSR_OK;
  }
  return multiply_batched(*desc, V, v_dtype, batch, OUT, out_dtype, variant, workspace, workspace_bytes,
                          (cudaStream_t)stream);
}

rsr_status rsr_multiply_host(const rsr_index_desc* desc, const void* v_host, rsr_dtype v_dtype, void* out_host,
                             rsr_dtype out_dtype, rsr_variant variant, void* d_v, void* d_out, void* stream) {
  rsr_status st = check_range(desc, 0, desc ? desc->nblocks : 0);
  if (st != RSR_OK) return st;
  if (!v_host || !out_host || !d_v || !d_out) return fail(RSR_ERR_INVALID, "null buffer");
  if (v_dtype == RSR_I64 || out_dtype == RSR_I64) return fail(RSR_ERR_INVALID, "rsr_multiply_host: int32, float32 or float64");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t vsz = v_dtype == RSR_F64 ? 8 : 4, osz = out_dtype == RSR_F64 ? 8 : 4;
  if ((st = cuda_check(cudaMemcpyAsync(d_v, v_host, desc->rows * vsz, cudaMemcpyHostToDevice, s), "H2D v")) != RSR_OK)
    return st;
  if ((st = multiply(*desc, d_v, v_dtype, d_out, out_dtype, variant, RSR_FORM_AUTO, 0, desc->nblocks, s)) != RSR_OK)
    return st;
  if ((st = cuda_check(cudaMemcpyAsync(out_host, d_out, desc->cols * osz, cudaMemcpyDeviceToHost, s), "D2H out")) !=
      RSR_OK)
    return st;
  return cuda_check(cudaStreamSynchronize(s), "stream sync");
}

rsr_status rsr_segmented_sum(const rsr_index_desc* desc, int32_t half, int32_t block, const void* v, rsr_dtype dtype,
                             void* u, void* stream) {
  rsr_status st = check_range(desc, 0, desc ? desc->nblocks : 0);
  if (st != RSR_OK) return st;
  if (half < 0 || half >= desc->halves || block < 0 || block >= desc->nblocks)
    return fail(RSR_ERR_INVALID, "half or block out of range");
  return segmented_sum(*desc, half, block, v, dtype, u, (cudaStream_t)stream);
}

size_t rsr_dense_plane_words(int64_t rows, int64_t cols) { return rows > 0 && cols > 0 ? dense_plane_words(rows, cols) : 0; }

rsr_status rsr_dense_pack_ternary(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* d_pos,
                                  uint32_t* d_neg, int32_t* d_bad_entries, void* stream) {
  return dense_pack_ternary(A, lda, rows, cols, d_pos, d_neg, d_bad_entries, (cudaStream_t)stream);
}

rsr_status rsr_dense_multiply(const uint32_t* d_pos, const uint32_t* d_neg, int64_t rows, int64_t cols, const void* v,
                              rsr_dtype dtype, void* out, void* stream) {
  return dense_multiply(d_pos, d_neg, rows, cols, v, dtype, out, (cudaStream_t)stream);
}

size_t rsr_dense_i8_words(int64_t rows, int64_t cols) { return rows > 0 && cols > 0 ? dense_i8_words(rows, cols) : 0; }

rsr_status rsr_dense_pack_ternary_i8(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* d_q,
                                     int32_t* d_bad_entries, void* stream) {
  return dense_pack_i8(A, lda, rows, cols, d_q, d_bad_entries, (cudaStream_t)stream);
}

rsr_status rsr_dense_multiply_i8(const uint32_t* d_q, int64_t rows, int64_t cols, const int8_t* v, int32_t* out,
                                 void* stream) {
  return dense_multiply_i8(d_q, rows, cols, v, out, (cudaStream_t)stream);
}

rsr_status rsr_naive_multiply_ternary(const int8_t* A, int64_t rows, int64_t cols, int64_t lda, const void* v,
                                      rsr_dtype dtype, void* out, void* stream) {
  if (!A || !v || !out || rows < 1 || cols < 1 || lda < cols) return fail(RSR_ERR_INVALID, "bad naive arguments");
  return naive_ternary(A, rows, cols, lda, v, dtype, out, (cudaStream_t)stream);
}

rsr_status rsr_block_product(const double* u, int32_t width, rsr_variant variant, double* buf, double* out,
                             void* stream) {
  if (!u || !buf || !out) return fail(RSR_ERR_INVALID, "null buffer");
  if (width < 1 || width > 30) return fail(RSR_ERR_INVALID, "sums length must be 2^" + std::to_string(width));
  if (variant != RSR_VARIANT_RSR && variant != RSR_VARIANT_RSRPP)
    return fail(RSR_ERR_INVALID, "variant must be rsr or rsrpp");
  return block_product(u, width, variant == RSR_VARIANT_RSRPP, buf, out, (cudaStream_t)stream);
}

}  // extern "C"
