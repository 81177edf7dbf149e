// Shared device helpers for the sm_100a RSR kernels: TMA bulk copies,
// mbarriers, warp scans and the C-ABI error plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/rsr_b200.h"

namespace rsr {

constexpr int kMaxDeviceK = 16;  // u16 buckets
constexpr int kSmSlots = 148;    // B200 SM count (runtime value is queried; this is the default)

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string& msg);
rsr_status fail(rsr_status st, const std::string& msg);
rsr_status cuda_check(cudaError_t e, const char* what);
int device_sm_count();
size_t device_max_smem_optin();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size)
rsr_status set_max_smem(const void* kernel, size_t smem);

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Make mbarrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Key-order schedule of the scatter kernel (k <= 11, csrc/preprocess.cu schedule_keys_kernel).
// Inside an aligned 8-row group the codes are stored in slot order; slot s holds row p[s]
// where p = butterfly8(identity, ctrl).  The 12 control bits live in bits 13-15 of the
// group's codes 0..3 (codes are <= 8188 for k <= 11): bits 3c..3c+2 in code c.
constexpr uint32_t kSchedCodeMask = 0x1fff1fffu;  // clears the control bits of two codes

__device__ __forceinline__ uint32_t sched_ctrl(uint32_t w0, uint32_t w1) {
  return ((w0 >> 13) & 7u) | ((w0 >> 26) & 0x38u) | (((w1 >> 13) & 7u) << 6) | ((w1 >> 20) & 0xe00u);
}

// Butterfly network on 8 values: stage st (0..2) swaps a[e] and a[e | 1 << st] for the four
// e with bit st clear (switch i = their rank) when control bit 4*st + i is set.
template <typename T>
__device__ __forceinline__ void butterfly8(T (&a)[8], uint32_t ctrl) {
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    int i = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (!(e & (1 << st))) {
        const bool sw = (ctrl >> (4 * st + i)) & 1u;
        const T x = a[e], y = a[e | (1 << st)];
        a[e] = sw ? y : x;
        a[e | (1 << st)] = sw ? x : y;
        ++i;
      }
  }
}

// Bulk prefetch of [src, src + bytes) into L2 (bytes % 16 == 0, src 16-byte aligned).
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Prefetch the line holding p into L1 (no register result, so the scheduler has no reason to
// sink it the way it sinks register loads).
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Inclusive warp scan.
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Device encoding of a bucket key (see multiply.cu): bank bits XOR-ed with the next five
// bits.  An involution, so the same function encodes and decodes.
__host__ __device__ __forceinline__ uint32_t key_swizzle(uint32_t j) { return j ^ ((j >> 5) & 31u); }

// Device code of a bucket key stored in the index: the swizzled key, pre-multiplied by 4
// (the byte offset of its histogram word) when k <= 14 so the scatter loop needs one ALU
// op per key.  k = 15, 16 keep the plain swizzled key (u16 range).
// Device code of a key: the byte offset of its histogram word (swz(key) << 2) for k <= 11 and
// k = 14, the word index swz(key) for k = 12, 13, 15, 16.  Codes of k <= 13 stay below 2^13, so
// bits 13-15 are free for the key schedule's control bits.
__host__ __device__ __forceinline__ int code_shift(int k) { return (k <= 11 || k == 14) ? 2 : 0; }
__host__ __device__ __forceinline__ bool sched_keys(int k) { return k <= 13; }
__host__ __device__ __forceinline__ uint32_t encode_key(uint32_t key, int k) {
  return key_swizzle(key) << code_shift(k);
}
__host__ __device__ __forceinline__ uint32_t decode_key(uint32_t code, int k) {
  return key_swizzle(code >> code_shift(k));
}

// Programmatic dependent launch (PDL): wait until the preceding grid in the stream has
// completed and flushed its memory; let the next grid start launching its CTAs.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Shared-memory reduction (no return value): ATOMS.ADD on sm_100.
__device__ __forceinline__ void red_add_shared(uint32_t addr, int32_t v) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Predicated form: the predicate lives inside the asm, so the reduction stays one predicated
// instruction (a C++ `if` around an asm statement becomes a divergent branch per reduction).
__device__ __forceinline__ void red_add_shared_if(uint32_t addr, int32_t v, bool p) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.shared.add.s32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
      "r"((int)p)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__host__ __device__ __forceinline__ int block_width(int64_t cols, int k, int b) {
  int64_t rem = cols - (int64_t)b * k;
  return rem < k ? (int)rem : k;
}

// Host-buffer sessions (csrc/host.cu): a single-split scatter multiply can take its vector from
// MAPPED host memory and deliver its results into mapped host memory itself, so one call is one
// kernel launch (tools/microbench/launch_latency.cu: a graph of one kernel node reaches the GPU
// in ~4.8 us, one with an H2D copy node ahead of it in ~17 us).
//  * pull (pull != nullptr): the staged payload (v, 4-byte elements, then the call's seq word at
//    byte seq_off) is copied by the kernel into `v` (device): CTA c copies chunk c and adds 1 to a
//    64-bit arrival counter at `sync`; every CTA waits until the counter reaches the end of its
//    launch's generation (each launch adds exactly grid: one counter per launch shape, never
//    reset) and, after 20 us, copies the payload itself (copies are identical): no co-residency
//    is assumed (a grid barrier could deadlock against a concurrent kernel holding SMs).
//  * tagged results: as soon as a block is folded, each of its columns is written to host memory
//    as one 64-bit store (seq << 32 | value, single-copy atomic); the host accepts a word once its
//    tag is the call's seq, so it converts results while later blocks are still running.
struct Publish {
  unsigned long long* tagged;  // device pointer of the mapped tagged-result buffer [cols]
  const void* pull;            // device pointer of the mapped staging payload, or nullptr (v already on the device)
  uint32_t pull_bytes;         // payload bytes (multiple of 16): v, then the seq word
  uint32_t seq_off;            // byte offset of the seq word in the payload
  uint32_t* sync;              // device 64-bit arrival counter (pull only), zero-initialised once
  uint32_t seq;                // tag of this call when pull == nullptr
  uint32_t steal_ns;           // pull: a CTA that waited this long for the chunks copies the payload itself
};

// Fused all-gather epilogue (multi-GPU, csrc/multiply.cu): as soon as a block is folded, every
// one of its int32 column values is stored into EVERY rank's gathered output (peer pointers into
// NVLink-mapped symmetric memory: P2P stores overlap the remaining blocks' reductions); each CTA
// then releases its stores at system scope and counts itself done, and the launch's last CTA
// adds 1 to every rank's signal word.  A rank's gathered vector is complete when its signal has
// counted one arrival per rank for this call (rsr_allgather_wait).  Single-split launches only.
constexpr int kMaxPeers = 8;
struct Gather {
  int32_t* out[kMaxPeers];              // each rank's gathered vector (device pointers, peer-mapped)
  unsigned long long* sig[kMaxPeers];   // each rank's signal word
  unsigned long long* done;             // this rank's CTA-completion counter (local, zero-initialised)
  int npeers;                           // 0: no gather
  int64_t col_base;                     // this rank's first column in the gathered vector
};

// True when multiply() of a vector of type vt (result type vt) on this index is one single-split
// scatter launch that can pull and publish (int32, or fp32 within the fixed-point limits).
bool publishes(const rsr_index_desc& d, rsr_dtype vt);

// multiply.cu: one fused multiply over blocks [b0, b1).  With `pub`, a single-split scatter
// launch with int32 / fp32 results also publishes them (then *published = true); otherwise the
// caller copies the results back.
// `independent`: this launch reads nothing the previous launch in the stream writes and writes
// nothing it touches (e.g. vector i > 0 of a batch), so the scatter kernel skips its grid
// dependency wait and overlaps the previous launch's tail.
rsr_status multiply(const rsr_index_desc& d, const void* v, rsr_dtype vt, void* out, rsr_dtype ot, rsr_variant var,
                    rsr_form form, int b0, int b1, cudaStream_t s, const Publish* pub = nullptr,
                    bool* published = nullptr, bool independent = false);
// int32 scatter multiply with the fused all-gather epilogue (see Gather); RSR_ERR_UNSUPPORTED when
// the launch would need row splits.
rsr_status multiply_allgather(const rsr_index_desc& d, const int32_t* v, int32_t* out, rsr_variant var, const Gather& g,
                              cudaStream_t s);

// multiply.cu, batched int32 path: the packed-pair guard and the pair multiply.
// pack_guard: res[0] = max over blocks [0, b1) and logical bins j >= 1 of the bucket load (rows of key j
// over both halves), res[1] = max |V| over nv activations (res caller-zeroed, device).
rsr_status pack_guard(const rsr_index_desc& d, int b1, const int32_t* V, int64_t nv, uint32_t* res, cudaStream_t s);
// va and vb in one scatter launch (v + vb * 2^16 per reduction): exact iff the guard's
// load * max|v| <= 32767.  int32 in, int32 out, blocks [0, b1).
rsr_status multiply_pair(const rsr_index_desc& d, int b1, const int32_t* va, const int32_t* vb, int32_t* outa, int32_t* outb,
                         rsr_variant var, cudaStream_t s, bool independent);

}  // namespace rsr
