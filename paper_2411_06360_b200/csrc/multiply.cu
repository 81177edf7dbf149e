// sm_100a multiply kernels for RSR / RSR++ (arxiv 2411.06360).
//
// Two formulations of the reference hot loop, both computing, per column block b of width w,
// the bucket sums u_b[j] and the block product r_b = u_b . Bin_w:
//
//  * SCATTER (int32, and fp32 as exact fixed point) — the reference's own fused driver
//    `_run_blocks` (kernels.py:127-177): u_b[key_b[r]] += v[r] over rows r.  One persistent
//    CTA per SM keeps its slice of v in REGISTERS for the whole launch, streams the per-block
//    key codes straight into registers (L2 bulk prefetch of the next block), and accumulates
//    a 2^k-bin histogram with shared-memory int32 reductions in a bank-conflict-minimising
//    key order chosen at preprocess time (butterfly schedule).  Ternary matrices add +v at
//    the positive key's bin and -v at the negative key's bin of ONE histogram: the fold is
//    linear, so fold(u+ - u-) equals the reference's `pos - neg` (kernels.py:206) exactly.
//    Dedicated fold warps reduce finished histograms (RSR++ pairwise compaction,
//    kernels.py:74-91, or the dense RSR product, kernels.py:63-71) while the scatter warps
//    fill the next buffer.
//
//  * GATHER (fp64, and fp32 / int32 beyond the scatter limits) — the paper's Eq. 4 form
//    (`_segment_sums`, kernels.py:50-60): u[j] = sum over sorted positions p in
//    [seg[j], seg[j+1]) of v[perm[p]], v staged in shared memory, bucket boundaries folded
//    with the RSR++ telescoping coefficients (bit_s(j-1) - bit_s(j)) of window-local prefix
//    sums, or (variant "rsr") the segment sum added to every column whose bit is set.  No
//    floating-point atomics: results are deterministic run to run.
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace rsr {

namespace {

#ifndef RSR_R
#define RSR_R 32
#endif
constexpr int kScatterR = RSR_R;  // rows per scatter thread (multiple of 8)
// scatter threads of a full CTA: kScatterR rows each, >= 16384 rows per CTA
constexpr int kScatterThreads = (16384 / kScatterR + 31) / 32 * 32;
#ifndef RSR_FW
#define RSR_FW 4
#endif
constexpr int kFoldWarps = RSR_FW;  // dedicated fold warps per CTA (full CTAs); 8 measured 9% slower
                                    // (80 registers, fold warps compete for issue and smem)
constexpr int kMaxK = 16;
#ifndef RSR_KA
#define RSR_KA 1
#endif
#ifndef RSR_TRIGGER_EARLY
#define RSR_TRIGGER_EARLY 1
#endif
constexpr int KA = RSR_KA;  // scatter kernel: 8-row key groups in flight per lane (divides R / 8)

// =====================================================================================
// Histogram layout.  Logical bin j lives at word key_swizzle(j) = j ^ ((j >> 5) & 31):
// the low five bits (the shared-memory bank) are XOR-ed with the next five, which
// flattens the skewed key distribution of a uniform ternary half (P[bit] = 1/3) from
// 13% of atomics on bank 0 to ~5%.  The device bucket array stores keys already
// swizzled, so the scatter loop adds no ALU work.  The swizzle only permutes bins
// inside aligned 32-bin groups, and inside each int4 it is an XOR by (c & 3).
// =====================================================================================

// Recursive-halving warp reduce-scatter of 16 values: afterwards lanes 2i and 2i+1 hold
// the warp total of a[i] (16 shuffles instead of 16 x 5).
template <typename T>
__device__ __forceinline__ T reduce_scatter16(T (&a)[16], int lane) {
#pragma unroll
  for (int step = 0; step < 4; ++step) {
    const int half = 8 >> step;  // values kept after this step
    const int bit = (lane >> (4 - step)) & 1;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const T keep = bit ? a[i + half] : a[i];
      const T send = bit ? a[i] : a[i + half];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16 >> step);
    }
  }
  return a[0] + __shfl_xor_sync(0xffffffffu, a[0], 1);
}

// =====================================================================================
// SCATTER kernel (int32)
// =====================================================================================

#ifdef RSR_TRACE
// Diagnostic build only (`make trace`, tools/trace_scatter.py): per-unit globaltimer stamps.
__device__ unsigned long long g_trace[148 * 512];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot) do { if (lane == 0 && blockIdx.x < 148) g_trace[blockIdx.x * 512 + (slot)] = gtimer(); } while (0)
}  // namespace
}  // namespace rsr
extern "C" int rsr_debug_trace_copy(unsigned long long* host, size_t n) {
  return (int)cudaMemcpyFromSymbol(host, rsr::g_trace, n * sizeof(unsigned long long));
}
namespace rsr {
namespace {
#else
#define TRACE(slot) do { } while (0)
#endif

// Work-count build only (`make count`, -DRSR_COUNT, the reference's counted twins
// kernels.py:240-320): every thread counts the accumulate steps it actually executes —
// [0] histogram reductions (one per row, half and block: the reference's segmented-sum adds),
// [1] fold adds (pairwise compaction, chunk and slot accumulation, output atomics),
// [2] lane adds inside warp reductions (31 per REDUX) — and adds them to g_count at exit.
#ifdef RSR_COUNT
__device__ unsigned long long g_count[4];
#define CNT(var, n) ((var) += (unsigned long long)(n))
}  // namespace
}  // namespace rsr
extern "C" int rsr_debug_count_copy(unsigned long long* host, int reset) {
  int e = (int)cudaMemcpyFromSymbol(host, rsr::g_count, sizeof(rsr::g_count));
  if (!e && reset) {
    static const unsigned long long z[4] = {0, 0, 0, 0};
    e = (int)cudaMemcpyToSymbol(rsr::g_count, z, sizeof(z));
  }
  return e;
}
namespace rsr {
namespace {
#else
#define CNT(var, n) ((void)0)
#endif

struct ScatterParams {
  const uint16_t* key[2];
  const int32_t* v;
  void* out;
  const int32_t* v2;  // PACK: second vector (bits 16-31 of each packed activation)
  void* out2;         // PACK: its output
  int64_t rows, cols, row_stride;
  int k, halves, b_begin, b_end;
  int rows_per_cta, n_splits, stages, atomic_out, nhist;
  int v_aligned;
  int scatter_warps;
  int sched;          // keys stored in scheduled order (k <= 13): butterfly control bits in the codes
  int codes;          // code format: 0 byte offsets in row order, 1 scheduled byte offsets, 2 scheduled word indices
  uint32_t code_mask; // mask of the group's first two code words (clears the control bits)
  Publish pub;        // tagged != nullptr: also stream the results into mapped host memory
  Gather gat;         // npeers > 0: fused all-gather epilogue (see common.cuh Gather)
  int independent;    // v not written by any launch still in flight: only the fold warps wait (PDL)
};

// Logical-order view of one int4 of swizzled bins: element e of the result is logical bin
// 4q + e, given c = swizzle constant of the 32-bin group (key_swizzle XORs the low 5 bits).
__device__ __forceinline__ int4 unswizzle4(int4 q, uint32_t c) {
  if (c & 1u) q = make_int4(q.y, q.x, q.w, q.z);
  if (c & 2u) q = make_int4(q.z, q.w, q.x, q.y);
  return q;
}

// Persistent CTA (one per SM at n >= 8192): up to 16 SCATTER warps + kFoldWarps FOLD warps.
//  * Scatter warp w, lane l owns rows w*32R + 256g + 8l + e (g < R/8, e < 8) of the CTA's row
//    slice: their v values live in registers for the whole launch.  Each scatter warp streams
//    its rows' key codes of every column block straight into registers (16-byte
//    ld.global.nc.L1::no_allocate per 8 rows, software-pipelined one half-block ahead) while
//    lane 0 prefetches the next block (S = 0 further ones) with cp.async.bulk.prefetch.L2.
//    Keys never touch shared memory: the smem data path (128 B/clk) is the kernel's bound and
//    belongs to the reductions (tools/microbench/red_stream.cu: TMA->smem->LDS streaming
//    costs 1.5x the LDG path against concurrent REDs).
//  * Both halves of a ternary index scatter into ONE 2^k-bin histogram (+v for the positive
//    key, -v for the negative key): the fold is linear, so fold(u+ - u-) is exactly the
//    reference's `pos - neg` (kernels.py:206) in integer arithmetic.
//  * The fold warps never scatter, so folding overlaps the scatter warps' reductions instead
//    of stalling them: for every block they wait on hfull (all scatter warps done), each
//    reads its quarter of the histogram (RSR++ pairwise compaction of the lane-local bits,
//    kernels.py:74-91, or the dense RSR product, kernels.py:63-71), reduces the lane bits with
//    REDUX, and adds its share of the k outputs with global reductions; then arrives on hfree.
//  * Histogram buffers are never zeroed: block u adds into buffer u % NH on top of block
//    u - NH; each fold lane keeps its previous fold of the buffer and adds the difference
//    (exact modulo 2^32).
// Quantization exponent for the FX path: the CTA max |v| (float bits in fxmax[0..n)) maps to
// just below 2^30, so |v_q| < 2^30 and every limb sum over <= 16384 rows fits in int32.
__device__ __forceinline__ int fx_exponent(const uint32_t* fxmax, int n) {
  uint32_t m = 0;
  for (int i = 0; i < n; ++i) m = max(m, fxmax[i]);
  if (m == 0) return 0;
  // ilogb of the max (finite, positive float bits), denormals included
  const int lg = (m >> 23) ? (int)(m >> 23) - 127 : (31 - __clz((int)m)) - 149;
  return 29 - lg;  // max < 2^(lg+1) -> |v| * 2^e < 2^30
}

// x * 2^e, exact (power-of-two scaling of a value whose result is normal): one or two
// multiplies by power-of-two constants built from the exponent bits (ldexpf is a software
// routine with special-case branches, measured ~3 us of the FX prologue at 4096 rows)
__device__ __forceinline__ float scale_pow2(float x, int e) {
  if (e >= -126 && e <= 127) return x * __int_as_float((127 + e) << 23);
  const int h = e / 2;
  return (x * __int_as_float((127 + h) << 23)) * __int_as_float((127 + (e - h)) << 23);
}
__device__ __forceinline__ double pow2d(int e) {  // 2^e for |e| <= 1022
  return __longlong_as_double((long long)(1023 + e) << 52);
}

// Session pull (see Publish): CTA c copies chunk c of the mapped payload into dst and adds 1 to a
// 64-bit arrival counter; thread 0 of every CTA waits until the counter reaches the end of its
// launch's generation (every launch on the counter adds exactly nch, so it never needs resetting).  A CTA
// that has waited kStealNs (some chunk's CTA not yet resident, e.g. SMs held by a concurrent
// kernel) copies the whole payload itself: copies are identical, so no CTA ever depends on
// another being scheduled.  Called by every thread.
// The first 16 bytes of this thread's part of its CTA's chunk, loaded at kernel entry so that the
// sysmem latency (~2.2 us, tools/microbench/pcie_latency.cu) overlaps the prologue.
struct PullHead {
  uint4 q;
  bool has;
};
__device__ __forceinline__ uint32_t pull_chunk_bytes(const Publish& pb) {
  return ((pb.pull_bytes + gridDim.x - 1) / gridDim.x + 15u) & ~15u;
}
__device__ __forceinline__ PullHead pull_begin(const Publish& pb) {
  PullHead h{make_uint4(0, 0, 0, 0), false};
  const uint32_t csz = pull_chunk_bytes(pb);
  const uint32_t lo = min(pb.pull_bytes, blockIdx.x * csz), hi = min(pb.pull_bytes, lo + csz);
  const uint32_t o = lo + 16u * threadIdx.x;
  if (o < hi) {
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(h.q.x), "=r"(h.q.y), "=r"(h.q.z), "=r"(h.q.w)
                 : "l"(reinterpret_cast<const char*>(pb.pull) + o));
    h.has = true;
  }
  return h;
}

template <typename Trace>
__device__ __forceinline__ void pull_payload(const Publish& pb, const PullHead& head, void* dst, Trace&& trace) {
  const unsigned long long kStealNs = pb.steal_ns;
  const uint32_t nch = gridDim.x;
  const uint32_t csz = pull_chunk_bytes(pb);
  const int t = threadIdx.x;
  const char* src = reinterpret_cast<const char*>(pb.pull);
  // .nc loads of the mapped payload (tools/microbench/pull_probe.cu: .cv is 8x slower on sysmem;
  // no launch ever saw a stale line of the rewritten payload with .ca / .cg / .nc)
  auto copy = [&](uint32_t lo, uint32_t hi) {
    for (uint32_t o = lo + 16u * (uint32_t)t; o < hi; o += 16u * blockDim.x) {
      uint4 q;
      asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(src + o));
      *reinterpret_cast<uint4*>((char*)dst + o) = q;
    }
  };
  __shared__ uint32_t sh_steal;
  {
    const uint32_t lo = min(pb.pull_bytes, blockIdx.x * csz), hi = min(pb.pull_bytes, lo + csz);
    if (head.has) *reinterpret_cast<uint4*>((char*)dst + lo + 16u * t) = head.q;
    copy(min(hi, lo + 16u * blockDim.x), hi);  // chunks longer than one load per thread (small grids)
  }
  __threadfence();
  __syncthreads();
  trace(502);
  if (t == 0) {
    // this launch's generation from my own arrival (launches on one counter are stream-ordered and
    // each adds exactly nch): no sysmem read (same-address sysmem reads from many SMs serialise)
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(pb.sync);
    const unsigned long long old = atomicAdd(ctr, 1ull);
    const unsigned long long target = (old / nch + 1) * nch;
    trace(505);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint32_t steal = 0;
    for (;;) {
      unsigned long long c;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(ctr) : "memory");
      if (c >= target) break;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > kStealNs) { steal = 1; break; }
    }
    __threadfence();  // acquire: the other CTAs' chunks before my v loads
    sh_steal = steal;
  }
  __syncthreads();
  trace(503);
  if (sh_steal) {
    trace(504);
    copy(0, pb.pull_bytes);
    __threadfence();
    __syncthreads();
  }
}

// FX (fp32 activations): v is quantized once per launch to 31-bit fixed point with a per-CTA
// power-of-two scale (2^-31 of max|v|, far below fp32 rounding) and accumulated EXACTLY as two
// 16-bit limbs in two int32 histograms (integer atomics are native; fp32 shared atomics are a
// CAS loop on sm_100).  Deterministic, and more accurate than fp32 summation.  Single row
// split only (one scale per output column).
// FW fold warps: 4 for full CTAs; 1 for small CTAs (<= 4 scatter warps, k <= 13) so that 4 of
// them fit on an SM (the register budget stays that of the largest CTA: 96 per thread)
// CODES: 0 = byte-offset codes in row order (k = 14), 1 = scheduled byte-offset codes (k <= 11),
// 2 = scheduled word-index codes (k = 12, 13; see common.cuh encode_key)
// PACK (int32 vector pairs, batched path): v2 rides in bits 16-31 of every activation, so one
// reduction serves two vectors.  Exact when every bucket sum of either vector fits in int16
// (the host guard: max bucket load x max |v| <= 32767, bin 0 excluded — the fold never adds
// logical bin 0 into an output); the fold warps split each bin into its two int16 halves,
// fold both in one int32 pass (the packed words and their high halves), and zero the buffer after reading
// (a per-block value per bin, no running total).
template <int R, bool FOLDPP, bool TERNARY, typename OutT, bool FX, int CODES, int FW, bool PACK = false>
__global__ void __launch_bounds__(kScatterThreads + 32 * kFoldWarps, 1) scatter_kernel(const ScatterParams p) {
  static_assert(FW == 1 || FW == 2 || FW == 4 || FW == 8, "fold warps");
  static_assert(!(PACK && FX) && (!PACK || std::is_same<OutT, int32_t>::value), "PACK: int32 only");
  constexpr int FB = FW == 8 ? 3 : FW == 4 ? 2 : FW == 2 ? 1 : 0;  // key bits spanned by the fold warps
  static_assert(R % 8 == 0 && R * kScatterThreads <= 32768, "rows per CTA");
  constexpr int LIMBS = FX ? 2 : 1;              // histogram limbs
  constexpr int OLIMBS = (FX || PACK) ? 2 : 1;   // fold results per slot
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int HALVES = TERNARY ? 2 : 1;
  constexpr int NG = R / 8;      // 8-row groups per lane
  constexpr int WROWS = 32 * R;  // rows per warp
  constexpr int MAXNH = 4;
  const int nwarps = p.scatter_warps;  // scatter warps; fold warps follow them
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int nbk = 1 << p.k;
  const int S = p.stages;
  const int NH = p.nhist;
  const int hist_words = (NH * LIMBS * nbk + 15) & ~15;
  int32_t* hist = reinterpret_cast<int32_t*>(smem);  // [NH][LIMBS][nbk]
  uint64_t* hfull = reinterpret_cast<uint64_t*>(smem + ((sizeof(int32_t) * hist_words + 127) & ~(size_t)127));
  uint64_t* hfree = hfull + NH;
  uint32_t* fxmax = reinterpret_cast<uint32_t*>(hfree + NH);                   // [32] per-warp max |v| bits
  long long* fxpart = reinterpret_cast<long long*>(fxmax + 32);                // [2][FW][16]

  const int split = blockIdx.x % p.n_splits;
  const int col_cta = blockIdx.x / p.n_splits;
  const int ncol = gridDim.x / p.n_splits;
  const int64_t r0 = (int64_t)split * p.rows_per_cta;
  const int nblk = p.b_end - p.b_begin;
  const int nunits = col_cta < nblk ? (nblk - col_cta + ncol - 1) / ncol : 0;
  const uint16_t* key0 = p.key[0];
  const uint16_t* key1 = p.key[1];
  OutT* out = reinterpret_cast<OutT*>(p.out);
  OutT* out2 = reinterpret_cast<OutT*>(p.out2);
  const bool is_fold = warp >= nwarps;
  if (warp == 0) TRACE(0);
  const PullHead pull_head = p.pub.pull ? pull_begin(p.pub) : PullHead{make_uint4(0, 0, 0, 0), false};
  unsigned long long cnt_red = 0, cnt_fold = 0, cnt_redux = 0;  // work counts (RSR_COUNT builds only)
  (void)cnt_red; (void)cnt_fold; (void)cnt_redux;

  // ---- prologue (index only: may overlap the previous kernel under PDL) ----
  const int64_t wr0 = r0 + (int64_t)warp * WROWS;  // first row of this (scatter) warp
  const int wcopy = is_fold ? 0 : (int)std::max<int64_t>(0, std::min<int64_t>(WROWS, p.row_stride - wr0));
  const uint32_t wbytes = (uint32_t)wcopy * 2u;  // multiple of 16 (row_stride % 8 == 0)
  auto prefetch_unit = [&](int u) {              // lane 0: both halves of unit u into L2
    const int b = p.b_begin + col_cta + u * ncol;
    for (int h = 0; h < HALVES; ++h) prefetch_l2_bulk((h ? key1 : key0) + (int64_t)b * p.row_stride + wr0, wbytes);
  };
  // before the PDL wait: the first S + 1 units' keys into L2, one bulk prefetch per lane (a bulk
  // prefetch costs its issuing thread ~0.15 us, so lane 0 alone spent ~1.2 us here)
  if (!is_fold && wbytes) {
    const int u = lane / HALVES, h = lane % HALVES;
    if (u <= S && u < nunits) {
      const int b = p.b_begin + col_cta + u * ncol;
      prefetch_l2_bulk((h ? key1 : key0) + (int64_t)b * p.row_stride + wr0, wbytes);
    }
  }
  if (warp == 0) TRACE(2);
  if (t == 0) {  // (no fence: the mbarriers are only used by this CTA's threads, never by TMA)
    for (int h = 0; h < NH; ++h) {
      mbar_init(&hfull[h], nwarps);
      mbar_init(&hfree[h], FW);
    }
  }
  for (int i = t; i < hist_words / 4; i += blockDim.x) reinterpret_cast<int4*>(hist)[i] = make_int4(0, 0, 0, 0);
  if (warp == 0) TRACE(3);
  // v and out may belong to the previous kernel in the stream: wait for it here (PDL).
  // Independent launches (the caller guarantees no kernel still in flight writes v) skip this:
  // their scatter warps start at once on SMs the previous launch has freed, and only the fold
  // warps wait, before their first access to out (zeroing included) — so out is ordered after
  // the previous launch and every launch still completes after its predecessor.
  if (!p.independent) grid_dependency_wait();
  if (warp == 0) TRACE(4);
  if (p.pub.pull) pull_payload(p.pub, pull_head, const_cast<int32_t*>(p.v), [&](int slot) { if (warp == 0) TRACE(slot); });
  auto zero_out = [&](int t0, int nt) {
    if (p.atomic_out) return;  // (row splits: the host zeroes out) a single-split launch owns its columns
    for (int i = t0; i < nunits * p.k; i += nt) {
      const int b = p.b_begin + col_cta + (i / p.k) * ncol;
      const int c = i % p.k;
      if (c < block_width(p.cols, p.k, b)) {
        out[(int64_t)b * p.k + c] = (OutT)0;
        if constexpr (PACK) out2[(int64_t)b * p.k + c] = (OutT)0;
      }
    }
  };
  if (!p.independent) zero_out(t, blockDim.x);

  if (!is_fold) {
    // =========================== scatter warps ===========================
    const bool warp_all_valid = wr0 + WROWS <= p.rows;  // every row of this warp is a matrix row
    const uint32_t hist_s = smem_u32(hist);
    // this lane's keys of 8-row group g of unit u, half h: kb[h] + u * ustride + 256 g
    const int64_t ustride = (int64_t)ncol * p.row_stride;
    const int64_t koff = (int64_t)(p.b_begin + col_cta) * p.row_stride + wr0 + 8 * lane;
    const uint16_t* kb0 = key0 + koff;
    const uint16_t* kb1 = TERNARY ? key1 + koff : nullptr;
    uint32_t gmask = 0;  // groups present in the key arrays (all but in the last warp)
#pragma unroll
    for (int g = 0; g < NG; ++g) gmask |= (wr0 + 256 * g + 8 * lane < p.row_stride) ? (1u << g) : 0u;
    // warp-uniform group classes of the warp holding the end of the rows: all 256 rows valid,
    // some valid (the one group holding row `rows`), none
    uint32_t full_groups = 0, part_groups = 0;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const int64_t g0 = wr0 + 256 * g;
      if (g0 + 256 <= p.rows) full_groups |= 1u << g;
      else if (g0 < p.rows) part_groups |= 1u << g;
    }
    // key register ring: KA groups in flight; slot g % KA holds group g's keys, refilled right
    // after its reductions with the keys of the group KA places later in the (unit, group) order
    uint4 q0[KA], q1[KA];
#pragma unroll
    for (int g = 0; g < KA; ++g) {
      const bool ld = nunits > 0 && ((gmask >> g) & 1u);
      q0[g] = ld ? ld_nc_v4(kb0 + 256 * g) : make_uint4(0, 0, 0, 0);
      q1[g] = (TERNARY && ld) ? ld_nc_v4(kb1 + 256 * g) : make_uint4(0, 0, 0, 0);
    }
    int32_t vr[R];
    const bool pulled = p.pub.pull != nullptr;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const int64_t row = wr0 + 256 * g + 8 * lane;
      const int32_t* vp = p.v + row;
      if (row + 8 <= p.rows && p.v_aligned) {
        // .nc shares the lines between the CTAs of an SM (small CTAs); .cg when a session pull
        // wrote v during this launch (the non-coherent path may not see it)
        const int4 a = pulled ? __ldcg(reinterpret_cast<const int4*>(vp)) : __ldg(reinterpret_cast<const int4*>(vp));
        const int4 c = pulled ? __ldcg(reinterpret_cast<const int4*>(vp) + 1) : __ldg(reinterpret_cast<const int4*>(vp) + 1);
        vr[8 * g + 0] = a.x; vr[8 * g + 1] = a.y; vr[8 * g + 2] = a.z; vr[8 * g + 3] = a.w;
        vr[8 * g + 4] = c.x; vr[8 * g + 5] = c.y; vr[8 * g + 6] = c.z; vr[8 * g + 7] = c.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) vr[8 * g + e] = (row + e < p.rows) ? (pulled ? __ldcg(vp + e) : __ldg(vp + e)) : 0;  // rows past the end: 0
      }
    }
    if constexpr (PACK) {  // packed = v + v2 * 2^16 (mod 2^32)
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const int64_t row = wr0 + 256 * g + 8 * lane;
        const int32_t* vp = p.v2 + row;
        int32_t b[8];
        if (row + 8 <= p.rows && p.v_aligned) {
          const int4 a = __ldg(reinterpret_cast<const int4*>(vp));
          const int4 c = __ldg(reinterpret_cast<const int4*>(vp) + 1);
          b[0] = a.x; b[1] = a.y; b[2] = a.z; b[3] = a.w; b[4] = c.x; b[5] = c.y; b[6] = c.z; b[7] = c.w;
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) b[e] = (row + e < p.rows) ? vp[e] : 0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) vr[8 * g + e] = (int32_t)((uint32_t)vr[8 * g + e] + ((uint32_t)b[e] << 16));
      }
    }
    if (warp == 0) TRACE(5);
    if constexpr (FX) {  // CTA max |v| -> quantization scale
      uint32_t m = 0;
#pragma unroll
      for (int i = 0; i < R; ++i) m = max(m, (uint32_t)vr[i] & 0x7fffffffu);
      m = __reduce_max_sync(0xffffffffu, m);
      if (lane == 0) fxmax[warp] = m;
    }
    __syncthreads();
    if constexpr (FX) {
      const int e = fx_exponent(fxmax, nwarps);
#pragma unroll
      for (int i = 0; i < R; ++i) vr[i] = __float2int_rn(scale_pow2(__int_as_float(vr[i]), e));
    }
    if (warp == 0) TRACE(1);
    constexpr bool SCHED = CODES != 0;
    constexpr uint32_t kMask = SCHED ? kSchedCodeMask : 0xffffffffu;
    // the reductions of one half of one group: slot s adds +-vp[s] into the bin of code s.
    // SKIP0 (the warp holding the end of the rows): rows past the end carry v = 0 and their
    // (padding or absent) codes are skipped; a zero contribution is a no-op for any row.
    auto reduce_group = [&](uint32_t Hs, const uint4& a, const int32_t (&vp)[8], bool neg, auto skip0) {
      constexpr bool SKIP0 = decltype(skip0)::value;
      const uint32_t w4[4] = {a.x & kMask, a.y & kMask, a.z, a.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int32_t x0 = vp[2 * e], x1 = vp[2 * e + 1];
        // byte offsets of the two bins (word-index codes are scaled here)
        const uint32_t c0 = CODES == 2 ? (w4[e] & 0xffffu) << 2 : w4[e] & 0xffffu;
        const uint32_t c1 = CODES == 2 ? (w4[e] >> 16) << 2 : w4[e] >> 16;
        // SKIP0: predicated inside the asm (an `if` around it would branch per reduction)
        auto red = [&](uint32_t a, int32_t val, int32_t x) {
          CNT(cnt_red, SKIP0 ? (x != 0) : 1);
          if constexpr (SKIP0) red_add_shared_if(a, val, x != 0);
          else red_add_shared(a, val);
        };
        if constexpr (FX) {
          const uint32_t lo_off = (uint32_t)nbk * 4u;
          red(Hs + c0, neg ? -(x0 >> 16) : (x0 >> 16), x0);
          red(Hs + lo_off + c0, neg ? -(x0 & 0xffff) : (x0 & 0xffff), x0);
          red(Hs + c1, neg ? -(x1 >> 16) : (x1 >> 16), x1);
          red(Hs + lo_off + c1, neg ? -(x1 & 0xffff) : (x1 & 0xffff), x1);
        } else {
          red(Hs + c0, neg ? -x0 : x0, x0);
          red(Hs + c1, neg ? -x1 : x1, x1);
        }
      }
    };
    // one unit's groups: the reductions of group g, then the keys of the group KA later (this
    // unit's group g + KA, or the next unit's group g + KA - NG) into the registers just consumed
    auto unit_groups = [&](uint32_t Hs, bool more, auto skip0) {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        uint4& q0g = q0[g % KA];
        [[maybe_unused]] uint4& q1g = q1[g % KA];
        // slot s of the group holds row p[s], p = butterfly of the control bits (k <= 11):
        // route the v registers the same way, once for both halves
        int32_t vp[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) vp[e] = vr[g * 8 + e];
        if constexpr (SCHED) butterfly8(vp, sched_ctrl(q0g.x, q0g.y));
        if (!decltype(skip0)::value || ((full_groups >> g) & 1u)) {  // every lane's 8 rows exist
          reduce_group(Hs, q0g, vp, false, std::false_type{});
          if constexpr (TERNARY) reduce_group(Hs, q1g, vp, true, std::false_type{});
        } else if ((part_groups >> g) & 1u) {  // the group holding the last row: predicated
          reduce_group(Hs, q0g, vp, false, std::true_type{});
          if constexpr (TERNARY) reduce_group(Hs, q1g, vp, true, std::true_type{});
        }  // else: every row of the group is past the end (warp-uniform skip)
        // branch-free (a shared guard lets the compiler merge the four loads and sink them to
        // the end of the unit, which leaves them no time): without a next unit, or for a group
        // past the key rows (its rows carry v = 0 and are skipped), load the array base instead
        const int gn = (g + KA) % NG;             // group to load (unrolled: constant)
        const bool next_unit = g + KA >= NG;      // ... of the next unit (kb0 points there)
        const bool ld = (!next_unit || more) && ((gmask >> gn) & 1u);
        const int64_t back = next_unit ? 0 : ustride;  // this unit = kb0 - ustride
        q0g = ld_nc_v4(ld ? kb0 - back + 256 * gn : key0);
        if constexpr (TERNARY) q1g = ld_nc_v4(ld ? kb1 - back + 256 * gn : key1);
      }
    };
    int hb = 0;            // histogram buffer of unit u (u % NH, kept incrementally)
    uint32_t hpar = 1;     // parity of hfree[hb]'s phase to wait for: ((u / NH) - 1) & 1
    for (int u = 0; u < nunits; ++u) {
      // PDL trigger: the next grid is launched (its CTAs wait for free SMs and take each one the
      // moment this grid's CTA on it exits).  Every CTA of this grid is resident by now (grids
      // never exceed one wave), so triggering early cannot starve it; triggering only at the
      // last unit left the next launch's latency exposed.
      if (u == (RSR_TRIGGER_EARLY ? 0 : nunits - 1)) grid_launch_dependents();
      if (lane == 0 && wbytes && u + 1 + S < nunits) prefetch_unit(u + 1 + S);
      const uint32_t Hs = hist_s + (uint32_t)(hb * LIMBS * nbk) * 4u;
      if (warp == 0 && u < 40) TRACE(8 + u * 8 + 0);
      if (u >= NH) mbar_wait(&hfree[hb], hpar);
      if (warp == 0 && u < 40) TRACE(8 + u * 8 + 1);
      const bool more = u + 1 < nunits;
      kb0 += ustride;
      if constexpr (TERNARY) kb1 += ustride;
      if (warp_all_valid) unit_groups(Hs, more, std::false_type{});
      else unit_groups(Hs, more, std::true_type{});
      __syncwarp();
      if (warp == 0 && u < 40) TRACE(8 + u * 8 + 2);
      if (lane == 0) {
        mbar_arrive(&hfull[hb]);  // release: this warp's reductions are visible to the fold warps
        if (warp == 0 && u < 40) TRACE(8 + u * 8 + 7);
      }
      if (++hb == NH) {
        hb = 0;
        hpar ^= 1u;
      }
    }
  } else {
    // ============================= fold warps =============================
    __syncthreads();
    const int fw = warp - nwarps;  // fold warp index (FB warp bits)
    if (p.independent) {  // out belongs to the stream order: wait, zero, then fold
      grid_dependency_wait();
      zero_out(t - nwarps * 32, 32 * FW);
      asm volatile("bar.sync 1, %0;" ::"r"(32 * FW) : "memory");
    }
    // logical bin j = (fw*32 + lane) * 2^lb + e; lane bits start at lb, fold-warp bits at lb + 5
    int lb = p.k - 5 - FB;  // <= 8
    if (lb < 0) lb = 0;
    const int fbase = (fw * 32 + lane) << lb;
    const bool active = fbase < nbk;
    int32_t prev[OLIMBS][MAXNH];
#pragma unroll
    for (int l = 0; l < OLIMBS; ++l)
#pragma unroll
      for (int i = 0; i < MAXNH; ++i) prev[l][i] = 0;
    int fx_e = 0;
    if constexpr (FX) fx_e = fx_exponent(fxmax, nwarps);
    // tag of the streamed results: the pulled payload's seq word (or the launch's own)
    const uint32_t pub_seq = p.pub.pull ? __ldcg(reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(p.v) + p.pub.seq_off))
                                        : p.pub.seq;
    // slot of lane i: 0-7 local bits (< lb), 8-12 lane bits, 13-14 fold-warp bits
    int sh = -1;
    if (lane < 8) sh = lane < lb ? lane : -1;
    else if (lane < 13) sh = lb + (lane - 8);
    else if (lane < 13 + FB) sh = lb + 5 + (lane - 13);
    // per-lane partials of my bins of one limb histogram, then REDUX over the warp: lane i -> slot i
    auto fold_limb = [&](const int32_t* H) -> int32_t {
      int32_t a[8];  // local-bit partials, lb <= 7
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = 0;
      int32_t X = 0;
      if (active) {
        const int4* H4 = reinterpret_cast<const int4*>(H);
        if (lb >= 2) {
          const int n4 = 1 << (lb - 2);
          for (int c4 = 0; c4 < n4; c4 += 4) {  // 4 int4 (16 bins) at a time
            int4 z[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j4 = (fbase >> 2) + c4 + i;  // logical int4 index
              const uint32_t c = ((uint32_t)j4 >> 3) & 31u;
              z[i] = (c4 + i < n4) ? unswizzle4(H4[j4 ^ (int)(c >> 2)], c) : make_int4(0, 0, 0, 0);
            }
            int32_t x[16] = {z[0].x, z[0].y, z[0].z, z[0].w, z[1].x, z[1].y, z[1].z, z[1].w,
                             z[2].x, z[2].y, z[2].z, z[2].w, z[3].x, z[3].y, z[3].z, z[3].w};
            int32_t tot = 0;
            if (FOLDPP) {  // pairwise compaction over the 4 bits inside the 16-bin chunk
#pragma unroll
              for (int L = 0; L < 4; ++L) {
                const int cnt = 8 >> L;
                int32_t odd = 0;
#pragma unroll
                for (int tt = 0; tt < 8; ++tt)
                  if (tt < cnt) {
                    odd += x[2 * tt + 1];
                    x[tt] = x[2 * tt] + x[2 * tt + 1];
                    CNT(cnt_fold, 2);
                  }
                a[L] += odd;
                CNT(cnt_fold, 1);
              }
              tot = x[0];
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
#pragma unroll
                for (int L = 0; L < 4; ++L) a[L] += ((e >> L) & 1) ? x[e] : 0;
                tot += x[e];
                CNT(cnt_fold, 1 + __popc(e & 15));
              }
            }
            // chunk bits 4.. (chunk index c4/4) are local bits too
            const int ci = c4 >> 2;
#pragma unroll
            for (int L = 4; L < 8; ++L) a[L] += ((ci >> (L - 4)) & 1) ? tot : 0;
            X += tot;
            CNT(cnt_fold, 1 + __popc(ci & 15));
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < (1 << lb)) {
              const int32_t x = H[key_swizzle((uint32_t)(fbase + e))];
              if (lb >= 1 && (e & 1)) a[0] += x;
              X += x;
              CNT(cnt_fold, 1 + (lb >= 1 && (e & 1)));
            }
        }
      }
      int32_t r = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < lb) {
          const int32_t tv = __reduce_add_sync(0xffffffffu, a[i]);
          if (lane == i) r = tv;
          CNT(cnt_redux, lane == 0 ? 31 : 0);
        }
#pragma unroll
      for (int bit = 0; bit < 5; ++bit) {
        const int32_t tv = __reduce_add_sync(0xffffffffu, ((lane >> bit) & 1) ? X : 0);
        if (lane == 8 + bit) r = tv;
        CNT(cnt_redux, lane == 0 ? 31 : 0);
      }
      const int32_t W = __reduce_add_sync(0xffffffffu, X);
      CNT(cnt_redux, lane == 0 && FB > 0 ? 31 : 0);
#pragma unroll
      for (int fb2 = 0; fb2 < FB; ++fb2)
        if (lane == 13 + fb2) r = ((fw >> fb2) & 1) ? W : 0;
      return r;
    };
    // PACK, one pass, int32 only: fold the packed words x themselves (wrapping: the sums are
    // lo + 2^16 hi modulo 2^32) and the high halves hi = (x - (int16)x) >> 16 (exact: every
    // partial sum is below 2^31 in magnitude); then lo = fold(x) - 2^16 fold(hi) modulo 2^32,
    // exact for the same reason.  Half the ALU of 64-bit (hi << 32) + lo accumulation.
    auto fold_pair = [&](const int32_t* H, int32_t& rlo, int32_t& rhi) {
      auto hi16 = [](int32_t x) -> int32_t { return (int32_t)((uint32_t)x - (uint32_t)(int32_t)(int16_t)x) >> 16; };
      int32_t a[8], b[8];  // local-bit partials of x and hi, lb <= 7
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = b[i] = 0;
      int32_t X = 0, Y = 0;
      if (active) {
        const int4* H4 = reinterpret_cast<const int4*>(H);
        if (lb >= 2) {
          const int n4 = 1 << (lb - 2);
          for (int c4 = 0; c4 < n4; c4 += 4) {  // 4 int4 (16 bins) at a time
            int4 z[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j4 = (fbase >> 2) + c4 + i;  // logical int4 index
              const uint32_t c = ((uint32_t)j4 >> 3) & 31u;
              z[i] = (c4 + i < n4) ? unswizzle4(H4[j4 ^ (int)(c >> 2)], c) : make_int4(0, 0, 0, 0);
            }
            int32_t x[16] = {z[0].x, z[0].y, z[0].z, z[0].w, z[1].x, z[1].y, z[1].z, z[1].w,
                             z[2].x, z[2].y, z[2].z, z[2].w, z[3].x, z[3].y, z[3].z, z[3].w};
            int32_t y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = hi16(x[i]);
            int32_t tot = 0, toty = 0;
            if (FOLDPP) {  // pairwise compaction over the 4 bits inside the 16-bin chunk
#pragma unroll
              for (int L = 0; L < 4; ++L) {
                const int cnt = 8 >> L;
                int32_t odd = 0, oddy = 0;
#pragma unroll
                for (int tt = 0; tt < 8; ++tt)
                  if (tt < cnt) {
                    odd += x[2 * tt + 1];
                    oddy += y[2 * tt + 1];
                    x[tt] = x[2 * tt] + x[2 * tt + 1];
                    y[tt] = y[2 * tt] + y[2 * tt + 1];
                  }
                a[L] += odd;
                b[L] += oddy;
              }
              tot = x[0];
              toty = y[0];
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
#pragma unroll
                for (int L = 0; L < 4; ++L) {
                  a[L] += ((e >> L) & 1) ? x[e] : 0;
                  b[L] += ((e >> L) & 1) ? y[e] : 0;
                }
                tot += x[e];
                toty += y[e];
              }
            }
            const int ci = c4 >> 2;  // chunk bits 4.. are local bits too
#pragma unroll
            for (int L = 4; L < 8; ++L) {
              a[L] += ((ci >> (L - 4)) & 1) ? tot : 0;
              b[L] += ((ci >> (L - 4)) & 1) ? toty : 0;
            }
            X += tot;
            Y += toty;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < (1 << lb)) {
              const int32_t x = H[key_swizzle((uint32_t)(fbase + e))];
              const int32_t y = hi16(x);
              if (lb >= 1 && (e & 1)) { a[0] += x; b[0] += y; }
              X += x;
              Y += y;
            }
        }
      }
      auto set = [&](int32_t tx, int32_t ty) {  // slot value of both vectors from fold(x), fold(hi)
        rhi = ty;
        rlo = (int32_t)((uint32_t)tx - ((uint32_t)ty << 16));
      };
      rlo = 0; rhi = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < lb) {
          const int32_t tx = __reduce_add_sync(0xffffffffu, a[i]), ty = __reduce_add_sync(0xffffffffu, b[i]);
          if (lane == i) set(tx, ty);
        }
#pragma unroll
      for (int bit = 0; bit < 5; ++bit) {
        const bool on = (lane >> bit) & 1;
        const int32_t tx = __reduce_add_sync(0xffffffffu, on ? X : 0), ty = __reduce_add_sync(0xffffffffu, on ? Y : 0);
        if (lane == 8 + bit) set(tx, ty);
      }
      const int32_t Wx = __reduce_add_sync(0xffffffffu, X), Wy = __reduce_add_sync(0xffffffffu, Y);
#pragma unroll
      for (int fb2 = 0; fb2 < FB; ++fb2)
        if (lane == 13 + fb2) {
          if ((fw >> fb2) & 1) set(Wx, Wy);
          else set(0, 0);
        }
    };
    int fb = 0;          // f % NH, kept incrementally
    uint32_t fpar = 0;   // (f / NH) & 1
    for (int f = 0; f < nunits; ++f, (++fb == NH ? (fb = 0, fpar ^= 1u) : 0u)) {
      const int32_t* H = hist + fb * LIMBS * nbk;
      if (fw == 0 && f < 40) TRACE(8 + f * 8 + 3);
      mbar_wait(&hfull[fb], fpar);
      if (fw == 0 && f < 40) TRACE(8 + f * 8 + 4);
      int32_t d[OLIMBS];  // this block's slot value per limb: fold(H now) - fold(H after block f - NH)
      if constexpr (PACK) {
        fold_pair(H, d[0], d[OLIMBS - 1]);  // one pass (two int16 passes measured 11% slower)
        if (active) {  // zero my bins: the next block in this buffer starts from 0
          int32_t* Hw = const_cast<int32_t*>(H);
          if (lb >= 2) {
            for (int c4 = 0; c4 < (1 << (lb - 2)); ++c4) {
              const int j4 = (fbase >> 2) + c4;
              reinterpret_cast<int4*>(Hw)[j4 ^ (int)((((uint32_t)j4 >> 3) & 31u) >> 2)] = make_int4(0, 0, 0, 0);
            }
          } else {
            for (int e = 0; e < (1 << lb); ++e) Hw[key_swizzle((uint32_t)(fbase + e))] = 0;
          }
        }
      } else {
#pragma unroll
        for (int l = 0; l < LIMBS; ++l) {
          const int32_t r = fold_limb(H + l * nbk);
          int32_t pv = 0;
#pragma unroll
          for (int i = 0; i < MAXNH; ++i)
            if (i == fb) { pv = prev[l][i]; prev[l][i] = r; }
          d[l] = r - pv;
        }
      }
      __syncwarp();
      if (fw == 0 && f < 40) TRACE(8 + f * 8 + 5);
      if (lane == 0) mbar_arrive(&hfree[fb]);  // release: my reads of the buffer are complete
      const int b = p.b_begin + col_cta + f * ncol;
      const int w = block_width(p.cols, p.k, b);
      if constexpr (FX) {
        // exact fixed-point slot values from the 4 fold warps, summed in a fixed order
        long long* fp = fxpart + (f & 1) * FW * 16;
        if (lane < 16) fp[fw * 16 + lane] = ((long long)d[0] << 16) + (long long)d[LIMBS - 1];
        asm volatile("bar.sync 1, %0;" ::"r"(32 * FW) : "memory");
        if (fw == 0 && sh >= 0 && sh < w) {
          long long tot = 0;
#pragma unroll
          for (int i = 0; i < FW; ++i) tot += fp[i * 16 + lane];
          const int64_t o = (int64_t)b * p.k + (w - 1 - sh);
          const float r = (float)((double)tot * pow2d(-fx_e));
          out[o] = (OutT)r;
          if (p.pub.tagged)  // streamed publish: this block's columns are final
            asm volatile("st.global.u64 [%0], %1;" ::"l"(p.pub.tagged + o),
                         "l"(((unsigned long long)pub_seq << 32) | __float_as_uint(r)) : "memory");
        }
      } else if (!PACK && (p.pub.tagged || p.gat.npeers)) {
        // streamed publish (single split: this CTA owns the block's columns): the fold warps'
        // slot values summed in shared memory, one store per column to out and to the host
        int32_t* ip = reinterpret_cast<int32_t*>(fxpart) + (f & 1) * FW * 16;
        if (lane < 16) ip[fw * 16 + lane] = d[0];
        asm volatile("bar.sync 1, %0;" ::"r"(32 * FW) : "memory");
        if (fw == 0 && sh >= 0 && sh < w) {
          int32_t tot = 0;
#pragma unroll
          for (int i = 0; i < FW; ++i) tot += ip[i * 16 + lane];
          const int64_t o = (int64_t)b * p.k + (w - 1 - sh);
          out[o] = (OutT)tot;
          if (p.pub.tagged)
            asm volatile("st.global.u64 [%0], %1;" ::"l"(p.pub.tagged + o),
                         "l"(((unsigned long long)pub_seq << 32) | (uint32_t)tot) : "memory");
          for (int r = 0; r < p.gat.npeers; ++r) p.gat.out[r][p.gat.col_base + o] = tot;  // P2P stores
        }
        CNT(cnt_fold, sh >= 0 && sh < w && d[0] != 0);
      } else {
        if (sh >= 0 && sh < w && d[0] != 0) atomicAdd(out + (int64_t)b * p.k + (w - 1 - sh), (OutT)d[0]);
        CNT(cnt_fold, sh >= 0 && sh < w && d[0] != 0);
        if constexpr (PACK)
          if (sh >= 0 && sh < w && d[OLIMBS - 1] != 0) atomicAdd(out2 + (int64_t)b * p.k + (w - 1 - sh), (OutT)d[OLIMBS - 1]);
      }
      if (fw == 0 && f < 40) TRACE(400 + f);
    }
    if (fw == 0) TRACE(6);
    if (p.gat.npeers && fw == 0) {
      // fused all-gather: my peer stores released at system scope, then the launch's last CTA
      // (cumulativity through the completion counter) signals every rank
      __syncwarp();
      if (lane == 0) {
        __threadfence_system();
        const unsigned long long old = atomicAdd(p.gat.done, 1ull);
        if (old % gridDim.x == gridDim.x - 1) {
          __threadfence_system();
          for (int r = 0; r < p.gat.npeers; ++r)
            asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(p.gat.sig[r]) : "memory");
        }
      }
    }
  }
  if (warp == 0) TRACE(7);
#ifdef RSR_COUNT
  if (cnt_red) atomicAdd(&g_count[0], cnt_red);
  if (cnt_fold) atomicAdd(&g_count[1], cnt_fold);
  if (cnt_redux) atomicAdd(&g_count[2], cnt_redux);
#endif
}

// =====================================================================================
// GATHER kernel (fp32 / fp64 / int32)
// =====================================================================================

struct GatherParams {
  const void* perm[2];
  const uint32_t* seg[2];
  const void* v;
  void* out;
  int64_t rows, cols, row_stride, seg_stride;
  int k, halves, b_begin, b_end;
  int perm_bytes, v_in_smem, seg_in_smem;
};

constexpr int kGatherWarps = 8;
constexpr int kMaxWin = 64;    // window-end records buffered per warp (expanded when full)

template <typename T>
__device__ __forceinline__ T vload(const T* vs, const T* vg, uint32_t row, bool smem) {
  return smem ? vs[row] : __ldg(vg + row);
}

// One CTA per column block at a time (persistent over blocks).  The 8 warps split the block's
// sorted positions: (half, part) = (warp / P, warp % P), P = 8 / halves contiguous position
// ranges per half.  Per 256-position window a warp gathers v[perm[p]] from shared memory (8
// positions per lane; perm streamed kPermAhead windows ahead with 16-byte loads) and forms
// window-local prefix sums with a warp scan (stored transposed: conflict-free).  Every bucket
// boundary j (position seg[j], seg staged in shared memory) contributes its prefix P with the
// RSR++ telescoping coefficients bit_s(j-1) - bit_s(j) — the pairwise compaction of Alg. 3
// applied to prefix sums: the lane adds P to its private slot B[ctz(j)], and at the range end
// column s receives sum_{t>s} B[t] - B[s] (two adds per bucket overall).  For variant "rsr"
// the boundary forms the segment sum u and adds it to every column whose bit is set (the dense
// product).  The bucket open at a window end contributes the window total with its bit
// pattern (one (bucket, total) record per window, expanded in parallel at the range end).
// Everything is linear, so the warps' partial column sums are combined in a fixed order:
// deterministic, no float atomics.
template <typename T, bool FOLDPP, bool PERM16>
__global__ void __launch_bounds__(kGatherWarps * 32) gather_kernel(const GatherParams p) {
  constexpr int AHEAD = PERM16 ? 12 : 6;  // perm windows in flight per warp (16-byte loads)
  constexpr int PW = PERM16 ? 1 : 2;      // uint4 per lane per window
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg_words = p.seg_in_smem ? (int)((p.seg_stride + 3) & ~3) : 0;
  uint32_t* segs = reinterpret_cast<uint32_t*>(smem);                       // [2][seg_words]
  T* pbuf_all = reinterpret_cast<T*>(segs + 2 * seg_words);                  // [8][256]
  T* pbuf = pbuf_all + warp * 256;
  T* part = pbuf_all + kGatherWarps * 256;                                   // [8][16]
  T* Bl_all = part + kGatherWarps * 16;                                      // [8][32 lanes][17] telescoping slots
  T* Bl = Bl_all + (warp * 32 + lane) * 17;
  T* etot_all = Bl_all + kGatherWarps * 32 * 17;                             // [8][kMaxWin] window-end totals
  int* ebkt_all = reinterpret_cast<int*>(etot_all + kGatherWarps * kMaxWin); // [8][kMaxWin] window-end buckets
  T* etot = etot_all + warp * kMaxWin;
  int* ebkt = ebkt_all + warp * kMaxWin;
  T* vs = reinterpret_cast<T*>(ebkt_all + kGatherWarps * kMaxWin);
  const T* vg = reinterpret_cast<const T*>(p.v);
  const bool vsm = p.v_in_smem != 0;
  if (vsm)
    for (int i = threadIdx.x; i < (int)p.rows; i += blockDim.x) vs[i] = vg[i];
  T* out = reinterpret_cast<T*>(p.out);
  const int P = kGatherWarps / p.halves;  // position ranges per half
  const int h = warp / P, part_i = warp % P;
  const int rows = (int)p.rows;
  const int plen = ((rows + P - 1) / P + 255) / 256 * 256;  // window-aligned range length
  const int P0 = part_i * plen;
  const int P1 = min(rows, P0 + plen);
  const uint32_t* seg0 = p.seg[0];
  const uint32_t* seg1 = p.seg[1];
  const void* perm_g = h ? p.perm[1] : p.perm[0];
  const T sgn = h ? T(-1) : T(1);

  for (int b = p.b_begin + blockIdx.x; b < p.b_end; b += gridDim.x) {
    const int w = block_width(p.cols, p.k, b);
    const int nbk = 1 << w;
    __syncthreads();  // previous block's segs / part are no longer read
    if (p.seg_in_smem)
      for (int i = threadIdx.x; i < p.halves * (nbk + 1); i += blockDim.x) {
        const int hh = i / (nbk + 1), j = i % (nbk + 1);
        segs[hh * seg_words + j] = (hh ? seg1 : seg0)[(int64_t)b * p.seg_stride + j];
      }
#pragma unroll
    for (int i = 0; i < 17; ++i) Bl[i] = T(0);
    __syncthreads();
    const uint32_t* seg = p.seg_in_smem ? segs + h * seg_words : (h ? seg1 : seg0) + (int64_t)b * p.seg_stride;
    T acc[kMaxK];  // dense ("rsr") accumulation only
#pragma unroll
    for (int s = 0; s < kMaxK; ++s) acc[s] = T(0);
    int nwin = 0;
    if (P0 < P1) {
      // first boundary after P0: jcur = 1 + #{j in [1, nbk] : seg[j] <= P0}
      int lo = 1, hi = nbk + 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int)seg[mid] <= P0) lo = mid + 1; else hi = mid;
      }
      int jcur = (P0 == 0) ? 1 : lo;
      T carry = T(0);
      const uint16_t* perm16 = reinterpret_cast<const uint16_t*>(perm_g) + (int64_t)b * p.row_stride;
      const uint32_t* perm32 = reinterpret_cast<const uint32_t*>(perm_g) + (int64_t)b * p.row_stride;
      auto load_perm = [&](int w0, uint4 (&q)[PW]) {
        const int pos0 = w0 + 8 * lane;
#pragma unroll
        for (int i = 0; i < PW; ++i) q[i] = make_uint4(0, 0, 0, 0);
        if (pos0 < P1) {
          if (PERM16) {
            q[0] = ld_nc_v4(perm16 + pos0);
          } else {
            q[0] = ld_nc_v4(perm32 + pos0);
            q[PW - 1] = ld_nc_v4(perm32 + pos0 + 4);
          }
        }
      };
      uint4 ring[AHEAD][PW];
#pragma unroll
      for (int i = 0; i < AHEAD; ++i) load_perm(P0 + 256 * i, ring[i]);
      for (int wb = P0; wb < P1; wb += 256 * AHEAD) {
#pragma unroll
        for (int ri = 0; ri < AHEAD; ++ri) {  // static ring slots: no register shuffling
          const int w0 = wb + 256 * ri;
          if (w0 < P1) {
            const int E = min(256, P1 - w0);
            const int pos0 = w0 + 8 * lane;
            uint32_t rowsel[8];
            if (PERM16) {
              const uint4 q0 = ring[ri][0];
              rowsel[0] = q0.x & 0xffffu; rowsel[1] = q0.x >> 16; rowsel[2] = q0.y & 0xffffu; rowsel[3] = q0.y >> 16;
              rowsel[4] = q0.z & 0xffffu; rowsel[5] = q0.z >> 16; rowsel[6] = q0.w & 0xffffu; rowsel[7] = q0.w >> 16;
            } else {
              const uint4 q0 = ring[ri][0], q1 = ring[ri][PW - 1];
              rowsel[0] = q0.x; rowsel[1] = q0.y; rowsel[2] = q0.z; rowsel[3] = q0.w;
              rowsel[4] = q1.x; rowsel[5] = q1.y; rowsel[6] = q1.z; rowsel[7] = q1.w;
            }
            T x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (pos0 + e < P1) ? vload(vs, vg, rowsel[e], vsm) : T(0);
            load_perm(w0 + 256 * AHEAD, ring[ri]);  // refill this slot
#pragma unroll
            for (int e = 1; e < 8; ++e) x[e] += x[e - 1];
            const T incl = warp_inclusive_scan(x[7], lane);
            const T base = incl - x[7];
            const T total = __shfl_sync(0xffffffffu, incl, 31);
            // transposed prefix buffer: position 8*lane + e lives at e*32 + lane (conflict-free)
#pragma unroll
            for (int e = 0; e < 8; ++e) pbuf[e * 32 + lane] = base + x[e];
            __syncwarp();
            int last_in = -1;
            T p_last = T(0);
            while (true) {
              const int jj = jcur + lane;
              const int sj = jj <= nbk ? (int)seg[jj] : 0x7fffffff;
              const bool in = sj <= w0 + E;
              const int cnt = __popc(__ballot_sync(0xffffffffu, in));
              T Pv = T(0);
              if (in) {
                const int q = sj - w0 - 1;
                Pv = q >= 0 ? pbuf[((q & 7) << 5) | (q >> 3)] : T(0);
              }
              if (FOLDPP) {
                if (in) {  // boundary j closes bucket j-1, opens bucket j: +P below ctz(j), -P at ctz(j)
                  const int tz = __ffs(jj) - 1;
                  Bl[tz] += sgn * Pv;
                }
              } else {
                const T prevP = __shfl_up_sync(0xffffffffu, Pv, 1);
                if (in) {
                  const T uj = (lane == 0) ? carry + Pv : Pv - prevP;
                  const int j = jj - 1;
#pragma unroll
                  for (int s = 0; s < kMaxK; ++s) acc[s] += ((j >> s) & 1) ? sgn * uj : T(0);
                }
                if (cnt > 0) {
                  p_last = __shfl_sync(0xffffffffu, Pv, cnt - 1);
                  carry = T(0);
                  last_in = cnt - 1;
                }
              }
              jcur += cnt;
              if (cnt < 32) break;
              if (!FOLDPP) carry = T(0) - p_last;
            }
            if (FOLDPP) {  // bucket open at the window end: its tail is the window total
              if (lane == 0) {
                ebkt[nwin] = jcur - 1;
                etot[nwin] = sgn * total;
              }
              ++nwin;
            } else {
              carry = (last_in >= 0) ? total - p_last : carry + total;
            }
            __syncwarp();
            if (FOLDPP && nwin == kMaxWin) {  // record buffer full (long ranges): expand it now
              for (int i = lane; i < nwin; i += 32) {
                const int g = ebkt[i];
                const T tt = etot[i];
#pragma unroll
                for (int s = 0; s < kMaxK; ++s) acc[s] += ((g >> s) & 1) ? tt : T(0);
              }
              nwin = 0;
              __syncwarp();
            }
          }
        }
      }
      if (!FOLDPP) {
        const int g = jcur - 1;  // the bucket still open at the range end gets the carried tail
        if (lane == 0 && P1 < rows) {
#pragma unroll
          for (int s = 0; s < kMaxK; ++s) acc[s] += ((g >> s) & 1) ? sgn * carry : T(0);
        }
      }
    }
    if (FOLDPP) {
      __syncwarp();
      // telescoping slots -> columns: acc[s] = sum_{t > s} B[t] - B[s]
      T suffix = T(0);
#pragma unroll
      for (int s = kMaxK; s >= 0; --s) {
        const T bs = Bl[s];
        if (s < kMaxK) acc[s] += suffix - bs;
        suffix += bs;
      }
      // window-end records, one per lane
      for (int i = lane; i < nwin; i += 32) {
        const int g = ebkt[i];
        const T tt = etot[i];
#pragma unroll
        for (int s = 0; s < kMaxK; ++s) acc[s] += ((g >> s) & 1) ? tt : T(0);
      }
    }
    const T r = reduce_scatter16(acc, lane);  // lanes 2s, 2s+1: warp total of column shift s
    if (!(lane & 1)) part[warp * 16 + (lane >> 1)] = r;
    __syncthreads();
    if (warp == 0 && lane < w) {
      T sum = T(0);
      for (int ww = 0; ww < kGatherWarps; ++ww) sum += part[ww * 16 + lane];
      out[(int64_t)b * p.k + (w - 1 - lane)] = sum;
    }
  }
}

// gather-form bucket sums of one block (segmented_sum, kernels.py:50-60, 94-101):
// one warp per bucket chunk, ascending-position accumulation per bucket.
template <typename T>
__global__ void segmented_sum_kernel(const void* perm, int perm_bytes, const uint32_t* seg, const T* v, int nbk,
                                     T* u) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nbk) return;
  const uint32_t lo = seg[j], hi = seg[j + 1];
  T acc = T(0);
  for (uint32_t q = lo; q < hi; ++q) {
    const uint32_t r = perm_bytes == 2 ? reinterpret_cast<const uint16_t*>(perm)[q]
                                       : reinterpret_cast<const uint32_t*>(perm)[q];
    acc += v[r];
  }
  u[j] = acc;
}

// Block products of one SegmentedSums vector (block_product_rsr / block_product_rsrpp,
// kernels.py:104-116): a single thread replays the reference loops in fp64 so the
// result is bitwise the reference's.  Utility op; the multiply kernels fold in-warp.
__global__ void block_product_kernel(const double* __restrict__ u, int w, int use_fold, double* __restrict__ buf,
                                     double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t nseg = (int64_t)1 << w;
  if (use_fold) {  // kernels.py:74-91
    int64_t half = nseg >> 1;
    double acc = 0.0;
    for (int64_t t = 0; t < half; ++t) {
      acc += u[2 * t + 1];
      buf[t] = u[2 * t] + u[2 * t + 1];
    }
    out[w - 1] = acc;
    int64_t size = half;
    for (int c = w - 2; c >= 0; --c) {
      half = size >> 1;
      acc = 0.0;
      for (int64_t t = 0; t < half; ++t) {
        acc += buf[2 * t + 1];
        buf[t] = buf[2 * t] + buf[2 * t + 1];
      }
      out[c] = acc;
      size = half;
    }
  } else {  // kernels.py:63-71
    for (int c = 0; c < w; ++c) {
      const int shift = w - 1 - c;
      double acc = 0.0;
      for (int64_t j = 0; j < nseg; ++j) acc += u[j] * (double)((j >> shift) & 1);
      out[c] = acc;
    }
  }
}

// Standard dense multiply (core.py:135-169) on the GPU: thread per column, rows ascending.
template <typename T>
__global__ void naive_ternary_kernel(const int8_t* __restrict__ A, int64_t rows, int64_t cols, int64_t lda,
                                     const T* __restrict__ v, T* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  T acc = T(0);
  for (int64_t i = 0; i < rows; ++i) {
    const int8_t a = A[i * lda + j];
    acc += (a == 1) ? v[i] : ((a == -1) ? -v[i] : T(0));
  }
  out[j] = acc;
}

// ------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------

// Programmatic dependent launch on by default (RSR_B200_PDL=0 disables it).
static bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RSR_B200_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <bool PP, typename OutT, bool FX, int FW, bool PACK>
rsr_status launch_scatter_t(const ScatterParams& p, int grid, size_t smem, int threads, cudaStream_t s) {
  auto pick = [&](auto ternary) {
    constexpr bool T = decltype(ternary)::value;
    return p.codes == 1 ? scatter_kernel<kScatterR, PP, T, OutT, FX, 1, FW, PACK>
           : p.codes == 2 ? scatter_kernel<kScatterR, PP, T, OutT, FX, 2, FW, PACK>
                          : scatter_kernel<kScatterR, PP, T, OutT, FX, 0, FW, PACK>;
  };
  auto kern = p.halves == 2 ? pick(std::true_type{}) : pick(std::false_type{});
  rsr_status st = set_max_smem((const void*)kern, smem);
  if (st != RSR_OK) return st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads + 32 * FW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, kern, p), "scatter_kernel launch");
}

template <bool PP, typename OutT, bool FX, bool PACK = false>
rsr_status launch_scatter_fw(const ScatterParams& p, int grid, size_t smem, int threads, int fw, cudaStream_t s) {
  return fw == 1   ? launch_scatter_t<PP, OutT, FX, 1, PACK>(p, grid, smem, threads, s)
         : fw == 2 ? launch_scatter_t<PP, OutT, FX, 2, PACK>(p, grid, smem, threads, s)
                   : launch_scatter_t<PP, OutT, FX, kFoldWarps, PACK>(p, grid, smem, threads, s);
}

rsr_status multiply_scatter(const rsr_index_desc& d, const void* v, bool fx, void* out, rsr_dtype out_dtype, bool pp,
                            int b0, int b1, cudaStream_t s, const Publish* pub, bool* published, bool independent,
                            const void* v2 = nullptr, void* out2 = nullptr, const Gather* gat = nullptr) {
  if (d.k > 14) return fail(RSR_ERR_UNSUPPORTED, "scatter multiply supports k <= 14");
  const bool pack = v2 != nullptr;
  if (pack && (fx || out_dtype != RSR_I32 || pub))
    return fail(RSR_ERR_INVALID, "packed pair multiply: int32 activations and output only");
  ScatterParams p{};
  p.v2 = reinterpret_cast<const int32_t*>(v2);
  p.out2 = out2;
  p.independent = independent ? 1 : 0;
  const bool publish = (pub && out_dtype != RSR_F64) || gat;  // single split only (decided below)
  for (int h = 0; h < d.halves; ++h) p.key[h] = d.half[h].bucket;
  p.v = reinterpret_cast<const int32_t*>(v);
  p.v_aligned = ((uintptr_t)v & 15) == 0 && ((uintptr_t)v2 & 15) == 0;
  p.out = out;
  p.rows = d.rows;
  p.cols = d.cols;
  p.row_stride = d.row_stride;
  p.k = d.k;
  p.halves = d.halves;
  p.b_begin = b0;
  p.b_end = b1;
  // R = 32 rows per thread; a power-of-two warp count (the fold maps warp-index bits onto key bits)
  const int R = kScatterR;
  int threads = 32;
  while (threads < kScatterThreads && (int64_t)threads * R < d.rows) threads *= 2;
  threads = std::min(threads, kScatterThreads);
  p.rows_per_cta = threads * R;
  p.scatter_warps = threads / 32;
  p.sched = sched_keys(d.k);
  p.codes = !p.sched ? 0 : code_shift(d.k) == 2 ? 1 : 2;
  p.code_mask = p.sched ? kSchedCodeMask : 0xffffffffu;
  p.n_splits = (int)((d.rows + p.rows_per_cta - 1) / p.rows_per_cta);
  p.atomic_out = p.n_splits > 1;
  if (gat) {
    if (p.n_splits != 1 || fx || out_dtype != RSR_I32)
      return fail(RSR_ERR_UNSUPPORTED, "all-gather epilogue: single-split int32 launches only");
    p.gat = *gat;
  } else if (publish && p.n_splits == 1) {
    p.pub = *pub;
    if (published) *published = true;
  } else if (pub && pub->pull) {
    return fail(RSR_ERR_INVALID, "session pull needs a publishing (single-split int32 / fp32) launch");
  }
  if (p.pub.pull || p.gat.npeers) p.independent = 0;  // a pull writes v; the all-gather signals peers
  if (p.pub.pull && (!p.v_aligned || (p.pub.pull_bytes & 15u) || ((uintptr_t)p.pub.pull & 15u)))
    return fail(RSR_ERR_INVALID, "session pull: 16-byte aligned payload expected");
  const size_t max_smem = device_max_smem_optin();
  const size_t limbs = fx ? 2 : 1;
  auto need = [&](int nh) {  // layout of scatter_kernel's dynamic smem
    return ((sizeof(int32_t) * ((((size_t)1 << d.k) * nh * limbs + 15) & ~(size_t)15) + 127) & ~(size_t)127) +
           8 * (2 * nh) + 128 /* fxmax */ + (fx || publish ? sizeof(long long) * 2 * kFoldWarps * 16 : 0) /* fxpart */;
  };
  // the deferred fold wants 3 histogram buffers (2 is the minimum)
  int nhist = need(3) <= max_smem ? 3 : 2;
  if (need(nhist) > max_smem) return fail(RSR_ERR_UNSUPPORTED, "scatter multiply: histograms do not fit in shared memory");
  // diagnostics overrides, read once (an environment scan per launch costs ~1 us of host time)
  static const int env_stages = getenv("RSR_B200_STAGES") ? std::max(0, atoi(getenv("RSR_B200_STAGES"))) : -1;
  static const int env_nhist = getenv("RSR_B200_NHIST") ? std::min(4, std::max(2, atoi(getenv("RSR_B200_NHIST")))) : -1;
  // L2 bulk prefetch distance in units beyond the next one: 0 (the next unit only) measured best
  // under independent launches (tools/ab.sh RSR_B200_STAGES: 16384^2 22.18 -> 21.68 us with 0
  // instead of 3, 14336 x 4096 7.35 -> 7.01, 4096 x 14336 6.62 -> 6.46, binary 14.66 -> 14.49)
  const int stages = env_stages >= 0 ? env_stages : 0;
  if (env_nhist > 0) nhist = env_nhist;
  p.stages = stages;
  p.nhist = nhist;
  const size_t smem = need(nhist);
  // small CTAs (few rows) share an SM: limits from threads, smem and registers (<= 96 per
  // thread under the launch bounds)
  // fold warps: threads < 128: one (so that FW = 4 means 4, 8 or 16 scatter warps and the fold
  // warps form one aligned warpgroup)
  static const int env_fw = getenv("RSR_B200_FOLD_WARPS") ? atoi(getenv("RSR_B200_FOLD_WARPS")) : 0;  // A/B only
  // 4 scatter warps (rows <= 4096): 2 fold warps for int32 (4096^2 3.74 vs 4.35 us with 1, 4096 x 14336
  // 7.90 vs 8.34 us with 4), 4 for the two-limb FX fold (4096^2 fp32 6.09 vs 7.20 us with 1)
  int fw = threads < 128 ? 1 : threads == 128 ? (fx ? kFoldWarps : 2) : kFoldWarps;
  const int nblk = b1 - b0;
  // RSR_B200_MAX_CTAS (read once): leave SMs free for a concurrent collective — the multi-GPU
  // bench runs the all-gather of step i on a comm stream beside the multiply of step i + 1, and
  // an NCCL kernel cannot start while a persistent 148-CTA grid holds every SM
  static const int env_max_ctas = getenv("RSR_B200_MAX_CTAS") ? atoi(getenv("RSR_B200_MAX_CTAS")) : 0;
  const int sms = env_max_ctas > 0 ? std::min(device_sm_count(), env_max_ctas) : device_sm_count();
  // independent launches overlap their neighbours' CTAs: fewer fold warps leave room for more
  // CTAs per SM (tools/fw_ab.sh, independent stream: 4096^2 fp32 5.32 -> 4.97 us with 2 instead
  // of 4; 4096 x 14336 int32, several CTA waves, 6.82 -> 6.63 us with 1 instead of 2)
  if (p.independent && threads == 128) fw = fx ? 2 : (nblk > 3 * sms ? 1 : 2);
  if (env_fw == 1 || env_fw == 2 || env_fw == kFoldWarps) fw = (threads < 128 && env_fw > 1) ? fw : env_fw;
  const int cta_threads = threads + 32 * fw;
  const int per_sm = std::max<int>(1, (int)std::min<size_t>(std::min(2048 / cta_threads, 65536 / (cta_threads * 96)),
                                                            (228u << 10) / (smem + 1024)));
  const int ncol = std::max(1, std::min(nblk, sms * per_sm / std::max(1, p.n_splits)));
  const int grid = ncol * p.n_splits;
  if (p.atomic_out) {
    const size_t esz = out_dtype == RSR_F64 ? 8 : 4;
    const int64_t c0 = (int64_t)b0 * d.k;
    const int64_t c1 = std::min<int64_t>(d.cols, (int64_t)b1 * d.k);
    rsr_status st = cuda_check(cudaMemsetAsync((char*)out + c0 * esz, 0, (c1 - c0) * esz, s), "memset out");
    if (st != RSR_OK) return st;
    if (pack) {
      st = cuda_check(cudaMemsetAsync((char*)out2 + c0 * esz, 0, (c1 - c0) * esz, s), "memset out2");
      if (st != RSR_OK) return st;
    }
  }
  if (pack)
    return pp ? launch_scatter_fw<true, int32_t, false, true>(p, grid, smem, threads, fw, s)
              : launch_scatter_fw<false, int32_t, false, true>(p, grid, smem, threads, fw, s);
  if (fx)
    return pp ? launch_scatter_fw<true, float, true>(p, grid, smem, threads, fw, s)
              : launch_scatter_fw<false, float, true>(p, grid, smem, threads, fw, s);
  if (out_dtype == RSR_F64)
    return pp ? launch_scatter_fw<true, double, false>(p, grid, smem, threads, fw, s)
              : launch_scatter_fw<false, double, false>(p, grid, smem, threads, fw, s);
  return pp ? launch_scatter_fw<true, int32_t, false>(p, grid, smem, threads, fw, s)
            : launch_scatter_fw<false, int32_t, false>(p, grid, smem, threads, fw, s);
}

template <typename T>
rsr_status multiply_gather_t(const rsr_index_desc& d, const void* v, void* out, bool pp, int b0, int b1,
                             cudaStream_t s) {
  GatherParams p{};
  for (int h = 0; h < d.halves; ++h) {
    p.perm[h] = d.half[h].perm;
    p.seg[h] = d.half[h].seg;
  }
  p.v = v;
  p.out = out;
  p.rows = d.rows;
  p.cols = d.cols;
  p.row_stride = d.row_stride;
  p.seg_stride = d.seg_stride;
  p.k = d.k;
  p.halves = d.halves;
  p.b_begin = b0;
  p.b_end = b1;
  p.perm_bytes = d.perm_bytes;
  const size_t max_smem = device_max_smem_optin();
  const size_t pbuf_bytes = sizeof(T) * (kGatherWarps * 256 + kGatherWarps * 16 + kGatherWarps * 32 * 17 +
                                         kGatherWarps * kMaxWin) + sizeof(int) * kGatherWarps * kMaxWin;
  if (d.rows > ((int64_t)1 << 30)) return fail(RSR_ERR_UNSUPPORTED, "gather multiply supports at most 2^30 rows");
  p.seg_in_smem = sizeof(uint32_t) * 2 * (size_t)((d.seg_stride + 3) & ~3) + pbuf_bytes <= (96u << 10);
  const size_t seg_words = p.seg_in_smem ? (size_t)((d.seg_stride + 3) & ~3) : 0;
  const size_t fixed = sizeof(uint32_t) * 2 * seg_words + pbuf_bytes;
  const size_t vbytes = sizeof(T) * (size_t)d.rows;
  p.v_in_smem = fixed + vbytes <= max_smem;
  const size_t smem = fixed + (p.v_in_smem ? vbytes : 0);
  const int per_sm = std::max<int>(1, (int)std::min<size_t>(4, (228u << 10) / (smem + 1024)));
  const int nblk = b1 - b0;
  const int grid = std::max(1, std::min(nblk, device_sm_count() * per_sm));
  auto kern = d.perm_bytes == 2 ? (pp ? gather_kernel<T, true, true> : gather_kernel<T, false, true>)
                                : (pp ? gather_kernel<T, true, false> : gather_kernel<T, false, false>);
  rsr_status st = set_max_smem((const void*)kern, smem);
  if (st != RSR_OK) return st;
  kern<<<grid, kGatherWarps * 32, smem, s>>>(p);
  return cuda_check(cudaGetLastError(), "gather_kernel launch");
}

}  // namespace

rsr_status multiply_allgather(const rsr_index_desc& d, const int32_t* v, int32_t* out, rsr_variant var, const Gather& g,
                              cudaStream_t s) {
  if (g.npeers < 1 || g.npeers > kMaxPeers) return fail(RSR_ERR_INVALID, "all-gather: 1 to 8 ranks");
  if (!publishes(d, RSR_I32)) return fail(RSR_ERR_UNSUPPORTED, "all-gather epilogue: single-split int32 launches only");
  return multiply_scatter(d, v, false, out, RSR_I32, var == RSR_VARIANT_RSRPP, 0, d.nblocks, s, nullptr, nullptr, false,
                          nullptr, nullptr, &g);
}

bool publishes(const rsr_index_desc& d, rsr_dtype vt) {
  return (vt == RSR_I32 || vt == RSR_F32) && d.k <= 14 && d.rows <= (int64_t)kScatterThreads * kScatterR;
}

rsr_status multiply(const rsr_index_desc& d, const void* v, rsr_dtype vt, void* out, rsr_dtype ot, rsr_variant var,
                    rsr_form form, int b0, int b1, cudaStream_t s, const Publish* pub, bool* published,
                    bool independent) {
  const bool pp = var == RSR_VARIANT_RSRPP;
  if (published) *published = false;
  if (b0 >= b1) return RSR_OK;
  // fp32 on the scatter kernel needs one quantization scale per output column: one row split
  const bool fx_ok = vt == RSR_F32 && ot == RSR_F32 && d.rows <= (int64_t)kScatterThreads * kScatterR && d.k <= 14;
  if (form == RSR_FORM_AUTO)
    form = ((vt == RSR_I32 && d.k <= 14) || fx_ok) ? RSR_FORM_SCATTER : RSR_FORM_GATHER;
  if (form == RSR_FORM_SCATTER) {
    if (vt == RSR_F32) {
      if (!fx_ok) return fail(RSR_ERR_INVALID, "fp32 scatter form needs rows <= 16384, k <= 14, fp32 output");
      return multiply_scatter(d, v, true, out, ot, pp, b0, b1, s, pub, published, independent);
    }
    if (vt != RSR_I32) return fail(RSR_ERR_INVALID, "scatter form needs int32 or fp32 activations");
    if (ot != RSR_I32 && ot != RSR_F64) return fail(RSR_ERR_INVALID, "int32 activations produce int32 or float64");
    return multiply_scatter(d, v, false, out, ot, pp, b0, b1, s, pub, published, independent);
  }
  if (vt != ot) return fail(RSR_ERR_INVALID, "gather form writes the activation dtype");
  switch (vt) {
    case RSR_I32: return multiply_gather_t<int32_t>(d, v, out, pp, b0, b1, s);
    case RSR_F32: return multiply_gather_t<float>(d, v, out, pp, b0, b1, s);
    case RSR_F64: return multiply_gather_t<double>(d, v, out, pp, b0, b1, s);
    default: break;
  }
  return fail(RSR_ERR_INVALID, "unknown dtype");
}

namespace {
// grid-stride over (block, bin) pairs, then over the activations; warp max, one atomic per warp
// grid (bins / 256, ceil(b1 / 4) + 128): rows below ceil(b1 / 4) cover 4 blocks' bins each
// (coalesced seg reads), the last 128 rows the activations (grid-stride); CTA max, then one
// atomic per CTA (same-address atomics from every warp serialise at L2)
__global__ void __launch_bounds__(256) pack_guard_kernel(const rsr_index_desc d, int b1, const int32_t* __restrict__ V,
                                                         int64_t nv, uint32_t* res) {
  constexpr int kBlocksPerRow = 4, kVRows = 128;
  uint32_t m = 0;
  const int brows = (b1 + kBlocksPerRow - 1) / kBlocksPerRow;
  const bool is_bins = (int)blockIdx.y < brows;
  if (is_bins) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int q = 0; q < kBlocksPerRow; ++q) {
      const int b = blockIdx.y * kBlocksPerRow + q;
      if (b < b1 && j >= 1 && j < ((int64_t)1 << block_width(d.cols, d.k, b))) {
        uint32_t load = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h)  // constant half index: the descriptor stays in param space
          if (h < d.halves) {
            const uint32_t* seg = d.half[h].seg + (int64_t)b * d.seg_stride;
            load += __ldg(seg + j + 1) - __ldg(seg + j);
          }
        m = max(m, load);
      }
    }
  } else {
    const int64_t stride = (int64_t)kVRows * gridDim.x * blockDim.x;
    for (int64_t i = ((int64_t)(blockIdx.y - brows) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
         i += stride) {
      const int32_t x = V[i];
      m = max(m, x < 0 ? 0u - (uint32_t)x : (uint32_t)x);
    }
  }
  __shared__ uint32_t wm[8];
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = max(m, wm[i]);
    if (m) atomicMax(res + (is_bins ? 0 : 1), m);
  }
}
}  // namespace

rsr_status pack_guard(const rsr_index_desc& d, int b1, const int32_t* V, int64_t nv, uint32_t* res, cudaStream_t s) {
  const dim3 grid((unsigned)std::max<int64_t>(8, (((int64_t)1 << d.k) + 255) / 256), (unsigned)((b1 + 3) / 4 + 128));
  pack_guard_kernel<<<grid, 256, 0, s>>>(d, b1, V, nv, res);
  return cuda_check(cudaGetLastError(), "pack_guard_kernel launch");
}

rsr_status multiply_pair(const rsr_index_desc& d, int b1, const int32_t* va, const int32_t* vb, int32_t* outa,
                         int32_t* outb, rsr_variant var, cudaStream_t s, bool independent) {
  return multiply_scatter(d, va, false, outa, RSR_I32, var == RSR_VARIANT_RSRPP, 0, b1, s, nullptr, nullptr,
                          independent, vb, outb);
}

rsr_status segmented_sum(const rsr_index_desc& d, int half, int block, const void* v, rsr_dtype dt, void* u,
                         cudaStream_t s) {
  const int w = block_width(d.cols, d.k, block);
  const int nbk = 1 << w;
  const void* perm = (const char*)d.half[half].perm + (size_t)block * d.row_stride * d.perm_bytes;
  const uint32_t* seg = d.half[half].seg + (size_t)block * d.seg_stride;
  const int grid = (nbk + 255) / 256;
  switch (dt) {
    case RSR_I32: segmented_sum_kernel<int32_t><<<grid, 256, 0, s>>>(perm, d.perm_bytes, seg, (const int32_t*)v, nbk, (int32_t*)u); break;
    case RSR_F32: segmented_sum_kernel<float><<<grid, 256, 0, s>>>(perm, d.perm_bytes, seg, (const float*)v, nbk, (float*)u); break;
    case RSR_F64: segmented_sum_kernel<double><<<grid, 256, 0, s>>>(perm, d.perm_bytes, seg, (const double*)v, nbk, (double*)u); break;
    default: return fail(RSR_ERR_INVALID, "segmented sum takes int32, float32 or float64");
  }
  return cuda_check(cudaGetLastError(), "segmented_sum_kernel launch");
}

rsr_status block_product(const double* u, int w, int use_fold, double* buf, double* out, cudaStream_t s) {
  block_product_kernel<<<1, 32, 0, s>>>(u, w, use_fold, buf, out);
  return cuda_check(cudaGetLastError(), "block_product_kernel launch");
}

rsr_status naive_ternary(const int8_t* A, int64_t rows, int64_t cols, int64_t lda, const void* v, rsr_dtype dt,
                         void* out, cudaStream_t s) {
  const unsigned grid = (unsigned)((cols + 255) / 256);
  switch (dt) {
    case RSR_I32: naive_ternary_kernel<int32_t><<<grid, 256, 0, s>>>(A, rows, cols, lda, (const int32_t*)v, (int32_t*)out); break;
    case RSR_F32: naive_ternary_kernel<float><<<grid, 256, 0, s>>>(A, rows, cols, lda, (const float*)v, (float*)out); break;
    case RSR_F64: naive_ternary_kernel<double><<<grid, 256, 0, s>>>(A, rows, cols, lda, (const double*)v, (double*)out); break;
    default: return fail(RSR_ERR_INVALID, "naive multiply takes int32, float32 or float64");
  }
  return cuda_check(cudaGetLastError(), "naive_ternary_kernel launch");
}

}  // namespace rsr
