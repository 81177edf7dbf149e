// Batch-native RSR / RSR++ multiply (BASELINE config 3: B activation vectors against ONE index).
//
// The reference has no batch API: it runs `multiply_ternary` (kernels.py:196-206) once per
// vector, i.e. the scatter loop `u[bucket[r]] += v[r]` (`_run_blocks`, kernels.py:127-177) and the
// fold (`_product_fold`, kernels.py:74-91) per vector.  Here the loop is turned so that the 32
// lanes of a warp span the VECTOR dimension: lane w holds the packed int16 pair of vectors 2w
// and 2w + 1 (v + v' * 2^16, the per-vector kernel's PACK trick), and one shared-memory
// reduction adds one row's 64 activations into the 32 consecutive words of ONE histogram slot.
// Those reductions never conflict (tools/microbench/batch_red.cu: 1 cycle per warp instruction
// against ~2 for 32 random words), the slot codes are warp-uniform (one broadcast load per
// 8 rows per block and half), and every activation row is read once per pass of P = 2 column
// blocks.  A slot is 128 bytes, so the histograms use a re-cut index, the BATCH PLAN:
//
//  * plan_rowkeys_kernel: row-order keys of every index block from perm + seg (the bucket of
//    sorted position p is the largest j with seg[j] <= p, indexer.py:176-186);
//  * plan_keys_kernel: the kb-bit key (MSB-first, indexer.py:215-219) of every row in every
//    kb-wide plan block, composed from the index keys' bits;
//  * plan_slots_kernel (one CTA per unit = plan block x row split): a bin whose rows over both
//    halves could push an int16 sum past 32767 for |v| <= vmax (load > 32767 / vmax) is split
//    into ceil(load / lmax) slots, its rows dealt round-robin by their rank (halves, then row
//    order), so every slot's sum fits int16 and the packed accumulation is exact.  Split slots
//    follow the 2^kb direct slots; `slot_bins` records their logical bin for the fold.
//
// lanes_kernel (persistent, one CTA per SM): 16 scatter warps stream the plan codes and the
// packed activations (software-pipelined two 8-row groups ahead, L2 bulk prefetch of the next
// unit's codes) into NBUF rotating histograms; one fold warp (mbarrier full / free handshake,
// like the per-vector kernel) reads each finished histogram in slot order, decodes every slot's
// int16 pair, applies the RSR++ pairwise compaction (Alg. 3; or the dense RSR product,
// kernels.py:63-71) lane-locally — each lane owns its two vectors, no cross-lane reduction —
// adds the split slots into their bins' columns and zeroes the buffer.  Slot codes are stored
// as u16 byte offsets (4 * slot) into a TRANSPOSED histogram (lane w's words of all slots form
// one row of an odd number of words, so a warp's 32 words of one slot sit in 32 distinct banks),
// so a reduction's address is one or two integer ops.  If max |V| > vmax (a device flag written by
// lanes_prep_kernel; no host synchronisation) the same kernel runs 32 int32 vectors per pass.
// Results: int32, exact modulo 2^32 (bit-exact whenever the true results fit), equal to the
// per-vector path.
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace rsr {

namespace {

constexpr int kPlanWarps = 16;
constexpr int kLaneWarps = 16;   // scatter warps
constexpr int kLaneFold = 4;     // fold warps (20 warps: 96 registers per thread)
constexpr int kPlanKb = 9;       // plan block width: 2^9 slots x 128 B = 64 KB per histogram
constexpr int kExtraCap = 48;    // slots beyond 2^kb (3 buffers of 560 slots = 210 KB)
constexpr int kVmax = 127;       // packed int16 pairs exact for |v| <= 127 (int8-range activations)
constexpr int kSplitRows = 16384;
constexpr int kMaxNbuf = 3;

__device__ __forceinline__ int find_bucket(const uint32_t* seg, int w, int64_t p) {
  int lo = 0, hi = (1 << w) - 1;  // largest j in [0, 2^w) with seg[j] <= p (seg[0] = 0)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)__ldg(seg + mid) <= p) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void plan_rowkeys_kernel(const rsr_index_desc d, uint16_t* __restrict__ keys) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y, h = blockIdx.z;
  if (p >= d.rows) return;
  const int w = block_width(d.cols, d.k, b);
  const uint32_t* seg = (h ? d.half[1].seg : d.half[0].seg) + (int64_t)b * d.seg_stride;
  const int64_t off = (int64_t)b * d.row_stride + p;
  const void* perm = h ? d.half[1].perm : d.half[0].perm;
  const int64_t row = d.perm_bytes == 2 ? (int64_t)__ldg(reinterpret_cast<const uint16_t*>(perm) + off)
                                        : (int64_t)__ldg(reinterpret_cast<const uint32_t*>(perm) + off);
  keys[((int64_t)h * d.nblocks + b) * d.rows + row] = (uint16_t)find_bucket(seg, w, p);
}

__global__ void plan_keys_kernel(const rsr_index_desc d, const rsr_batch_plan pl, const uint16_t* __restrict__ keys) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int pb = blockIdx.y, h = blockIdx.z;
  if (r >= pl.row_stride) return;
  uint32_t key = 0;
  if (r < d.rows) {
    const int64_t c0 = (int64_t)pb * pl.kb;
    const int wb = (int)std::min<int64_t>(pl.kb, d.cols - c0);
    int bprev = -1;
    uint32_t kk = 0;
    int w = 0;
    for (int i = 0; i < wb; ++i) {
      const int64_t c = c0 + i;
      const int b = (int)(c / d.k), j = (int)(c % d.k);
      if (b != bprev) {
        kk = keys[((int64_t)h * d.nblocks + b) * d.rows + r];
        w = block_width(d.cols, d.k, b);
        bprev = b;
      }
      key |= ((kk >> (w - 1 - j)) & 1u) << (wb - 1 - i);  // MSB-first in both
    }
  }
  pl.codes[((int64_t)h * pl.nblocks + pb) * pl.row_stride + r] = (uint16_t)key;
}

// One CTA per unit (plan block, row split).  Dynamic smem: cnt [halves][16][nbins] u32, then
// nsub [nbins], base [nbins].
__global__ void __launch_bounds__(kPlanWarps * 32) plan_slots_kernel(const rsr_batch_plan pl, int lmax, uint32_t* emax) {
  extern __shared__ uint32_t psm[];
  const int nbins = 1 << pl.kb;  // counter layout; keys of this unit's block are < 2^wb
  uint32_t* cnt = psm;
  uint32_t* nsub = cnt + 2 * kPlanWarps * nbins;
  uint32_t* base = nsub + nbins;
  const int unit = blockIdx.x;
  const int pb = unit / pl.nsplits, q = unit % pl.nsplits;
  const int nbw = 1 << (int)std::min<int64_t>(pl.kb, pl.cols - (int64_t)pb * pl.kb);  // direct slots
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr = pl.split_rows / kPlanWarps;
  const int64_t r0 = (int64_t)q * pl.split_rows + (int64_t)warp * wr;
  for (int i = threadIdx.x; i < 2 * kPlanWarps * nbins; i += blockDim.x) cnt[i] = 0;
  for (int e = threadIdx.x; e < pl.extra_cap; e += blockDim.x) pl.slot_bins[(int64_t)unit * pl.extra_cap + e] = 0;
  __syncthreads();
  for (int h = 0; h < pl.halves; ++h) {
    const uint16_t* c = pl.codes + ((int64_t)h * pl.nblocks + pb) * pl.row_stride + r0;
    for (int i = lane; i < wr; i += 32) atomicAdd(&cnt[(h * kPlanWarps + warp) * nbins + c[i]], 1u);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nbins; j += blockDim.x) {  // exclusive rank prefix in (half, warp) order
    uint32_t run = 0;
    for (int h = 0; h < pl.halves; ++h)
      for (int w = 0; w < kPlanWarps; ++w) {
        uint32_t& x = cnt[(h * kPlanWarps + w) * nbins + j];
        const uint32_t t = x;
        x = run;
        run += t;
      }
    nsub[j] = j == 0 ? 1u : max(1u, (run + lmax - 1) / lmax);
  }
  __syncthreads();
  if (warp == 0) {  // base[j] = 2^wb + exclusive prefix of (nsub - 1): split slots follow the direct ones
    uint32_t carry = 0;
    for (int j0 = 0; j0 < nbins; j0 += 32) {
      const int j = j0 + lane;
      const uint32_t x = j < nbins ? nsub[j] - 1 : 0;
      const uint32_t inc = warp_inclusive_scan(x, lane);
      if (j < nbins) base[j] = (uint32_t)nbw + carry + inc - x;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    // slots beyond 2^kb this unit needs (a narrow last block reuses its unused direct slots)
    if (lane == 0) atomicMax(emax, carry > (uint32_t)pl.extra_cap ? 0xffffu : (uint32_t)max(0, nbw + (int)carry - nbins));
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nbins; j += blockDim.x)
    for (uint32_t t = 1; t < nsub[j]; ++t) {
      const uint32_t e = base[j] - nbw + t - 1;
      if (e < (uint32_t)pl.extra_cap) pl.slot_bins[(int64_t)unit * pl.extra_cap + e] = (uint16_t)j;
    }
  // ranks -> slots, in place (each lane rewrites the codes it read)
  for (int h = 0; h < pl.halves; ++h) {
    uint16_t* c = pl.codes + ((int64_t)h * pl.nblocks + pb) * pl.row_stride + r0;
    uint32_t* wc = cnt + (h * kPlanWarps + warp) * nbins;
    for (int i0 = 0; i0 < wr; i0 += 32) {
      const int i = i0 + lane;
      const uint32_t key = i < wr ? c[i] : 0xffffffffu;
      const uint32_t mask = __match_any_sync(0xffffffffu, key);
      const uint32_t lower = __popc(mask & ((1u << lane) - 1u));
      const uint32_t rank = i < wr ? wc[key] + lower : 0;
      __syncwarp();
      if (i < wr && lower == 0) wc[key] += __popc(mask);
      __syncwarp();
      if (i < wr) {
        const uint32_t s = nsub[key], t = rank % s;
        c[i] = (uint16_t)((t == 0 ? key : base[key] + t - 1) << 2);  // byte offset of the slot in a lane's histogram row
      }
    }
  }
}

// V [batch][rows] int32 -> packed pairs VP [nslice64][row_stride / 4][32] uint4 (word w of a row =
// V[64 s + 2w] + V[64 s + 2w + 1] * 2^16) and int32 lanes VW [2 nslice64][row_stride / 4][32] uint4
// (lane w of slice s = vector 32 s + w); padding rows and vectors are 0.  vmax_seen: max |V|.
__global__ void lanes_prep_kernel(const int32_t* __restrict__ V, int64_t rows, int64_t batch, int64_t row_stride,
                                  int nslice64, uint4* __restrict__ vp, uint4* __restrict__ vw, uint32_t* vmax_seen) {
  const int64_t n4 = row_stride / 4;
  const int64_t total = (int64_t)nslice64 * n4 * 32;
  uint32_t m = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(t & 31);
    const int64_t r4 = (t >> 5) % n4;
    const int s = (int)((t >> 5) / n4);
    const int64_t va = (int64_t)s * 64 + 2 * w, vb = va + 1;
    int32_t a[4], b[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t r = 4 * r4 + e;
      a[e] = (va < batch && r < rows) ? __ldg(V + va * rows + r) : 0;
      b[e] = (vb < batch && r < rows) ? __ldg(V + vb * rows + r) : 0;
      m = max(m, max(a[e] < 0 ? 0u - (uint32_t)a[e] : (uint32_t)a[e], b[e] < 0 ? 0u - (uint32_t)b[e] : (uint32_t)b[e]));
    }
    vp[((int64_t)s * n4 + r4) * 32 + w] =
        make_uint4((uint32_t)a[0] + ((uint32_t)b[0] << 16), (uint32_t)a[1] + ((uint32_t)b[1] << 16),
                   (uint32_t)a[2] + ((uint32_t)b[2] << 16), (uint32_t)a[3] + ((uint32_t)b[3] << 16));
    const int s32 = 2 * s + (w >= 16), l = (2 * w) & 31;
    vw[((int64_t)s32 * n4 + r4) * 32 + l] = make_uint4(a[0], a[1], a[2], a[3]);
    vw[((int64_t)s32 * n4 + r4) * 32 + l + 1] = make_uint4(b[0], b[1], b[2], b[3]);
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(vmax_seen, m);
}

struct LanesParams {
  const uint16_t* codes;
  const uint16_t* slot_bins;
  const uint4* vp;
  const uint4* vw;
  const uint32_t* vmax_seen;
  int32_t* out;
  int64_t cols, row_stride, batch;
  int kb, nblocks, halves, split_rows, nsplits, slots, extra_cap, vmax, nbuf, atomic_out;
};

__device__ __forceinline__ int32_t hi16(int32_t x) {  // high half of a packed pair whose low half is int16
  return (int32_t)((uint32_t)x - (uint32_t)(int32_t)(int16_t)x) >> 16;
}

template <bool FOLDPP, bool TERNARY>
__global__ void __launch_bounds__((kLaneWarps + kLaneFold) * 32, 1) lanes_kernel(const LanesParams p) {
  // 16 scatter warps (16 x 1024 rows of a 16384-row split) + 4 fold warps
  extern __shared__ __align__(128) unsigned char smem[];
  const int NBUF = p.nbuf;
  const int slot_words = p.slots * 32;
  int32_t* hist = reinterpret_cast<int32_t*>(smem);  // [NBUF][slots][32]
  uint64_t* hfull = reinterpret_cast<uint64_t*>(smem + (size_t)NBUF * slot_words * 4);
  uint64_t* hfree = hfull + kMaxNbuf;
  int32_t* fpart = reinterpret_cast<int32_t*>(hfree + kMaxNbuf);  // [2][kLaneFold][2][kPlanKb][32] fold partials
  // per scatter warp: the codes of one 64-row chunk, [4 streams][64 rows] u16, read back with
  // warp-uniform (broadcast) 16-byte loads (tools/microbench/lds_broadcast.cu: 8 codes per 2.24
  // cycles against 2 codes per 1.47 cycles for a shuffle)
  uint16_t* cstage = reinterpret_cast<uint16_t*>(fpart + 2 * kLaneFold * 2 * kPlanKb * 32);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&hfull[b], kLaneWarps);
      mbar_init(&hfree[b], kLaneFold);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < NBUF * slot_words / 4; i += blockDim.x) reinterpret_cast<int4*>(hist)[i] = make_int4(0, 0, 0, 0);
  // the prep kernel (activations, max |V|) must be complete (PDL: the prologue above overlaps it)
  grid_dependency_wait();
  const bool packed = *reinterpret_cast<const volatile uint32_t*>(p.vmax_seen) <= (uint32_t)p.vmax;  // grid-uniform
  const int vper = packed ? 64 : 32;
  const int nslices = (int)((p.batch + vper - 1) / vper);
  const int npass = (p.nblocks + 1) / 2;
  const int nunits = nslices * p.nsplits * npass;
  const int64_t n4 = p.row_stride / 4;
  __syncthreads();
  auto unit_of = [&](int u, int& q, int& pp, int& s) {
    s = u % nslices;
    const int r = u / nslices;
    pp = r % npass;
    q = r / npass;
  };
  // Work items: full units for the whole rounds of the grid, then the remainder units split by
  // rows into `S` parts each, so the last round keeps every CTA busy (1821 plan blocks = 911
  // passes over 148 CTAs would otherwise leave a 7th round on 23 CTAs).  Split items add their
  // columns atomically (the output is zeroed first).
  const int G = gridDim.x;
  const int F = nunits / G, R = nunits - F * G;
  const int S = (R == 0 || F == 0) ? 1 : min(8, max(1, G / R));
  const int nitems = F * G + R * S;
  auto item_of = [&](int i, int& q, int& pp, int& s, int& part, int& nparts) {
    int u = i;
    part = 0;
    nparts = 1;
    if (i >= F * G) {
      const int k = i - F * G;
      u = F * G + k / S;
      part = k % S;
      nparts = S;
    }
    unit_of(u, q, pp, s);
  };
  // scatter warp w of an item: its share of the item's 8-row groups (part `part` of `nparts` of
  // the split's split_rows / 8 groups)
  const int gsplit = p.split_rows / 8;
  auto warp_groups = [&](int part, int nparts, int& g0, int& n) {
    const int p0 = part * gsplit / nparts, p1 = (part + 1) * gsplit / nparts;  // the part's groups
    g0 = p0 + warp * (p1 - p0) / kLaneWarps;
    n = p0 + (warp + 1) * (p1 - p0) / kLaneWarps - g0;
  };

  if (warp < kLaneWarps) {
    // =============================== scatter warps ===============================
    // transposed histogram: lane w's words of every slot form one row of `slots` words (odd), so
    // the 32 lanes of a reduction hit 32 distinct banks whatever the slot
    const uint32_t hs = smem_u32(hist) + (uint32_t)lane * p.slots * 4u;
    int t = 0;  // block sequence number of this CTA (2 per item)
    for (int it = blockIdx.x; it < nitems; it += G, t += 2) {
      int q, pp, s, part, nparts, gw0, ng;
      item_of(it, q, pp, s, part, nparts);
      warp_groups(part, nparts, gw0, ng);
      const int wr = 8 * ng;  // rows of this warp
      const int bA = 2 * pp;
      const bool hasB = bA + 1 < p.nblocks;
      const int bufA = t % NBUF, bufB = (t + 1) % NBUF;
      const int64_t r0 = (int64_t)q * p.split_rows + 8 * (int64_t)gw0;
      // code streams (byte offsets 4 * slot in a lane's histogram row): A+, A-, B+, B-
      const uint16_t* cAp = p.codes + (int64_t)bA * p.row_stride + r0;
      const int64_t hstride = (int64_t)p.nblocks * p.row_stride;
      const uint4* vrow = (packed ? p.vp : p.vw) + ((int64_t)s * n4 + r0 / 4) * 32 + lane;
      // L2 prefetch of the next unit's code rows of this warp (the code stream comes from HBM)
      if (lane == 0 && it + G < nitems) {
        int q2, pp2, s2, part2, nparts2, g02, n2;
        item_of(it + G, q2, pp2, s2, part2, nparts2);
        warp_groups(part2, nparts2, g02, n2);
        const int64_t r02 = (int64_t)q2 * p.split_rows + 8 * (int64_t)g02;
        for (int b = 2 * pp2; b < 2 * pp2 + 2 && b < p.nblocks; ++b)
          for (int h = 0; h < (TERNARY ? 2 : 1); ++h)
            prefetch_l2_bulk(p.codes + (int64_t)h * hstride + (int64_t)b * p.row_stride + r02, (uint32_t)n2 * 16u);
      }
      if (t >= NBUF) mbar_wait(&hfree[bufA], (uint32_t)((t / NBUF) - 1) & 1u);
      if (t + 1 >= NBUF) mbar_wait(&hfree[bufB], (uint32_t)(((t + 1) / NBUF) - 1) & 1u);
      const uint32_t HA = hs + (uint32_t)bufA * slot_words * 4u;
      const uint32_t HB = hs + (uint32_t)bufB * slot_words * 4u;
      auto pass = [&](auto with_b) {
        constexpr bool WB = decltype(with_b)::value;
        constexpr int NC = (TERNARY ? 2 : 1) * (WB ? 2 : 1);  // code streams A+ (A-) (B+ B-)
        // Codes are warp-uniform, so they are loaded lane-distributed — lane l holds 8 codes of
        // stream l / 8 for rows 8 (l % 8) .. + 7 of a 64-row chunk (one coalesced 16-byte load
        // per lane) — and handed out with shuffles, two codes per shuffle: a broadcast load
        // would cost a full data-pipe pass per 16 bytes (tools/microbench/batch_red.cu).
        const int c_l = lane >> 3;
        const uint16_t* cl = cAp + (c_l >= (TERNARY ? 2 : 1) ? p.row_stride : 0) +
                             ((TERNARY && (c_l & 1)) ? hstride : 0) + 8 * (lane & 7);
        const bool c_on = c_l < NC;
        auto load_codes = [&](int ch) -> uint4 {  // chunk ch: groups 8 ch .. 8 ch + 7
          const int g = 8 * ch + (lane & 7);
          return (c_on && g < ng) ? __ldg(reinterpret_cast<const uint4*>(cl + 64 * ch)) : make_uint4(0, 0, 0, 0);
        };
        auto load_v = [&](int g, uint4 (&q)[2]) {
          q[0] = __ldg(vrow + (int64_t)(2 * g) * 32);
          q[1] = __ldg(vrow + (int64_t)(2 * g + 1) * 32);
        };
        const int nch = (ng + 7) / 8;
        uint4 qn = load_codes(0);
        uint4 qv[2][2];
        load_v(0, qv[0]);
        if (ng > 1) load_v(1, qv[1]);
        uint16_t* stg = cstage + warp * (4 * 64);
        const uint32_t stg_s = smem_u32(stg);
        for (int ch = 0; ch < nch; ++ch) {
          const uint4 qc = qn;
          if (ch + 1 < nch) qn = load_codes(ch + 1);
          __syncwarp();  // the previous chunk's broadcast reads are done
          if (c_on) *reinterpret_cast<uint4*>(stg + c_l * 64 + 8 * (lane & 7)) = qc;
          __syncwarp();
#pragma unroll
          for (int gg = 0; gg < 8; ++gg) {
            const int g = 8 * ch + gg;
            if (g >= ng) break;
            const int d = gg & 1;  // v ring: group g in slot g & 1, refilled with group g + 2
            const uint32_t x8[8] = {qv[d][0].x, qv[d][0].y, qv[d][0].z, qv[d][0].w,
                                    qv[d][1].x, qv[d][1].y, qv[d][1].z, qv[d][1].w};
            if (g + 2 < ng) load_v(g + 2, qv[d]);
            uint4 cw[NC];  // this group's 8 codes of every stream (warp-uniform 16-byte loads)
#pragma unroll
            for (int c = 0; c < NC; ++c)
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(cw[c].x), "=r"(cw[c].y), "=r"(cw[c].z), "=r"(cw[c].w)
                           : "r"(stg_s + (uint32_t)(c * 128 + 16 * gg)));
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // rows 2k, 2k + 1 of the group
              uint32_t w[NC];
#pragma unroll
              for (int c = 0; c < NC; ++c) w[c] = k == 0 ? cw[c].x : k == 1 ? cw[c].y : k == 2 ? cw[c].z : cw[c].w;
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int32_t x = (int32_t)x8[2 * k + hh];
                const int32_t nx = -x;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                  const uint32_t off = hh ? (w[c] >> 16) : (w[c] & 0xffffu);
                  const uint32_t H = c >= (TERNARY ? 2 : 1) ? HB : HA;
                  red_add_shared(H + off, (TERNARY && (c & 1)) ? nx : x);
                }
              }
            }
          }
        }
      };
      if (hasB) pass(std::true_type{});
      else pass(std::false_type{});
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&hfull[bufA]);
        mbar_arrive(&hfull[bufB]);
      }
    }
  } else {
    // ================================= fold warps =================================
    // fold warp f takes the 16-slot chunks f, f + 4, ... and the split slots e = f mod 4; the four
    // warps' partial columns are summed in a fixed order by fold warp 0
    const int f = warp - kLaneWarps;
    int t = 0;
    for (int it = blockIdx.x; it < nitems; it += G) {
      int q, pp, s, part, nparts;
      item_of(it, q, pp, s, part, nparts);
      const bool atomic_out = p.nsplits > 1 || nparts > 1;
      for (int half_pass = 0; half_pass < 2; ++half_pass, ++t) {
        const int b = 2 * pp + half_pass;
        const int buf = t % NBUF;
        mbar_wait(&hfull[buf], (uint32_t)(t / NBUF) & 1u);
        if (b >= p.nblocks) {  // a pass with one block: its second buffer stayed clean
          __syncwarp();
          if (lane == 0) mbar_arrive(&hfree[buf]);
          continue;
        }
        int32_t* Hl = hist + (size_t)buf * slot_words + lane * p.slots;  // this lane's histogram row
        const int wb = (int)std::min<int64_t>(p.kb, p.cols - (int64_t)b * p.kb);
        const int nbw = 1 << wb;  // direct slots of this block; split slots follow
        int32_t ax[kPlanKb], ay[kPlanKb];
#pragma unroll
        for (int L = 0; L < kPlanKb; ++L) ax[L] = ay[L] = 0;
        for (int c0 = 16 * f; c0 < nbw; c0 += 16 * kLaneFold) {  // 16 slots at a time, in bin order
          int32_t x[16], y[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int j = c0 + i;
            const bool in = j < nbw;
            x[i] = (in && j != 0) ? Hl[j] : 0;  // logical bin 0 feeds no column
            if (in) Hl[j] = 0;
            y[i] = packed ? hi16(x[i]) : 0;
          }
          if (FOLDPP) {  // pairwise compaction over the 4 bits inside the chunk (Alg. 3)
#pragma unroll
            for (int L = 0; L < 4; ++L) {
              const int cnt = 8 >> L;
              int32_t ox = 0, oy = 0;
#pragma unroll
              for (int tt = 0; tt < 8; ++tt)
                if (tt < cnt) {
                  ox += x[2 * tt + 1];
                  oy += y[2 * tt + 1];
                  x[tt] = x[2 * tt] + x[2 * tt + 1];
                  y[tt] = y[2 * tt] + y[2 * tt + 1];
                }
              ax[L] += ox;
              ay[L] += oy;
            }
            const int ci = c0 >> 4;  // chunk bits: bin bits 4..
#pragma unroll
            for (int L = 4; L < kPlanKb; ++L)
              if ((ci >> (L - 4)) & 1) {
                ax[L] += x[0];
                ay[L] += y[0];
              }
          } else {  // dense product: every bin adds into the columns of its set bits
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int j = c0 + i;
#pragma unroll
              for (int L = 0; L < kPlanKb; ++L)
                if ((j >> L) & 1) {
                  ax[L] += x[i];
                  ay[L] += y[i];
                }
            }
          }
        }
        // split slots (heavy bins): each adds into its bin's columns
        const uint16_t* sb = p.slot_bins + ((int64_t)b * p.nsplits + q) * p.extra_cap;
        for (int e = f; e < p.extra_cap; e += kLaneFold) {
          const int bin = __ldg(sb + e);
          if (!bin) break;  // split slots are listed contiguously
          int32_t* w = Hl + nbw + e;
          const int32_t xv = *w;
          *w = 0;
          const int32_t yv = packed ? hi16(xv) : 0;
#pragma unroll
          for (int L = 0; L < kPlanKb; ++L)
            if ((bin >> L) & 1) {
              ax[L] += xv;
              ay[L] += yv;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&hfree[buf]);  // my part of the buffer read and zeroed
        int32_t* pt = fpart + (t & 1) * (kLaneFold * 2 * kPlanKb * 32);
#pragma unroll
        for (int L = 0; L < kPlanKb; ++L) {
          pt[((f * 2 + 0) * kPlanKb + L) * 32 + lane] = ax[L];
          pt[((f * 2 + 1) * kPlanKb + L) * 32 + lane] = ay[L];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kLaneFold) : "memory");
        if (f != 0) continue;
#pragma unroll
        for (int L = 0; L < kPlanKb; ++L) {
          if (L >= wb) break;
          int32_t sx = 0, sy = 0;
#pragma unroll
          for (int ff = 0; ff < kLaneFold; ++ff) {
            sx += pt[((ff * 2 + 0) * kPlanKb + L) * 32 + lane];
            sy += pt[((ff * 2 + 1) * kPlanKb + L) * 32 + lane];
          }
          const int64_t col = (int64_t)b * p.kb + (wb - 1 - L);  // MSB-first
          if (packed) {
            const int64_t v0 = (int64_t)s * 64 + 2 * lane;
            const int32_t lo = (int32_t)((uint32_t)sx - ((uint32_t)sy << 16));
            if (v0 < p.batch) {
              if (atomic_out) atomicAdd(p.out + v0 * p.cols + col, lo);
              else p.out[v0 * p.cols + col] = lo;
            }
            if (v0 + 1 < p.batch) {
              if (atomic_out) atomicAdd(p.out + (v0 + 1) * p.cols + col, sy);
              else p.out[(v0 + 1) * p.cols + col] = sy;
            }
          } else {
            const int64_t v0 = (int64_t)s * 32 + lane;
            if (v0 < p.batch) {
              if (atomic_out) atomicAdd(p.out + v0 * p.cols + col, sx);
              else p.out[v0 * p.cols + col] = sx;
            }
          }
        }
      }
    }
  }
}

size_t lanes_smem(int slots, int nbuf) {
  return (size_t)nbuf * slots * 128 + 2 * kMaxNbuf * 8 + 2 * (size_t)kLaneFold * 2 * kPlanKb * 32 * 4 +
         (size_t)kLaneWarps * 4 * 64 * 2 /* code staging */;
}

}  // namespace

rsr_status batch_plan_layout(const rsr_index_desc& d, rsr_batch_plan* pl, size_t* code_bytes, size_t* map_bytes,
                             size_t* ws_bytes) {
  std::memset(pl, 0, sizeof(*pl));
  pl->rows = d.rows;
  pl->cols = d.cols;
  pl->kb = kPlanKb;
  pl->nblocks = (int32_t)((d.cols + kPlanKb - 1) / kPlanKb);
  pl->halves = d.halves;
  pl->split_rows = (int32_t)std::min<int64_t>(kSplitRows, (d.rows + 8 * kPlanWarps - 1) / (8 * kPlanWarps) * (8 * kPlanWarps));
  pl->nsplits = (int32_t)((d.rows + pl->split_rows - 1) / pl->split_rows);
  pl->extra_cap = (1 << kPlanKb) + kExtraCap;  // split slots a unit may list (narrow blocks reuse direct slots)
  pl->vmax = kVmax;
  pl->row_stride = (int64_t)pl->nsplits * pl->split_rows;
  if (code_bytes) *code_bytes = (size_t)d.halves * pl->nblocks * pl->row_stride * 2;
  if (map_bytes) *map_bytes = (size_t)pl->nblocks * pl->nsplits * pl->extra_cap * 2;
  // row-order index keys (temporary) + the extra-slot maximum
  if (ws_bytes) *ws_bytes = (((size_t)d.halves * d.nblocks * d.rows * 2 + 255) & ~(size_t)255) + 256;
  if (d.rows >= 65536 * 1024LL) return fail(RSR_ERR_UNSUPPORTED, "batch plan: too many rows");
  return RSR_OK;
}

rsr_status batch_plan_build(const rsr_index_desc& d, rsr_batch_plan* pl, void* ws, size_t ws_bytes, cudaStream_t s) {
  size_t need = 0;
  rsr_batch_plan chk;
  rsr_status st = batch_plan_layout(d, &chk, nullptr, nullptr, &need);
  if (st != RSR_OK) return st;
  if (!ws || ws_bytes < need) return fail(RSR_ERR_INVALID, "batch plan: workspace too small");
  if (!pl->codes || !pl->slot_bins || pl->kb != chk.kb || pl->row_stride != chk.row_stride)
    return fail(RSR_ERR_INVALID, "batch plan: arrays missing or layout does not match the index");
  uint16_t* keys = reinterpret_cast<uint16_t*>(ws);
  uint32_t* emax = reinterpret_cast<uint32_t*>((char*)ws + ((((size_t)d.halves * d.nblocks * d.rows * 2) + 255) & ~(size_t)255));
  if ((st = cuda_check(cudaMemsetAsync(emax, 0, 4, s), "plan memset")) != RSR_OK) return st;
  plan_rowkeys_kernel<<<dim3((unsigned)((d.rows + 255) / 256), (unsigned)d.nblocks, (unsigned)d.halves), 256, 0, s>>>(d, keys);
  if ((st = cuda_check(cudaGetLastError(), "plan_rowkeys_kernel launch")) != RSR_OK) return st;
  plan_keys_kernel<<<dim3((unsigned)((pl->row_stride + 255) / 256), (unsigned)pl->nblocks, (unsigned)d.halves), 256, 0, s>>>(
      d, *pl, keys);
  if ((st = cuda_check(cudaGetLastError(), "plan_keys_kernel launch")) != RSR_OK) return st;
  const size_t psmem = (size_t)(2 * kPlanWarps + 2) * (1u << pl->kb) * 4;
  if ((st = set_max_smem((const void*)plan_slots_kernel, psmem)) != RSR_OK) return st;
  const int lmax = 32767 / pl->vmax;
  plan_slots_kernel<<<(unsigned)(pl->nblocks * pl->nsplits), kPlanWarps * 32, psmem, s>>>(*pl, lmax, emax);
  if ((st = cuda_check(cudaGetLastError(), "plan_slots_kernel launch")) != RSR_OK) return st;
  uint32_t e = 0;
  if ((st = cuda_check(cudaMemcpyAsync(&e, emax, 4, cudaMemcpyDeviceToHost, s), "plan extra copy")) != RSR_OK) return st;
  if ((st = cuda_check(cudaStreamSynchronize(s), "plan sync")) != RSR_OK) return st;
  pl->extra = (int32_t)e;
  if (e > (uint32_t)kExtraCap)
    return fail(RSR_ERR_UNSUPPORTED, "batch plan: a unit needs " + std::to_string(e) + " slots beyond 2^" +
                                         std::to_string(pl->kb) + " (capacity " + std::to_string(kExtraCap) + ")");
  return RSR_OK;
}

size_t batched_plan_workspace_bytes(const rsr_batch_plan& pl, int64_t batch) {
  const int64_t ns64 = std::max<int64_t>(1, (batch + 63) / 64);
  const size_t vp = (size_t)ns64 * pl.row_stride * 128;
  return 256 + vp + 2 * vp;
}

rsr_status multiply_batched_plan(const rsr_index_desc& d, const rsr_batch_plan& pl, const int32_t* V, int64_t batch,
                                 int32_t* out, rsr_variant var, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (batch <= 0) return RSR_OK;
  if (pl.rows != d.rows || pl.cols != d.cols || pl.halves != d.halves || !pl.codes || !pl.slot_bins)
    return fail(RSR_ERR_INVALID, "batch plan does not belong to this index");
  if (pl.extra > kExtraCap || pl.extra < 0) return fail(RSR_ERR_INVALID, "batch plan not built");
  if (!ws || ws_bytes < batched_plan_workspace_bytes(pl, batch) || ((uintptr_t)ws & 255))
    return fail(RSR_ERR_INVALID, "batched plan multiply: workspace too small or misaligned");
  const int ns64 = (int)((batch + 63) / 64);
  uint32_t* vmax_seen = reinterpret_cast<uint32_t*>(ws);
  uint4* vp = reinterpret_cast<uint4*>((char*)ws + 256);
  uint4* vw = vp + (size_t)ns64 * pl.row_stride * 8;
  rsr_status st = cuda_check(cudaMemsetAsync(vmax_seen, 0, 4, s), "memset vmax");
  if (st != RSR_OK) return st;
  const int sms = device_sm_count();
  const int64_t prep_threads = (int64_t)ns64 * (pl.row_stride / 4) * 32;
  lanes_prep_kernel<<<(unsigned)std::min<int64_t>(8 * sms, (prep_threads + 255) / 256), 256, 0, s>>>(
      V, d.rows, batch, pl.row_stride, ns64, vp, vw, vmax_seen);
  if ((st = cuda_check(cudaGetLastError(), "lanes_prep_kernel launch")) != RSR_OK) return st;
  LanesParams p{};
  p.codes = pl.codes;
  p.slot_bins = pl.slot_bins;
  p.vp = vp;
  p.vw = vw;
  p.vmax_seen = vmax_seen;
  p.out = out;
  p.cols = d.cols;
  p.row_stride = pl.row_stride;
  p.batch = batch;
  p.kb = pl.kb;
  p.nblocks = pl.nblocks;
  p.halves = pl.halves;
  p.split_rows = pl.split_rows;
  p.nsplits = pl.nsplits;
  p.slots = ((1 << pl.kb) + pl.extra) | 1;  // odd row length: conflict-free transposed histogram
  p.extra_cap = pl.extra_cap;

  p.vmax = pl.vmax;
  p.atomic_out = pl.nsplits > 1;
  const size_t max_smem = device_max_smem_optin();
  p.nbuf = lanes_smem(p.slots, 3) <= max_smem ? 3 : 2;
  const size_t smem = lanes_smem(p.slots, p.nbuf);
  if (smem > max_smem) return fail(RSR_ERR_UNSUPPORTED, "batched plan multiply: histograms do not fit");
  // outputs of row-split items are added atomically: start from zero (4 bytes per result)
  if ((st = cuda_check(cudaMemsetAsync(out, 0, (size_t)batch * d.cols * 4, s), "memset out")) != RSR_OK) return st;
  const bool pp = var == RSR_VARIANT_RSRPP;
  auto kern = d.halves == 2 ? (pp ? lanes_kernel<true, true> : lanes_kernel<false, true>)
                            : (pp ? lanes_kernel<true, false> : lanes_kernel<false, false>);
  if ((st = set_max_smem((const void*)kern, smem)) != RSR_OK) return st;
  // units: an upper bound (the int32-lane form has twice the slices); idle CTAs exit at once
  const int64_t units = (int64_t)((batch + 31) / 32) * pl.nsplits * ((pl.nblocks + 1) / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(sms, units)));
  cfg.blockDim = dim3((kLaneWarps + kLaneFold) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, kern, p), "lanes_kernel launch");
}

}  // namespace rsr
