// GPU preprocessing: ternary/binary matrix -> per-block keys -> stable counting
// sort (perm) + cumulative segmentation (seg).
//
// Reference algorithm (indexer.py:251-286, core.py:124-128):
//   for each half (A == +1, A == -1) and each column block of width w:
//     key(r)  = MSB-first bits of row r inside the block            (indexer.py:215-219)
//     perm    = np.argsort(key, kind="stable")                       (indexer.py:269)
//     seg     = [0, cumsum(bincount(key, minlength=2^w))]            (indexer.py:274-276)
// B200 design: one kernel turns the int8 matrix into both halves' keys for all
// blocks (smem-tiled so global reads and key writes are coalesced); a second
// kernel gives each (half, block) to one warp, which builds the histogram in a
// warp-private shared-memory counter array, scans it into `seg`, and then walks
// the rows in ascending order 32 at a time, ranking equal keys with
// __match_any_sync so the scatter into `perm` is stable by construction.
#include <cstdlib>

#include "common.cuh"

namespace rsr {

namespace {

constexpr int kKeyRowsPerTile = 64;
constexpr int kKeyThreads = 256;
constexpr int kKeyTileBytes = 512;  // max columns per tile

// Grid: x = row tiles, y = block tiles.  Each block tile holds `bt` column blocks.
__global__ void __launch_bounds__(kKeyThreads) keys_ternary_kernel(const int8_t* __restrict__ A, int64_t lda,
                                                                     int64_t rows, int64_t cols, int k, int bt,
                                                                     int64_t row_stride, uint16_t* __restrict__ kpos,
                                                                     uint16_t* __restrict__ kneg,
                                                                     int32_t* __restrict__ bad) {
  // Row pitch: an odd number of 4-byte words keeps the per-lane row accesses on distinct banks.
  __shared__ int8_t tile[kKeyRowsPerTile * (kKeyTileBytes + 4)];
  const int pitch = kKeyTileBytes + 4;
  const int64_t r0 = (int64_t)blockIdx.x * kKeyRowsPerTile;
  const int b0 = blockIdx.y * bt;
  const int64_t c0 = (int64_t)b0 * k;
  const int tw = (int)std::min<int64_t>((int64_t)bt * k, cols - c0);
  const int nr = (int)std::min<int64_t>(kKeyRowsPerTile, rows - r0);
  int nbad = 0;
  for (int idx = threadIdx.x; idx < nr * tw; idx += kKeyThreads) {
    int r = idx / tw, c = idx - r * tw;
    int8_t x = A[(r0 + r) * lda + c0 + c];
    nbad += (x < -1 || x > 1);
    tile[r * pitch + c] = x;
  }
  if (nbad) atomicAdd(bad, nbad);
  __syncthreads();
  const int nblk = (tw + k - 1) / k;
  for (int p = threadIdx.x; p < kKeyRowsPerTile * nblk; p += kKeyThreads) {
    int r = p % kKeyRowsPerTile, bl = p / kKeyRowsPerTile;
    if (r >= nr) continue;
    int w = min(k, tw - bl * k);
    const int8_t* src = tile + r * pitch + bl * k;
    unsigned kp = 0, kn = 0;
    for (int c = 0; c < w; ++c) {
      int8_t x = src[c];
      kp = (kp << 1) | (unsigned)(x == 1);
      kn = (kn << 1) | (unsigned)(x == -1);
    }
    int64_t o = (int64_t)(b0 + bl) * row_stride + r0 + r;
    kpos[o] = (uint16_t)encode_key(kp, k);
    kneg[o] = (uint16_t)encode_key(kn, k);
  }
}

// BinaryMatrix bits (core.py:53-99): row-major bytes, MSB-first within a byte.
__global__ void keys_binary_kernel(const uint8_t* __restrict__ bits, int64_t ldb, int64_t rows, int64_t cols, int k,
                                   int nblocks, int64_t row_stride, uint16_t* __restrict__ keys) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint8_t* row = bits + r * ldb;
  for (int b = blockIdx.y; b < nblocks; b += gridDim.y) {
    int w = block_width(cols, k, b);
    int64_t c0 = (int64_t)b * k;
    unsigned key = 0;
    for (int c = 0; c < w; ++c) {
      int64_t cc = c0 + c;
      key = (key << 1) | ((row[cc >> 3] >> (7 - (cc & 7))) & 1u);
    }
    keys[(int64_t)b * row_stride + r] = (uint16_t)encode_key(key, k);
  }
}

// One warp per (half, block): histogram -> exclusive scan (seg) -> stable ranked scatter (perm).
template <typename PermT>
__global__ void sort_blocks_kernel(rsr_index_desc d, uint32_t* __restrict__ gcnt, int use_smem, int warps_per_cta) {
  extern __shared__ uint32_t scnt[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t unit = (int64_t)blockIdx.x * warps_per_cta + wib;  // (half, block)
  const int64_t nunits = (int64_t)d.halves * d.nblocks;
  if (unit >= nunits) return;
  const int h = (int)(unit / d.nblocks);
  const int b = (int)(unit % d.nblocks);
  const int w = block_width(d.cols, d.k, b);
  const int nbk = 1 << w;
  uint32_t* cnt = use_smem ? scnt + ((size_t)wib << d.k) : gcnt + ((size_t)unit << d.k);
  const uint16_t* key = d.half[h].bucket + (int64_t)b * d.row_stride;
  uint32_t* seg = d.half[h].seg + (int64_t)b * d.seg_stride;
  PermT* perm = reinterpret_cast<PermT*>(d.half[h].perm) + (int64_t)b * d.row_stride;
  const int64_t rows = d.rows;

  for (int j = lane; j < nbk; j += 32) cnt[j] = 0;
  __syncwarp();
  for (int64_t r = lane; r < rows; r += 32) atomicAdd(&cnt[decode_key(key[r], d.k)], 1u);
  __syncwarp();
  // Exclusive scan of cnt[0..nbk): lane owns a contiguous chunk.
  const int chunk = (nbk + 31) / 32;
  const int j0 = min(nbk, lane * chunk), j1 = min(nbk, j0 + chunk);
  uint32_t local = 0;
  for (int j = j0; j < j1; ++j) local += cnt[j];
  uint32_t incl = warp_inclusive_scan(local, lane);
  uint32_t run = incl - local;
  for (int j = j0; j < j1; ++j) {
    uint32_t c = cnt[j];
    seg[j] = run;
    cnt[j] = run;  // becomes the per-key write cursor
    run += c;
  }
  for (int64_t j = nbk + lane; j < d.seg_stride; j += 32) seg[j] = (uint32_t)rows;  // sentinel (+ unused tail)
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t r0 = 0; r0 < rows; r0 += 32) {
    const int64_t r = r0 + lane;
    const bool active = r < rows;
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (active) {
      const unsigned kk = decode_key(key[r], d.k);
      const unsigned peers = __match_any_sync(act, kk);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == leader) {
        base = cnt[kk];
        cnt[kk] = base + __popc(peers);
      }
      base = __shfl_sync(act, base, leader);
      perm[base + __popc(peers & lt)] = (PermT)r;
    }
    __syncwarp();
  }
}

rsr_status launch_sort(const rsr_index_desc& d, void* workspace, size_t ws_bytes, cudaStream_t s) {
  const size_t per_warp = sizeof(uint32_t) << d.k;
  const int64_t nunits = (int64_t)d.halves * d.nblocks;
  int wpc = (int)std::min<size_t>(8, (160u << 10) / per_warp);
  const bool use_smem = wpc >= 1;
  if (!use_smem) {
    wpc = 8;
    if (ws_bytes < per_warp * (size_t)nunits) return fail(RSR_ERR_INVALID, "preprocess workspace too small");
  }
  const size_t smem = use_smem ? per_warp * wpc : 0;
  const unsigned grid = (unsigned)((nunits + wpc - 1) / wpc);
  if (d.perm_bytes == 2) {
    auto kern = sort_blocks_kernel<uint16_t>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * wpc, smem, s>>>(d, (uint32_t*)workspace, use_smem, wpc);
  } else {
    auto kern = sort_blocks_kernel<uint32_t>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * wpc, smem, s>>>(d, (uint32_t*)workspace, use_smem, wpc);
  }
  return cuda_check(cudaGetLastError(), "sort_blocks_kernel launch");
}

// ---------------------------------------------------------------------------------------
// Key-order scheduling for the scatter kernel's shared-memory reductions (k <= 13).
// The scatter kernel issues one reduction instruction per (8-row group, slot s) with lane l
// handling one row of its group 256c + 8l + [0, 8) of 256-row chunk c; the cost of an
// instruction is the number of bank wavefronts = the largest number of lanes that hit one
// bank.  A lane may process its 8 rows in any order reachable by a 3-stage butterfly with 12
// independent switches (common.cuh butterfly8; 4096 orders, shared by both halves).  One warp
// per (block, chunk) picks every lane's 12 control bits by coordinate descent: lanes take
// turns; for the active lane, 12 lanes each evaluate one switch flip against the other lanes'
// bank counts (cost sum of c(c+1) over the slots' banks, i.e. the growth of sum c^3, which
// penalises the maximum), the best improving flip is applied, until none improves.  Codes are
// stored in slot order with the control bits in bits 13-15 of codes 0..3.  Simulated on
// uniform ternary keys: 3.66 wavefronts per reduction in row order, 2.77 with a per-lane XOR
// order, 2.26 with this butterfly schedule.  Results are unchanged (integer sums are
// order-free).
constexpr int kSchedWarps = 8;

__global__ void __launch_bounds__(kSchedWarps * 32) schedule_keys_kernel(rsr_index_desc d, int sweeps) {
  __shared__ int cnt_all[kSchedWarps][2][8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nchunks = d.row_stride / 256;  // only whole 256-row chunks are scheduled
  const int64_t task = (int64_t)blockIdx.x * kSchedWarps + wib;
  if (task >= (int64_t)d.nblocks * nchunks) return;
  const int b = (int)(task / nchunks);
  const int64_t c = task % nchunks;
  int (*cnt)[8][32] = cnt_all[wib];
  const int H = d.halves;
  const int cs = code_shift(d.k);  // code -> histogram word index: code >> cs
  uint16_t* code[2] = {nullptr, nullptr};
  uint32_t kc[2][8] = {};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h >= H) break;
    code[h] = d.half[h].bucket + (int64_t)b * d.row_stride + c * 256 + 8 * lane;
    const uint4 q = *reinterpret_cast<const uint4*>(code[h]);
    const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      kc[h][2 * e] = w4[e] & 0xffffu;
      kc[h][2 * e + 1] = w4[e] >> 16;
    }
  }
  for (int i = lane; i < 2 * 8 * 32; i += 32) (&cnt[0][0][0])[i] = 0;
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (h < H) atomicAdd(&cnt[h][e][(kc[h][e] >> cs) & 31], 1);
  __syncwarp();
  uint32_t ctrl = 0;  // this lane's switches
  for (int sweep = 0; sweep < sweeps; ++sweep) {
    for (int l = 0; l < 32; ++l) {
      uint32_t bk[2][8];  // lane l's banks in row order, broadcast
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 8; ++e) bk[h][e] = __shfl_sync(0xffffffffu, (kc[h][e] >> cs) & 31, l);
      uint32_t cur = __shfl_sync(0xffffffffu, ctrl, l);
      auto slot_banks = [&](uint32_t cc, uint32_t (&sb)[2][8]) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int e = 0; e < 8; ++e) sb[h][e] = bk[h][e];
          butterfly8(sb[h], cc);
        }
      };
      if (lane == l) {  // take lane l out of the counts
        uint32_t sb[2][8];
        slot_banks(cur, sb);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2)
            if (h < H) cnt[h][s2][sb[h][s2]] -= 1;
      }
      __syncwarp();
      for (int round = 0; round < 12; ++round) {
        // lane j < 12 evaluates flipping switch j, lane 12 the current order
        int cost = 0x7fffffff;
        if (lane <= 12) {
          const uint32_t cc = lane < 12 ? cur ^ (1u << lane) : cur;
          uint32_t sb[2][8];
          slot_banks(cc, sb);
          int cst = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2)
              if (h < H) {
                const int n = cnt[h][s2][sb[h][s2]];
                cst += n * (n + 1);
              }
          cost = cst * 16 + (lane < 12 ? lane + 1 : 0);  // ties keep the current order
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cost = min(cost, __shfl_xor_sync(0xffffffffu, cost, o));
        const int pick = cost & 15;
        if (pick == 0) break;
        cur ^= 1u << (pick - 1);
      }
      if (lane == l) {  // put lane l back with its new order
        ctrl = cur;
        uint32_t sb[2][8];
        slot_banks(cur, sb);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2)
            if (h < H) cnt[h][s2][sb[h][s2]] += 1;
      }
      __syncwarp();
    }
  }
  // write the codes in slot order with the control bits in codes 0..3
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h >= H) break;
    uint32_t o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = kc[h][e];
    butterfly8(o, ctrl);
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) o[s2] |= ((ctrl >> (3 * s2)) & 7u) << 13;
    *reinterpret_cast<uint4*>(code[h]) =
        make_uint4(o[0] | (o[1] << 16), o[2] | (o[3] << 16), o[4] | (o[5] << 16), o[6] | (o[7] << 16));
  }
}

rsr_status launch_schedule(const rsr_index_desc& d, cudaStream_t s) {
  if (!sched_keys(d.k)) return RSR_OK;  // no spare code bits: keys stay in row order
  if (const char* e = getenv("RSR_B200_NOSCHED"))
    if (e[0] == '1') return RSR_OK;  // diagnostics
  const int64_t tasks = (int64_t)d.nblocks * (d.row_stride / 256);
  if (tasks == 0) return RSR_OK;
  const unsigned grid = (unsigned)((tasks + kSchedWarps - 1) / kSchedWarps);
  static const int env_sweeps = getenv("RSR_B200_SCHED_SWEEPS") ? atoi(getenv("RSR_B200_SCHED_SWEEPS")) : -1;
  schedule_keys_kernel<<<grid, kSchedWarps * 32, 0, s>>>(d, env_sweeps > 0 ? env_sweeps : 4);  // 4 sweeps: 2.277 -> 2.258 wavefronts per reduction (converged)
  return cuda_check(cudaGetLastError(), "schedule_keys_kernel launch");
}

// ---------------------------------------------------------------------------------------
// Import of a stored index (`.rsx`, store.py:49-101): per block a u32 permutation and 2^w
// u32 segment starts.  One warp per (half, block) validates the invariants the reference's
// RsrIndex.from_blocks checks (indexer.py:89-129) — permutation a bijection (a seen-bitmap
// with atomicOr), segmentation starting at 0, non-decreasing, <= rows — writes our layout
// (u16/u32 perm, u32 seg + sentinel) and rebuilds every row's key code from the segments on
// the device (lane j walks bucket j), replacing the host-side `_buckets_from_segments`
// (indexer.py:176-186).  err[0] |= flags, err[1] = min failing block.
enum : int { kImpPermRange = 1, kImpPermDup = 2, kImpSeg0 = 4, kImpSegOrder = 8 };

__global__ void import_blocks_kernel(rsr_index_desc d, int h, const uint32_t* __restrict__ perm_in,
                                     const uint32_t* __restrict__ seg_in, int64_t seg_in_stride,
                                     uint32_t* __restrict__ seen, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= d.nblocks) return;
  const int w = block_width(d.cols, d.k, b);
  const int nbk = 1 << w;
  const int64_t rows = d.rows;
  const uint32_t* pin = perm_in + (int64_t)b * rows;
  const uint32_t* sin = seg_in + (int64_t)b * seg_in_stride;
  uint32_t* seg = d.half[h].seg + (int64_t)b * d.seg_stride;
  uint16_t* key = d.half[h].bucket + (int64_t)b * d.row_stride;
  uint32_t* my_seen = seen + (int64_t)b * ((rows + 31) / 32);
  int flags = 0;
  for (int j = lane; j < nbk; j += 32) {
    const uint32_t sj = sin[j];
    if (j == 0 && sj != 0) flags |= kImpSeg0;
    if ((j > 0 && sin[j - 1] > sj) || sj > (uint64_t)rows) flags |= kImpSegOrder;
    seg[j] = sj;
  }
  for (int64_t j = nbk + lane; j < d.seg_stride; j += 32) seg[j] = (uint32_t)rows;  // sentinel (+ unused tail)
  for (int64_t p = lane; p < rows; p += 32) {
    const uint32_t r = pin[p];
    if (r >= rows) {
      flags |= kImpPermRange;
      continue;
    }
    if (d.perm_bytes == 2) reinterpret_cast<uint16_t*>(d.half[h].perm)[(int64_t)b * d.row_stride + p] = (uint16_t)r;
    else reinterpret_cast<uint32_t*>(d.half[h].perm)[(int64_t)b * d.row_stride + p] = r;
    const uint32_t bit = 1u << (r & 31);
    if (atomicOr(&my_seen[r >> 5], bit) & bit) flags |= kImpPermDup;
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (flags) {  // do not walk a broken segmentation
    if (lane == 0) {
      atomicOr(&err[0], flags);
      atomicMin(&err[1], b);
    }
    return;
  }
  // key codes: rows of bucket j are pin[sin[j] .. sin[j+1])
  for (int j = lane; j < nbk; j += 32) {
    const uint32_t e = j + 1 < nbk ? sin[j + 1] : (uint32_t)rows;
    const uint16_t code = (uint16_t)encode_key((uint32_t)j, d.k);
    for (uint32_t q = sin[j]; q < e; ++q) key[pin[q]] = code;
  }
}

rsr_status clear_index(const rsr_index_desc& d, cudaStream_t s) {
  for (int h = 0; h < d.halves; ++h) {
    size_t nb = (size_t)d.nblocks * d.row_stride;
    rsr_status st = cuda_check(cudaMemsetAsync(d.half[h].bucket, 0, nb * 2, s), "memset bucket");
    if (st != RSR_OK) return st;
    st = cuda_check(cudaMemsetAsync(d.half[h].perm, 0, nb * d.perm_bytes, s), "memset perm");
    if (st != RSR_OK) return st;
  }
  return RSR_OK;
}

rsr_status check_desc(const rsr_index_desc* d) {
  if (!d) return fail(RSR_ERR_INVALID, "null index descriptor");
  if (d->rows < 1 || d->cols < 1) return fail(RSR_ERR_INVALID, "index dimensions must be at least 1x1");
  if (d->k < 1 || d->k > kMaxDeviceK) return fail(RSR_ERR_UNSUPPORTED, "k exceeds the device limit of 16");
  for (int h = 0; h < d->halves; ++h)
    if (!d->half[h].perm || !d->half[h].seg || !d->half[h].bucket)
      return fail(RSR_ERR_INVALID, "index descriptor has null arrays");
  return RSR_OK;
}

}  // namespace

size_t preprocess_workspace_bytes(const rsr_index_desc* d) {
  const size_t per_warp = sizeof(uint32_t) << d->k;
  if ((160u << 10) / per_warp >= 1) return 0;
  return per_warp * (size_t)d->halves * d->nblocks;
}

rsr_status preprocess_ternary(const int8_t* A, int64_t lda, const rsr_index_desc* d, int32_t* bad, void* ws,
                              size_t ws_bytes, cudaStream_t s) {
  rsr_status st = check_desc(d);
  if (st != RSR_OK) return st;
  if (d->halves != 2) return fail(RSR_ERR_INVALID, "ternary preprocess needs a two-half index");
  if (!A || !bad || lda < d->cols) return fail(RSR_ERR_INVALID, "bad ternary matrix arguments");
  if ((st = clear_index(*d, s)) != RSR_OK) return st;
  const int bt = std::max(1, kKeyTileBytes / d->k);
  dim3 grid((unsigned)((d->rows + kKeyRowsPerTile - 1) / kKeyRowsPerTile), (unsigned)((d->nblocks + bt - 1) / bt));
  keys_ternary_kernel<<<grid, kKeyThreads, 0, s>>>(A, lda, d->rows, d->cols, d->k, bt, d->row_stride,
                                                   d->half[0].bucket, d->half[1].bucket, bad);
  if ((st = cuda_check(cudaGetLastError(), "keys_ternary_kernel launch")) != RSR_OK) return st;
  if ((st = launch_sort(*d, ws, ws_bytes, s)) != RSR_OK) return st;
  return launch_schedule(*d, s);
}

rsr_status preprocess_binary(const uint8_t* bits, int64_t ldb, const rsr_index_desc* d, void* ws, size_t ws_bytes,
                             cudaStream_t s) {
  rsr_status st = check_desc(d);
  if (st != RSR_OK) return st;
  if (d->halves != 1) return fail(RSR_ERR_INVALID, "binary preprocess needs a one-half index");
  if (!bits || ldb < (d->cols + 7) / 8) return fail(RSR_ERR_INVALID, "bad binary matrix arguments");
  if ((st = clear_index(*d, s)) != RSR_OK) return st;
  dim3 grid((unsigned)((d->rows + 255) / 256), (unsigned)std::min(d->nblocks, 65535));
  keys_binary_kernel<<<grid, 256, 0, s>>>(bits, ldb, d->rows, d->cols, d->k, d->nblocks, d->row_stride,
                                          d->half[0].bucket);
  if ((st = cuda_check(cudaGetLastError(), "keys_binary_kernel launch")) != RSR_OK) return st;
  if ((st = launch_sort(*d, ws, ws_bytes, s)) != RSR_OK) return st;
  return launch_schedule(*d, s);
}

size_t index_import_workspace_bytes(const rsr_index_desc* d) {
  return d ? (size_t)d->halves * d->nblocks * (size_t)((d->rows + 31) / 32) * 4 : 0;
}

rsr_status index_import(const rsr_index_desc* d, const uint32_t* perm0, const uint32_t* seg0, const uint32_t* perm1,
                        const uint32_t* seg1, int64_t seg_in_stride, void* ws, size_t ws_bytes, int32_t* err,
                        cudaStream_t s) {
  rsr_status st = check_desc(d);
  if (st != RSR_OK) return st;
  if (!perm0 || !seg0 || (d->halves == 2 && (!perm1 || !seg1)) || !err)
    return fail(RSR_ERR_INVALID, "null import arrays");
  if (seg_in_stride < ((int64_t)1 << d->k)) return fail(RSR_ERR_INVALID, "segment stride must be >= 2^k");
  if (!ws || ws_bytes < index_import_workspace_bytes(d)) return fail(RSR_ERR_INVALID, "import workspace too small");
  if ((st = clear_index(*d, s)) != RSR_OK) return st;
  if ((st = cuda_check(cudaMemsetAsync(ws, 0, index_import_workspace_bytes(d), s), "memset import bitmap")) != RSR_OK)
    return st;
  const int wpc = 8;
  const unsigned grid = (unsigned)((d->nblocks + wpc - 1) / wpc);
  const size_t half_words = (size_t)d->nblocks * ((d->rows + 31) / 32);
  for (int h = 0; h < d->halves; ++h) {
    import_blocks_kernel<<<grid, 32 * wpc, 0, s>>>(*d, h, h ? perm1 : perm0, h ? seg1 : seg0, seg_in_stride,
                                                    (uint32_t*)ws + h * half_words, err);
    if ((st = cuda_check(cudaGetLastError(), "import_blocks_kernel launch")) != RSR_OK) return st;
  }
  return launch_schedule(*d, s);
}

}  // namespace rsr
