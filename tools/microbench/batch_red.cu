// Microbenchmark for a batch-native RSR scatter (BASELINE config 3, B = 64): lanes span the
// vector dimension (lane w owns the packed int16 pair of vectors 2w, 2w+1), so each
// reduction instruction adds one row's 64 activations into the 32 consecutive words of ONE
// histogram slot (conflict-free).  Per pass a CTA streams the packed activations of its 16384
// rows once (VP [rows/4][32][4] u32, L2-resident) and applies each row to P column blocks x 2
// halves (4 reductions for P = 2).  Slot codes are synthetic and uniform over NSLOT slots.
//   mode 0: u16 slot codes, broadcast 16-byte loads (2 rows x 4 codes), extracted in registers
//   mode 1: u32 byte-offset codes (4 per row, one broadcast 16-byte load per row)
//   mode 2: mode 0 without the activation loads (registers only): the RED + code path alone
//   mode 3: mode 0 without the reductions: the load path alone
//   mode 4: reductions only (addresses from a register hash, conflict-free 32-word rows)
//   mode 5: reductions only, 32 random words (the B = 1 kernel's access pattern)
//   mode 7: mode 0 software-pipelined (codes and v one group ahead, L2 bulk prefetch of codes)
//   mode 8: mode 7 without the activation loads
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_s(uint32_t a, int v) { asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

constexpr int WARPS = 16, ROWS = 16384, P = 2, NSLOT = 528;

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) kern(const uint4* __restrict__ vp, const void* __restrict__ codes,
                                                       int passes, int* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  int* hist = reinterpret_cast<int*>(smem);  // [3][NSLOT][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 3 * NSLOT * 32; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const uint32_t hs = su32(hist) + lane * 4;
  const int r0 = warp * (ROWS / WARPS);
  int acc = 0;
  for (int u = 0; u < passes; ++u) {
    const int pass = blockIdx.x + u * gridDim.x;
    const uint32_t hbase[P] = {hs + (uint32_t)((2 * u) % 3) * NSLOT * 128, hs + (uint32_t)((2 * u + 1) % 3) * NSLOT * 128};
    if (MODE == 9 || MODE == 10) {
      // codes lane-distributed (lane l: stream l / 8, rows 64 u + 8 (l % 8) .. + 7 as 8 u16 = one
      // coalesced 16-byte load per lane per 64 rows) and handed to the warp with SHFL (two codes
      // per shuffle); transposed histogram (odd row of NSLOT_T words per lane), codes = 4 * slot
      constexpr int NT = NSLOT | 1;
      const uint32_t hl = su32(hist) + (uint32_t)lane * NT * 4u;
      const uint32_t hA = hl + (uint32_t)((2 * u) % 3) * NT * 128u, hB = hl + (uint32_t)((2 * u + 1) % 3) * NT * 128u;
      const uint16_t* cb = reinterpret_cast<const uint16_t*>(codes) + ((size_t)pass * ROWS + r0) * 4;
      const uint4* vb0 = vp + (size_t)(r0 / 4) * 32 + lane;
      const int nchunks = ROWS / WARPS / 64;
      uint4 qn = ldg_nc(reinterpret_cast<const uint4*>(cb) + lane);  // chunk 0 (stream-major 4 x 64 rows)
      for (int ch = 0; ch < nchunks; ++ch) {
        const uint4 qc = qn;
        if (ch + 1 < nchunks) qn = ldg_nc(reinterpret_cast<const uint4*>(cb) + (ch + 1) * 32 + lane);
        uint4 va[2], vb[2];
        va[0] = __ldg(vb0 + (size_t)(16 * ch) * 32);
        va[1] = __ldg(vb0 + (size_t)(16 * ch + 1) * 32);
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          if (g + 1 < 8) {
            vb[0] = __ldg(vb0 + (size_t)(16 * ch + 2 * g + 2) * 32);
            vb[1] = __ldg(vb0 + (size_t)(16 * ch + 2 * g + 3) * 32);
          }
          const uint32_t x8[8] = {va[0].x, va[0].y, va[0].z, va[0].w, va[1].x, va[1].y, va[1].z, va[1].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // row pair (2k, 2k + 1) of group g
            const uint32_t src = k == 0 ? qc.x : k == 1 ? qc.y : k == 2 ? qc.z : qc.w;
            uint32_t w[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) w[c] = MODE == 9 ? __shfl_sync(0xffffffffu, src, c * 8 + g) : src;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int x = (int)x8[2 * k + h];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const uint32_t off = h ? (w[c] >> 16) : (w[c] & 0xffffu);
                red_s((c < 2 ? hA : hB) + off, (c & 1) ? -x : x);
              }
            }
          }
          va[0] = vb[0];
          va[1] = vb[1];
        }
      }
      continue;
    }
    if (MODE >= 4) {
      // 16 precomputed addresses per lane, cycled: conflict-free rows (mode 4), random words
      // (mode 5: ~3.5-way worst bank per instruction), or one bank per instruction (mode 6)
      uint32_t ad[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        uint32_t x = (uint32_t)(blockIdx.x * 7919 + warp * 104729 + q * 31337 + u) * 2654435761u;
        if (MODE == 4) ad[q] = hbase[q & 1] + (((x >> 8) % NSLOT) << 7);
        else if (MODE == 11)  // transposed: lane w's words of all slots form one odd-length row
          ad[q] = (hbase[q & 1] - lane * 4) + (uint32_t)lane * (NSLOT | 1) * 4 + ((x >> 8) % NSLOT) * 4;
        else if (MODE == 5) ad[q] = (hbase[q & 1] - lane * 4) + ((((x >> 3) ^ (lane * 2246822519u)) >> 7) % (NSLOT * 32)) * 4;
        else ad[q] = hbase[q & 1];
      }
      for (int r = r0; r < r0 + ROWS / WARPS; r += 4) {
#pragma unroll
        for (int q = 0; q < 16; ++q) red_s(ad[q], r + q);
      }
      continue;
    }
    if (MODE == 7 || MODE == 8) {
      const uint16_t* cb = reinterpret_cast<const uint16_t*>(codes) + ((size_t)pass * ROWS + r0) * 4;
      const uint4* vb0 = vp + (size_t)(r0 / 4) * 32 + lane;
      constexpr int D = 2;  // groups in flight
      uint4 qc[D][4], qv[D][2];
      if (lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cb), "r"((uint32_t)(ROWS / WARPS) * 8) : "memory");
#pragma unroll
      for (int d = 0; d < D; ++d) {
#pragma unroll
        for (int i = 0; i < 4; ++i) qc[d][i] = ldg_nc(cb + d * 32 + 8 * i);
        qv[d][0] = ldg_nc(vb0 + (2 * d) * 32);
        qv[d][1] = ldg_nc(vb0 + (2 * d + 1) * 32);
      }
      const int ng = ROWS / WARPS / 8;
      for (int g = 0; g < ng; g += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const uint32_t v8[8] = {qv[d][0].x, qv[d][0].y, qv[d][0].z, qv[d][0].w, qv[d][1].x, qv[d][1].y, qv[d][1].z, qv[d][1].w};
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) { w[4 * i] = qc[d][i].x; w[4 * i + 1] = qc[d][i].y; w[4 * i + 2] = qc[d][i].z; w[4 * i + 3] = qc[d][i].w; }
          const int gn = g + d + D < ng ? g + d + D : g + d;
#pragma unroll
          for (int i = 0; i < 4; ++i) qc[d][i] = ldg_nc(cb + gn * 32 + 8 * i);
          if (MODE == 7) {
            qv[d][0] = ldg_nc(vb0 + (2 * gn) * 32);
            qv[d][1] = ldg_nc(vb0 + (2 * gn + 1) * 32);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int x = (int)v8[e];
            const uint32_t a0 = w[2 * e] & 0xffffu, a1 = w[2 * e] >> 16, a2 = w[2 * e + 1] & 0xffffu, a3 = w[2 * e + 1] >> 16;
            red_s(hbase[0] + (a0 << 7), x);
            red_s(hbase[0] + (a1 << 7), -x);
            red_s(hbase[1] + (a2 << 7), x);
            red_s(hbase[1] + (a3 << 7), -x);
          }
        }
      }
      continue;
    }
    for (int r = r0; r < r0 + ROWS / WARPS; r += 8) {
      uint4 va, vb;  // rows r..r+3, r+4..r+7: word `lane`
      if (MODE != 2) {
        va = ldg_nc(vp + (size_t)(r / 4) * 32 + lane);
        vb = ldg_nc(vp + (size_t)(r / 4 + 1) * 32 + lane);
      } else {
        va = make_uint4(r, r + 1, r + 2, r + 3);
        vb = make_uint4(r ^ lane, r + 5, r + 6, r + 7);
      }
      const uint32_t v8[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
      if (MODE == 1) {
        const uint32_t* c = reinterpret_cast<const uint32_t*>(codes) + ((size_t)pass * ROWS + r) * 4;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint4 q = ldg_nc(c + 4 * e);  // broadcast: 4 byte-offset codes of row r + e
          red_s(hbase[0] + q.x, (int)v8[e]);
          red_s(hbase[0] + q.y, -(int)v8[e]);
          red_s(hbase[1] + q.z, (int)v8[e]);
          red_s(hbase[1] + q.w, -(int)v8[e]);
        }
      } else {
        const uint16_t* c = reinterpret_cast<const uint16_t*>(codes) + ((size_t)pass * ROWS + r) * 4;
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const uint4 q = ldg_nc(c + 4 * e);  // broadcast: 2 rows x 4 slot codes
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int x = (int)v8[e + h];
            const uint32_t a0 = w[2 * h] & 0xffffu, a1 = w[2 * h] >> 16, a2 = w[2 * h + 1] & 0xffffu, a3 = w[2 * h + 1] >> 16;
            if (MODE == 3) {
              acc += x ^ (int)(a0 + a1 + a2 + a3);
            } else {
              red_s(hbase[0] + (a0 << 7), x);
              red_s(hbase[0] + (a1 << 7), -x);
              red_s(hbase[1] + (a2 << 7), x);
              red_s(hbase[1] + (a3 << 7), -x);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (MODE == 3 && acc == 0x12345) sink[0] = acc;
  if (threadIdx.x == 0) sink[blockIdx.x] = hist[lane];
}

int main() {
  const int sms = 148, passes = 6;  // 148 x 6 = 888 passes ~ ceil(1821 / 2)
  std::vector<uint32_t> hv((size_t)ROWS * 32);
  for (size_t i = 0; i < hv.size(); ++i) hv[i] = (uint32_t)(i * 2654435761u) & 0x00ff00ffu;
  uint4* dvp;
  cudaMalloc(&dvp, hv.size() * 4);
  cudaMemcpy(dvp, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice);
  const size_t ncodes = (size_t)sms * passes * ROWS * 4;
  std::vector<uint16_t> c16(ncodes);
  std::vector<uint32_t> c32(ncodes);
  uint32_t s = 12345;
  for (size_t i = 0; i < ncodes; ++i) {
    s = s * 1664525u + 1013904223u;
    c16[i] = (uint16_t)((s >> 8) % NSLOT);
    c32[i] = (uint32_t)c16[i] * 128u;
  }
  std::vector<uint16_t> c16t(ncodes);  // 4 * slot offsets for the transposed histogram
  for (size_t i = 0; i < ncodes; ++i) c16t[i] = (uint16_t)(c16[i] * 4u);
  void *d16, *d32, *d16t;
  cudaMalloc(&d16t, ncodes * 2);
  cudaMemcpy(d16t, c16t.data(), ncodes * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&d16, ncodes * 2);
  cudaMalloc(&d32, ncodes * 4);
  cudaMemcpy(d16, c16.data(), ncodes * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(d32, c32.data(), ncodes * 4, cudaMemcpyHostToDevice);
  int* sink;
  cudaMalloc(&sink, 4096);
  const size_t smem = 3 * (NSLOT | 1) * 128;
  auto run = [&](auto kfn, const void* codes, const char* name) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 3; ++i) kfn<<<sms, WARPS * 32, smem>>>(dvp, codes, passes, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) kfn<<<sms, WARPS * 32, smem>>>(dvp, codes, passes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    // one launch = 888 passes = 888 x 2 column blocks of 9 columns for 64 vectors
    printf("%-34s %8.1f us / launch  (%.1f us per 64-vector batch at 16384^2, k=9: 1821 blocks)  err=%s\n", name, us,
           us * 1821.0 / (2.0 * sms * passes), cudaGetErrorString(cudaGetLastError()));
  };
  run(kern<0>, d16, "u16 codes + v loads + REDs");
  run(kern<1>, d32, "u32 byte-offset codes + v + REDs");
  run(kern<2>, d16, "u16 codes + REDs (v in registers)");
  run(kern<3>, d16, "u16 codes + v loads (no REDs)");
  run(kern<4>, d16, "REDs only, conflict-free rows");
  run(kern<5>, d16, "REDs only, random words");
  run(kern<11>, d16, "REDs only, transposed rows (odd)");
  run(kern<9>, d16t, "lane codes + SHFL + v + REDs (transposed)");
  run(kern<10>, d16t, "lane codes (no SHFL) + v + REDs");
  return 0;
}
