/*
 * rsr_b200.h — C ABI of the B200-native RSR / RSR++ library (librsr_b200.so).
 *
 * The reference (arxiv 2411.06360, /root/reference/pkg/src/rsr) is a Python +
 * Numba package with no C ABI; its compiled entry points are Numba functions
 * called from Python.  Each function below replaces one of them (cited
 * file:line), with plain pointers and sizes and no torch types, so any host
 * (Python ctypes, C, C++) can bind it.  INTEGRATION.md shows the ctypes stub
 * the reference's `rsr.kernels` would use.
 *
 * Conventions
 *  - Device pointers unless a name ends in `_host`.  Kernels are enqueued on
 *    `stream` (a cudaStream_t, NULL = legacy default stream); nothing
 *    synchronizes except the `_host` entry points.
 *  - Every call returns an rsr_status; rsr_b200_last_error() returns a
 *    thread-local message for the last failure.  RSR_ERR_INVALID messages use
 *    the reference's wording ("does not match", "variant", "k must be in ...")
 *    so the Python layer can raise the same ValueError.
 *  - No CPU fallback exists: if there is no usable sm_100 device the call
 *    fails with RSR_ERR_CUDA.
 */
#ifndef RSR_B200_H_
#define RSR_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSR_B200_ABI_VERSION 3

typedef enum rsr_status {
  RSR_OK = 0,
  RSR_ERR_INVALID = 1,     /* bad argument (maps to ValueError) */
  RSR_ERR_UNSUPPORTED = 2, /* valid for the reference but beyond a device limit (e.g. k > 15) */
  RSR_ERR_CUDA = 3,        /* CUDA runtime failure */
} rsr_status;

typedef enum rsr_dtype { RSR_I32 = 0, RSR_F32 = 1, RSR_F64 = 2, RSR_I64 = 3 } rsr_dtype;

/* kernels.py:14-21 `_VARIANTS`: "rsr" -> dense block product, "rsrpp"/"rsr++" -> fold. */
typedef enum rsr_variant { RSR_VARIANT_RSR = 0, RSR_VARIANT_RSRPP = 1 } rsr_variant;

/* Multiply formulation.  AUTO picks SCATTER for int32 activations and GATHER
 * otherwise (no native fp32 shared-memory atomic add exists on sm_100). */
typedef enum rsr_form { RSR_FORM_AUTO = 0, RSR_FORM_SCATTER = 1, RSR_FORM_GATHER = 2 } rsr_form;

/* One binary matrix's index: the device image of the reference RsrIndex
 * (indexer.py:47-139).  Arrays are block-major; block b covers columns
 * [b*k, b*k + w_b), w_b = min(k, cols - b*k) (column_blocks, indexer.py:193-199). */
typedef struct rsr_half_index {
  void* perm;       /* [nblocks][row_stride] u16 if rows <= 65536 else u32:
                       stable row order per block (indexer.py:269); entries >= rows are 0 */
  uint32_t* seg;    /* [nblocks][seg_stride]: seg[j] = #rows with key < j for
                       j < 2^w, seg[2^w] = rows (indexer.py:274-276 incl. sentinel) */
  uint16_t* bucket; /* [nblocks][row_stride]: key of every row, MSB-first
                       (indexer.py:270 `_buckets`), as a device code:
                       code = swz(key) << 2 for k <= 11 and k = 14 (the byte offset of the
                       key's histogram word), swz(key) for k = 12, 13, 15, 16 (its word
                       index), where swz(key) = key ^ ((key >> 5) & 31) is a shared-memory
                       bank swizzle (an involution); padding rows hold 0.  For k <= 13 the codes
                       of every aligned 8-row group of whole 256-row chunks are stored in
                       the scatter kernel's slot order: slot s holds row p[s], p = a
                       3-stage butterfly of 12 control bits kept in bits 13-15 of the
                       group's codes 0..3 (csrc/common.cuh butterfly8 / sched_ctrl;
                       indexer.unschedule_codes restores row order) */
} rsr_half_index;

typedef struct rsr_index_desc {
  int64_t rows, cols;
  int32_t k;          /* block width, 1 <= k <= 16 on the device */
  int32_t nblocks;    /* ceil(cols / k) */
  int32_t perm_bytes; /* 2 or 4 */
  int32_t halves;     /* 1 = binary index; 2 = ternary (half[0] positive, half[1] negative) */
  int64_t row_stride; /* rows rounded up to a multiple of 8 (16-byte aligned 8-row groups) */
  int64_t seg_stride; /* 2^k + 1 */
  rsr_half_index half[2];
} rsr_index_desc;

int rsr_b200_abi_version(void);
const char* rsr_b200_last_error(void);

/* Fill the size fields of `desc` (pointers untouched) and report the bytes of each
 * array per half.  Validates k as `_check_k` does (indexer.py:19-23). */
rsr_status rsr_index_layout(int64_t rows, int64_t cols, int32_t k, int32_t halves,
                            rsr_index_desc* desc, size_t* perm_bytes, size_t* seg_bytes,
                            size_t* bucket_bytes);

/* Device workspace bytes rsr_preprocess_* needs for this index. */
size_t rsr_preprocess_workspace_bytes(const rsr_index_desc* desc);

/* Replaces preprocess_ternary (indexer.py:281-286) = decompose_ternary
 * (core.py:124-128) + preprocess (indexer.py:251-278) for both halves.
 * A: int8 [rows][lda] row-major, entries must be -1/0/+1.  Any other entry sets
 * *d_bad_entries (device int32, caller-zeroed) to a nonzero count — the
 * TernaryMatrix alphabet check (core.py:33). */
rsr_status rsr_preprocess_ternary(const int8_t* A, int64_t lda, const rsr_index_desc* desc,
                                  int32_t* d_bad_entries, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* Replaces preprocess (indexer.py:251-278) for a BinaryMatrix stored as the
 * reference stores it (core.py:53-99): bits [rows][ldb] bytes, MSB-first. */
rsr_status rsr_preprocess_binary(const uint8_t* bits, int64_t ldb, const rsr_index_desc* desc,
                                 void* workspace, size_t workspace_bytes, void* stream);

/* Replaces `_run_blocks` over blocks [block_begin, block_end) of every half
 * (kernels.py:127-177) followed by the `pos - neg` of multiply_ternary
 * (kernels.py:196-206) or the single half of multiply_rsr (kernels.py:185-193).
 * v: [rows] of v_dtype.  out: [cols] of out_dtype; only columns of the block
 * range are written (multiply_parallel's disjoint slices, kernels.py:209-239).
 * int32 accumulation is exact modulo 2^32 (bit-exact whenever the true result
 * fits); out_dtype may be F64 for int32 input (reference result type). */
rsr_status rsr_multiply(const rsr_index_desc* desc, const void* v, rsr_dtype v_dtype, void* out,
                        rsr_dtype out_dtype, rsr_variant variant, rsr_form form,
                        int32_t block_begin, int32_t block_end, void* stream);

/* rsr_multiply with launch flags.  RSR_MULTIPLY_INDEPENDENT: the caller guarantees that no
 * kernel still in flight on `stream` writes v (e.g. a stream of matvecs on resident inputs, or
 * layers sharing one input).  The scatter launch then starts its reductions on the SMs the
 * previous launch has already freed (programmatic dependent launch) instead of waiting for that
 * launch to finish; only its writes to out wait, so out keeps stream order and launches still
 * complete in stream order.  Other forms ignore the flag.  Same results as rsr_multiply. */
#define RSR_MULTIPLY_INDEPENDENT 1u
rsr_status rsr_multiply_ex(const rsr_index_desc* desc, const void* v, rsr_dtype v_dtype, void* out,
                           rsr_dtype out_dtype, rsr_variant variant, rsr_form form,
                           int32_t block_begin, int32_t block_end, uint32_t flags, void* stream);

/* Replaces `load_index` -> RsrIndex.from_blocks (store.py:49-101, indexer.py:89-129): import
 * a stored index whose per-block arrays are already on the device — d_perm{0,1}: u32
 * [nblocks][rows] stable row orders, d_seg{0,1}: u32 [nblocks][seg_stride] segment starts
 * (2^w used per block, no sentinel), half 1 only for a ternary desc.  Validates the
 * invariants on the device (d_error[0] |= 1 perm out of range, 2 perm not a bijection,
 * 4 segmentation does not start at 0, 8 segmentation decreasing or > rows; d_error[1] =
 * lowest failing block; the caller initializes d_error to {0, INT32_MAX} and reads it after
 * the stream), writes the device layout of `desc` (arrays from rsr_index_layout) including
 * the key codes rebuilt from the segments, and schedules the keys.  `workspace` needs
 * rsr_index_import_workspace_bytes(desc) device bytes. */
size_t rsr_index_import_workspace_bytes(const rsr_index_desc* desc);
rsr_status rsr_index_import(const rsr_index_desc* desc, const uint32_t* d_perm0, const uint32_t* d_seg0,
                            const uint32_t* d_perm1, const uint32_t* d_seg1, int64_t seg_stride,
                            void* workspace, size_t workspace_bytes, int32_t* d_error, void* stream);

/* Dense 2-bit ternary GEMV — the paper's "standard" multiply (naive_multiply, core.py:135-169)
 * on the GPU, kept as the honest comparator of the RSR path.
 * rsr_dense_pack_ternary: int8 A [rows][lda] (device) -> bit-planes d_pos / d_neg, each
 * rsr_dense_plane_words(rows, cols) u32 laid out [ceil(rows/32)][cols] (bit i of word
 * [w][j] = A[32w+i][j] is +1 / -1); entries outside {-1,0,1} are counted into d_bad_entries.
 * rsr_dense_multiply: out[cols] = v[rows] . A for int32 (exact) or fp32 v. */
size_t rsr_dense_plane_words(int64_t rows, int64_t cols);
rsr_status rsr_dense_pack_ternary(const int8_t* A, int64_t lda, int64_t rows, int64_t cols,
                                  uint32_t* d_pos, uint32_t* d_neg, int32_t* d_bad_entries, void* stream);
rsr_status rsr_dense_multiply(const uint32_t* d_pos, const uint32_t* d_neg, int64_t rows, int64_t cols,
                              const void* v, rsr_dtype dtype, void* out, void* stream);

/* The same comparator at HBM speed for int8-range activations (the reference's own vectors are
 * integers in [-100, 100]): 2 bits per entry laid out so that IDP4A does four entries per two
 * instructions.  rsr_dense_pack_ternary_i8: int8 A -> d_q, rsr_dense_i8_words(rows, cols) u32
 * ([ceil(rows/16)][cols]; entry (16r + 4t + k, j) = 2-bit field t of byte k: 01 = +1, 11 = -1).
 * rsr_dense_multiply_i8: out[cols] int32 = v[rows] int8 . A, exact. */
size_t rsr_dense_i8_words(int64_t rows, int64_t cols);
rsr_status rsr_dense_pack_ternary_i8(const int8_t* A, int64_t lda, int64_t rows, int64_t cols, uint32_t* d_q,
                                     int32_t* d_bad_entries, void* stream);
rsr_status rsr_dense_multiply_i8(const uint32_t* d_q, int64_t rows, int64_t cols, const int8_t* v, int32_t* out,
                                 void* stream);

/* Batched multiply: V [batch][rows] -> OUT [batch][cols] on the current stream (SURVEY.md
 * §8(d) config 3; the reference has no batch API and runs `multiply_ternary`,
 * kernels.py:196-206, once per vector).  int32 and fp32 need `workspace` of
 * rsr_multiply_batched_workspace_bytes() bytes (device, 16-byte aligned); out_dtype must equal
 * v_dtype.  Forms: index beyond L2 -> the batched gather kernel (each index byte read once per
 * slice of up to 128 vectors, V transposed into the workspace); index L2-resident -> scatter
 * launches, for int32 two vectors per launch (v + v' * 2^16 per reduction) when a device guard
 * proves every bucket sum fits in int16 — that guard is ONE host synchronisation of `stream`
 * per call, skipped (per-vector launches) while the stream is being captured.  Results are
 * exact for int32 in every form.  fp64 runs one multiply per vector (workspace unused). */
size_t rsr_multiply_batched_workspace_bytes(const rsr_index_desc* desc, int64_t batch, rsr_dtype v_dtype);
rsr_status rsr_multiply_batched(const rsr_index_desc* desc, const void* V, rsr_dtype v_dtype,
                                int64_t batch, void* OUT, rsr_dtype out_dtype,
                                rsr_variant variant, void* workspace, size_t workspace_bytes,
                                void* stream);

/* Exact wide-integer multiply (int64 activations): the reference computes in fp64
 * (core.py:110-117), exact for every integer vector whose partial sums stay below 2^53
 * (SPEC.md:276), while int32 accumulation is exact only while sum_r |v_r| <= 2^31 - 1.  v is
 * split into L balanced base-2^s digit vectors (rows * 2^(s-1) <= 2^31 - 1), each runs through
 * the int32 multiply, and the limb results recombine in 128-bit integers (csrc/wide.cu).
 * v: int64 [rows] (device); max_abs: a bound on |v| (0 = the whole int64 range; it sets L);
 * out: [cols] int64 (wraps modulo 2^64) or float64 (the exact integer, rounded once); only the
 * block range's columns are written.  workspace: rsr_multiply_wide_workspace_bytes() device
 * bytes, 256-byte aligned. */
size_t rsr_multiply_wide_workspace_bytes(const rsr_index_desc* desc, uint64_t max_abs);
rsr_status rsr_multiply_wide(const rsr_index_desc* desc, const int64_t* v, uint64_t max_abs, void* out,
                             rsr_dtype out_dtype, rsr_variant variant, int32_t block_begin, int32_t block_end,
                             void* workspace, size_t workspace_bytes, void* stream);
/* Fixed-point fp64 (non-integer float64 activations, kernels.py:196-206 computes in fp64):
 * v_q = round(v * 2^exp2) as int64 (|v_q| <= max_abs < 2^62), multiplied exactly like
 * rsr_multiply_wide, each column's exact integer rounded once to fp64 and scaled by 2^-exp2.
 * The host session chooses exp2 so every nonzero |v| keeps >= 41 significant bits (else the fp64
 * gather kernel runs); the same workspace as rsr_multiply_wide. */
rsr_status rsr_multiply_fixed(const rsr_index_desc* desc, const int64_t* v_q, uint64_t max_abs, int32_t exp2,
                              double* out, rsr_variant variant, int32_t block_begin, int32_t block_end, void* workspace,
                              size_t workspace_bytes, void* stream);

/* Batch plan: the index re-cut for the batch-native kernel (BASELINE config 3, many vectors
 * against one index; the reference has no batch API and runs `multiply_ternary`,
 * kernels.py:196-206, once per vector).  The batch kernel's lanes span the VECTOR dimension:
 * lane w owns the packed int16 pair of vectors 2w, 2w+1 (v + v' * 2^16), so one shared-memory
 * reduction adds a row's 64 activations into the 32 consecutive words of ONE histogram slot —
 * conflict-free, where the per-vector kernel's 32 random rows are not.  A slot is 128 bytes,
 * so the plan uses narrower column blocks (kb, 9 at 16384 rows) than the index, and every
 * row's bin becomes a SLOT: bins whose rows (both halves) could exceed int16 for |v| <= vmax
 * are split into several slots (rows dealt round-robin by rank), so every slot's sum fits
 * int16 and the packed accumulation is exact; the fold adds a split bin's slots back
 * together in int32.  Built on the device from any index (perm + seg) by
 * rsr_batch_plan_build; `extra` (the largest number of split slots of a unit) is read back
 * once, at build time. */
typedef struct rsr_batch_plan {
  int64_t rows, cols;
  int32_t kb;          /* plan block width */
  int32_t nblocks;     /* ceil(cols / kb) */
  int32_t halves;      /* 1 binary, 2 ternary */
  int32_t split_rows;  /* rows per unit (multiple of 8); units = (plan block, row split) */
  int32_t nsplits;     /* ceil(rows / split_rows) */
  int32_t extra_cap;   /* entries per unit in slot_bins (split slots follow the unit's 2^w direct slots) */
  int32_t extra;       /* histogram slots beyond 2^kb the widest unit needs (set by rsr_batch_plan_build) */
  int32_t vmax;        /* packed form valid for |v| <= vmax (else int32 lanes, 32 vectors per pass) */
  int64_t row_stride;  /* nsplits * split_rows */
  uint16_t* codes;     /* [halves][nblocks][row_stride]: 4 * slot of each row (the slot's byte offset
                          in a lane's histogram row; slot 0 = logical bin 0, never read) */
  uint16_t* slot_bins; /* [nblocks * nsplits][extra_cap]: logical bin of split slot 2^w + e (0 ends the list) */
} rsr_batch_plan;

/* Fill the plan's size fields for an index (pointers untouched) and the device bytes of its
 * arrays; RSR_ERR_UNSUPPORTED when the batch kernel does not apply (e.g. k < 2). */
rsr_status rsr_batch_plan_layout(const rsr_index_desc* desc, rsr_batch_plan* plan, size_t* code_bytes,
                                 size_t* map_bytes, size_t* workspace_bytes);
/* Build the plan's arrays from the index (device kernels, then ONE host synchronisation of
 * `stream` to read `extra`); RSR_ERR_UNSUPPORTED if a unit needs more split slots than fit. */
rsr_status rsr_batch_plan_build(const rsr_index_desc* desc, rsr_batch_plan* plan, void* workspace,
                                size_t workspace_bytes, void* stream);
/* Batch-native multiply through a plan: V int32 [batch][rows] -> OUT int32 [batch][cols]
 * (int32 arithmetic, exact modulo 2^32 like rsr_multiply).  No host synchronisation (CUDA
 * graph capturable): a device flag picks the packed form (max |V| <= vmax) or int32 lanes.
 * workspace: rsr_multiply_batched_plan_workspace_bytes() device bytes, 256-byte aligned. */
size_t rsr_multiply_batched_plan_workspace_bytes(const rsr_batch_plan* plan, int64_t batch);
rsr_status rsr_multiply_batched_plan(const rsr_index_desc* desc, const rsr_batch_plan* plan, const int32_t* V,
                                     int64_t batch, int32_t* OUT, rsr_variant variant, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* Fused all-gather epilogue (multi-GPU column shards; replaces the
 * multiply_parallel shard launch + the all-gather of the output slices): int32 multiply of all
 * blocks of `desc` (single row split: rows <= 16384) that ALSO stores every folded block's column
 * values into peer_out[r][col_base + column] for r < npeers — device pointers of every rank's
 * gathered vector in peer-mapped (symmetric) memory — then releases its stores at system scope
 * and adds 1 to every rank's peer_sig[r].  `done` is this rank's local completion counter
 * (zero-initialised, reused every call).  A rank's gathered vector holds every rank's slice of
 * call c once its signal reaches c * npeers: rsr_allgather_wait enqueues that wait on a stream
 * (traps after 4 s if a peer never arrives).  `out` receives this rank's own slice too. */
rsr_status rsr_multiply_allgather(const rsr_index_desc* desc, const int32_t* v, int32_t* out, rsr_variant variant,
                                  int32_t* const* peer_out, unsigned long long* const* peer_sig, int32_t npeers,
                                  int64_t col_base, unsigned long long* done, void* stream);
rsr_status rsr_allgather_wait(const unsigned long long* sig, unsigned long long target, void* stream);

/* End-to-end entry with HOST buffers (the call a reference-side binding makes):
 * copies v_host -> d_v, multiplies all blocks, copies d_out -> out_host and
 * synchronizes the stream.  d_v / d_out are caller-owned device scratch of the
 * right size; v_host / out_host should be pinned for async copies.  int32 / float32 / float64
 * vectors only, computed in that type (int32 wraps modulo 2^32: see the session below for the
 * exact reference contract). */
rsr_status rsr_multiply_host(const rsr_index_desc* desc, const void* v_host, rsr_dtype v_dtype,
                             void* out_host, rsr_dtype out_dtype, rsr_variant variant,
                             void* d_v, void* d_out, void* stream);

/* Host-buffer session (the e2e call `multiply_ternary(numpy v, idx)`, kernels.py:185-206):
 * mapped pinned staging, device copies of v and of the result, and mapped pinned result memory,
 * allocated once for one index on the current device.  rsr_host_session_multiply takes v_host
 * [rows] of any element type, v_bytes = its size, and writes out_host [cols] (out_bytes = its size)
 * as float64 (the reference's result type) or as the vector type.  Staging classifies v in the
 * same pass that copies it (csrc/host_stage.cpp), so the result is exact wherever the
 * reference's fp64 result is:
 *   - integer-valued v (int32 / int64, or float64 holding integers) with sum |v| <= 2^31 - 1:
 *     int32 scatter multiply (bit-exact); with rows <= 16384 the call is ONE kernel launch that
 *     pulls v from the mapped staging itself and streams each folded block's results into the
 *     mapped buffer as seq-tagged words (no H2D / D2H copy, no stream synchronize);
 *   - other integer-valued v (|v| < 2^63): the exact wide multiply above;
 *   - float32: fp32 (exact fixed-point scatter while rows <= 16384, else the gather kernel);
 *   - other float64: the fp64 gather kernel.
 * A non-finite entry fails with RSR_ERR_INVALID "vector entries must be finite" (core.py:115).
 * out_dtype = int32 with int32 v keeps int32 arithmetic (modulo 2^32).  One call at a time per
 * session (use one session per thread). */
typedef struct rsr_host_session rsr_host_session;
rsr_status rsr_host_session_create(const rsr_index_desc* desc, rsr_host_session** out);
void rsr_host_session_destroy(rsr_host_session* session);
rsr_status rsr_host_session_multiply(rsr_host_session* session, const void* v_host, rsr_dtype v_dtype,
                                     size_t v_bytes, void* out_host, rsr_dtype out_dtype, size_t out_bytes,
                                     rsr_variant variant, void* stream);
/* Replaces segmented_sum / `_segment_sums` (kernels.py:50-60, 94-101): gather-form
 * bucket sums u[0..2^w) of one block of one half. */
rsr_status rsr_segmented_sum(const rsr_index_desc* desc, int32_t half, int32_t block,
                             const void* v, rsr_dtype dtype, void* u, void* stream);

/* Replaces block_product_rsr / block_product_rsrpp (kernels.py:104-116, loops at
 * kernels.py:63-91) for one SegmentedSums vector u[0..2^width) (fp64); buf holds
 * 2^(width-1) doubles of scratch, out receives `width` doubles. */
rsr_status rsr_block_product(const double* u, int32_t width, rsr_variant variant, double* buf, double* out,
                             void* stream);

/* Replaces naive_multiply (core.py:135-169) for a ternary int8 matrix: the
 * "standard" dense multiply, on the GPU (the honest dense comparator). */
rsr_status rsr_naive_multiply_ternary(const int8_t* A, int64_t rows, int64_t cols, int64_t lda,
                                      const void* v, rsr_dtype dtype, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RSR_B200_H_ */
