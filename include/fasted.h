/*
 * fasted.h -- C ABI of libfasted.so, the B200 (sm_100a) FaSTED epsilon
 * self-join engine.
 *
 * Plain pointers and sizes only.  Every data pointer is DEVICE memory owned
 * by the caller (torch tensors in the Python drop-in); every call is
 * asynchronous on `stream` (a cudaStream_t passed as void*, NULL = legacy
 * default stream) unless stated otherwise.  Thread-safe: one host thread per
 * device may call concurrently (all state is per call).
 *
 * Status codes mirror the reference's exception classes
 * (/root/reference/pkg/src/mpjoin/errors.py:4-29 and the CLI exit-code map,
 * cli.py:56-59,588-607):
 *   0 FASTED_OK
 *   2 FASTED_ERR_ARGUMENT   -> ArgumentError / ConfigError
 *   3 FASTED_ERR_RANGE      -> RangeError (FP16 overflow in quantisation)
 *   4 FASTED_ERR_CAPACITY   -> result buffer too small (count still exact)
 *   5 FASTED_ERR_CUDA       -> CUDA runtime / launch failure
 *   6 FASTED_ERR_UNSUPPORTED-> device is not sm_100 (no silent fallback)
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/mpjoin):
 *   fasted_quantize  : dataset.to_half            dataset.py:164-193
 *                      + _kernel.squared_norms_rz _kernel.py:79-93
 *   fasted_quantize_async : the same, stream-ordered (device overflow word)
 *   fasted_norms     : dataset.compute_squared_norms dataset.py:159-161
 *   fasted_join      : tiling.self_join's sweep   tiling.py:307-344
 *                      (work queue + compute_block_tile tiling.py:199-285
 *                       + _kernel.accumulate_panel _kernel.py:57-76
 *                       + combine_distance mma.py:143-157); a 128x128 range
 *                      is compute_block_tile itself
 *   fasted_sort_pairs: tiling.make_result_set     tiling.py:116-122
 *                      (and the merge, tiling.py:346-351)
 *   fasted_fp64_rows : oracle.brute_force_fp64    oracle.py:43-64 (sampled rows,
 *                      for analysis.overlap_accuracy at scale)
 */
#ifndef FASTED_H_
#define FASTED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FASTED_ABI_VERSION 2

enum {
    FASTED_OK = 0,
    FASTED_ERR_ARGUMENT = 2,
    FASTED_ERR_RANGE = 3,
    FASTED_ERR_CAPACITY = 4,
    FASTED_ERR_CUDA = 5,
    FASTED_ERR_UNSUPPORTED = 6
};

/* fasted_join flags */
enum {
    FASTED_JOIN_TC = 0,     /* tcgen05/TMEM fused kernel (the product path)          */
    FASTED_JOIN_EXACT = 1,  /* CUDA-core FFMA.RZ kernel, bit-exact with the reference */
    FASTED_JOIN_COUNT = 2,  /* OR-able: count only, write no records                 */
    /* OR-able, tcgen05 only, needs row range == column range: compute only the
     * tiles on or above the diagonal and write every off-diagonal pair in both
     * orientations, (i, j) and (j, i), with the same dist_sq -- half the MMA
     * work for the same record set (and the set is exactly symmetric). */
    FASTED_JOIN_SYMMETRIC = 4,
    /* OR-able hint: the caller expects <= 128 pairs per row.  Only picks the
     * kernel form (results are identical): at d_pad > 256 on large joins the
     * CTA-pair form, faster at low selectivity under the 1 kW power cap. */
    FASTED_JOIN_LOW_OUTPUT = 8,
    /* OR-able: do not zero `count`; the launch appends to the records and
     * totals an earlier launch left in out_records / count (same buffer,
     * same capacity), e.g. one row range swept in column segments while the
     * dataset is still arriving (engine.stream_join). */
    FASTED_JOIN_APPEND = 16,
    /* OR-able hint: the caller expects at most one pair per 8192 examined
     * (row x column) pairs.  Only picks the kernel form (results are
     * identical): the tcgen05 kernels then hand candidate rows to two hit
     * warps instead of running the rare path in the epilogue warps (1M x
     * 128: 1137 vs 992 TFLOPS; at ~1 pair per 1000 examined the hit warps
     * cannot keep up, 2x slower). */
    FASTED_JOIN_SPARSE = 32
};
/* Every other flag bit is rejected (FASTED_ERR_ARGUMENT): no flag, and no
 * environment setting, changes which pairs are returned. */

int fasted_abi_version(void);
const char* fasted_strerror(int status);
/* Message of the last failing call on this host thread ("" if none). */
const char* fasted_last_error(void);
/* 0 if `device` is an sm_100 part this library can drive, else 6. */
int fasted_device_check(int device);

/*
 * FP32 [n, d] row-major -> FP16 [n_pad, d_pad] row-major (RNE, zero padded)
 * plus per-row FP32 squared norms accumulated round-toward-zero in
 * ascending k over all d_pad columns (bit-exact with to_half).
 * n_pad >= n, d_pad >= d, d_pad % 8 == 0.
 * On FP16 overflow returns FASTED_ERR_RANGE after the stream syncs, with
 * *first_overflow_host = row-major flat index (i*d + k) of the first value
 * whose cast is +-inf (the point/dimension RangeError names).  This call
 * synchronises `stream` to read the overflow flag.
 */
int fasted_quantize(const float* x, int64_t n, int64_t d, uint16_t* values16,
                    int64_t n_pad, int64_t d_pad, float* norms,
                    int64_t* first_overflow_host, void* stream);

/*
 * fasted_quantize without the synchronisation (same kernel, same bits): the
 * overflow index is atomicMin'ed into the DEVICE word *first_overflow_dev,
 * which the caller sets to ~0 before the call and reads after the stream
 * reaches it (~0: no overflow).  For pipelines that quantise in chunks and
 * check once (bench.py's 5M x 384 generation, the per-kernel timing).
 */
int fasted_quantize_async(const float* x, int64_t n, int64_t d, uint16_t* values16,
                          int64_t n_pad, int64_t d_pad, float* norms,
                          unsigned long long* first_overflow_dev, void* stream);

/* RZ squared norms of an existing FP16 [n_pad, d_pad] matrix. */
int fasted_norms(const uint16_t* values16, int64_t n_pad, int64_t d_pad, float* norms,
                 void* stream);

/*
 * Epsilon join over point rows [row_begin, row_end) x columns
 * [col_begin, col_end) of the FP16 matrix; all four bounds multiples of 128
 * (or the end == n_pad), n_pad % 128 == 0, d_pad % 16 == 0.
 * A pair (i, j) qualifies iff i, j < n_logical and
 *   max(((-2 a_ij) + s_i) + s_j, 0) <= eps_sq           (tiling.py:273-279)
 * with i == j forced to distance 0 (the reference's self-distance is
 * exactly 0, tiling.py:13-14).  Records are 16 bytes, {uint32 i, uint32 j,
 * float dist_sq, uint32 0} with 1-based i, j, written to out_records in
 * UNSPECIFIED order.  Each warp fills private runs of FASTED_RECORD_CHUNK
 * slots, so the record array may contain unused slots, marked i == 0
 * (fasted_sort_pairs drops them).
 * The tcgen05 path reads only the rows of [row_begin, row_end) and
 * [col_begin, col_end) (plus the padding of their last tiles, whose results
 * are masked), so a launch may run while other rows are still being copied.
 * `count` is DEVICE memory for two uint64 (zeroed by this call unless
 * FASTED_JOIN_APPEND):
 *   count[0] = exact number of qualifying pairs,
 *   count[1] = chunks taken; slots used = count[1] * FASTED_RECORD_CHUNK.
 * Slots >= capacity are not written; if slots used > capacity the caller
 * resizes (count[0] + FASTED_RECORD_CHUNK * 32 * SMs always suffices) and
 * reruns.  With FASTED_JOIN_COUNT the out_* pointers may be NULL.
 */
#define FASTED_RECORD_CHUNK 256
int fasted_join(const uint16_t* values16, const float* norms, int64_t n_logical,
                int64_t n_pad, int64_t d_pad, int64_t row_begin, int64_t row_end,
                int64_t col_begin, int64_t col_end, float eps_sq, int flags,
                void* out_records, uint64_t capacity, unsigned long long* count,
                void* stream);

/*
 * Canonical (i, j) order (the reference's lexsort) of `slots` join records
 * (16-byte records from fasted_join; slots with i == 0 are unused and
 * dropped) whose i lie in [row_begin+1, row_end] and j in [1, n_cols].
 * Writes the valid records, sorted, to out_i/out_j/out_d (SoA, length >=
 * number of valid records).  tmp is 8-byte aligned scratch of tmp_bytes >=
 * 8 bytes per valid record (the row-bucketed (j, dist_sq) pairs).
 * workspace must hold fasted_sort_workspace_bytes(row_end - row_begin,
 * n_cols) bytes.  (ABI version 2: version 1 took two 4-byte scratch arrays.)
 */
size_t fasted_sort_workspace_bytes(int64_t n_rows, int64_t n_cols);
int fasted_sort_pairs(const void* records, uint64_t slots, int64_t row_begin, int64_t row_end,
                      int64_t n_cols, uint32_t* out_i, uint32_t* out_j, float* out_d,
                      void* tmp, size_t tmp_bytes, void* workspace, size_t workspace_bytes,
                      void* stream);

/*
 * FP64 ground truth for `nq` sampled query rows (device int64 indices,
 * 0-based) of the ORIGINAL FP32 dataset x [n, d]: every (q, j) with
 * sqrt(sum_k (x_qk - x_jk)^2) <= epsilon, accumulated in FP64 in ascending
 * k exactly as the reference's oracle (oracle.py:26-64, numpy order, no
 * FMA).  Records are 16 bytes {uint32 q+1, uint32 j+1, float64 dist_sq},
 * unordered; *count (device uint64, zeroed here) is the exact total.
 * Used to report pair accuracy vs FP64 (the paper's Eq. 3) at scale.
 */
int fasted_fp64_rows(const float* x, int64_t n, int64_t d, const int64_t* qrows, int64_t nq,
                     double epsilon, void* out_records, uint64_t capacity,
                     unsigned long long* count, void* stream);

/* Name of the join kernel fasted_join launches for this d_pad, row and
 * column counts and flags (the same selection rule, environment overrides
 * included; for reports). */
const char* fasted_join_kernel_name(int64_t d_pad, int64_t rows, int64_t cols, int flags);

/* Number of SMs and device name of the current device (for reports). */
int fasted_device_info(int* sm_count, char* name, int name_len);

#ifdef __cplusplus
}
#endif

#endif /* FASTED_H_ */
