/*
 * spca.h — C ABI of the B200 sketch pass (libspca.so).
 *
 * This is the drop-in boundary for the one hot path of the reference
 * package `streampca` (arXiv 1704.07669, Algorithm 4 steps 4-8): the single
 * streaming pass over A (m x n, row blocks A_i) that accumulates
 *
 *     G_i = A_i Omega          (m x l, one row per data row)
 *     H  += A_i^T G_i          (n x l)
 *     col_sums += 1^T A_i      (n)
 *     rows_seen += rows(A_i)
 *
 * Entry points replace, one for one, the reference seam
 *   sketch_pass(stream, omega, block_rows=None, fixed_order=False,
 *               compensated=False) -> SketchState
 * (/root/reference/pkg/src/streampca/sketch.py:52-116):
 *   spca_sketch_create   <- argument checks + accumulator allocation, sketch.py:68-83
 *   spca_sketch_push     <- one iteration of `for block in stream.blocks(...)`,
 *                           _check_block sketch.py:40-49 and the two GEMMs +
 *                           column sum sketch.py:102-113
 *   spca_sketch_finish   <- `np.vstack(g_parts)` + SketchState(...), sketch.py:115-116
 *   spca_center_correct  <- center_correct, sketch.py:119-139
 *   spca_last_error      <- the exception taxonomy of errors.py:4-69
 *                           (StreamFormatError / DataError(row=...))
 * Plain pointers and sizes only; no torch or numpy types cross this line.
 *
 * Threading: a handle is single-consumer — one handle per
 * host thread and per GPU. All work is ordered on the handle's CUDA stream.
 *
 * Determinism: the library re-chunks the pushed rows into canonical chunks
 * of `spca_sketch_chunk_rows()` rows aligned to absolute row 0, and reduces
 * every partial sum in a fixed order (no float atomics). Results are
 * therefore bitwise identical for ANY sequence of push sizes and run to run
 * — the GPU analogue of the reference's fixed_order contract
 * (pkg/README.md:179-196, test_acceptance.py:223-255).
 */
#ifndef SPCA_H_
#define SPCA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPCA_ABI_VERSION 1

typedef struct spca_sketch *spca_handle_t;

/* element type of A (and of the device-side G) */
enum spca_dtype { SPCA_F32 = 0, SPCA_F64 = 1 };

/* arithmetic used for the two contractions */
enum spca_precision {
  SPCA_PREC_AUTO = 0, /* best available: TC split for f32, DFMA for f64    */
  SPCA_PREC_SIMT = 1, /* CUDA-core FFMA (f32) / DFMA (f64), fp32|fp64 accum */
  SPCA_PREC_TC = 2    /* tcgen05 tensor cores, split precision (f32 only)   */
};

/* where a pointer lives */
enum spca_mem {
  SPCA_MEM_DEVICE = 0,   /* device memory of the handle's GPU               */
  SPCA_MEM_PINNED = 1,   /* page-locked host memory (cudaHostAlloc/Register) */
  SPCA_MEM_PAGEABLE = 2  /* ordinary host memory (staged through pinned)    */
};

/* status codes; the Python layer maps them onto errors.py classes */
enum spca_status {
  SPCA_OK = 0,
  SPCA_ERR_FORMAT = 1,     /* StreamFormatError  (sketch.py:69-75, 41-44)   */
  SPCA_ERR_DATA = 2,       /* DataError(row=)    (sketch.py:45-49)          */
  SPCA_ERR_CAPABILITY = 3, /* CapabilityError    (errors.py:36-38)          */
  SPCA_ERR_CONFIG = 4,     /* ConfigError        (errors.py:41-42)          */
  SPCA_ERR_CUDA = 5,       /* CUDA runtime failure                           */
  SPCA_ERR_OOM = 6,        /* device or pinned allocation failed             */
  SPCA_ERR_STATE = 7,      /* call out of order (e.g. push after finish)     */
  SPCA_ERR_EMPTY = 8       /* EmptyStreamError   (sketch.py:133-134)        */
};

/* Library version (SPCA_ABI_VERSION) and build info string. */
int spca_abi_version(void);
const char *spca_build_info(void);

/* Create a sketch accumulator for A with n columns and sketch width l.
 *  omega        : n x l row-major float64 test matrix (the reference draws it
 *                 with linalg.gaussian_matrix, linalg.py:46-56); copied.
 *  omega_where  : SPCA_MEM_DEVICE or a host kind.
 *  device       : CUDA ordinal; stream: cudaStream_t (NULL = a private
 *                 non-blocking stream owned by the handle).
 *  rows_hint    : expected m (0 = unknown, G grows geometrically).
 *  compensated  : Kahan summation of col_sums across chunks (sketch.py:82,107-111).
 * Errors: SPCA_ERR_FORMAT for n<1 or l<1 (omega.ndim != 2, sketch.py:69-70). */
int spca_sketch_create(spca_handle_t *out, int64_t n, int64_t l, int dtype,
                       int precision, const double *omega, int omega_where,
                       int device, void *stream, int64_t rows_hint,
                       int compensated);

/* Append `rows` rows of A (row stride `ld` elements, ld >= n) whose first
 * row is absolute row `first_row`, which must equal the rows pushed so far
 * (RowStream blocks are consecutive, streams.py:31-52).
 * Asynchronous: device and pinned sources must stay valid until the next
 * spca_sketch_sync / finish. Non-finite values are detected on the device;
 * the first offending absolute row is reported by sync/finish as
 * SPCA_ERR_DATA (DataError(row=...), sketch.py:45-49). */
int spca_sketch_push(spca_handle_t h, const void *a, int64_t rows, int64_t ld,
                     int64_t first_row, int where);

/* spca_sketch_push for the last block of the stream (the final iteration of
 * `for block in stream.blocks(...)`, sketch.py:85-113): the trailing partial
 * chunk is processed with the rest of the block instead of waiting in the
 * staging buffer for spca_sketch_finish. Results are bitwise identical to
 * push + finish (the canonical chunk boundaries do not move); pushes after a
 * final push fail with SPCA_ERR_STATE until spca_sketch_reset. */
int spca_sketch_push_final(spca_handle_t h, const void *a, int64_t rows, int64_t ld,
                           int64_t first_row, int where);

/* The arithmetic the handle runs: SPCA_PREC_SIMT or SPCA_PREC_TC (what
 * SPCA_PREC_AUTO resolved to for this dtype, shape and device); -1 on a null handle. */
int spca_sketch_precision(spca_handle_t h);

/* Start a new pass on the same handle (same n, l, Omega): zero the
 * accumulators and the row counter, keep every allocation. Lets a caller
 * run repeated passes (or a second pass of power_refine with the same Omega)
 * without re-uploading Omega. */
int spca_sketch_reset(spca_handle_t h);

/* Wait for all queued work; returns SPCA_ERR_DATA if a non-finite row was seen. */
int spca_sketch_sync(spca_handle_t h);

/* Rows accepted so far (rows_seen) and the canonical chunk size. */
int spca_sketch_rows(spca_handle_t h, int64_t *rows_seen);
int64_t spca_sketch_chunk_rows(spca_handle_t h);

/* Complete the pass and copy the state out in float64:
 *   g_out  rows_seen x l row-major, h_out n x l row-major, colsum_out n.
 * Any output pointer may be NULL (skipped). out_where: device or host.
 * After finish the handle accepts no more pushes (it may still be read
 * again with finish or used by spca_center_correct / spca_device_views). */
int spca_sketch_finish(spca_handle_t h, double *g_out, double *h_out,
                       double *colsum_out, int64_t *rows_seen, int out_where);

/* Device views of the accumulators after finish (for the GPU post-pass and
 * for an NCCL all-reduce of [H | colsum] across ranks). H and colsum are
 * one contiguous float64 buffer of n*(l+1) elements: H row-major n x l,
 * then colsum. G is float64 rows_seen x l. Pointers stay owned by h. */
int spca_device_views(spca_handle_t h, double **g_dev, double **hcs_dev);


/* Multi-GPU exchange: sum the finished [H | col_sums] of
 * every rank of `nccl_comm` (an ncclComm_t of the caller's NCCL, one rank per
 * GPU, each handle on its own GPU) in place with ncclAllReduce on the handle's
 * stream, and return the global row count. G stays row-sharded. libnccl.so.2
 * is resolved at run time (SPCA_ERR_CAPABILITY when absent); the row shards
 * are the reference's consecutive RowStream blocks split by rank. */
int spca_allreduce(spca_handle_t h, void *nccl_comm, int64_t *rows_total);

/* center_correct (sketch.py:119-139) on the finished device state, in
 * place: mu = colsum / m_total; G -= 1 (mu^T Omega); H -= mu (1^T G) where
 * 1^T G is `gsum` (l values, already summed over every rank's rows; NULL =
 * use this handle's own G); colsum <- 0. m_total = rows over all ranks.
 * Writes mu (n values) to mean_out if non-NULL (host or device per where). */
int spca_center_correct(spca_handle_t h, int64_t m_total, const double *gsum,
                        double *mean_out, int mean_where);

/* Omega exactly as the pass used it (n x l float64 row-major: the fp32
 * rounding of the caller's Omega for SPCA_F32) — the test matrix the post-pass
 * must pair with G and H (blocked_qb, qb.py:59-135). out_where: device or host. */
int spca_omega_used(spca_handle_t h, double *out, int out_where);

/* Column sums of the finished G (l values, float64) — for center_correct. */
int spca_g_colsum(spca_handle_t h, double *out, int out_where);

/* Sketch the rows as normalize_rows would leave them (NormalizedRowStream,
 * sketch.py:142-182): each row minus its mean, divided by its centered norm.
 * Must precede the first push of a pass (SPCA_ERR_STATE otherwise). On the
 * tensor-core path the normalisation is fused into the pass (row shifts and
 * norms folded into G, H and col_sums); on the SIMT path each chunk is
 * normalized into a workspace first. */
int spca_sketch_set_normalize(spca_handle_t h, int on);

/* Column shift: with on != 0 the pass sketches A - 1 c^T, c = the mean of
 * the first (up to 256) rows of the pass's first push (a non-finite mean as
 * 0), and finish adds the shift back in
 * fp64 (G += 1 (Omega^T c)^T, H += col_sums' w^T + c (1^T G')^T + m c w^T, or
 * H += c (1^T L)^T with a co-sketch operand; col_sums += m c), so the results
 * are the sketch of A itself. The fp32 accumulators then hold values of the
 * size of A's deviation from c rather than of A: post-hoc centering
 * (center_correct, sketch.py:119-139) no longer cancels fp32 rounding of a
 * large column mean. Must precede the first push of a pass; exclusive with
 * spca_sketch_set_normalize (SPCA_ERR_CONFIG). */
int spca_sketch_set_shift(spca_handle_t h, int on);

/* Co-sketch operand: with L set (rows x l row-major float64, device or host),
 * the pass accumulates H += A_i^T L[first_row .. first_row + rows(A_i)) in
 * place of A_i^T G_i; G = A Omega and col_sums are formed as usual. This is
 * the second contraction of the reference's other two passes:
 *   legacy_single_pass  Yt += vals^T omega_t[r0:r0+rows]   (algorithms.py:344-346)
 *   basic_rand_svd      B  += q[r0:r0+rows]^T vals          (algorithms.py:247-250, as H = B^T)
 * L is converted like Omega (rounded to float32 for SPCA_F32) and kept by the
 * handle across spca_sketch_reset; spca_center_correct then subtracts
 * mu (1^T L)^T from H (algorithms.py:251-252, 356-357). Must precede the first
 * push of a pass (SPCA_ERR_STATE); pushing more rows than L has fails with
 * SPCA_ERR_CAPABILITY. rows = 0 (or left = NULL) restores the plain sketch. */
int spca_sketch_set_left(spca_handle_t h, const double *left, int64_t rows, int where);

/* normalize_rows (sketch.py:142-153) on device rows: each row minus its
 * mean, divided by its Euclidean norm (a constant row becomes zero), fp64
 * arithmetic; dtype SPCA_F32 / SPCA_F64 for both src and dst (device
 * pointers, row strides in elements; dst may equal src). Enqueued on
 * `stream` (a cudaStream_t, NULL = legacy default); errors are reported
 * through spca_last_error(NULL, ...). */
int spca_normalize_rows(const void *src, int64_t rows, int64_t n, int64_t ld_src, void *dst,
                        int64_t ld_dst, int dtype, void *stream);

/* Last error of the handle (or of the calling thread when h == NULL):
 * code, offending absolute row (or -1) and a message. */
/* ---- post-pass: one block of the blocked QB on the device (fp64) --------
 * Replaces the tall-skinny work of one iteration of blocked_qb
 * (/root/reference/pkg/src/streampca/qb.py:93-118, with qr_unpivoted's
 * CholeskyQR2 form of linalg.py:71-98 for well-conditioned blocks):
 *   y = G_i - Q X (X = B Omega_i, c0 x b, computed by the caller),
 *   Q_i R_i = qr(y), Q_i Rt = qr(Q_i - Q (Q^T Q_i)), R_i <- Rt R_i.
 * Q is m x ldq row-major: columns [0, c0) are read, [c0, c0 + b) written.
 * G_i points at the block's first column (row stride ldg). On return (stream
 * ordered): p_out = [y^T Q | y^T y] (b x (c0 + b), row-major), factors =
 * ten b x b upper-triangular matrices R1, R2, r_i, R3, R4, R_i, R1^-1,
 * R1^-1 R2^-1, R3^-1, R3^-1 R4^-1, then an eleventh b x b scratch whose first
 * two entries flag a skipped second CholeskyQR pass (R2 = I / R4 = I: a block
 * with cond_F(R) <= 16, where one pass is accurate to ~1e-13; SPCA_QB_CQ2=1
 * forces both passes) (R_i = factors[5] feeds the
 * caller's B_i = R_i^-T (H_i^T - (y^T Q) B - (Omega_i^T B^T) B)), and *flag
 * set to 1 if any test of the optimistic path failed (Cholesky breakdown,
 * CholeskyQR2 defect >= 1e-5, |r_jj| < *tol (qb.py:100), solve_rt's
 * singularity guard (linalg.py:131-135)): the caller then redoes the
 * factorization on the general path. Every pointer is device memory; b even,
 * 2 <= b <= 16, c0 even, c0 + b <= 256, ldq and ldg even, 16-byte aligned
 * operands. ws: spca_qb_workspace_elems(m, c0, b) doubles. */
int64_t spca_qb_workspace_elems(int64_t m, int c0_max, int b);
int spca_qb_block(int64_t m, int c0, int b, double *q, int64_t ldq, const double *g, int64_t ldg,
                  const double *x, double *ybuf, double *ws, int64_t ws_elems, double *p_out,
                  double *factors, int *flag, const double *tol, void *stream);

/* ---- the reference's seeded Gaussian draw on the device ----------------
 * Replaces gaussian_matrix (/root/reference/pkg/src/streampca/linalg.py:46-56):
 * writes the first `count` values of numpy's
 *   Generator(Philox(key=[seed, stream])).standard_normal()
 * bit for bit into `out` (device fp64; an n x l Omega is the first n*l values
 * in row-major order). w, k, f, r_tail, inv_r: numpy's ziggurat constants
 * (host arrays of 256; paper_1704_07669_b200/ziggurat.py recovers them).
 * Enqueued on `stream`; returns after one host synchronization (tail values
 * are recomputed on the host with libm's log1p). SPCA_ERR_STATE when the
 * device cannot vouch for every value (a layer or tail test within 1e-12 of
 * its threshold, or the speculative walk failing its chain check): the
 * caller then draws on the host. */
int spca_gaussian_device(double *out, int64_t count, uint64_t seed, uint64_t stream_id, const double *w,
                         const uint64_t *k, const double *f, double r_tail, double inv_r, void *stream);

/* ---- post-pass: the B side of one QB block (qb.py:96 and :115-118) -----
 * spca_qb_omega_proj: X = B[:c0] Omega_i (c0 x b, row-major), B row-major
 * (row stride ldb), omega pointing at column c0 of Omega (row stride ldo);
 * ws: spca_qb_omega_proj_ws(n, c0, b) doubles (fixed-order split-K partials).
 * spca_qb_b_rows: rows [c0, c0 + b) of B,
 *   B_i = R_i^-T (H[:, c0:c0+b]^T - (y^T Q + X^T) B[:c0]),
 * h pointing at column c0 of H (row stride ldh), p_out = spca_qb_block's
 * [y^T Q | y^T y] (b x (c0 + b)), r_i = its factors[5], b_out pointing at
 * row c0 of B (row stride ldb). Device pointers, b even in [2, 16]. */
int64_t spca_qb_omega_proj_ws(int64_t n, int c0_max, int b);
int spca_qb_omega_proj(int64_t n, int c0, int b, const double *bm, int64_t ldb, const double *omega, int64_t ldo,
                       double *x, double *ws, int64_t ws_elems, void *stream);
int spca_qb_b_rows(int64_t n, int c0, int b, const double *bm, int64_t ldb, const double *h, int64_t ldh,
                   const double *p_out, const double *x, const double *r_i, double *b_out, void *stream);

int spca_last_error(spca_handle_t h, int *code, int64_t *bad_row, char *msg,
                    size_t msg_len);

/* Number of kernels this handle launched so far (bench evidence). */
int64_t spca_kernel_launches(spca_handle_t h);

/* Device time (ms) spent in the dominant kernel (the contraction kernels),
 * measured with CUDA events on the handle's stream when timing is enabled. */
int spca_enable_kernel_timing(spca_handle_t h, int enable);
int spca_kernel_time_ms(spca_handle_t h, double *ms, int64_t *launches);

void spca_sketch_destroy(spca_handle_t h);

#ifdef __cplusplus
}
#endif

#endif /* SPCA_H_ */
