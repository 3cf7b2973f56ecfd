/*
 * libstarm -- C ABI of the B200 (sm_100a) t-SVDM hot path.
 *
 * The reference (arxiv 2605.16058 package `starm`, /root/reference/pkg) is
 * pure Python over numpy/scipy; it has no FFI of its own.  These entry
 * points sit UNDER the reference's Python operators and replace the
 * numpy/LAPACK calls each one names.  The Python package
 * paper_2605_16058_b200 binds them with ctypes.
 *
 * Collectives: the multi-GPU split (paper_2605_16058_b200/sharded.py) runs
 * its all-to-all / all-gathers through torch.distributed over NCCL; no entry
 * point here takes an ncclComm_t.  Every kernel below operates on the
 * calling rank's buffers only.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated otherwise; the caller
 *    allocates every buffer (outputs and workspace) and owns it.  Nothing
 *    here allocates or frees caller memory.
 *  - Tensors are column-major (Fortran) float64 exactly like the
 *    reference's DenseTensor (tensor.py:76-98): frontal slice i of an
 *    (m, p, N) tensor is the contiguous m x p column-major block at element
 *    offset i*m*p.
 *  - `stream` is a cudaStream_t passed as void*; every call is
 *    stream-ordered and asynchronous unless documented otherwise.
 *  - Return value: STARM_OK or an error code; the message is available
 *    from starm_last_error().  Per-slice failures (non-finite data,
 *    non-convergence) are reported through a device int32 status pair so
 *    the host can raise the reference's exceptions naming the slice
 *    (slicesvd.py:49-50,58-61).
 */
#ifndef STARM_H_
#define STARM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STARM_ABI_VERSION 1

enum starm_status {
  STARM_OK = 0,
  STARM_INVALID_ARG = 1,      /* -> ValueError                              */
  STARM_NONFINITE_SLICE = 2,  /* -> ValueError("slice {i} contains ...")    */
  STARM_NOCONVERGE = 3,       /* -> np.linalg.LinAlgError                   */
  STARM_CUDA = 4,             /* -> RuntimeError                            */
  STARM_UNSUPPORTED = 5       /* -> ValueError (shape outside kernel range) */
};

/* SVD jobs for starm_svd_f64 */
enum starm_svd_job {
  STARM_SVD_VALUES = 0,     /* slicesvd.py:139-177 svd_values_only            */
  STARM_SVD_FULL = 1,       /* slicesvd.py:115-136 svd_all_slices             */
  STARM_SVD_TRUNCATED = 2,  /* slicesvd.py:259-292 svd_truncated_slices       */
  /* Two-pass form of tsvdm_tolerance (tsvdm.py:268-321): VALUES_STATE is a
   * values pass over every slice that also keeps each slice's factorisation
   * (bidiagonal, logged right-side transformations) in `ws`; a following
   * TRUNCATED_STATE call with the SAME ws, shapes and s computes the packed
   * factors of `slice_ids` from that state without refactoring (the device
   * analogue of the reference's compute-efficient strategy). */
  STARM_SVD_VALUES_STATE = 3,
  STARM_SVD_TRUNCATED_STATE = 4
};

int starm_abi_version(void);

/* Number of kernel launches issued by the library since the last call
 * (CUB device-wide primitives count as one each); resets the counter. */
long long starm_launch_count_reset(void);

/* Copies the calling thread's last error message into buf (NUL-terminated,
 * truncated to len); returns the full message length. */
size_t starm_last_error(char* buf, size_t len);

/* ---------------------------------------------------------------- K1 TTM
 * Replaces ttm.py:113-135 (`_dispatch`, np.matmul -> OpenBLAS DGEMM).
 * View of the column-major buffer: `batch` row-major blocks
 * src[b] (inner x rows), dst[b] (out_cols x rows); computes
 *     dst[b] = mat @ src[b]            for b in [0, batch)
 * with `mat` ROW-MAJOR out_cols x inner (mat[j*inner + l]).  This is the
 * mode-k product of ttm.py:87-104 for rows = prod(dims[:k]),
 * inner = dims[k], batch = prod(dims[k+1:]) (TTMPlan, ttm.py:59-69).
 * FP64 DMMA tiles, cp.async shared-memory staging. */
int starm_ttm_f64(const double* src, const double* mat, double* dst, int64_t rows,
                  int64_t inner, int64_t batch, int64_t out_cols, void* stream);
/* starm_ttm_f64 (batch 1) restricted to the fibre block [f0, f0 + nf): src
 * and dst are the full tensors' buffers (leading dimension `rows`).  The
 * drop-in tsvdm_fixed_rank / tsvdm_tolerance on a host DenseTensor transform
 * each block behind the host-to-device copy of the next. */
int starm_ttm_block_f64(const double* src, const double* mat, double* dst, int64_t rows,
                        int64_t inner, int64_t out_cols, int64_t f0, int64_t nf, void* stream);

/* float32 twin of starm_ttm_f64 (same view and semantics, f32 in / f32
 * out): the operands are upcast on the device and contracted in FP64 on the
 * DMMA path, so the result is the f64 product rounded once to f32 (the
 * reference itself computes in f64: tensor.py:87 upcasts f32 input).
 * ws: starm_ttm_f32_workspace_bytes(rows, inner, batch, out_cols) bytes. */
size_t starm_ttm_f32_workspace_bytes(int64_t rows, int64_t inner, int64_t batch, int64_t out_cols);
int starm_ttm_f32(const float* src, const float* mat, float* dst, int64_t rows, int64_t inner,
                  int64_t batch, int64_t out_cols, void* ws, size_t ws_bytes, void* stream);
/* The DenseTensor upcast (tensor.py:87) on the device: dst[i] = (double)src[i]
 * (lets a float32 tensor cross PCIe at half the bytes). */
int starm_upcast_f32_f64(const float* src, double* dst, int64_t count, void* stream);

/* ------------------------------------------------------- K1b fast DCT
 * The DCT transform of the reference (transforms.py dct matrix applied by
 * the mode-k product, ttm.py:87-104) computed in O(n log n) per fiber:
 * the same (rows, n, batch) column-major view as starm_ttm_f64 with
 * inner = out_cols = n, and mat = the orthonormal DCT-II matrix
 * (inverse = 0) or its transpose, the DCT-III (inverse = 1).  n must be a
 * power of two in [2, 4096] (STARM_UNSUPPORTED otherwise); src != dst. */
int starm_dct_f64(const double* src, double* dst, int64_t rows, int64_t n, int64_t batch,
                  int inverse, void* stream);

/* -------------------------------------------- K1c reference-operator residual
 * The DCT kind of the reference is a DENSE product with the float64 matrix
 * dct_matrix() builds (transforms.py:75-91 applied by ttm.py:113-135).  Its
 * entries differ from the exact DCT-II by Delta (rounding of the cos
 * argument, ~2.4e-14 at n = 1024).  starm_dct_f64 computes the exact
 * transform; this call then adds the residual so the result is the
 * reference's operator applied to src (to a few u):
 *     dst[b] += 2^-log2_scale * (Delta_s @ src[b])       b < batch
 * in the (rows, n, batch) view of starm_dct_f64.  delta_bf16 is the
 * ROW-MAJOR n x n matrix Delta * 2^log2_scale in bfloat16 bits (the scale
 * keeps it in bf16's normal range); the product runs on the tcgen05 tensor
 * cores (kind::f16, fp32 accumulate, TMA-staged), which is exact enough
 * because |Delta| is ~1e-14.  n must be a multiple of 256; ws and
 * delta_bf16 128-byte aligned; ws of starm_ttm_residual_workspace_bytes. */
size_t starm_ttm_residual_workspace_bytes(int64_t rows, int64_t n, int64_t batch);
/* The reference's DCT operator in one call: starm_dct_f64 followed by
 * starm_ttm_residual_bf16 (inverse = 1 takes Delta^T as delta_bf16).  For
 * n = 1024 forward the FFT kernel writes the bf16 operand itself, so the
 * input is read once.  Same workspace as starm_ttm_residual_bf16. */
int starm_dct_residual_f64(const double* src, double* dst, int64_t rows, int64_t n, int64_t batch,
                           int inverse, const uint16_t* delta_bf16, int log2_scale, void* ws,
                           size_t ws_bytes, void* stream);
/* The same two halves separately, so a caller can correct only some output
 * columns (the pruned tolerance path corrects only the slices it keeps):
 * starm_dct_pack_f64 = the exact FFT DCT into dst and the bf16 operand into
 * ws; starm_residual_apply_f64 then adds 2^-e Dsel @ x to dst, where Dsel is
 * an nout x n row-major bf16 matrix (rows of Delta * 2^e, padded with zero
 * rows to a multiple of 256 and 128-byte aligned) and dst holds nout output
 * columns per batch block (dst[b * rows * nout + f + j * rows]). */
int starm_dct_pack_f64(const double* src, double* dst, int64_t rows, int64_t n, int64_t batch,
                       int inverse, void* ws, size_t ws_bytes, void* stream);
/* starm_dct_pack_f64 restricted to the fibre block [f0, f0 + nf) of a
 * (rows x n) tensor (batch 1, forward), transformed where it lies: src, dst
 * and ws are the FULL tensor's buffers.  Blocks start on multiples of 128
 * fibres and end on one or at `rows`; after every block has run the three
 * buffers are exactly those starm_dct_pack_f64 leaves.  The drop-in
 * tsvdm_tolerance(DenseTensor) uses it to transform each block behind the
 * host-to-device copy of the next (the reference's np.matmul in
 * ttm.py:113-135 has the whole tensor in memory at once). */
int starm_dct_pack_block_f64(const double* src, double* dst, int64_t rows, int64_t n, int64_t f0,
                             int64_t nf, void* ws, size_t ws_bytes, void* stream);
int starm_residual_apply_f64(const void* ws, const uint16_t* delta_bf16, int log2_scale,
                             double* dst, int64_t rows, int64_t n, int64_t nout, int64_t batch,
                             void* stream);
int starm_ttm_residual_bf16(const double* src, const uint16_t* delta_bf16, int log2_scale,
                            double* dst, int64_t rows, int64_t n, int64_t batch, void* ws,
                            size_t ws_bytes, void* stream);

/* ------------------------------------------------ data-driven transform
 * G = unfold(k) unfold(k)^T (inner x inner, column-major, exactly
 * symmetric) over the (rows, inner, batch) view of the mode-k product: the
 * Gram matrix whose eigenvectors (starm_svd_f64 on G) are the left singular
 * vectors data_driven_transform takes (transforms.py:94-110).  FP64 DMMA,
 * deterministic split-K.  ws: starm_gram_workspace_bytes bytes. */
size_t starm_gram_workspace_bytes(int64_t rows, int64_t inner, int64_t batch);
int starm_gram_f64(const double* a, int64_t rows, int64_t inner, int64_t batch, double* g, void* ws,
                   size_t ws_bytes, void* stream);

/* ----------------------------------------------------- K11 facewise GEMM
 * Replaces _facewise_matmul (tsvdm.py:205-216): for each slice i,
 *   C_i (m x l) = A_i (m x p) * B_i (p x l), all column-major, slice
 *   strides m*p, p*l, m*l. */
int starm_facewise_gemm_f64(const double* a, const double* b, double* c, int64_t m,
                            int64_t p, int64_t l, int64_t nslices, void* stream);

/* ------------------------------------------------------ K3-K6 slice SVD
 * Replaces _slice_svd/LAPACK dgesvd over slices (slicesvd.py:42-62 and the
 * three drivers named by `job`).  Slices whose 16-column panel fits in
 * shared memory take the bidiagonal path: Householder QR + band reduction
 * (FP64 DMMA compact-WY updates), Householder bulge chasing to upper
 * bidiagonal, bisection for sigma, inverse iteration + back-transformation
 * for vectors.  Others run a blocked one-sided Jacobi SVD (Gram tiles on
 * DMMA).  One CTA per slice, persistent grids, global workspace.
 *
 *  ahat       (m, p, nslices) column-major input, never modified.
 *  slice_ids  optional device int64 list of slices to factor (count
 *             entries); NULL means all slices 0..nslices-1 (count ignored).
 *  s          (r, nslices) column-major singular values, descending per
 *             slice, r = min(m, p).  Required for VALUES/FULL, optional
 *             (may be NULL) for TRUNCATED.
 *  u, v       FULL: (m, r, nslices) and (p, r, nslices) column-major,
 *             slice i reconstructs as u_i diag(s_i) v_i^T (SliceSVDSet).
 *  ranks, u_off, g_off, u_data, g_data
 *             TRUNCATED: packed VariableRankFactors (slicesvd.py:180-256):
 *             u_data[u_off[i] ...] = U_i[:, :k] (m x k col-major),
 *             g_data[g_off[i] ...] = diag(s[:k]) V_i[:, :k]^T (k x p col-major),
 *             k = ranks[i]; offsets from starm_pack_offsets.
 *  status     device int32[2]: status[0] = lowest slice index with a
 *             non-finite entry, status[1] = lowest slice that did not
 *             converge; both INT32_MAX when clean.  Reset by this call.
 *  ws         device workspace of starm_svd_workspace_bytes(m, p, nslices,
 *             count, job) bytes (count = number of slices factored).
 * All-zero slices yield s = 0, U = eye(m, r), V = eye(p, r) (slicesvd.py:51-54). */
size_t starm_svd_workspace_bytes(int64_t m, int64_t p, int64_t nslices, int64_t count, int job);
/* Tuning / diagnostics (process-wide; a value < 0 leaves a knob unchanged):
 * inner Jacobi sweeps per pair step (default 1), sweep cap (60), values
 * path (1 = QR + band reduction + bulge chasing + bisection whenever a
 * 16-column panel of the slice fits in shared memory, 0 = Jacobi only,
 * 2 = as 1 with the bulge-chase window in global memory, 3 = diagnostic
 * for timing the band-reduction kernel alone: the call returns after it
 * with undefined outputs), kernel counters on/off.  starm_svd_stats copies 16 counters (slices,
 * sweeps, pairs, rotated pairs, cycles in gram / eig / apply / qr /
 * finalize / load / band / bulge) to host memory, synchronising the device. */
int starm_svd_tune(int max_inner, int max_sweeps, int mode, int stats);
int starm_svd_stats(unsigned long long* host16, int reset);
int starm_svd_f64(const double* ahat, int64_t m, int64_t p, int64_t nslices,
                  const int64_t* slice_ids, int64_t count, int job, double* s, double* u,
                  double* v, const int64_t* ranks, const int64_t* u_off, const int64_t* g_off,
                  double* u_data, double* g_data, int32_t* status, void* ws, size_t ws_bytes,
                  void* stream);

/* -------------------------------------------------------- K7 threshold
 * Replaces compute_threshold (tsvdm.py:85-115) with identical semantics:
 * squares, ascending sort, SEQUENTIAL running sums (np.cumsum), j =
 * searchsorted(w, eps^2*total, 'left'), tau = v[j-1], strict keep
 * sq > tau, discarded = numpy pairwise sum of the dropped squares in
 * C order of the (r, N) matrix, tie-retain rule, ranks per slice.
 *  s          (r, nslices) column-major, finite, >= 0, each column
 *             descending (as produced by starm_svd_f64).
 *  v_out,w_out optional (may be NULL) r*nslices sorted squares / sums.
 *  ranks_out  int64[nslices].
 *  scal_out   double[3] = {tau, discarded, total};  j_out int64[1].
 * Output scalars are device-resident; the call is asynchronous. */
size_t starm_threshold_workspace_bytes(int64_t r, int64_t nslices);
int starm_threshold_f64(const double* s, int64_t r, int64_t nslices, double epsilon,
                        double* v_out, double* w_out, int64_t* ranks_out, double* scal_out,
                        int64_t* j_out, void* ws, size_t ws_bytes, void* stream);

/* Pruned form of the same threshold for tsvdm_tolerance: `s` holds the
 * singular values of a SUBSET of the slices; the left-out slices have total
 * energy e0 and every one of their sigma^2 is <= tbound (callers use the
 * slice's Frobenius norm squared, starm_slice_energy_f64).  The running sum
 * starts at e0, total = e0 + sum of the subset's squares, discarded
 * includes e0.  cert_out (device int32) = 1 when the crossing value v[j]
 * exceeds tbound: then every value <= tbound is discarded by the reference's
 * rule whatever its exact size, so the left-out slices have rank 0 and the
 * subset's ranks are the reference's.  cert_out = 0: recompute unpruned.
 * Same workspace as starm_threshold_f64 for (r, nslices). */
int starm_threshold_pruned_f64(const double* s, int64_t r, int64_t nslices, double epsilon,
                               double e0, double tbound, int64_t* ranks_out, double* scal_out,
                               int64_t* j_out, int32_t* cert_out, void* ws, size_t ws_bytes,
                               void* stream);

/* Per-slice energy f[i] = ||slice i||_F^2 (slice_elems contiguous doubles per
 * slice), deterministic: the bound sigma_max^2 <= f used for pruning. */
int starm_slice_energy_f64(const double* a, int64_t slice_elems, int64_t nslices, double* f_out,
                           void* stream);

/* Partial energies over the fibre block [f0, f0 + nf) of every slice
 * (f_out[i] = sum_{f0 <= q < f0 + nf} a[i * slice_elems + q]^2). */
int starm_slice_energy_block_f64(const double* a, int64_t slice_elems, int64_t nslices, int64_t f0,
                                 int64_t nf, double* f_out, void* stream);

/* Strided host-to-device copy (cudaMemcpy2DAsync, pitches and width in
 * bytes): one fibre block of a host DenseTensor (tensor.py:76-98 layout)
 * into the same place of its device copy; asynchronous for page-locked
 * host memory. */
int starm_copy2d_h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                     size_t height, void* stream);

/* ---------------------------------------------------------- K8 offsets
 * slicesvd.py:208-211: u_off[0]=g_off[0]=0, u_off[i+1] = u_off[i] +
 * ranks[i]*m, g_off likewise with p.  Arrays hold nslices+1 int64. */
int starm_pack_offsets(const int64_t* ranks, int64_t nslices, int64_t m, int64_t p,
                       int64_t* u_off, int64_t* g_off, void* stream);

/* ------------------------------------------- K9 facewise reconstruction
 * tsvdm.py:346-355: chat_i = U_i G_i for ranks[i] > 0, zero otherwise.
 * chat is (m, p, nslices) column-major and fully overwritten. */
int starm_unpack_facewise_f64(const double* u_data, const double* g_data, const int64_t* ranks,
                              const int64_t* u_off, const int64_t* g_off, int64_t m, int64_t p,
                              int64_t nslices, double* chat, void* stream);

/* ---------------------------------------------------- K10 error sums
 * out2[0] = sum (a - b)^2, out2[1] = sum a^2 over `count` elements, with a
 * fixed (deterministic) reduction tree.  Used for the relative
 * reconstruction error of tests/helpers.py:44-47 and cli.py:185-197. */
size_t starm_error_sums_workspace_bytes(int64_t count);
int starm_error_sums_f64(const double* a, const double* b, int64_t count, double* out2,
                         void* ws, size_t ws_bytes, void* stream);


/* ------------------------------ K9 + inverse transform + K10, fused (3-way)
 * Replaces reconstruct (tsvdm.py:342-357) followed by the relative error of
 * tests/helpers.py:44-47 / cli.py:185-197, in one stream-ordered call:
 *     chat_i = U_i G_i                   for the nnz slices in nz_ids (ranks > 0)
 *     out_(3) = minv @ chat_(3)          (only the nnz columns of minv meet a
 *                                         nonzero slice: a K = nnz DMMA GEMM)
 *     err2 = {sum (a - out)^2, sum a^2}  accumulated in that GEMM's epilogue
 *                                         (deterministic), when a != NULL
 *  minv   ROW-MAJOR n x n inverse operator: M^T for an orthonormal M (what
 *         from_transform_domain applies, ttm.py:147-153; for the DCT kind the
 *         reference's own dense matrix, not the exact DCT-III), or an explicit
 *         M^-1 (the config-4 restatement).
 *  nz_ids device int64 list of the nnz slices with ranks > 0 (any order);
 *         nnz = 0 writes zeros.  out is the (m, p, n) tensor (m*p*n doubles).
 *  ws     starm_reconstruct_workspace_bytes(m, p, n, nnz) bytes. */
size_t starm_reconstruct_workspace_bytes(int64_t m, int64_t p, int64_t n, int64_t nnz);
int starm_reconstruct_f64(const double* u_data, const double* g_data, const int64_t* ranks,
                          const int64_t* u_off, const int64_t* g_off, int64_t m, int64_t p,
                          int64_t n, const int64_t* nz_ids, int64_t nnz, const double* minv,
                          const double* a, double* out, double* err2, void* ws, size_t ws_bytes,
                          void* stream);

/* ------------------------------------------------- K8b pack from full
 * _pack_from_full (tsvdm.py:324-339): from full factors (s (r,N), u
 * (m,r,N), v (p,r,N)) write u_data block i = u_i[:, :k] and g_data block
 * i = diag(s_i[:k]) v_i[:, :k]^T, k = ranks[i].  With ranks == r it also
 * forms the operands of the lossless full_tsvdm reconstruction
 * (tsvdm.py:190-202). */
int starm_pack_from_full_f64(const double* s, const double* u, const double* v, int64_t m,
                             int64_t p, int64_t nslices, const int64_t* ranks,
                             const int64_t* u_off, const int64_t* g_off, double* u_data,
                             double* g_data, void* stream);

/* ------------------------------------------------ fixed-rank energies
 * tsvdm.py:260-262: out2[0] = sum_{j >= rank} s[j,i]^2 (discarded),
 * out2[1] = sum s^2 (total), deterministic single-CTA reduction. */
int starm_tail_energy_f64(const double* s, int64_t r, int64_t nslices, int64_t rank,
                          double* out2, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STARM_H_ */
