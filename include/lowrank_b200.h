/*
 * lowrank_b200 -- C ABI of the B200-native randomized range finder / SVD.
 *
 * This is the drop-in boundary for the passes over A of the reference
 * package `lowrank` (/root/reference/pkg/src/lowrank).  The reference is
 * pure Python; its plug-in point is the MatVecOperator protocol
 * (core.py:343-380) plus the dense kernels the range finders call.  Each
 * entry point below replaces one of those call sites; the Python package
 * paper_0909_4061_b200 binds them with ctypes (INTEGRATION.md shows the
 * binding a maintainer of the reference would add).
 *
 * Conventions
 *   - All matrices are row-major (C order, as numpy arrays in the
 *     reference); `ld*` is the row stride in elements.
 *   - All pointers are device pointers owned by the caller; the library
 *     never frees caller memory.  Scratch comes from a handle-owned pool.
 *   - Every call is stream-ordered and asynchronous on the handle's stream
 *     unless documented as synchronizing (composites that must make a
 *     host-side decision say "syncs").
 *   - Return value: LR_OK (0) or an lr_status code; lr_last_error() gives a
 *     thread-local message.  Codes map to the reference's exceptions:
 *     LR_EINVAL -> ValueError, LR_ECONV -> ConvergenceError (core.py:25-30).
 *   - One handle per (host thread, device); handles are not thread-safe.
 */
#ifndef LOWRANK_B200_H
#define LOWRANK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LR_ABI_VERSION 1

typedef struct lr_handle_s* lr_handle_t;

typedef enum { LR_F32 = 0, LR_F64 = 1, LR_C64 = 2, LR_C128 = 3 } lr_dtype_t;
typedef enum { LR_OP_N = 0, LR_OP_T = 1, LR_OP_C = 2 } lr_op_t;
typedef enum {
  LR_OK = 0,
  LR_EINVAL = 1,       /* ValueError */
  LR_ECONV = 2,        /* ConvergenceError */
  LR_ENOTPSD = 3,      /* NotPSDError */
  LR_ECUDA = 4,        /* CUDA runtime failure */
  LR_ENOMEM = 5,       /* device allocation failed */
  LR_EUNSUPPORTED = 6  /* dtype/shape combination not built */
} lr_status_t;

/* fp32 GEMM arithmetic schemes (LR_F32 only) */
typedef enum {
  LR_F32_SPLIT3 = 0,   /* default: 3-product split on tcgen05 kind::f16 */
  LR_F32_SIMT = 1      /* plain fp32 FFMA (reference arithmetic check) */
} lr_f32_mode_t;

int lr_abi_version(void);
const char* lr_last_error(void);
/* Number of kernels this library has launched in the process (evidence
 * for bench.py's "gpu_launches"). */
uint64_t lr_launch_count(void);

/* Handle: device + stream + scratch pool.  `stream` is a cudaStream_t (or
 * NULL for the legacy default stream). */
int lr_create(int device, void* stream, lr_handle_t* out);
int lr_destroy(lr_handle_t h);
int lr_set_stream(lr_handle_t h, void* stream);
int lr_set_f32_mode(lr_handle_t h, int mode);
/* Bytes currently reserved by the scratch pool. */
int64_t lr_workspace_bytes(lr_handle_t h);
/* Scratch-pool generation: incremented whenever pool chunks are freed
 * (the pool merges its chunks after a call outgrew it).  Work captured in a
 * CUDA graph holds raw pool addresses, so a graph recorded at generation g
 * must not be replayed once the handle's generation differs. */
uint64_t lr_pool_generation(lr_handle_t h);
/* Pre-size the scratch pool (needed before CUDA-graph capture). */
int lr_reserve(lr_handle_t h, int64_t bytes);

/* K1/K2 -- one pass over A (replaces DenseOperator._apply / _apply_adjoint,
 * reference core.py:391-395):
 *   op = LR_OP_N :  Y (m x ell)  = A   (m x n) . X (n x ell)
 *   op = LR_OP_T :  Y (n x ell)  = A^T (n x m) . X (m x ell)
 *   op = LR_OP_C :  Y (n x ell)  = A^H (n x m) . X (m x ell)
 * Deterministic: split-K partials are reduced in a fixed order. */
int lr_gemm(lr_handle_t h, int dtype, int op, int64_t m, int64_t n, int64_t ell,
            const void* A, int64_t lda, const void* X, int64_t ldx,
            void* Y, int64_t ldy);

/* lr_gemm for a pass over an operator whose max |a_ij| is known (from the
 * as_matrix validation pass, lr_check_finite): fp32 / complex64 passes run
 * on the tcgen05 tensor cores with the three-product scaled-fp16 split
 * (DESIGN.md "fp32 passes"); a_amax < 0 means unknown (computed here, one
 * extra read of A).  fp64 / complex128 behave exactly like lr_gemm. */
int lr_gemm_scaled(lr_handle_t h, int dtype, int op, int64_t m, int64_t n, int64_t ell,
                   const void* A, int64_t lda, double a_amax, const void* X, int64_t ldx,
                   void* Y, int64_t ldy);

/* A pass over an fp32 A with exact products and fp64 accumulation (DMMA on
 * fp32 operands widened at fragment load): Y (fp64) = A X (op N) or A^T X
 * (op T), X fp32.  The posterior estimator's narrow pass (reference
 * posterior_error_estimate, rangefinder.py:65-82, r = 10 probes) uses it for
 * fp32 operators: the residual it measures is ~1e-5 of |A w| at config 4,
 * below the tensor-core split's rounding. */
int lr_gemm_f64acc(lr_handle_t h, int op, int64_t m, int64_t n, int64_t ell, const float* A,
                   int64_t lda, const float* X, int64_t ldx, double* Y, int64_t ldy);

/* fp64 passes on the int8 tensor cores (Ozaki digit slicing, exact int32
 * products; accuracy of an fp64 GEMM, bitwise deterministic).  Replaces the
 * same reference call as lr_gemm (DenseOperator._apply / _apply_adjoint,
 * core.py:391-395) for float64 A.  lr_ozaki_prepare builds, once per
 * operator, the 8 int8 digit planes of A as the two tiled shared-memory
 * images the pass kernel streams (planes: 16 x MP x ldp bytes, MP = m and
 * ldp = n rounded up to multiples of 256, device memory owned by the
 * caller) and the
 * row exponents (row_exp: m int32).  The digits are fixed-point relative to
 * each row's maximum: |error_ij| <= 2^-50 max_k|A_ik| sum_k|X_kj| (fp64
 * accuracy relative to the row scale).  wide_rows (device int32, nullable,
 * accumulated with +=) counts graded rows -- more than 1/8 of the nonzeros
 * below 2^-32 of the row maximum; for such a matrix the caller keeps the
 * passes on lr_gemm (DMMA, error relative to |A||X| entrywise).  lr_gemm_ozaki then computes
 * Y = A X (op N: X n x ell, Y m x ell) or Y = A^T X (op T: X m x ell,
 * Y n x ell), ell <= 256, from the planes. */
int lr_ozaki_prepare(lr_handle_t h, int64_t m, int64_t n, const double* A, int64_t lda,
                     int8_t* planes, int64_t ldp, int32_t* row_exp, int32_t* wide_rows);
/* lr_ozaki_prepare for rows [i0, i1) only (A still points at row 0; i0 a
 * multiple of 128, i1 a multiple of 128 or m): a row-chunked upload prepares
 * each chunk as it arrives; the chunk ending at m also zero-fills the padding. */
int lr_ozaki_prepare_rows(lr_handle_t h, int64_t m, int64_t n, int64_t i0, int64_t i1,
                          const double* A, int64_t lda, int8_t* planes, int64_t ldp,
                          int32_t* row_exp, int32_t* wide_rows);
int lr_gemm_ozaki(lr_handle_t h, int op, int64_t m, int64_t n, int64_t ell,
                  const int8_t* planes, int64_t ldp, const int32_t* row_exp, const double* X,
                  int64_t ldx, double* Y, int64_t ldy);

/* Gram matrix G = Y^H Y (ell x ell), accumulated in fp64 (real dtypes) or
 * complex128 (complex dtypes) regardless of the input precision.  G is
 * written as double / double2 row-major with leading dimension ell.  Used
 * by lr_orth and, between ranks, by the row-sharded path (all-reduce of G). */
int lr_gram(lr_handle_t h, int dtype, int64_t m, int64_t ell,
            const void* Y, int64_t ldy, void* G);

/* Gram of an fp32 panel on the tcgen05 tensor cores, G (ell x ell fp64,
 * row-major) = Y^T Y, at fp32-level accuracy: Y scaled by 2^log2_scale and
 * split into fp16 hi + lo, fp32 accumulation in TMEM per row block, the
 * blocks summed in fp64.  Used for the second CholeskyQR pass of an fp32
 * panel (reference orthonormalize_double_gs, core.py:84-115, whose second
 * projection it replaces); an entry with |y| 2^log2_scale >= 2^15 sets bit 1
 * of *status (device int32, nullable).  ell <= 256, m >= 4096. */
int lr_gram_tc(lr_handle_t h, int64_t m, int64_t ell, const float* Y, int64_t ldy, double* G,
               int log2_scale, int32_t* status);

/* Cholesky with column deletion on a Gram matrix G = Y^H Y (fp64 / c128,
 * row-major) -- the rank decision of orthonormalize_double_gs (reference
 * core.py:104-106); the pivot d_j is the squared residual of column j after
 * projection onto the kept columns before it.  With t = trace(G) = ||Y||_F^2:
 *   G_jj += shift_coef * t                 (shifted CholeskyQR; 0 = none)
 *   d_j <= drop_tol^2 * t (or non-finite)  -> column j dropped
 *   d_j <= unres_rel * G_jj (kept)         -> counted as unresolved (too small
 *                                             to be trusted from a Gram; the
 *                                             caller falls back to CGS2)
 * Outputs (device): P (ell x ell, row-major, ld ell): Q = Y . P[:, :rank];
 * R (ell x ell upper, kept rows/cols only, others 0); info[0] = rank,
 * info[1] = unresolved pivots, info[2] = non-finite pivots.  Async.  Used
 * by the row-sharded path on an all-reduced G. */
int lr_chol_drop(lr_handle_t h, int dtype, int64_t ell, const void* G,
                 double drop_tol, double unres_rel, double shift_coef,
                 void* P, void* R, int32_t* info);

/* PSD Cholesky of the reference (cholesky, core.py:249-272) as used by
 * eig_nystrom (factor.py:300-335): G (ell x ell, fp64/complex128, Hermitian)
 * = C^H C with pivots in [-neg_tol, 0] clamped to zero (zero row of C) and
 * positive pivots kept; info[3] = number of pivots below -neg_tol (the
 * caller raises NotPSDError / takes the eigen fallback).  P = C~^{-1}
 * uncompacted: column j zero for a clamped pivot j, so A Q P is the
 * reference's F = B1 C^{-1} with solve_triangular_trunc's zero components.
 * info: {rank, 0, non-finite pivots, pivots < -neg_tol}.  ell <= 200 real /
 * 140 complex (LR_EUNSUPPORTED above). */
int lr_chol_psd(lr_handle_t h, int dtype, int64_t ell, const void* G, double neg_tol,
                void* P, void* R, int32_t* info);

/* Hermitian part of a small matrix (small_eig_hermitian symmetrizes,
 * core.py:239-240): H = (B + B^H)/2 + s I with s = shift_mult ||(B+B^H)/2||_F
 * (s = 1 for a zero matrix when shift_mult > 0); out2[0] = s, and with
 * power_iters > 0 out2[1] = ||(B+B^H)/2||_2 by power iteration (the scale of
 * the reference's PSD tolerance, core.py:259).  fp64 / complex128. */
int lr_herm_prep(lr_handle_t h, int dtype, int64_t n, const void* B, int64_t ldb, void* H,
                 double shift_mult, int power_iters, double* out2);

/* Eigenpairs from the SVD of the shifted SPD matrix H = U diag(S) U^H:
 * lam = S - *shift ordered as the reference's small_eig_hermitian
 * (core.py:245: descending |lam|, ties descending lam), V the matching
 * columns of U.  fp64 / complex128. */
int lr_eig_finish(lr_handle_t h, int dtype, int64_t n, const double* S, const double* shift,
                  const void* U, double* lam, void* V);

/* Host-sync-free lr_chol_drop for pipelines that decide later (the
 * row-sharded orthonormalization, dist.py): flags as lr_orth_fast are ORed
 * into *status (device int32): 1 = unresolved pivot, 2 = column dropped,
 * 4 = non-finite.  near_thr > 0 (with shift_coef == 0) takes the first-order
 * factor of a near-identity Gram (second CholeskyQR pass) when
 * max |G - I| <= near_thr, the exact factorization otherwise -- decided on
 * the device. */
int lr_chol_drop_fast(lr_handle_t h, int dtype, int64_t ell, const void* G,
                      double drop_tol, double unres_rel, double shift_coef, double near_thr,
                      void* P, void* R, int32_t* info, int32_t* status);

/* Orthonormalize the columns of Y (m x ell) -- replaces
 * orthonormalize_double_gs (reference core.py:84-115).  CholeskyQR2 with a
 * fp64 Gram; guarded fallbacks (shifted CholeskyQR3, then column-wise CGS2
 * on the device) when pivots cannot be resolved.  Writes Q (m x rank) into
 * Q (ld ldq, may alias Y) and the rank into *rank_out.  Syncs. */
int lr_orth(lr_handle_t h, int dtype, int64_t m, int64_t ell, const void* Y, int64_t ldy,
            void* Q, int64_t ldq, double tol, int64_t* rank_out);

/* Speculative (host-sync-free) variant of lr_orth for pipelines that are
 * enqueued ahead / captured in a CUDA graph: CholeskyQR2 with the drop rule
 * and the pivot-resolvability test evaluated on the device.  Writes Q
 * (m x ell) and ORs flags into *status (device int32): 1 = a pivot too
 * small to be resolved from the Gram, 2 = a column was dropped, 4 =
 * non-finite input.  status == 0 afterwards means Q is exactly what lr_orth
 * returns with rank == ell; otherwise the caller re-runs with lr_orth.
 * Q must not alias Y. */
int lr_orth_fast(lr_handle_t h, int dtype, int64_t m, int64_t ell, const void* Y, int64_t ldy,
                 void* Q, int64_t ldq, double tol, int32_t* status);
/* lr_orth_fast without its last product: Q1 (m x ell, ld ell, dtype) and P2
 * (ell x ell, float64 / complex128) with Q = Q1 P2.  For a subspace step
 * whose next product is A^H Q the caller forms (A^H Q1) P2 on the n side.
 * Same speculative flags as lr_orth_fast in *status. */
int lr_orth_fast_deferred(lr_handle_t h, int dtype, int64_t m, int64_t ell, const void* Y,
                          int64_t ldy, void* Q1, void* P2, double tol, int32_t* status);

/* Speculative variant of lr_small_svd (no host sync; Bh is not modified);
 * flags as lr_orth_fast plus 8 = Jacobi sweep limit reached. */
int lr_small_svd_fast(lr_handle_t h, int dtype, int64_t ell, int64_t ncols, const void* Bh,
                      void* U, double* S, void* V, int32_t* status);

/* Small SVD of B (ell x ncols, ell <= ncols) given through Bh = B^H
 * (ncols x ell, row-major) -- which is exactly what the adjoint pass of
 * direct_svd produces (reference factor.py:163-164, core.py:199-230).
 * Outputs: U (ell x ell), S (ell, double), V (ncols x ell) with
 * B = U diag(S) V^H, S descending, and the reference sign convention (first
 * entry with |u| > 1e-10 max|u| of each U column real positive).  Bh is
 * overwritten.  Syncs. */
int lr_small_svd(lr_handle_t h, int dtype, int64_t ell, int64_t ncols,
                 void* Bh, void* U, double* S, void* V);

/* One-sided Jacobi SVD of a square ell x ell matrix M (row-major):
 * M = W diag(S) J^H.  Outputs W, S (descending), J, sign-fixed so that J's
 * columns follow the reference convention.  info[0] = sweeps used
 * (negative if not converged). */
int lr_jacobi_svd(lr_handle_t h, int dtype, int64_t ell, const void* M,
                  void* W, double* S, void* J, int32_t* info);

/* Posterior estimator tail (reference rangefinder.py:79-82): given
 * Z = A W (m x r) and Q (m x k), compute
 * alpha sqrt(2/pi) max_i ||(I - QQ^H) z_i|| into *est (device double). */
int lr_estimate_tail(lr_handle_t h, int dtype, int64_t m, int64_t k, int64_t r,
                     const void* Q, int64_t ldq, void* Z, int64_t ldz,
                     double alpha, double* est);

/* SRFT sketch (reference sketch.py:306-320): for complex A (m x n, any n),
 * Y[:, t] = scale * (F_unitary (A_i * d))[picks[t]]. */
int lr_srft(lr_handle_t h, int dtype, int64_t m, int64_t n, int64_t ell,
            const void* A, int64_t lda, const void* d, const int32_t* picks,
            double scale, void* Y, int64_t ldy);

/* lr_srft given the operator's max |a| (from lr_check_finite).  complex64
 * with ell <= 128 runs the SRFT as one tensor-core pass over A against the
 * ell picked columns of diag(d) F (the lr_gemm_scaled kernel); a_amax < 0
 * means unknown (reduced on the device). */
int lr_srft_scaled(lr_handle_t h, int dtype, int64_t m, int64_t n, int64_t ell,
                   const void* A, int64_t lda, double a_amax, const void* d,
                   const int32_t* picks, double scale, void* Y, int64_t ldy);

/* The ell picked columns of the Givens-chain SRFT (reference
 * sketch.py:221-337, gsrft_operator / gsrft_apply):
 *   Omega = D_outer Theta_outer D_mid Theta_inner D_inner F R scale,
 *   Theta = P G_0 ... G_{n-2} (row-vector convention: x -> x[:, perm], then
 *   column pairs (i, i+1) rotated by [[cos t_i, sin t_i], [-sin t_i, cos t_i]]).
 * Inputs (device): d_* complex128 (n), perm_* int32 (n), thetas_* double
 * (n-1), picks int32 (ell).  Output X (n x ell, row-major, dtype LR_C64 or
 * LR_C128) such that gsrft_apply(A) = A X (one lr_gemm_scaled pass). */
int lr_gsrft_matrix(lr_handle_t h, int dtype, int64_t n, int64_t ell, const void* d_outer,
                    const int32_t* perm_outer, const double* thetas_outer, const void* d_mid,
                    const int32_t* perm_inner, const double* thetas_inner, const void* d_inner,
                    const int32_t* picks, double scale, void* X);

/* Unitary DFT of each row of X (rows x n, any n), in place (reference
 * sketch.py:179-200; radix-2 FFT for powers of two, the dense DFT product
 * otherwise -- the linear map of the reference's Bluestein path). */
int lr_dft_rows(lr_handle_t h, int dtype, int64_t rows, int64_t n, void* X, int64_t ldx);

/* CSR SpMM (config 5): Y (m x ell) = S . X (n x ell) with int64 row
 * pointers and int32 column indices.  For S^T . X pass the CSR of S^T. */
int lr_csr_spmm(lr_handle_t h, int dtype, int64_t m, int64_t n, int64_t ell,
                const int64_t* rowptr, const int32_t* colidx, const void* vals,
                const void* X, int64_t ldx, void* Y, int64_t ldy, int accumulate);

/* Input validation of as_matrix (reference core.py:44-49) fused with a max
 * |a| reduction: info[0] = number of non-finite entries, amax[0] = max |a|. */
int lr_check_finite(lr_handle_t h, int dtype, int64_t m, int64_t n, const void* A,
                    int64_t lda, int64_t* nonfinite, double* amax);

/* dst (rows x cols, dst_dtype) = src (src_dtype), or src^H when
 * conj_transpose (then src is cols x rows).  Real -> complex casts zero the
 * imaginary part.  Layout plumbing for the Python layer (e.g. B -> B^H for
 * small_svd, reference core.py:211). */
int lr_copy(lr_handle_t h, int src_dtype, const void* src, int64_t lds, int dst_dtype,
            void* dst, int64_t ldd, int64_t rows, int64_t cols, int conj_transpose);

/* Reference sign convention on U (rows x cols): the first entry of each
 * column with |u| > 1e-10 max|u| is rotated onto the positive real axis and
 * V's matching column absorbs the same phase (core.py:221-229). */
int lr_sign_fix(lr_handle_t h, int dtype, int64_t rows, int64_t vrows, int64_t cols, void* U,
                int64_t ldu, void* V, int64_t ldv);

/* max |imag(Y)| over a complex matrix (fast_range_finder's
 * diagnostics["max_imag_sample"], reference rangefinder.py:261-262). */
int lr_max_abs_imag(lr_handle_t h, int dtype, int64_t m, int64_t n, const void* Y, int64_t ldy,
                    double* out);

/* The reference's Gaussian draws on the device (replaces the host draw of
 * gaussian_matrix, reference sketch.py:32-42,96-100, and of the estimator
 * probes, rangefinder.py:78): writes the first `count` values of numpy's
 * Generator(Philox(key)).standard_normal stream -- Philox4x64-10 with the
 * 128-bit key (key_lo = seed, key_hi = stream | index << 32) and numpy's
 * 256-layer ziggurat -- as f64 or f32 (rounded like numpy's astype).
 * Flags ORed into *status (device, may be NULL): 16 = a tail attempt
 * exceeded 63 draws, 32 = internal stream margin too short.  Async. */
int lr_gaussian(lr_handle_t h, uint64_t key_lo, uint64_t key_hi, int64_t count, int dtype,
                void* out, int32_t* status);

/* Row interpolative decomposition M ~= X M[J, :] (reference row_id /
 * _column_id, factor.py:198-246, with the Businger-Golub pivoted QR of
 * core.py:133-186): M m x ncols (float64 / complex128, row-major, ldm),
 * k <= ncols skeleton rows, perm
 * (device int32, m): out = the column order of B = M^H (perm[:k] = J);
 * forced = 1 takes perm as the given order (the Gu-Eisenstat refinement's
 * recomputation).  X m x k (ldx): X[J] = I, X[free] = (R11^{-1} R12)^H with
 * truncated back substitution (rows |r_ii| <= 1e-12 max give zero);
 * *tmax (device double) = max |X[free]|, the refinement test. */
int lr_row_id(lr_handle_t h, int dtype, int64_t m, int64_t ncols, int64_t k, const void* M,
              int64_t ldm, int32_t* perm, int forced, void* X, int64_t ldx, double* tmax);

/* Collectives for the row-sharded path without torch.distributed (SURVEY.md
 * §8b/§8e; reference analogue: the row-block sums of
 * accumulate_two_sided_samples, io.py:364-388, turned into all-reduces).
 * Rank r holds rows of A; the passes A_r X are local (lr_gemm), A^H Y is the
 * sum of the ranks' n x ell partials (lr_comm_allreduce), and a row-sharded
 * m x ell panel is orthonormalized by lr_orth_sharded: CholeskyQR2 with both
 * Grams all-reduced, every rank computing the same factors.  NCCL is loaded
 * at run time (libnccl.so.2).
 *   lr_comm_unique_id: LR_COMM_ID_BYTES bytes on rank 0, shared by the caller;
 *   lr_comm_init:      attach a communicator of nranks to the handle;
 *   lr_comm_allreduce: in-place sum of count float64 / complex128 elements
 *                      on the handle's stream;
 *   lr_orth_sharded:   the speculative orthonormalization (flags as
 *                      lr_orth_fast, identical on every rank). */
#define LR_COMM_ID_BYTES 128
int lr_comm_unique_id(void* id_out);
int lr_comm_init(lr_handle_t h, const void* id, int nranks, int rank);
int lr_comm_destroy(lr_handle_t h);
int lr_comm_allreduce(lr_handle_t h, int dtype, int64_t count, void* buf);
int lr_orth_sharded(lr_handle_t h, int dtype, int64_t m_local, int64_t ell, const void* Y,
                    int64_t ldy, void* Q, int64_t ldq, double tol, int32_t* status);

/* One-pass sketches (reference io.py:364-388 accumulate_two_sided_samples,
 * factor.py:364-401 svd_one_pass_general):
 *   lr_axpy_add:      Z (rows x cols) += T    (fp64 / complex128) -- the
 *                     row-block accumulation Y~ += block^H Omega~[rows];
 *   lr_sylvester_div: C_ij /= (d2_i + d1_j), 0 where the sum <= floor -- the
 *                     diagonalized normal equations B (P P^H) + (S S^H) B = C
 *                     of the one-pass least-squares problem.
 * d1, d2: device float64; C row-major k x kt (ldc). */
int lr_axpy_add(lr_handle_t h, int dtype, int64_t rows, int64_t cols, const void* T,
                int64_t ldt, void* Z, int64_t ldz);
int lr_sylvester_div(lr_handle_t h, int dtype, int64_t k, int64_t kt, void* C, int64_t ldc,
                     const double* d2, const double* d1, double floor);

/* BLAS-1 helpers for the column-wise paths (device CGS2 / the unsafeguarded
 * Gram-Schmidt of power_iteration_range(safeguarded=False), reference
 * rangefinder.py:169-184):  Z -= T;  out[j] = sum_i |Z_ij|^2 (fp64, fixed
 * reduction order);  dst[:, 0] = src[:, 0] * inv. */
int lr_axpy_sub(lr_handle_t h, int dtype, int64_t rows, int64_t cols, const void* T, int64_t ldt,
                void* Z, int64_t ldz);
int lr_col_sumsq(lr_handle_t h, int dtype, int64_t m, int64_t r, const void* Z, int64_t ldz,
                 double* out);
int lr_scale_col(lr_handle_t h, int dtype, int64_t rows, const void* src, int64_t lds, double inv,
                 void* dst, int64_t ldd);

#ifdef __cplusplus
}
#endif

#endif /* LOWRANK_B200_H */
