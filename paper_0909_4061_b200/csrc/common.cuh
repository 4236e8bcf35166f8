// Shared runtime pieces of liblowrank_b200: handle, scratch pool, errors.
#pragma once

#include <cuda_runtime.h>
#include <cuComplex.h>
#include <stdint.h>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lowrank_b200.h"

namespace lr {

// ---------------------------------------------------------------------------
// errors: thread-local message + status code

void set_error(const std::string& msg);
const char* get_error();

struct Error {
  int code;
  std::string msg;
};

#define LR_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::lr::Error{LR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

extern unsigned long long g_launches;
#define LR_CHECK_LAUNCH()                 \
  do {                                    \
    __atomic_add_fetch(&::lr::g_launches, 1ULL, __ATOMIC_RELAXED); \
    LR_CUDA(cudaGetLastError());          \
  } while (0)

#define LR_REQUIRE(cond, code, msg)              \
  do {                                           \
    if (!(cond)) throw ::lr::Error{(code), (msg)}; \
  } while (0)

// ---------------------------------------------------------------------------
// handle + scratch pool.  The pool is a list of device chunks with a bump
// pointer; reset() at the start of every API call rewinds it (stream order
// makes reuse across calls safe).  If one call needs more than the current
// chunk, a new chunk is appended; at the next reset the chunks are merged
// into one (after a stream sync), so steady state is one cudaMalloc total.

struct Pool {
  struct Chunk {
    char* base;
    size_t size;
  };
  std::vector<Chunk> chunks;
  size_t cur = 0;     // index of chunk in use
  size_t off = 0;     // bump offset within chunk
  size_t peak = 0;    // bytes needed by the largest call so far
  size_t used = 0;    // bytes handed out in this call
  // bumped whenever chunks are freed (merge at reset): a CUDA graph captured
  // over this pool's addresses is stale once the generation moves
  uint64_t generation = 0;
};

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  int f32_mode = LR_F32_SPLIT3;
  Pool pool;
  int32_t* status = nullptr;   // speculative-path flags (device, set per call)
  int32_t* d_info = nullptr;   // small device scratch for composite decisions
  int32_t* h_info = nullptr;   // pinned mirror
  double* d_dscratch = nullptr;
  // device int read by the Cholesky kernels at entry: when set and *gate == 0
  // the launch returns at once (the near-identity fast path already produced
  // the factor; see chol_near_identity).  Host-sync free.
  const int32_t* gate = nullptr;
  // float bits of max|A| of the next fp32 tensor-core product's left operand,
  // already reduced on the device by an earlier kernel (sketch_rows.cu): the
  // split then skips its own max pass over the panel
  const unsigned int* amax_bits_hint = nullptr;
  // row-sharded calls (lr_comm_init / lr_orth_sharded): the NCCL communicator
  // of this rank; `sharded` makes the orthonormalization all-reduce its Grams
  void* nccl_comm = nullptr;
  int nranks = 1, rank = 0;
  bool sharded = false;
};

void pool_reset(Handle* h);
// comm.cu: in-place sum all-reduce of `count` elements of the wide dtype
// (float64 / complex128) over the handle's communicator, on h->stream; a
// no-op without one
void comm_allreduce_wide(Handle* h, int dtype_wide, int64_t count, void* buf);
void comm_destroy(Handle* h);
void comm_unique_id(void* out);
void comm_init(Handle* h, const void* id, int nranks, int rank);

// Every API entry runs on the handle's device (restoring the caller's):
// kernel attributes and the pool belong to that device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      cudaSetDevice(dev);
    } else {
      prev = -1;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// per-device "attribute already set" flags for kernels that raise their
// dynamic shared-memory limit once (cudaFuncSetAttribute is per device)
struct AttrOnce {
  bool done[16] = {};
  template <typename F>
  void operator()(F&& set) {
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= 16) {
      set();
      return;
    }
    if (!done[d]) {
      set();
      done[d] = true;
    }
  }
};
void* pool_alloc(Handle* h, size_t bytes);
template <typename T>
T* pool_alloc_t(Handle* h, size_t count) {
  return reinterpret_cast<T*>(pool_alloc(h, count * sizeof(T)));
}

inline int elem_size(int dtype) {
  switch (dtype) {
    case LR_F32: return 4;
    case LR_F64: return 8;
    case LR_C64: return 8;
    case LR_C128: return 16;
  }
  return 0;
}
inline bool is_complex(int dtype) { return dtype == LR_C64 || dtype == LR_C128; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// kernels launched from capi.cu (defined in the per-kernel .cu files)

// gemm_f64.cu ---------------------------------------------------------------
int64_t choose_splits(int sm_count, int64_t tiles, int64_t K);
// gemm_f64_ozaki.cu: fp64 passes on the int8 tensor cores (digit planes of A)
// wide_rows (nullable): += number of graded rows (> 1/8 of the nonzeros
// below 2^-32 of the row maximum; the caller keeps the matrix on DMMA)
void ozaki_prepare(Handle* h, int64_t m, int64_t n, const double* A, int64_t lda, int8_t* planes,
                   int64_t ldp, int32_t* row_exp, int32_t* wide_rows);
void ozaki_prepare_rows(Handle* h, int64_t m, int64_t n, int64_t i0, int64_t i1, const double* A,
                        int64_t lda, int8_t* planes, int64_t ldp, int32_t* row_exp,
                        int32_t* wide_rows);
void ozaki_gemm(Handle* h, bool trans, int64_t m, int64_t n, int64_t N, const int8_t* planes,
                int64_t ldp, const int32_t* row_exp, const double* X, int64_t ldx, double* C,
                int64_t ldc);
// C (M x N) = op(A) . B, op(A) = A (A M x K, lda) or A^T (A K x M, lda);
// B is K x N (ldb); C M x N (ldc).  conjA applies for complex.
void gemm_f64(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const double* A,
              int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc);
void gemm_c128(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
               const double2* A, int64_t lda, const double2* B, int64_t ldb, double2* C,
               int64_t ldc);

// gemm_f32.cu (tcgen05) -----------------------------------------------------
void gemm_f32(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
              int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc);
void gemm_c64(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
              const float2* A, int64_t lda, const float2* B, int64_t ldb, float2* C,
              int64_t ldc);
// gemm_simt.cu: honest-fp32 SIMT fallbacks (LR_F32_SIMT)
void gemm_f32_simt(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc);
void gemm_c64_simt(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
                   const float2* A, int64_t lda, const float2* B, int64_t ldb, float2* C,
                   int64_t ldc);
// passes over A with the operator's max|A| (a_amax < 0: unknown)
void gemm_f32_hint(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                   int64_t lda, double a_amax, const float* B, int64_t ldb, float* C,
                   int64_t ldc);
void gemm_c64_hint(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
                   const float2* A, int64_t lda, double a_amax, const float2* B, int64_t ldb,
                   float2* C, int64_t ldc);
// gram_tc.cu: G = Y^T Y of an fp32 panel (ell <= 256) on tcgen05 with
// fp32-level accuracy (second CholeskyQR pass); entries must satisfy
// |y| 2^log2_scale < 2^15, else *status |= 1 (status may be null)
// sketch_rows.cu: sparse-sign row sketch S Y (fp64, d x ell) of a tall fp32 panel
int64_t sketch_rows_dim();
bool sketch_rows_supported(int64_t m, int64_t ell);
void sketch_rows_f32(Handle* h, int64_t m, int64_t ell, const float* Y, int64_t ldy,
                     uint64_t seed, double* SY, unsigned int* amax_bits);
bool gram_tc_supported(int64_t m, int64_t ell, const float* Y, int64_t ldy);
void gram_tc_f32(Handle* h, int64_t m, int64_t ell, const float* Y, int64_t ldy, double* G,
                 int log2_scale, int32_t* status);
// fp64-accumulated Gram of fp32 / complex64 panels
void gram_f32(Handle* h, int64_t m, int64_t ell, const float* Y, int64_t ldy, double* G);
// C (M x N, ldc) = sum over S dense M x N partials, fixed order
void splitk_reduce(Handle* h, int64_t M, int64_t N, int S, const double* part, double* C,
                   int64_t ldc);
// gemm_small.cu: fp64 products small in every dimension (one 32 x 32 tile per CTA)
bool gemm_small_ok(int64_t M, int64_t N, int64_t K);
void gemm_small_f64(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const double* A,
                    int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc);
// gemm_skinny.cu: A^T B for K >> M, N <= 64 (fp64)
bool gemm_skinny_ok(bool transA, int64_t M, int64_t N, int64_t K);
void gemm_skinny_tn(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc);
bool gemm_skinny_wide_ok(bool transA, int64_t M, int64_t N, int64_t K, const double* C,
                         int64_t ldc);
void gemm_skinny_wide(Handle* h, bool tri, int64_t M, int64_t N, int64_t K, const double* A,
                      int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc);
bool gemm_skinny_tri_ok(int64_t M, int64_t N, int64_t K, const double* C, int64_t ldc);
void gemm_skinny_tri(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc);
bool gemm_skinny_nn_ok(bool transA, int64_t M, int64_t N, int64_t K, const double* C,
                       int64_t ldc);
void gemm_skinny_nn(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc);
bool gemm_f64_tma_ok(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb);
bool gemm_f64_tma_pick(bool transA, int64_t N, int64_t K);
bool gemm_f64_tma_f32_ok(bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                         int64_t lda, const float* B, int64_t ldb);
void gemm_f64_tma_f32(Handle* h, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb, double* C, int64_t ldc);
void gemm_f64_tma(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc);
void gemm_f64_from_f32(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                       int64_t lda, const float* B, int64_t ldb, double* C, int64_t ldc);
void gram_c64(Handle* h, int64_t m, int64_t ell, const float2* Y, int64_t ldy, double2* G);

// chol.cu ---------------------------------------------------------------------
// Cholesky with column deletion + triangular inverse, single CTA.
// drop threshold = drop_tol^2 * trace(G); shift = shift_coef * trace(G).
void chol_drop_f64(Handle* h, int64_t ell, const double* G, double drop_tol,
                   double unres_rel, double shift_coef, double* P, double* R, int32_t* info);
void chol_drop_c128(Handle* h, int64_t ell, const double2* G, double drop_tol,
                    double unres_rel, double shift_coef, double2* P, double2* R, int32_t* info);

// jacobi.cu -------------------------------------------------------------------
// M (rows x n, rows >= n) = W diag(S) J^H; W rows x n, J n x n.
void jacobi_svd_f64(Handle* h, int64_t rows, int64_t n, const double* M, double* W, double* S,
                    double* J, int32_t* info);
void jacobi_svd_c128(Handle* h, int64_t rows, int64_t n, const double2* M, double2* W,
                     double* S, double2* J, int32_t* info);

// chol_tiled.cu: register-tiled Cholesky with deletion for ell <= 128
// (by size; LR_CHOL=smem|tiled forces one kernel)
bool chol_tiled_supported(int64_t n, bool cplx);
// chol_panel.cu: panel-blocked Cholesky with deletion (default, ell <= 200 / 140)
int chol_mode();
bool chol_panel_supported(int64_t n, bool cplx);
void chol_panel_f64(Handle* h, int64_t n, const double* G, int64_t ldg, double drop_tol,
                    double unres_rel, double shift_coef, double* P, double* R, int32_t* info,
                    const double* trace_dev, const double* diag_src, int64_t diag_stride,
                    bool compact, double psd_neg = -1.0);
void chol_panel_c128(Handle* h, int64_t n, const double2* G, int64_t ldg, double drop_tol,
                     double unres_rel, double shift_coef, double2* P, double2* R, int32_t* info,
                     const double* trace_dev, const double2* diag_src, int64_t diag_stride,
                     bool compact, double psd_neg = -1.0);
// stageb.cu: Hermitian helpers of the Stage-B variants (factor.py:168-335)
void herm_prep(Handle* h, int dtype_wide, int64_t n, const void* B, int64_t ldb, void* H,
               double shift_mult, int power_iters, double* out2);
void eig_finish(Handle* h, int dtype_wide, int64_t n, const double* S, const double* shift,
                const void* U, double* lam, void* V);
bool chol_blocked_supported(int64_t n);
// Cholesky-with-deletion of a Gram that is expected to be I + E (second
// CholeskyQR pass): first-order factor when max|E| <= thr (its O(E^2) error
// must sit below the panel's rounding: 1e-8 for fp64 panels, 1e-4 for fp32),
// exact otherwise (decided on the device, no host synchronization).
void chol_near_identity(Handle* h, int dtype, int64_t n, const void* G, double drop_tol,
                        double unres_rel, void* P, void* R, int32_t* info, double thr);
void chol_blocked_f64(Handle* h, int64_t n, const double* G, double drop_tol, double unres_rel,
                      double shift_coef, double* P, double* R, int32_t* info);
void chol_blocked_c128(Handle* h, int64_t n, const double2* G, double drop_tol,
                       double unres_rel, double shift_coef, double2* P, double2* R,
                       int32_t* info);
void gemm_any(Handle* h, int dtype, bool trans, bool conj, int64_t M, int64_t N, int64_t K,
              const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc);
void chol_tiled_f64(Handle* h, int64_t n, const double* G, double drop_tol, double unres_rel,
                    double shift_coef, double* P, double* R, int32_t* info);
void chol_tiled_c128(Handle* h, int64_t n, const double2* G, double drop_tol, double unres_rel,
                     double shift_coef, double2* P, double2* R, int32_t* info);
// jacobi_blk.cu: block variant of the register-resident Jacobi (default;
// LR_JACOBI=round selects the column round-robin kernel of jacobi_reg.cu)
bool jacobi_blk_enabled();
void jacobi_blk_f64(Handle* h, int64_t n, const double* R, double* Mout, double* sig,
                    int32_t* info);
void jacobi_blk_c128(Handle* h, int64_t n, const double2* R, double2* Mout, double* sig,
                     int32_t* info);
// jacobi_reg.cu: register-resident Jacobi (R J = M, M unsorted) + finalize
bool jacobi_reg_supported(int64_t n, bool cplx);
void jacobi_reg_f64(Handle* h, int64_t n, const double* R, double* Mout, double* sig,
                    int32_t* info);
void jacobi_reg_c128(Handle* h, int64_t n, const double2* R, double2* Mout, double* sig,
                     int32_t* info);
void svd_finalize(Handle* h, int dtype_wide, int64_t n, const void* Jun, const void* Mun,
                  const double* sig, void* U, double* S, void* W, bool swap = false);

// misc.cu ---------------------------------------------------------------------
// G <- 1.5 I - 0.5 G  (Newton-Schulz coefficient matrix, n x n wide dtype)
void ns_coef(Handle* h, int dtype_wide, int64_t n, void* G);
void cast_copy(Handle* h, int src_dtype, const void* src, int64_t lds, int dst_dtype,
               void* dst, int64_t ldd, int64_t rows, int64_t cols, bool conj_transpose);
void col_sumsq(Handle* h, int dtype, int64_t m, int64_t r, const void* Z, int64_t ldz,
               double* out);
void estimate_finish(Handle* h, int64_t r, const double* sumsq, double alpha, double* est);
void check_finite(Handle* h, int dtype, int64_t m, int64_t n, const void* A, int64_t lda,
                  int64_t* nonfinite, double* amax);
void trmm_upper(Handle* h, int dtype, int64_t n, const void* R2, const void* R1, void* R);
void sign_fix(Handle* h, int dtype, int64_t rows, int64_t vrows, int64_t cols, void* U,
              int64_t ldu, void* V, int64_t ldv);
void max_abs_imag(Handle* h, int dtype, int64_t m, int64_t n, const void* Y, int64_t ldy,
                  double* out);
// Z (rows x cols) -= T ; Z[:, j] = src / s  helpers for CGS2 / estimator
void axpy_sub(Handle* h, int dtype, int64_t rows, int64_t cols, const void* T, int64_t ldt,
              void* Z, int64_t ldz);
void scale_col(Handle* h, int dtype, int64_t rows, const void* src, int64_t lds, double inv,
               void* dst, int64_t ldd);
// Z += T (fp64 / complex128); C_ij /= (d2_i + d1_j), 0 where d2_i + d1_j <= floor
void axpy_add(Handle* h, int dtype, int64_t rows, int64_t cols, const void* T, int64_t ldt,
              void* Z, int64_t ldz);
void sylvester_div(Handle* h, int dtype, int64_t k, int64_t kt, void* C, int64_t ldc,
                   const double* d2, const double* d1, double floor);

// srft.cu ---------------------------------------------------------------------
// n x ell picked columns of the Givens-chain SRFT (c64 or c128 output)
void gsrft_matrix(Handle* h, int dtype, int64_t n, int64_t ell, const double2* d_outer,
                  const int32_t* perm_outer, const double* thetas_outer, const double2* d_mid,
                  const int32_t* perm_inner, const double* thetas_inner, const double2* d_inner,
                  const int32_t* picks, double scale, void* Xout);
void srft_c64(Handle* h, int64_t m, int64_t n, int64_t ell, const float2* A, int64_t lda,
              const float2* d, const int32_t* picks, float scale, float2* Y, int64_t ldy,
              double a_amax = -1.0);
void srft_c128(Handle* h, int64_t m, int64_t n, int64_t ell, const double2* A, int64_t lda,
               const double2* d, const int32_t* picks, double scale, double2* Y, int64_t ldy);
void dft_rows(Handle* h, int dtype, int64_t rows, int64_t n, void* X, int64_t ldx);

// rowid.cu: row interpolative decomposition (pivoted-QR skeleton + T)
void row_id(Handle* h, int dtype, int64_t m, int64_t kc, int64_t k, const void* M, int64_t ldm,
            int32_t* perm, int forced, void* X, int64_t ldx, double* tmax_dev);

// gauss.cu ----------------------------------------------------------------------
// first `count` draws of numpy Generator(Philox(key)).standard_normal
void gaussian_stream(Handle* h, uint64_t key_lo, uint64_t key_hi, int64_t count, int out_dtype,
                     void* out);

// spmm.cu -----------------------------------------------------------------------
void csr_spmm_f64(Handle* h, int64_t m, int64_t n, int64_t ell, const int64_t* rowptr,
                  const int32_t* colidx, const double* vals, const double* X, int64_t ldx,
                  double* Y, int64_t ldy, bool accumulate);

}  // namespace lr
