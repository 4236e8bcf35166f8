// fp32 / complex64 passes over A: dispatch to the tcgen05 split kernel
// (gemm_f32_tc.cu) when the shape qualifies, else to the SIMT kernel.
// Complex64 products use the same real-view identities as gemm_c128.
#include "common.cuh"

namespace lr {

bool gemm_f32_tc_supported(bool transA, int64_t N, const float* A, int64_t lda);
void gemm_f32_tc(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                 int64_t lda, double a_amax, const float* B, int64_t ldb, float* C,
                 int64_t ldc);

namespace {

__global__ void cplx_expand_b_f32(int64_t K, int64_t N, const float2* __restrict__ B, int64_t ldb,
                                  float* __restrict__ Bt) {
  const int64_t total = K * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / N, j = i % N;
    const float2 b = B[k * ldb + j];
    float* r0 = Bt + (2 * k) * (2 * N) + 2 * j;
    float* r1 = r0 + 2 * N;
    r0[0] = b.x;  r0[1] = b.y;
    r1[0] = -b.y; r1[1] = b.x;
  }
}

__global__ void cplx_combine_t_f32(int64_t M, int64_t N, const float* __restrict__ D, bool conj,
                                   float2* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, j = i % N;
    const float* d0 = D + (2 * r) * (2 * N) + 2 * j;
    const float* d1 = d0 + 2 * N;
    float2 c;
    if (conj) { c.x = d0[0] + d1[1]; c.y = d0[1] - d1[0]; }
    else      { c.x = d0[0] - d1[1]; c.y = d0[1] + d1[0]; }
    C[r * ldc + j] = c;
  }
}

}  // namespace

void gemm_f32_hint(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                   int64_t lda, double a_amax, const float* B, int64_t ldb, float* C,
                   int64_t ldc) {
  if (h->f32_mode == LR_F32_SPLIT3 && gemm_f32_tc_supported(transA, N, A, lda) && K >= 1) {
    gemm_f32_tc(h, transA, M, N, K, A, lda, a_amax, B, ldb, C, ldc);
    return;
  }
  gemm_f32_simt(h, transA, M, N, K, A, lda, B, ldb, C, ldc);
}

// generic fp32 products (orthonormalization applies Y R^{-1}, U = Q U~,
// Q^T Z): large ones on the tcgen05 split with a device-side max|A| scale
// and per-column scales of B (so the columns of an ill-conditioned R^{-1}
// keep their low fp16 pieces); small ones on the SIMT kernel.
void gemm_f32(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
              int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc) {
  const bool big = double(M) * double(N) * double(K) >= double(1 << 26) &&
                   (transA ? K : M) >= 1024;
  if (big && h->f32_mode == LR_F32_SPLIT3 && gemm_f32_tc_supported(transA, N, A, lda)) {
    gemm_f32_tc(h, transA, M, N, K, A, lda, -1.0, B, ldb, C, ldc);
    return;
  }
  gemm_f32_simt(h, transA, M, N, K, A, lda, B, ldb, C, ldc);
}

void gemm_c64_hint(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
                   const float2* A, int64_t lda, double a_amax, const float2* B, int64_t ldb,
                   float2* C, int64_t ldc) {
  if (M == 0 || N == 0) return;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 4096)));
  if (!transA) {
    float* Bt = pool_alloc_t<float>(h, size_t(4) * K * N);
    cplx_expand_b_f32<<<blocks, 256, 0, h->stream>>>(K, N, B, ldb, Bt);
    LR_CHECK_LAUNCH();
    gemm_f32_hint(h, false, M, 2 * N, 2 * K, reinterpret_cast<const float*>(A), 2 * lda, a_amax,
                  Bt, 2 * N, reinterpret_cast<float*>(C), 2 * ldc);
  } else {
    float* D = pool_alloc_t<float>(h, size_t(4) * M * N);
    gemm_f32_hint(h, true, 2 * M, 2 * N, K, reinterpret_cast<const float*>(A), 2 * lda, a_amax,
                  reinterpret_cast<const float*>(B), 2 * ldb, D, 2 * N);
    cplx_combine_t_f32<<<blocks, 256, 0, h->stream>>>(M, N, D, conjA, C, ldc);
    LR_CHECK_LAUNCH();
  }
}

void gemm_c64(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
              const float2* A, int64_t lda, const float2* B, int64_t ldb, float2* C,
              int64_t ldc) {
  // large products on the tcgen05 split (real view: 2N <= 256 columns), the
  // rest on the SIMT kernel -- as gemm_f32
  const bool big = double(M) * double(N) * double(K) >= double(1 << 24) &&
                   (transA ? K : M) >= 1024 && 2 * N <= 256;
  if (big && h->f32_mode == LR_F32_SPLIT3 && (lda % 2) == 0 &&
      (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    gemm_c64_hint(h, transA, conjA, M, N, K, A, lda, -1.0, B, ldb, C, ldc);
    return;
  }
  gemm_c64_simt(h, transA, conjA, M, N, K, A, lda, B, ldb, C, ldc);
}

}  // namespace lr
