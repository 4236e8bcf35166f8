// fp32 / complex64 passes over A.  Placeholder routing to the SIMT kernel
// until the tcgen05 split kernel lands.
#include "common.cuh"

namespace lr {

void gemm_f32(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
              int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc) {
  gemm_f32_simt(h, transA, M, N, K, A, lda, B, ldb, C, ldc);
}

void gemm_c64(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
              const float2* A, int64_t lda, const float2* B, int64_t ldb, float2* C,
              int64_t ldc) {
  gemm_c64_simt(h, transA, conjA, M, N, K, A, lda, B, ldb, C, ldc);
}

}  // namespace lr
