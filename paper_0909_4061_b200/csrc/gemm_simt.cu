// SIMT (FFMA / DFMA) tall-skinny GEMM for fp32 / complex64 operands.
//
// Two uses:
//  * gram_f32 / gram_c64: G = Y^H Y of an fp32 panel with exact products and
//    fp64 accumulation (each fp32 x fp32 product is exact in fp64), the
//    "fp64 Gram" CholeskyQR2 needs for ill-conditioned fp32 panels
//    (DESIGN.md "orthonormalization").
//  * LR_F32_SIMT mode: honest fp32 arithmetic for the passes over A (the
//    arithmetic-parity check of the tensor-core split kernel).
// Tile 64 x 64 x 16, 256 threads, 4 x 4 outputs per thread, split-K with a
// fixed-order reduction.
#include "common.cuh"

namespace lr {
namespace {

constexpr int TM = 64, TN = 64, TK = 16, TTH = 256;

template <bool TRANS, typename TA>
__global__ void __launch_bounds__(TTH)
simt_gemm_kernel(int64_t M, int64_t N, int64_t K, const float* __restrict__ A, int64_t lda,
                 const float* __restrict__ B, int64_t ldb, TA* __restrict__ C, int64_t ldc,
                 int64_t kchunk, int64_t cstride) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = int64_t(blockIdx.x) * TM, n0 = int64_t(blockIdx.y) * TN;
  const int64_t kb = int64_t(blockIdx.z) * kchunk, ke = min(K, kb + kchunk);
  TA acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = TA(0);
  for (int64_t k0 = kb; k0 < ke; k0 += TK) {
    for (int e = threadIdx.x; e < TK * TM; e += TTH) {
      int kk, mm;
      float v = 0.f;
      if (!TRANS) {
        mm = e / TK; kk = e % TK;
        if (m0 + mm < M && k0 + kk < ke) v = A[(m0 + mm) * lda + k0 + kk];
      } else {
        kk = e / TM; mm = e % TM;
        if (m0 + mm < M && k0 + kk < ke) v = A[(k0 + kk) * lda + m0 + mm];
      }
      As[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < TK * TN; e += TTH) {
      const int kk = e / TN, nn = e % TN;
      float v = 0.f;
      if (n0 + nn < N && k0 + kk < ke) v = B[(k0 + kk) * ldb + n0 + nn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      TA a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = TA(As[kk][ty + 16 * i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = TA(Bs[kk][tx + 16 * j]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  TA* Cz = C + int64_t(blockIdx.z) * cstride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + ty + 16 * i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + tx + 16 * j;
      if (c < N) Cz[r * ldc + c] = acc[i][j];
    }
  }
}

template <typename TP, typename TO>
__global__ void reduce_slices(int64_t M, int64_t N, int S, const TP* __restrict__ part,
                              TO* __restrict__ out, int64_t ldo) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    TP s = TP(0);
    for (int k = 0; k < S; ++k) s += part[int64_t(k) * total + i];
    out[(i / N) * ldo + (i % N)] = TO(s);
  }
}

// C (M x N, TO) = op(A) B with accumulation type TA
template <typename TA, typename TO>
void simt_gemm(Handle* h, bool trans, int64_t M, int64_t N, int64_t K, const float* A,
               int64_t lda, const float* B, int64_t ldb, TO* C, int64_t ldc) {
  const int64_t mt = ceil_div(M, TM), nt = ceil_div(N, TN);
  int64_t splits = 1;
  {
    const int64_t want = int64_t(h->sm_count) * 4;
    if (mt * nt < want) splits = std::min<int64_t>(ceil_div(want, mt * nt), ceil_div(K, 4 * TK));
    splits = std::max<int64_t>(1, std::min<int64_t>(splits, 256));
  }
  const int64_t kchunk = ceil_div(ceil_div(K, splits), TK) * TK;
  splits = ceil_div(K, kchunk);
  TA* part = pool_alloc_t<TA>(h, size_t(splits) * M * N);
  dim3 grid{unsigned(mt), unsigned(nt), unsigned(splits)};
  if (trans)
    simt_gemm_kernel<true, TA><<<grid, TTH, 0, h->stream>>>(M, N, K, A, lda, B, ldb, part, N,
                                                            kchunk, M * N);
  else
    simt_gemm_kernel<false, TA><<<grid, TTH, 0, h->stream>>>(M, N, K, A, lda, B, ldb, part, N,
                                                             kchunk, M * N);
  LR_CHECK_LAUNCH();
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 8192)));
  reduce_slices<TA, TO><<<blocks, 256, 0, h->stream>>>(M, N, int(splits), part, C, ldc);
  LR_CHECK_LAUNCH();
}

// complex helpers (float2), same real-view identities as gemm_c128
__global__ void cplx_expand_b_f(int64_t K, int64_t N, const float2* __restrict__ B, int64_t ldb,
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

template <typename TD, typename TO2>
__global__ void cplx_combine_t_any(int64_t M, int64_t N, const TD* __restrict__ D, bool conj,
                                   TO2* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, j = i % N;
    const TD* d0 = D + (2 * r) * (2 * N) + 2 * j;
    const TD* d1 = d0 + 2 * N;
    TO2 c;
    if (conj) { c.x = d0[0] + d1[1]; c.y = d0[1] - d1[0]; }
    else      { c.x = d0[0] - d1[1]; c.y = d0[1] + d1[0]; }
    C[r * ldc + j] = c;
  }
}

}  // namespace

void gemm_f32_simt(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc) {
  simt_gemm<float, float>(h, transA, M, N, K, A, lda, B, ldb, C, ldc);
}

void gram_f32(Handle* h, int64_t m, int64_t ell, const float* Y, int64_t ldy, double* G) {
  simt_gemm<double, double>(h, true, ell, ell, m, Y, ldy, Y, ldy, G, ell);
}

void gram_c64(Handle* h, int64_t m, int64_t ell, const float2* Y, int64_t ldy, double2* G) {
  // D (2 ell x 2 ell) = Y_real^T Y_real; G = combine(conj)
  double* D = pool_alloc_t<double>(h, size_t(4) * ell * ell);
  const float* Yr = reinterpret_cast<const float*>(Y);
  // DMMA on the real view (fp32 staged, widened to fp64: exact products)
  gemm_f64_from_f32(h, true, 2 * ell, 2 * ell, m, Yr, 2 * ldy, Yr, 2 * ldy, D, 2 * ell);
  const int blocks = int(std::max<int64_t>(1, ceil_div(ell * ell, 256)));
  cplx_combine_t_any<double, double2><<<blocks, 256, 0, h->stream>>>(ell, ell, D, true, G, ell);
  LR_CHECK_LAUNCH();
}

void gemm_c64_simt(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
                   const float2* A, int64_t lda, const float2* B, int64_t ldb, float2* C,
                   int64_t ldc) {
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 4096)));
  if (!transA) {
    float* Bt = pool_alloc_t<float>(h, size_t(4) * K * N);
    cplx_expand_b_f<<<blocks, 256, 0, h->stream>>>(K, N, B, ldb, Bt);
    LR_CHECK_LAUNCH();
    simt_gemm<float, float>(h, false, M, 2 * N, 2 * K, reinterpret_cast<const float*>(A),
                            2 * lda, Bt, 2 * N, reinterpret_cast<float*>(C), 2 * ldc);
  } else {
    float* D = pool_alloc_t<float>(h, size_t(4) * M * N);
    simt_gemm<float, float>(h, true, 2 * M, 2 * N, K, reinterpret_cast<const float*>(A),
                            2 * lda, reinterpret_cast<const float*>(B), 2 * ldb, D, 2 * N);
    cplx_combine_t_any<float, float2><<<blocks, 256, 0, h->stream>>>(M, N, D, conjA, C, ldc);
    LR_CHECK_LAUNCH();
  }
}

}  // namespace lr
