// C (M x N) = op(A) B in fp64 for SMALL products -- the ell x ell x ell
// products around the Cholesky / Jacobi kernels (R^{-1} = P1 P2, J = R^{-1} M,
// the 2 x 2 blocked Cholesky's block products, U = Ut (1.5 I - 0.5 Ut^H Ut), ...;
// reference: the dense algebra inside small_svd / orthonormalize_double_gs,
// core.py:84-115, 190-230).
//
// The pass kernel (gemm_f64.cu: 128-row tiles, split-K + a reduction launch)
// runs these in 12 + 3.5 us at ell = 256 and 21-25 us at ell = 110 (ncu launch
// lists of configs 4 and 2): a 256^3 product is 4 tiles, so it is split 8
// ways along K to find 32 CTAs and then reduced.  Here every CTA owns one
// 32 x 32 tile of C over the whole K (64 CTAs at 256^2, no split, no
// reduction), 256 threads x (2 x 2) outputs, 32-deep k steps staged through
// shared memory with the next step's loads in flight in registers.  SIMT DFMA:
// 32 x 32 x K FMAs per CTA is ~2 us of one SM's fp64 rate at K = 256; the
// products are latency-bound, not pipe-bound.
#include "common.cuh"

namespace lr {
namespace {

constexpr int ST = 32;        // tile edge
constexpr int SKD = 32;       // k per step
constexpr int SPAD = ST + 1;  // smem row stride (bank spread for the transposed reads)

template <bool TRANS>
__global__ void __launch_bounds__(256)
gemm_small_kernel(int M, int N, int K, const double* __restrict__ A, int64_t lda,
                  const double* __restrict__ B, int64_t ldb, double* __restrict__ C,
                  int64_t ldc) {
  // As[k][i] = op(A)(m0 + i, k0 + k), Bs[k][j] = B(k0 + k, n0 + j)
  __shared__ double As[SKD][SPAD];
  __shared__ double Bs[SKD][SPAD];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * ST, n0 = blockIdx.y * ST;
  const int tx = tid & 15, ty = tid >> 4;          // outputs (ty + 16 a, tx + 16 b)
  // loader mapping: 1024 elements per tile, 4 per thread, 32 consecutive
  // elements of a global row per warp (coalesced 256 B)
  const int lr_ = tid >> 5, lc = tid & 31;         // rows lr_ + 8 u, column lc
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = lr_ + 8 * u;
      if (TRANS) {   // A is K x M: global row k0 + r, column m0 + lc
        ra[u] = (k0 + r < K && m0 + lc < M) ? A[int64_t(k0 + r) * lda + m0 + lc] : 0.0;
      } else {       // A is M x K: global row m0 + r, column k0 + lc
        ra[u] = (m0 + r < M && k0 + lc < K) ? A[int64_t(m0 + r) * lda + k0 + lc] : 0.0;
      }
      rb[u] = (k0 + r < K && n0 + lc < N) ? B[int64_t(k0 + r) * ldb + n0 + lc] : 0.0;
    }
  };
  load(0);
  for (int k0 = 0; k0 < K; k0 += SKD) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = lr_ + 8 * u;
      if (TRANS) As[r][lc] = ra[u];
      else As[lc][r] = ra[u];
      Bs[r][lc] = rb[u];
    }
    __syncthreads();
    if (k0 + SKD < K) load(k0 + SKD);
#pragma unroll
    for (int k = 0; k < SKD; ++k) {
      const double a0 = As[k][ty], a1 = As[k][ty + 16];
      const double b0 = Bs[k][tx], b1 = Bs[k][tx + 16];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int i = m0 + ty + 16 * a, j = n0 + tx + 16 * b;
      if (i < M && j < N) C[int64_t(i) * ldc + j] = acc[a][b];
    }
}

}  // namespace

// small in every dimension, yet enough tiles to be worth a grid
bool gemm_small_ok(int64_t M, int64_t N, int64_t K) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("LR_GEMM_SMALL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on && M <= 512 && N <= 512 && K <= 512 && M >= 16 && N >= 16 && K >= 1;
}

void gemm_small_f64(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const double* A,
                    int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc) {
  dim3 grid(unsigned(ceil_div(M, ST)), unsigned(ceil_div(N, ST)));
  if (transA)
    gemm_small_kernel<true><<<grid, 256, 0, h->stream>>>(int(M), int(N), int(K), A, lda, B, ldb, C,
                                                         ldc);
  else
    gemm_small_kernel<false><<<grid, 256, 0, h->stream>>>(int(M), int(N), int(K), A, lda, B, ldb,
                                                          C, ldc);
  LR_CHECK_LAUNCH();
}

}  // namespace lr
