// C (M x N) = A^T B for tall, narrow fp64 panels: K >> M, N <= 64 -- the
// Grams of an m x ell panel with ell <= 64 and the R^T X / L^T Y products of
// config 5's implicit low-rank term (reference: the DenseOperator products
// of core.py:391-395 and the Gram inside orthonormalize_double_gs' role,
// core.py:84-115).
//
// The 128-row tiles of the pass kernels compute on padding here (M = 32 or
// 48 of 128 rows: 62-75 % of the DMMA work wasted, 1.05 ms for a 2^21 x 48
// Gram, ncu launch list of config 5).  This kernel gives every warp a run of
// rows of A and B: per 4 rows it loads its m16n8k4 fragments straight from
// global memory (8 consecutive doubles per fragment row, several k-steps in
// flight) and issues MF x NF8 DMMAs on exactly the M x N output; the 8 warp
// partials are summed in shared memory in a fixed order, one partial per CTA
// goes to the split-K buffer, and splitk_reduce sums the CTAs in a fixed
// order (deterministic).  Bound: HBM (K (M + N) 8 bytes) or the DMMA pipe on
// M x N x K useful FMAs, whichever is larger.
#include "common.cuh"

namespace lr {
namespace {

constexpr int SK_THREADS = 256;
constexpr int SK_WARPS = SK_THREADS / 32;
// k4 steps with loads in flight: as many as the register file allows
// (accumulators MF x NF8 x 4 doubles + U x (2 MF + NF8) operands)
template <int MF, int NF8>
__host__ __device__ constexpr int sk_unroll() { return MF * NF8 <= 12 ? 4 : 2; }

__device__ __forceinline__ void dmma_sk(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// grid.x = CTAs, each owns rows [blockIdx.x * rows_per, ...) of A and B.
// SYM (A == B, a Gram): tiles entirely below the diagonal (8 nf + 7 < 16 mf)
// are skipped -- 12 of 18 tiles at 48 x 48 -- and mirrored after the reduction.
template <int MF, int NF8, bool SYM>
__global__ void __launch_bounds__(SK_THREADS)
skinny_tn_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ part,
                 int64_t rows_per) {
  __shared__ double red[MF * 16][NF8 * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per;
  const int64_t r1 = min(K, r0 + rows_per);
  double acc[MF][NF8][4];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  // SYM with NF8 == 2 MF: the B fragments ARE the A fragments (lane (g, t)
  // holds Y[k + t][16 mf + g (+ 8)] either way), so B is never loaded and the
  // registers go to a deeper unroll -- the Gram was latency-bound at 39 % of
  // HBM with two k4-steps in flight per warp (24 KB per SM)
  constexpr bool REUSE = SYM && NF8 == 2 * MF;
  // two register buffers of fragments (software pipeline) where they fit
  constexpr bool PIPE = REUSE || MF * NF8 <= 12;
  constexpr int SK_UNROLL = REUSE ? 4 : (PIPE ? 2 : sk_unroll<MF, NF8>());
  // warp w takes k4-steps w, w + 8, ... of the CTA's rows, SK_UNROLL at a time
  const int64_t nsteps = (r1 - r0 + 3) / 4;
  auto load = [&](int64_t s0, double (&a)[SK_UNROLL][MF][2], double (&b)[SK_UNROLL][REUSE ? 1 : NF8]) {
#pragma unroll
    for (int u = 0; u < SK_UNROLL; ++u) {
      const int64_t k = r0 + (s0 + u) * 4 + t;
      const bool kin = (s0 + u) < nsteps && k < r1;
      const double* ar = A + k * lda;
#pragma unroll
      for (int mf = 0; mf < MF; ++mf) {
        const int i0 = mf * 16 + g, i1 = i0 + 8;
        a[u][mf][0] = (kin && i0 < M) ? __ldg(ar + i0) : 0.0;
        a[u][mf][1] = (kin && i1 < M) ? __ldg(ar + i1) : 0.0;
      }
      if constexpr (!REUSE) {
        const double* br = B + k * ldb;
#pragma unroll
        for (int nf = 0; nf < NF8; ++nf) {
          const int j = nf * 8 + g;
          b[u][nf] = (kin && j < N) ? __ldg(br + j) : 0.0;
        }
      }
    }
  };
  auto mma = [&](double (&a)[SK_UNROLL][MF][2], double (&b)[SK_UNROLL][REUSE ? 1 : NF8]) {
#pragma unroll
    for (int u = 0; u < SK_UNROLL; ++u)
#pragma unroll
      for (int nf = 0; nf < NF8; ++nf)
#pragma unroll
        for (int mf = 0; mf < MF; ++mf)
          if (!SYM || 8 * nf + 7 >= 16 * mf) {
            const double bv = REUSE ? a[u][nf >> 1][nf & 1] : b[u][REUSE ? 0 : nf];
            dmma_sk(acc[mf][nf], a[u][mf][0], a[u][mf][1], bv);
          }
  };
  const int64_t sstride = int64_t(SK_WARPS) * SK_UNROLL;
  if constexpr (PIPE) {
    // software pipeline: the next batch of fragments is in flight while this
    // batch's DMMAs run (without it every batch paid a full HBM round trip:
    // 289 us for the 805 MB Gram, 43 % of the copy rate)
    constexpr int NB = REUSE ? 1 : NF8;
    double a0[SK_UNROLL][MF][2], a1[SK_UNROLL][MF][2], b0[SK_UNROLL][NB], b1[SK_UNROLL][NB];
    int64_t s0 = int64_t(warp) * SK_UNROLL;
    load(s0, a0, b0);
    for (; s0 < nsteps; s0 += 2 * sstride) {
      load(s0 + sstride, a1, b1);
      mma(a0, b0);
      load(s0 + 2 * sstride, a0, b0);
      mma(a1, b1);
    }
  } else {
    for (int64_t s0 = int64_t(warp) * SK_UNROLL; s0 < nsteps; s0 += sstride) {
      double a[SK_UNROLL][MF][2], b[SK_UNROLL][NF8];
      load(s0, a, b);
      mma(a, b);
    }
  }
  // accumulator layout (m16n8 fp64): c0,c1 at (g, 2t..2t+1), c2,c3 at (g+8, 2t..2t+1);
  // warps add their partials in a fixed order (deterministic)
  for (int w = 0; w < SK_WARPS; ++w) {
    if (warp == w) {
#pragma unroll
      for (int mf = 0; mf < MF; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF8; ++nf) {
          const int i = mf * 16 + g, j = nf * 8 + 2 * t;
          if (w == 0) {
            red[i][j] = acc[mf][nf][0];
            red[i][j + 1] = acc[mf][nf][1];
            red[i + 8][j] = acc[mf][nf][2];
            red[i + 8][j + 1] = acc[mf][nf][3];
          } else {
            red[i][j] += acc[mf][nf][0];
            red[i][j + 1] += acc[mf][nf][1];
            red[i + 8][j] += acc[mf][nf][2];
            red[i + 8][j + 1] += acc[mf][nf][3];
          }
        }
    }
    __syncthreads();
  }
  double* out = part + int64_t(blockIdx.x) * M * N;
  for (int e = threadIdx.x; e < M * N; e += SK_THREADS) {
    const int i = e / int(N), j = e - i * int(N);
    out[e] = red[i][j];
  }
}

__global__ void skinny_mirror_kernel(int n, double* __restrict__ C, int64_t ldc) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e / n, j = e - i * n;
    if (j < i) C[int64_t(i) * ldc + j] = C[int64_t(j) * ldc + i];
  }
}

template <int MF, int NF8>
void launch_skinny(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc) {
  // one CTA per SM (up to 232 registers per thread), each a run of >= 1024 rows
  int64_t ctas = std::min<int64_t>(h->sm_count, std::max<int64_t>(1, K / 1024));
  const int64_t rows_per = ((ceil_div(K, ctas) + 3) / 4) * 4;
  ctas = ceil_div(K, rows_per);
  double* part = pool_alloc_t<double>(h, size_t(ctas) * M * N);
  const bool sym = (A == B && lda == ldb && M == N);
  if (sym)
    skinny_tn_kernel<MF, NF8, true><<<unsigned(ctas), SK_THREADS, 0, h->stream>>>(
        M, N, K, A, lda, B, ldb, part, rows_per);
  else
    skinny_tn_kernel<MF, NF8, false><<<unsigned(ctas), SK_THREADS, 0, h->stream>>>(
        M, N, K, A, lda, B, ldb, part, rows_per);
  LR_CHECK_LAUNCH();
  splitk_reduce(h, M, N, int(ctas), part, C, ldc);
  if (sym) {
    skinny_mirror_kernel<<<unsigned(ceil_div(M * N, 256)), 256, 0, h->stream>>>(int(M), C, ldc);
    LR_CHECK_LAUNCH();
  }
}

// C (M x N) = A (M x K) B (K x N) for M >> K, N <= 64 (the applies Y P of a
// narrow panel and config 5's L Z): B staged in shared memory once per CTA,
// every warp streams 16-row tiles of A (fragments straight from global),
// K/4 x NF8 DMMAs per tile, 16-byte stores of the accumulator pairs.
// TRI: B is upper triangular (an inverse Cholesky factor): output columns
// 8 nf .. 8 nf + 7 only take k <= 8 nf + 7, i.e. the k4 steps ks <= 2 nf + 1 --
// 42 of 72 DMMAs at 48 x 48, which moves the product from the DMMA pipe's bound
// to HBM's.
template <int NF8, int KS, bool TRI>   // KS = k4 steps (K <= 4 KS)
__global__ void __launch_bounds__(SK_THREADS)
skinny_nn_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ C,
                 int64_t ldc) {
  __shared__ double bs[4 * KS][NF8 * 8 + 1];
  for (int e = threadIdx.x; e < 4 * KS * NF8 * 8; e += SK_THREADS) {
    const int k = e / (NF8 * 8), j = e - k * (NF8 * 8);
    bs[k][j] = (k < K && j < N) ? B[int64_t(k) * ldb + j] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t ntiles = (M + 15) / 16;
  const int64_t stride = int64_t(gridDim.x) * SK_WARPS;
  // software pipeline: the next tile's A fragments are in flight while the
  // current tile's DMMAs and stores run (the loop is latency-bound otherwise)
  auto load = [&](int64_t tile, double (&a)[KS][2]) {
    const int64_t r0 = tile * 16 + g, r1 = r0 + 8;
    const double* a0p = A + r0 * lda;
    const double* a1p = A + r1 * lda;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + t;
      a[ks][0] = (tile < ntiles && r0 < M && k < K) ? __ldg(a0p + k) : 0.0;
      a[ks][1] = (tile < ntiles && r1 < M && k < K) ? __ldg(a1p + k) : 0.0;
    }
  };
  int64_t tile = int64_t(blockIdx.x) * SK_WARPS + warp;
  double a[KS][2], an[KS][2];
  load(tile, a);
  for (; tile < ntiles; tile += stride) {
    load(tile + stride, an);
    const int64_t r0 = tile * 16 + g, r1 = r0 + 8;
    double acc[NF8][4];
#pragma unroll
    for (int nf = 0; nf < NF8; ++nf)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nf][e] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nf = 0; nf < NF8; ++nf)
        if (!TRI || ks <= 2 * nf + 1) dmma_sk(acc[nf], a[ks][0], a[ks][1], bs[4 * ks + t][nf * 8 + g]);
#pragma unroll
    for (int nf = 0; nf < NF8; ++nf) {
      const int64_t j = nf * 8 + 2 * t;
      if (j + 1 < N) {
        if (r0 < M) *reinterpret_cast<double2*>(C + r0 * ldc + j) = make_double2(acc[nf][0], acc[nf][1]);
        if (r1 < M) *reinterpret_cast<double2*>(C + r1 * ldc + j) = make_double2(acc[nf][2], acc[nf][3]);
      } else if (j < N) {
        if (r0 < M) C[r0 * ldc + j] = acc[nf][0];
        if (r1 < M) C[r1 * ldc + j] = acc[nf][2];
      }
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      a[ks][0] = an[ks][0];
      a[ks][1] = an[ks][1];
    }
  }
}

template <int NF8, int KS, bool TRI = false>
void launch_skinny_nn(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                      const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int64_t ntiles = ceil_div(M, 16);
  const int64_t ctas = std::min<int64_t>(4 * h->sm_count, ceil_div(ntiles, SK_WARPS));
  skinny_nn_kernel<NF8, KS, TRI><<<unsigned(ctas), SK_THREADS, 0, h->stream>>>(M, N, K, A, lda, B,
                                                                               ldb, C, ldc);
  LR_CHECK_LAUNCH();
}


// Wider B (64 < N <= 128, K <= 128): config 2's panel applies Y P / Q U~ with
// ell = 110 (reference orthonormalize_double_gs / direct_svd, core.py:84-115,
// factor.py:154-165).  The 128-row tiled kernel runs them on 64 CTAs at ~26 us
// (8192 x 110 x 110: 0.2 GFLOP, 14 MB -- under 10 us of either roofline).  Here
// a warp owns a 16-row tile over all N columns (14 x 4 accumulators); the K
// extent is walked in chunks of 8 k4-steps with the next chunk's A fragments
// in flight; B sits in shared memory (dynamic, K x (N8 + 1) doubles).  TRI as
// in skinny_nn_kernel.  4 warps per CTA so that 8192 rows already fill 128 SMs.
constexpr int SW_THREADS = 128;
constexpr int SW_KC = 8;   // k4-steps per chunk

template <int NF8, bool TRI>
__global__ void __launch_bounds__(SW_THREADS)
skinny_nn_wide_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
                      const double* __restrict__ B, int64_t ldb, double* __restrict__ C,
                      int64_t ldc) {
  extern __shared__ double bsw[];             // [Kp][BS], Kp = K rounded up to 4
  constexpr int BS = NF8 * 8 + 1;
  const int Kp = int((K + 3) / 4) * 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t ntiles = (M + 15) / 16;
  const int nks = Kp / 4;                     // k4-steps
  const int nch = (nks + SW_KC - 1) / SW_KC;  // chunks
  bool staged = false;
  auto stage = [&]() {
    // staging: thread j streams column j, 16 rows in flight (the flat loop with a
    // division per element kept ~4 loads in flight: ~10 us for 99 KB, longer than
    // the tile's own work)
    if (threadIdx.x < NF8 * 8) {
      const int j = threadIdx.x;
      const bool jin = j < N;
      const double* bj = B + (jin ? j : 0);
#pragma unroll 1
      for (int k0 = 0; k0 < Kp; k0 += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (jin && k0 + u < K) ? __ldg(bj + int64_t(k0 + u) * ldb) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (k0 + u < Kp) bsw[(k0 + u) * BS + j] = v[u];
      }
    }
    __syncthreads();
  };
  for (int64_t tile = int64_t(blockIdx.x) * (SW_THREADS / 32) + warp; tile < ntiles;
       tile += int64_t(gridDim.x) * (SW_THREADS / 32)) {
    const int64_t r0 = tile * 16 + g, r1 = r0 + 8;
    const double* a0p = A + r0 * lda;
    const double* a1p = A + r1 * lda;
    auto load = [&](int ch, double (&a)[SW_KC][2]) {
#pragma unroll
      for (int u = 0; u < SW_KC; ++u) {
        const int k = 4 * (ch * SW_KC + u) + t;
        a[u][0] = (ch < nch && r0 < M && k < K) ? __ldg(a0p + k) : 0.0;
        a[u][1] = (ch < nch && r1 < M && k < K) ? __ldg(a1p + k) : 0.0;
      }
    };
    double acc[NF8][4];
#pragma unroll
    for (int nf = 0; nf < NF8; ++nf)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nf][e] = 0.0;
    double a[SW_KC][2], an[SW_KC][2];
    load(0, a);
    if (!staged) {   // B is staged while the first tile's first fragments are in flight
      stage();
      staged = true;
    }
    for (int ch = 0; ch < nch; ++ch) {
      load(ch + 1, an);
#pragma unroll
      for (int u = 0; u < SW_KC; ++u) {
        const int ks = ch * SW_KC + u;
        if (ks < nks) {
          const double* brow = bsw + (4 * ks + t) * BS + g;
#pragma unroll
          for (int nf = 0; nf < NF8; ++nf)
            if (!TRI || ks <= 2 * nf + 1) dmma_sk(acc[nf], a[u][0], a[u][1], brow[nf * 8]);
        }
      }
#pragma unroll
      for (int u = 0; u < SW_KC; ++u) {
        a[u][0] = an[u][0];
        a[u][1] = an[u][1];
      }
    }
#pragma unroll
    for (int nf = 0; nf < NF8; ++nf) {
      const int64_t j = nf * 8 + 2 * t;
      if (j + 1 < N) {
        if (r0 < M) *reinterpret_cast<double2*>(C + r0 * ldc + j) = make_double2(acc[nf][0], acc[nf][1]);
        if (r1 < M) *reinterpret_cast<double2*>(C + r1 * ldc + j) = make_double2(acc[nf][2], acc[nf][3]);
      } else if (j < N) {
        if (r0 < M) C[r0 * ldc + j] = acc[nf][0];
        if (r1 < M) C[r1 * ldc + j] = acc[nf][2];
      }
    }
  }
  if (!staged) stage();   // a warp without a tile still joins the CTA barrier
}

template <int NF8, bool TRI>
void launch_skinny_wide(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int Kp = int(ceil_div(K, 4) * 4);
  const size_t smem = size_t(Kp) * (NF8 * 8 + 1) * sizeof(double);
  auto kern = skinny_nn_wide_kernel<NF8, TRI>;
  static AttrOnce once;
  once([&] {
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 129 * 8));
  });
  const int64_t ntiles = ceil_div(M, 16);
  const int64_t ctas = std::min<int64_t>(2 * h->sm_count, ceil_div(ntiles, SW_THREADS / 32));
  kern<<<unsigned(ctas), SW_THREADS, smem, h->stream>>>(M, N, K, A, lda, B, ldb, C, ldc);
  LR_CHECK_LAUNCH();
}

}  // namespace

// LR_SKINNY=0 disables (A/B against the tiled DMMA kernels)
bool gemm_skinny_ok(bool transA, int64_t M, int64_t N, int64_t K) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("LR_SKINNY");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  return !off && transA && ceil_div(M, 16) * ceil_div(N, 8) <= 18 && M <= 48 && N <= 64 &&
         K >= 16384;
}

void gemm_skinny_tn(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int mf = int(ceil_div(M, 16)), nf = int(ceil_div(N, 8));
  // instantiate the shapes the configurations use; round up the others
  if (mf <= 1 && nf <= 2) launch_skinny<1, 2>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else if (mf <= 2 && nf <= 4) launch_skinny<2, 4>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else if (mf <= 2 && nf <= 6) launch_skinny<2, 6>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else if (mf <= 3 && nf <= 6) launch_skinny<3, 6>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else launch_skinny<2, 8>(h, M, N, K, A, lda, B, ldb, C, ldc);   // M <= 32, N <= 64
}

}  // namespace lr

namespace lr {

// M >> K, N: 16-byte aligned C rows for the paired stores
bool gemm_skinny_nn_ok(bool transA, int64_t M, int64_t N, int64_t K, const double* C,
                       int64_t ldc) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("LR_SKINNY");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  // measured (config 5 launch lists): 328 vs 394 us at K = 32, but 453 vs 394
  // at K = 48 where the tiled kernel's larger warp tile wins -- K <= 32 only
  return !off && !transA && K <= 32 && N <= 64 && M >= 65536 && (ldc % 2) == 0 &&
         (reinterpret_cast<uintptr_t>(C) & 15) == 0;
}

// C = A B with B (K x N, K == N) upper triangular: a tall panel times an
// inverse Cholesky factor (orthonormalize_double_gs' Y R^{-1}, core.py:84-115)
bool gemm_skinny_tri_ok(int64_t M, int64_t N, int64_t K, const double* C, int64_t ldc) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("LR_SKINNY");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  return !off && K == N && N <= 64 && N >= 8 && M >= 65536 && (ldc % 2) == 0 &&
         (reinterpret_cast<uintptr_t>(C) & 15) == 0;
}

void gemm_skinny_tri(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int nf = int(ceil_div(N, 8));
  if (nf <= 4) launch_skinny_nn<4, 8, true>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else if (nf <= 6) launch_skinny_nn<6, 12, true>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else launch_skinny_nn<8, 16, true>(h, M, N, K, A, lda, B, ldb, C, ldc);
}

// 64 < N <= 128, K <= 128, tall A (the ell = 110 panel applies of config 2)
bool gemm_skinny_wide_ok(bool transA, int64_t M, int64_t N, int64_t K, const double* C,
                         int64_t ldc) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("LR_SKINNY");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  return !off && !transA && N > 64 && N <= 128 && K >= 8 && K <= 128 && M >= 4096 &&
         (ldc % 2) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
}

void gemm_skinny_wide(Handle* h, bool tri, int64_t M, int64_t N, int64_t K, const double* A,
                      int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int nf = int(ceil_div(N, 8));
  if (nf <= 12) {
    if (tri) launch_skinny_wide<12, true>(h, M, N, K, A, lda, B, ldb, C, ldc);
    else launch_skinny_wide<12, false>(h, M, N, K, A, lda, B, ldb, C, ldc);
  } else if (nf <= 14) {
    if (tri) launch_skinny_wide<14, true>(h, M, N, K, A, lda, B, ldb, C, ldc);
    else launch_skinny_wide<14, false>(h, M, N, K, A, lda, B, ldb, C, ldc);
  } else {
    if (tri) launch_skinny_wide<16, true>(h, M, N, K, A, lda, B, ldb, C, ldc);
    else launch_skinny_wide<16, false>(h, M, N, K, A, lda, B, ldb, C, ldc);
  }
}

void gemm_skinny_nn(Handle* h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int nf = int(ceil_div(N, 8));
  if (nf <= 4) launch_skinny_nn<4, 8>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else if (nf <= 6) launch_skinny_nn<6, 8>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else launch_skinny_nn<8, 8>(h, M, N, K, A, lda, B, ldb, C, ldc);
}

}  // namespace lr
