// K1/K2 in fp64: tall-skinny GEMM on the FP64 tensor pipe (DMMA).
//
// Replaces DenseOperator._apply / _apply_adjoint (reference core.py:391-395)
// for float64 A, and the small products of the orthonormalization and
// Stage B (Q = Y P, U = Q U~, Gram Y^T Y).
//
// tcgen05 has no f64 kind, so fp64 uses mma.sync m16n8k4 .f64 (SASS DMMA).
// Shape: C (M x N) = op(A) (M x K) . B (K x N) with N = ell small (<= 128
// per CTA tile) and M, K large.  A is streamed from HBM exactly once per
// pass when N fits one tile; B (the sketch / basis) is re-read from L2.
//   transA = false: A is M x K row-major (pass A.X, K contiguous)
//   transA = true : A is K x M row-major (pass A^T.X, M contiguous)
// CTA tile 128 x (16*NF), BK = 16, 3-stage cp.async ring, 8 warps (4 x 2),
// each warp 32 x 8*NF.  Split-K over blockIdx.z writes fp64 partials that a
// second kernel sums in a fixed order (deterministic; no atomics).
#include "common.cuh"

namespace lr {
namespace {

constexpr int BM = 128;
#ifndef LR_DMMA_BK
#define LR_DMMA_BK 16
#endif
#ifndef LR_DMMA_STAGES
#define LR_DMMA_STAGES 3
#endif
constexpr int BK = LR_DMMA_BK;
constexpr int STAGES = LR_DMMA_STAGES;
constexpr int THREADS = 256;
constexpr int AS_NN = BK + 4;    // row stride (f64) of the A tile, non-transposed
constexpr int AS_TN = BM + 4;    // row stride of the A tile, transposed

template <int NF, typename TIN = double>
struct Smem {
  static constexpr int BN = 16 * NF;
  static constexpr int BS = BN + 4;
  static constexpr int A_ELEMS = (BM * AS_NN > BK * AS_TN) ? BM * AS_NN : BK * AS_TN;
  static constexpr int B_ELEMS = BK * BS;
  static constexpr size_t bytes = size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(TIN);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
template <typename TIN>
__device__ __forceinline__ void cp_async_elem(TIN* smem, const TIN* gmem, int valid) {
  if constexpr (sizeof(TIN) == 8) cp_async8(smem, gmem, valid * 8);
  else cp_async4(smem, gmem, valid * 4);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Copy a rows x cols block starting at g (row stride ld) into smem (row
// stride ss), zero-filling out-of-range rows/cols.  vec: 16-byte chunks
// allowed (ld and the base 16-byte aligned).  fp32 inputs (the Gram of an fp32
// panel) are staged as fp32 and widened to fp64 when the fragments are loaded:
// products of fp32 values are exact in fp64.
template <typename TIN>
__device__ __forceinline__ void load_tile(TIN* s, int ss, const TIN* g, int64_t ld, int rows,
                                          int cols, int rows_ok, int cols_ok, bool vec) {
  constexpr int V = 16 / sizeof(TIN);   // elements per 16-byte chunk
  if (vec) {
    const int cpr = cols / V;
    for (int c = threadIdx.x; c < rows * cpr; c += THREADS) {
      int r = c / cpr, cc = (c % cpr) * V;
      int valid = (r < rows_ok) ? max(0, min(V, cols_ok - cc)) : 0;
      const TIN* src = valid ? g + int64_t(r) * ld + cc : g;
      cp_async16(s + r * ss + cc, src, valid * int(sizeof(TIN)));
    }
  } else {
    for (int c = threadIdx.x; c < rows * cols; c += THREADS) {
      int r = c / cols, cc = c % cols;
      int valid = (r < rows_ok && cc < cols_ok) ? 1 : 0;
      const TIN* src = valid ? g + int64_t(r) * ld + cc : g;
      cp_async_elem(s + r * ss + cc, src, valid);
    }
  }
}

template <bool TRANS, int NF, typename TIN = double>
__global__ void __launch_bounds__(THREADS, 1)
gemm_f64_kernel(int64_t M, int64_t N, int64_t K, const TIN* __restrict__ A, int64_t lda,
                const TIN* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc,
                int64_t kchunk, int64_t cstride, bool a16, bool b16) {
  using S = Smem<NF, TIN>;
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  TIN* As = reinterpret_cast<TIN*>(smem_bytes);
  TIN* Bs = As + STAGES * S::A_ELEMS;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;

  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t n0 = int64_t(blockIdx.y) * S::BN;
  const int64_t kbeg = int64_t(blockIdx.z) * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  const int nk = int((kend - kbeg + BK - 1) / BK);

  const int m_ok = int(min(int64_t(BM), M - m0));
  const int n_ok = int(min(int64_t(S::BN), N - n0));

  auto issue = [&](int kt, int stage) {
    const int64_t k0 = kbeg + int64_t(kt) * BK;
    const int k_ok = int(min(int64_t(BK), kend - k0));
    TIN* as = As + stage * S::A_ELEMS;
    TIN* bs = Bs + stage * S::B_ELEMS;
    if (!TRANS)
      load_tile(as, AS_NN, A + m0 * lda + k0, lda, BM, BK, m_ok, k_ok, a16);
    else
      load_tile(as, AS_TN, A + k0 * lda + m0, lda, BK, BM, k_ok, m_ok, a16);
    load_tile(bs, S::BS, B + k0 * ldb + n0, ldb, BK, S::BN, k_ok, n_ok, b16);
  };

  double acc[2][NF][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = kt + STAGES - 1;
      if (nxt < nk) issue(nxt, nxt % STAGES);
      cp_commit();
    }
    const int stage = kt % STAGES;
    const TIN* as = As + stage * S::A_ELEMS;
    const TIN* bs = Bs + stage * S::B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[2][2];
#pragma unroll
      for (int mf = 0; mf < 2; ++mf) {
        const int r = wm * 32 + mf * 16 + g;
        const int k = kk * 4 + t;
        if (!TRANS) {
          a[mf][0] = double(as[r * AS_NN + k]);
          a[mf][1] = double(as[(r + 8) * AS_NN + k]);
        } else {
          a[mf][0] = double(as[k * AS_TN + r]);
          a[mf][1] = double(as[k * AS_TN + r + 8]);
        }
      }
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        const double b = double(bs[(kk * 4 + t) * S::BS + wn * NF * 8 + nf * 8 + g]);
        dmma(acc[0][nf], a[0][0], a[0][1], b);
        dmma(acc[1][nf], a[1][0], a[1][1], b);
      }
    }
  }
  cp_wait<0>();

  // epilogue: C fragment (row g / g+8, cols 2t, 2t+1)
#pragma unroll
  for (int mf = 0; mf < 2; ++mf) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int r = wm * 32 + mf * 16 + g + half * 8;
      if (r >= m_ok) continue;
      double* crow = C + int64_t(blockIdx.z) * cstride + (m0 + r) * ldc + n0;
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        const int c = wn * NF * 8 + nf * 8 + 2 * t;
        if (c < n_ok) crow[c] = acc[mf][nf][half * 2];
        if (c + 1 < n_ok) crow[c + 1] = acc[mf][nf][half * 2 + 1];
      }
    }
  }
}

// out (M x N, ldo) = sum_s part[s] (M x N, dense ld N) in order s = 0..S-1
__global__ void splitk_reduce_f64(int64_t M, int64_t N, int S, const double* __restrict__ part,
                                  double* __restrict__ out, int64_t ldo) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[int64_t(k) * total + i];
    out[(i / N) * ldo + (i % N)] = s;
  }
}

// Many splits (one-tile Grams: up to one per SM) over few outputs: 8 threads
// per output element each sum a fixed stride of the partials, then a fixed
// order combine in shared memory (deterministic, 8x the parallelism of the
// one-thread-per-element sum whose 148 dependent loads were latency-bound).
__global__ void splitk_reduce_wide(int64_t M, int64_t N, int S, const double* __restrict__ part,
                                   double* __restrict__ out, int64_t ldo) {
  __shared__ double red[8][33];
  const int64_t total = M * N;
  const int64_t i = int64_t(blockIdx.x) * 32 + threadIdx.x;
  double s = 0.0;
  if (i < total)
    for (int k = threadIdx.y; k < S; k += 8) s += part[int64_t(k) * total + i];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && i < total) {
    double t = 0.0;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
    out[(i / N) * ldo + (i % N)] = t;
  }
}

}  // namespace

void splitk_reduce(Handle* h, int64_t M, int64_t N, int S, const double* part, double* C,
                   int64_t ldc) {
  const int64_t total = M * N;
  if (S >= 16) {
    splitk_reduce_wide<<<unsigned(ceil_div(total, 32)), dim3(32, 8), 0, h->stream>>>(
        M, N, S, part, C, ldc);
  } else {
    const int blocks = int(std::min<int64_t>(ceil_div(total, 256), int64_t(h->sm_count) * 8));
    splitk_reduce_f64<<<blocks, 256, 0, h->stream>>>(M, N, S, part, C, ldc);
  }
  LR_CHECK_LAUNCH();
}

namespace {

template <bool TRANS, int NF, typename TIN>
void launch_nf(Handle* h, int64_t M, int64_t N, int64_t K, const TIN* A, int64_t lda,
               const TIN* B, int64_t ldb, double* C, int64_t ldc) {
  using S = Smem<NF, TIN>;
  auto kern = gemm_f64_kernel<TRANS, NF, TIN>;
  static AttrOnce attr_once;
  attr_once([&] {
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(S::bytes)));
  });
  const int64_t mt = ceil_div(M, BM), nt = ceil_div(N, S::BN);
  // (one-tile products -- the Gram of config 2's 8192 x 110 panels -- keep one
  // split per SM: capping the splits at >= 128 / 256 / 512 rows each measured
  // 5.21 / 5.44 / 5.89 ms per config-2 step against 5.18)
  const int64_t splits_wanted = choose_splits(h->sm_count, mt * nt, K);
  const int64_t kchunk = ceil_div(ceil_div(K, splits_wanted), BK) * BK;
  const int64_t splits = std::max<int64_t>(1, ceil_div(K, kchunk));
  constexpr int V = 16 / sizeof(TIN);
  const bool a16 = (lda % V == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool b16 = (ldb % V == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
  dim3 grid{unsigned(mt), unsigned(nt), unsigned(splits)};
  if (splits == 1) {
    kern<<<grid, THREADS, S::bytes, h->stream>>>(M, N, K, A, lda, B, ldb, C, ldc, kchunk, 0,
                                                   a16, b16);
    LR_CHECK_LAUNCH();
    return;
  }
  double* part = pool_alloc_t<double>(h, size_t(splits) * M * N);
  kern<<<grid, THREADS, S::bytes, h->stream>>>(M, N, K, A, lda, B, ldb, part, N, kchunk, M * N,
                                                 a16, b16);
  LR_CHECK_LAUNCH();
  splitk_reduce(h, M, N, int(splits), part, C, ldc);
}

template <bool TRANS, typename TIN>
void launch_trans(Handle* h, int64_t M, int64_t N, int64_t K, const TIN* A, int64_t lda,
                  const TIN* B, int64_t ldb, double* C, int64_t ldc) {
  // N beyond one 128-wide tile is handled by grid.y (A re-read per N tile).
  const int nf = int(std::min<int64_t>(8, ceil_div(N, 16)));
  switch (nf) {
    case 1: launch_nf<TRANS, 1, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    case 2: launch_nf<TRANS, 2, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    case 3: launch_nf<TRANS, 3, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    case 4: launch_nf<TRANS, 4, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    case 5: launch_nf<TRANS, 5, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    case 6: launch_nf<TRANS, 6, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    case 7: launch_nf<TRANS, 7, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
    default: launch_nf<TRANS, 8, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc); break;
  }
}

// B~ (2K x 2N real) for the non-transposed complex product: row 2k = [br, bi]
// interleaved (= B's own row), row 2k+1 = [-bi, br] interleaved.
__global__ void cplx_expand_b(int64_t K, int64_t N, const double2* __restrict__ B, int64_t ldb,
                              double* __restrict__ Bt) {
  const int64_t total = K * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / N, j = i % N;
    const double2 b = B[k * ldb + j];
    double* r0 = Bt + (2 * k) * (2 * N) + 2 * j;
    double* r1 = r0 + 2 * N;
    r0[0] = b.x;  r0[1] = b.y;
    r1[0] = -b.y; r1[1] = b.x;
  }
}

// Combine the (2M x 2N) real product D of the transposed complex case into
// C (M x N complex): conj -> (D00 + D11) + i(D01 - D10), else (D00 - D11) + i(D01 + D10).
__global__ void cplx_combine_t(int64_t M, int64_t N, const double* __restrict__ D, bool conj,
                               double2* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, j = i % N;
    const double* d0 = D + (2 * r) * (2 * N) + 2 * j;
    const double* d1 = d0 + 2 * N;
    double2 c;
    if (conj) { c.x = d0[0] + d1[1]; c.y = d0[1] - d1[0]; }
    else      { c.x = d0[0] - d1[1]; c.y = d0[1] + d1[0]; }
    C[r * ldc + j] = c;
  }
}

}  // namespace

int64_t choose_splits(int sm_count, int64_t tiles, int64_t K) {
  // Fill the machine with whole waves (1 CTA / SM); each split keeps >= 4
  // k-tiles; each extra wave costs a little (split-K partial traffic).  Few
  // tiles (Gram / Q^T Z of a tall panel: one or two tiles) take up to one
  // split per SM.
  // A product of only a few tiles with a short K (the ell x ell x ell
  // products of the small SVD: one CTA, 24 us at ell = 110) splits down to
  // 2 k-tiles per CTA.
  const int64_t min_k = (tiles <= 4 && K < 1024) ? 2 * BK : 4 * BK;
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(4096, K / min_k));
  int64_t best_s = 1;
  double best = -1.0;
  for (int64_t s = 1; s <= max_s; ++s) {
    const double ctas = double(tiles * s);
    const double waves = ctas / double(sm_count);
    const double eff = waves / std::ceil(waves);
    const double score = eff - 0.01 * std::ceil(waves);
    if (score > best + 1e-9) {
      best = score;
      best_s = s;
    }
    if (ctas >= 8.0 * sm_count) break;
  }
  return best_s;
}

void gemm_f64(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const double* A,
              int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc) {
  if (M == 0 || N == 0) return;
  if (K == 0) {
    for (int64_t r = 0; r < M; ++r)
      LR_CUDA(cudaMemsetAsync(C + r * ldc, 0, N * sizeof(double), h->stream));
    return;
  }
  if (gemm_small_ok(M, N, K)) {
    gemm_small_f64(h, transA, M, N, K, A, lda, B, ldb, C, ldc);
    return;
  }
  if (gemm_skinny_wide_ok(transA, M, N, K, C, ldc)) {
    gemm_skinny_wide(h, false, M, N, K, A, lda, B, ldb, C, ldc);
    return;
  }
  if (gemm_skinny_nn_ok(transA, M, N, K, C, ldc)) {
    gemm_skinny_nn(h, M, N, K, A, lda, B, ldb, C, ldc);
    return;
  }
  if (gemm_skinny_ok(transA, M, N, K)) {
    gemm_skinny_tn(h, M, N, K, A, lda, B, ldb, C, ldc);
    return;
  }
  if (gemm_f64_tma_ok(M, N, K, A, lda, B, ldb) && gemm_f64_tma_pick(transA, N, K)) {
    gemm_f64_tma(h, transA, M, N, K, A, lda, B, ldb, C, ldc);
    return;
  }
  if (transA) launch_trans<true, double>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else        launch_trans<false, double>(h, M, N, K, A, lda, B, ldb, C, ldc);
}

// C (fp64) = op(A) B for fp32 A, B on the FP64 tensor pipe: exact products,
// fp64 accumulation (the Gram of an fp32 panel).
void gemm_f64_from_f32(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                       int64_t lda, const float* B, int64_t ldb, double* C, int64_t ldc) {
  if (M == 0 || N == 0) return;
  if (K == 0) {
    for (int64_t r = 0; r < M; ++r)
      LR_CUDA(cudaMemsetAsync(C + r * ldc, 0, N * sizeof(double), h->stream));
    return;
  }
  if (gemm_f64_tma_f32_ok(transA, M, N, K, A, lda, B, ldb)) {
    gemm_f64_tma_f32(h, M, N, K, A, lda, B, ldb, C, ldc);
    return;
  }
  if (transA) launch_trans<true, float>(h, M, N, K, A, lda, B, ldb, C, ldc);
  else        launch_trans<false, float>(h, M, N, K, A, lda, B, ldb, C, ldc);
}

void gemm_c128(Handle* h, bool transA, bool conjA, int64_t M, int64_t N, int64_t K,
               const double2* A, int64_t lda, const double2* B, int64_t ldb, double2* C,
               int64_t ldc) {
  if (M == 0 || N == 0) return;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 4096)));
  if (!transA) {
    // C (M x 2N real view) = A_real (M x 2K) . B~ (2K x 2N)
    double* Bt = pool_alloc_t<double>(h, size_t(4) * K * N);
    cplx_expand_b<<<blocks, 256, 0, h->stream>>>(K, N, B, ldb, Bt);
    LR_CHECK_LAUNCH();
    gemm_f64(h, false, M, 2 * N, 2 * K, reinterpret_cast<const double*>(A), 2 * lda, Bt, 2 * N,
             reinterpret_cast<double*>(C), 2 * ldc);
  } else {
    // D (2M x 2N) = A_real^T (2M x K) . B_real (K x 2N); then combine
    double* D = pool_alloc_t<double>(h, size_t(4) * M * N);
    gemm_f64(h, true, 2 * M, 2 * N, K, reinterpret_cast<const double*>(A), 2 * lda,
             reinterpret_cast<const double*>(B), 2 * ldb, D, 2 * N);
    cplx_combine_t<<<blocks, 256, 0, h->stream>>>(M, N, D, conjA, C, ldc);
    LR_CHECK_LAUNCH();
  }
}

}  // namespace lr
