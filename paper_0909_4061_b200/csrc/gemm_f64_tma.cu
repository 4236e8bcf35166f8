// K1/K2 in fp64, TMA-fed and warp-specialized (the default pass kernel).
//
// Same mathematics and tiling as gemm_f64.cu (DMMA mma.sync.m16n8k4 .f64,
// 128 x 16*NF CTA tile, 8 consumer warps 4 x 2, split-K with fixed-order
// partial sums), but the operand staging is done by ONE producer warp with
// TMA (cp.async.bulk.tensor) into a 6-stage mbarrier ring.  ncu on the
// cp.async kernel (profiles/round1_summary.md) showed the DMMA pipe only
// ~71 % busy, with ~20 % of the issued instructions being address arithmetic
// of the per-thread cp.async copies and a CTA barrier every k-stage; here the
// consumer warps issue only shared loads, DMMA and one mbarrier arrive per
// stage.
//   NN (A X):   A tile = box {16 k, 128 m} of the row-major A, 128-byte
//               swizzle (conflict-free fragment loads);
//   TN (A^T Y): A tile = box {128 m, 16 k} (m contiguous), no swizzle;
//   B tile   = box {BN n, 16 k} of the row-major X, no swizzle.
#include "common.cuh"
#include "tma.cuh"

namespace lr {
namespace {

constexpr int BM = 128;
constexpr int BK = 16;
#ifndef LR_TMA_ST
#define LR_TMA_ST 6
#endif
constexpr int ST = LR_TMA_ST;
constexpr int CONSUMERS = 8;
constexpr int THREADS = (CONSUMERS + 1) * 32;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                      int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

template <int NF, typename TIN = double>
struct Cfg {
  static constexpr int BN = 16 * NF;
  static constexpr int A_BYTES = BM * BK * int(sizeof(TIN));   // 16 KB (fp64)
  static constexpr int B_BYTES = BK * BN * int(sizeof(TIN));
  static constexpr int STAGE = A_BYTES + B_BYTES;              // multiple of 1024
  static constexpr size_t SMEM = size_t(ST) * STAGE + 1024 + 2 * ST * 8;
};

// TIN = float: fp32 operands (the Gram of an fp32 / complex64 panel) staged
// as fp32 and widened to fp64 at fragment load (exact products).  sym: C is
// the Gram of one operand (A == B, M == N): CTA tiles strictly below the
// diagonal are skipped and mirrored afterwards.
template <bool TRANS, int NF, typename TIN = double>
__global__ void __launch_bounds__(THREADS, 1)
gemm_f64_tma_kernel(const __grid_constant__ CUtensorMap mapA,
                    const __grid_constant__ CUtensorMap mapB, int64_t M, int64_t N, int64_t K,
                    double* __restrict__ C, int64_t ldc, int64_t kchunk, int64_t cstride,
                    bool sym) {
  using G = Cfg<NF, TIN>;
  if (sym && int64_t(blockIdx.y + 1) * G::BN <= int64_t(blockIdx.x) * BM) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + ST * G::STAGE);
  uint64_t* empty = full + ST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t n0 = int64_t(blockIdx.y) * G::BN;
  const int64_t kbeg = int64_t(blockIdx.z) * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  const int nk = kend > kbeg ? int((kend - kbeg + BK - 1) / BK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], CONSUMERS * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONSUMERS) {
    // ---------------- producer: one lane issues the TMA copies
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % ST;
        const uint32_t ph = uint32_t(kt / ST) & 1u;
        bar_wait(&empty[s], ph ^ 1u);
        bar_expect(&full[s], uint32_t(G::STAGE));
        const int k0 = int(kbeg + int64_t(kt) * BK);
        unsigned char* st = base + s * G::STAGE;
        if (!TRANS) tma2d(st, &mapA, &full[s], k0, int(m0));
        else        tma2d(st, &mapA, &full[s], int(m0), k0);
        tma2d(st + G::A_BYTES, &mapB, &full[s], int(n0), k0);
      }
    }
    return;
  }

  // ---------------- 8 consumer warps (4 x 2), warp tile 32 x 8 NF
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
  double acc[2][NF][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  // symmetric result: a warp whose 32 x 8NF tile lies strictly below the
  // diagonal issues no DMMA (mirrored afterwards), so a diagonal CTA tile
  // costs the SM's DMMA pipe 6/8 of a full one (BN = 128)
  const bool idle = sym && n0 + int64_t(wn + 1) * NF * 8 - 1 < m0 + int64_t(wm) * 32;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % ST;
    bar_wait(&full[s], uint32_t(kt / ST) & 1u);
    if (idle) {
      bar_arrive(&empty[s]);
      continue;
    }
    const TIN* as = reinterpret_cast<const TIN*>(base + s * G::STAGE);
    const TIN* bs = reinterpret_cast<const TIN*>(base + s * G::STAGE + G::A_BYTES);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int k = kk * 4 + t;
      double a[2][2];
#pragma unroll
      for (int mf = 0; mf < 2; ++mf) {
        const int r = wm * 32 + mf * 16 + g;
        if (!TRANS) {
          // 128-B swizzle: 16-B chunk c of row r lives at chunk c ^ (r & 7)
          // (fp64 only: the fp32 path is transposed-only)
          const int c = k >> 1, w = k & 1;
          a[mf][0] = double(as[r * 16 + ((c ^ (r & 7)) << 1) + w]);
          a[mf][1] = double(as[(r + 8) * 16 + ((c ^ ((r + 8) & 7)) << 1) + w]);
        } else {
          a[mf][0] = double(as[k * BM + r]);
          a[mf][1] = double(as[k * BM + r + 8]);
        }
      }
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        const double b = double(bs[k * G::BN + wn * NF * 8 + nf * 8 + g]);
        dmma(acc[0][nf], a[0][0], a[0][1], b);
        dmma(acc[1][nf], a[1][0], a[1][1], b);
      }
    }
    // every consumer thread releases the stage itself: an arrive by lane 0
    // after __syncwarp let the TMA overwrite a stage while loads of other lanes
    // were still reading it (intermittent wrong rows, tools/flaky_probe.py).
    // The release must also order this thread's own shared loads (generic
    // proxy, possibly still in flight: the arrive does not depend on them)
    // before the TMA refill (async proxy): proxy fence first.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bar_arrive(&empty[s]);
  }

  const int m_ok = int(min(int64_t(BM), M - m0));
  const int n_ok = int(min(int64_t(G::BN), N - n0));
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

// strictly-lower entries of a symmetric result <- transposed upper entries
// (the skipped CTA tiles and the idle warps' parts of the diagonal tiles)
__global__ void mirror_lower(int64_t n, double* __restrict__ C, int64_t ldc) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    if (j < i) C[i * ldc + j] = C[j * ldc + i];
  }
}

template <bool TRANS, int NF, typename TIN = double>
void launch(Handle* h, int64_t M, int64_t N, int64_t K, const TIN* A, int64_t lda,
            const TIN* B, int64_t ldb, double* C, int64_t ldc, bool sym = false) {
  using G = Cfg<NF, TIN>;
  auto kern = gemm_f64_tma_kernel<TRANS, NF, TIN>;
  constexpr CUtensorMapDataType DT =
      sizeof(TIN) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  static AttrOnce attr_once;
  attr_once([&] {
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(G::SMEM)));
  });
  constexpr uint64_t ES = sizeof(TIN);
  const CUtensorMap mapA =
      !TRANS ? make_map_2d(DT, A, uint64_t(K), uint64_t(M), uint64_t(lda) * ES, BK, BM,
                           CU_TENSOR_MAP_SWIZZLE_128B)
             : make_map_2d(DT, A, uint64_t(M), uint64_t(K), uint64_t(lda) * ES, BM, BK,
                           CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap mapB = make_map_2d(DT, B, uint64_t(N), uint64_t(K), uint64_t(ldb) * ES,
                                       G::BN, BK, CU_TENSOR_MAP_SWIZZLE_NONE);
  const int64_t mt = ceil_div(M, BM), nt = ceil_div(N, G::BN);
  // a symmetric result computes only the tiles reaching the diagonal: size
  // the split-K waves for those (the others exit at entry)
  int64_t live = mt * nt;
  if (sym) {
    live = 0;
    for (int64_t x = 0; x < mt; ++x)
      for (int64_t y = 0; y < nt; ++y) live += ((y + 1) * G::BN > x * BM) ? 1 : 0;
  }
  const int64_t want = choose_splits(h->sm_count, live, K);
  const int64_t kchunk = ceil_div(ceil_div(K, want), BK) * BK;
  const int64_t splits = std::max<int64_t>(1, ceil_div(K, kchunk));
  // (measured: giving the diagonal tiles, whose lower warps idle, 4/3 longer
  // k-chunks made config 4's Gram slower, 3.35 vs 2.99 ms -- a CTA's stage
  // time does not shrink with its DMMA count: uniform chunks)
  dim3 grid{unsigned(mt), unsigned(nt), unsigned(splits)};
  if (splits == 1) {
    kern<<<grid, THREADS, G::SMEM, h->stream>>>(mapA, mapB, M, N, K, C, ldc, kchunk, 0, sym);
    LR_CHECK_LAUNCH();
  } else {
    double* part = pool_alloc_t<double>(h, size_t(splits) * M * N);
    kern<<<grid, THREADS, G::SMEM, h->stream>>>(mapA, mapB, M, N, K, part, N, kchunk, M * N,
                                                sym);
    LR_CHECK_LAUNCH();
    splitk_reduce(h, M, N, int(splits), part, C, ldc);
  }
  if (sym) {
    mirror_lower<<<unsigned(std::min<int64_t>(ceil_div(M * N, 256), 4096)), 256, 0, h->stream>>>(
        M, C, ldc);
    LR_CHECK_LAUNCH();
  }
}

template <bool TRANS, typename TIN = double>
void launch_nf(Handle* h, int64_t M, int64_t N, int64_t K, const TIN* A, int64_t lda,
               const TIN* B, int64_t ldb, double* C, int64_t ldc, bool sym = false) {
  const int nf = int(std::min<int64_t>(8, ceil_div(N, 16)));
  switch (nf) {
    case 1: launch<TRANS, 1, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    case 2: launch<TRANS, 2, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    case 3: launch<TRANS, 3, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    case 4: launch<TRANS, 4, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    case 5: launch<TRANS, 5, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    case 6: launch<TRANS, 6, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    case 7: launch<TRANS, 7, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
    default: launch<TRANS, 8, TIN>(h, M, N, K, A, lda, B, ldb, C, ldc, sym); break;
  }
}

}  // namespace

// TMA needs 16-byte aligned bases and row strides; small products stay on the
// cp.async kernel (a descriptor encode per launch costs a few microseconds).
bool gemm_f64_tma_ok(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("LR_DMMA_TMA");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  if (off) return false;
  const bool aligned = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                       (lda % 2) == 0 && (ldb % 2) == 0;
  return aligned && double(M) * double(N) * double(K) >= double(1 << 28);
}

// measured (tools/gemm_probe.py, 16384 x 8192): TMA 32.6 / 33.0 TF at ell =
// 110 (NN / TN) against 25.0 / 25.2 for the cp.async kernel; for narrow TN
// products (ell = 30: 21 vs 27 TF) the cp.async kernel stays faster
// deep K only: a CTA needs enough k-stages to amortize its barrier setup and
// pipeline fill (the K = 32 / 110 products of the low-rank term and of Y R^{-1}
// stay on the cp.async kernel)
bool gemm_f64_tma_pick(bool transA, int64_t N, int64_t K) {
  return K >= 512 && (!transA || N >= 64);
}

void gemm_f64_tma(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc) {
  const bool sym = transA && A == B && M == N && lda == ldb;
  if (transA) launch_nf<true>(h, M, N, K, A, lda, B, ldb, C, ldc, sym);
  else        launch_nf<false>(h, M, N, K, A, lda, B, ldb, C, ldc);
}

// Gram-type products of fp32 panels (C = A^T B, fp64 out): TMA + DMMA with
// fp32 staging; symmetric results computed on the upper tiles only.
bool gemm_f64_tma_f32_ok(bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                         int64_t lda, const float* B, int64_t ldb) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("LR_DMMA_TMA");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  if (off || !transA || K < 512) return false;
  const bool aligned = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                       (lda % 4) == 0 && (ldb % 4) == 0;
  return aligned && double(M) * double(N) * double(K) >= double(1 << 26);
}

void gemm_f64_tma_f32(Handle* h, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb, double* C, int64_t ldc) {
  const bool sym = A == B && M == N && lda == ldb;
  launch_nf<true, float>(h, M, N, K, A, lda, B, ldb, C, ldc, sym);
}

}  // namespace lr
