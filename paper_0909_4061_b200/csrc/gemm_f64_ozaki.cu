// K1/K2 in fp64 on the int8 tensor cores (tcgen05.mma kind::i8): the passes
// over a float64 A (reference DenseOperator._apply / _apply_adjoint,
// core.py:391-395) as an exact-integer emulation of the fp64 product (Ozaki
// scheme, digit-sliced operands).
//
// B200's FP64 tensor pipe (DMMA) peaks near 36 TF/s, which makes a pass of
// config 2 (16384 x 8192 x 110) compute-bound at ~0.9 ms against 0.16 ms of
// HBM time.  The int8 pipe is ~100x faster, so the product is rebuilt from
// exact integer products:
//   A_ik = 2^eA_i * sum_{s=1..8} a_s,ik 2^-(6 + 7(s-1)),   |a_s| <= 64
//   X_kj = 2^eX_j * sum_{t=1..8} x_t,kj 2^-(6 + 7(t-1))
// (eA_i: exponent of row i's max, eX_j: of column j's max; the digits are
// exact fp64 rint remainders, 55 bits of each entry relative to its row /
// column maximum), and
//   (A X)_ij = 2^(eA_i + eX_j) * sum_{d=2..9} 2^-(12 + 7(d-2)) acc_d,ij,
//   acc_d = sum_{s+t=d} sum_k a_s,ik x_t,kj      (int32, exact)
// The 36 digit-plane products with s + t <= 9 are the only ones whose
// weight reaches fp64 resolution: the first dropped diagonal (d = 10) is
// 2^-53 of the |A||X| bound, the same size as the rounding of one fp64
// product -- the result has the accuracy of an fp64 GEMM (tests compare it
// with the DMMA kernels), and it is bitwise deterministic (integer sums).
//
// Data: the 8 digit planes of A are built once per operator
// (lr_ozaki_prepare, 8 bytes per entry like A itself) with row scaling; the
// same planes serve A^T Y, whose summation index is the row index: the row
// scales fold into Y (Y'_ik = 2^eA_i Y_ik, exact), and the A tile is read
// MN-major.  X / Y' are sliced per pass (small).
//
// Kernel: CTA = 128 rows x BN (32 or 64) columns, 8 int32 TMEM accumulators
// (one per diagonal d, 8 * BN <= 512 columns), k-stage = 32 (one UMMA K),
// 4-deep TMA ring of {8 A planes, 8 X planes} (48 KB per stage at BN = 64),
// warp-specialized: warp 0 TMA, warp 1 MMA issuer (36 UMMAs per stage),
// warp 2 TMEM allocator, warps 4-7 epilogue (TMEM -> fp64 combine -> scaled
// coalesced stores or a split-K slice).
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace lr {
namespace {

constexpr int OZ_S = 8;             // digit planes per operand
constexpr int OZ_ND = 8;            // diagonals d = 2..9
constexpr int OBM = 128;            // UMMA M
constexpr int OBK = 32;             // k per stage (= UMMA K for kind::i8)
#ifndef LR_OZ_ST
#define LR_OZ_ST 4
#endif
constexpr int OST = LR_OZ_ST;       // ring depth
constexpr int OTHREADS = 256;
constexpr int A_PLANE = OBM * OBK;  // 4 KB
constexpr int A_STAGE = OZ_S * A_PLANE;
// int32 headroom: at most 8 digit pairs per diagonal, |digit| <= 64, so one
// accumulator grows by <= 8 x 64^2 = 2^15 per k: K <= 2^15 keeps it < 2^30
constexpr int64_t OZ_KMAX = 32768;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (one request for a whole pre-swizzled tile)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
// byte offsets inside the shared-memory images the UMMA descriptors read:
// K-major SWIZZLE_32B (rows of 32 B; 16-B chunk c of row r at c ^ ((r >> 2) & 1))
__host__ __device__ __forceinline__ int img_k32(int r, int k) {
  return r * 32 + ((((k >> 4) ^ (r >> 2)) & 1) << 4) + (k & 15);
}
// MN-major SWIZZLE_128B (rows of 128 B along M, one row per k; chunk c at c ^ (k & 7))
__host__ __device__ __forceinline__ int img_mn128(int k, int mm) {
  return k * 128 + ((((mm >> 4) ^ k) & 7) << 4) + (mm & 15);
}

// K-major, 32-byte swizzle: rows of 32 B (one UMMA K of int8), 8-row groups 256 B apart
__device__ __forceinline__ uint64_t desc_k_sw32(const void* p) {
  return ((uint64_t(su32(p)) >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t(256 >> 4) << 32) |
         (1ull << 46) | (6ull << 61);
}
// MN-major, 128-byte swizzle: 128 M-elements (bytes) per K-row, 8-row groups
// 1024 B apart (one MN atom covers M = 128 int8)
__device__ __forceinline__ uint64_t desc_mn_sw128(const void* p) {
  return ((uint64_t(su32(p)) >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

// the 8 signed 7-bit digits of r in (-1, 1): r = sum_s d_s 2^-(6 + 7(s-1)) + O(2^-56)
__device__ __forceinline__ void digits8(double r, int8_t (&d)[OZ_S]) {
  double x = r * 64.0;
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) {
    const double q = rint(x);
    d[s] = static_cast<int8_t>(static_cast<int>(q));
    x = (x - q) * 128.0;
  }
}

__device__ __forceinline__ int exp_of(double amax) {
  if (!(amax > 0.0)) return 0;
  int e;
  frexp(amax, &e);   // amax = f 2^e, f in [0.5, 1): |v| 2^-e < 1
  return e;
}

// ---------------------------------------------------------------------------
// A planes (once per operator): row exponents, then digits

// Digits are fixed-point relative to each row's maximum, so an entry 2^-e
// below its row maximum keeps 55 - e bits: the pass is row-wise normwise
// accurate, |err_ij| <= 2^-50 max_k|A_ik| sum_k|X_kj|.  A graded row -- more
// than 1/8 of its nonzeros below 2^-OZ_RANGE of the row maximum, i.e. keeping
// fewer than 23 bits (fp32 precision) -- is counted in *wide_rows, and the
// caller keeps such a matrix on the DMMA passes, whose error is relative to
// |A||X| entrywise.  (Isolated tiny entries, as in Gaussian data, carry no
// weight and do not count.)
constexpr int OZ_RANGE = 32;

__global__ void oz_row_exp_kernel(int64_t m, int64_t n, const double* __restrict__ A, int64_t lda,
                                  int32_t* __restrict__ row_exp, int64_t i0,
                                  int32_t* __restrict__ wide_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = i0 + blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < m;
       i += warps) {
    double mx = 0.0;
    const double* row = A + i * lda;
    for (int64_t k = lane; k < n; k += 32) mx = fmax(mx, fabs(row[k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int e = exp_of(mx);
    if (lane == 0) row_exp[i] = e;
    if (wide_rows && mx > 0.0) {
      const double thr = ldexp(1.0, e - OZ_RANGE);
      int small = 0, nz = 0;
      for (int64_t k = lane; k < n; k += 32) {
        const double v = fabs(row[k]);
        nz += v > 0.0;
        small += (v > 0.0 && v < thr);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        small += __shfl_xor_sync(0xffffffffu, small, o);
        nz += __shfl_xor_sync(0xffffffffu, nz, o);
      }
      if (lane == 0 && 8 * small > nz) atomicAdd(wide_rows, 1);
    }
  }
}

// The digit planes of A are stored as the exact shared-memory images the
// pass kernel consumes, so every pipeline stage is ONE contiguous bulk copy
// (a tensor-map box of 32-byte rows split each stage into ~1024 sector
// requests, capping the A stream near 25 GB/s per SM):
//   imgN (A X):   tile (mt = i / 128, kt = k / 32), plane s: 128 rows x 32 B,
//                 K-major SWIZZLE_32B, at ((mt * KT + kt) * 8 + s) * 4 KB
//   imgT (A^T Y): tile (jt = k / 128, it = i / 32), plane s: 32 rows (i) x
//                 128 B (k), MN-major SWIZZLE_128B, at ((jt * IT + it) * 8 + s) * 4 KB
// with m, n padded to multiples of 128 (KT = NP / 32, IT = MP / 32); padding
// is zero.  Each image holds 8 * MP * NP bytes.
constexpr int OZB = 128;
constexpr int OZP = 256;          // m, n padding (the 2-SM kernel pairs 128-row tiles)
constexpr int64_t TILE = 4096;   // bytes of one plane of one stage tile

__global__ void oz_slice_a_kernel(int64_t m, int64_t n, const double* __restrict__ A, int64_t lda,
                                  const int32_t* __restrict__ row_exp, int8_t* __restrict__ imgN,
                                  int8_t* __restrict__ imgT, int64_t MP, int64_t NP, int64_t i0,
                                  int64_t i1) {
  // rows [i0, i1) of the padded MP x NP matrix; one thread: 4 consecutive k of
  // one row i (4-byte stores into imgN)
  const int64_t groups = NP / 4, total = (i1 - i0) * groups;
  const int64_t KT = NP / 32, IT = MP / 32;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = i0 + g / groups, k0 = (g % groups) * 4;
    const int e = i < m ? row_exp[i] : 0;
    uint32_t packed[OZ_S];
    int8_t dd[4][OZ_S];
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) packed[s] = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u;
      digits8((i < m && k < n) ? ldexp(A[i * lda + k], -e) : 0.0, dd[u]);
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) packed[s] |= uint32_t(uint8_t(dd[u][s])) << (8 * u);
    }
    // imgN: 4 consecutive k stay inside one 16-B chunk
    int8_t* tn = imgN + ((i / OZB) * KT + k0 / 32) * OZ_S * TILE + img_k32(int(i % OZB), int(k0 % 32));
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(tn + s * TILE) = packed[s];
    // imgT: byte (i, k) -> tile (k / 128, i / 32), row i % 32, column k % 128
    int8_t* tt = imgT + ((k0 / OZB) * IT + i / 32) * OZ_S * TILE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int off = img_mn128(int(i % 32), int((k0 + u) % OZB));
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) tt[s * TILE + off] = dd[u][s];
    }
  }
}

// ---------------------------------------------------------------------------
// X / Y' planes (per pass): column exponents of X' = diag(2^row_exp) X, then
// the digits transposed to [t][j][k] (K-major B operand), rows j >= N zero

__global__ void oz_col_max_kernel(int64_t K, int64_t N, const double* __restrict__ X, int64_t ldx,
                                  const int32_t* __restrict__ row_exp,
                                  unsigned long long* __restrict__ bits) {
  // block (32 x 8): columns tx + 32 c, rows ty + 8 r of the block's row range;
  // the 8 row lanes combine through shared memory, one atomic per column
  __shared__ double red[8][33];
  const int64_t rows_per = (K + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = blockIdx.x * rows_per, k1 = min(K, k0 + rows_per);
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int64_t j0 = 0; j0 < N; j0 += 32) {
    const int64_t j = j0 + tx;
    double mx = 0.0;
    if (j < N) {
#pragma unroll 4
      for (int64_t k = k0 + ty; k < k1; k += 8) {
        const double v = X[k * ldx + j];
        mx = fmax(mx, fabs(row_exp ? ldexp(v, row_exp[k]) : v));
      }
    }
    red[ty][tx] = mx;
    __syncthreads();
    if (ty == 0 && j < N) {
#pragma unroll
      for (int r = 1; r < 8; ++r) mx = fmax(mx, red[r][tx]);
      if (mx > 0.0) atomicMax(bits + j, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
    __syncthreads();
  }
}

__global__ void oz_col_exp_kernel(int64_t N, const unsigned long long* __restrict__ bits,
                                  int32_t* __restrict__ col_exp) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < N;
       j += int64_t(gridDim.x) * blockDim.x)
    col_exp[j] = exp_of(__longlong_as_double(static_cast<long long>(bits[j])));
}

// digits of X' into the B-operand images: tile (nt = j / BN, kt = k / 32),
// plane t: BN rows (j) x 32 B (k), K-major SWIZZLE_32B, at
// ((nt * KTB + kt) * 8 + t) * BN * 32; j >= N and k >= K are zero.  One
// block: 32 k x 32 j through shared memory (coalesced X reads).
__global__ void oz_slice_b_kernel(int64_t K, int64_t N, int64_t Np, int BNmax, int64_t KTB,
                                  const double* __restrict__ X, int64_t ldx,
                                  const int32_t* __restrict__ row_exp,
                                  const int32_t* __restrict__ col_exp, int8_t* __restrict__ img) {
  __shared__ int8_t t8[OZ_S][32][33];
  const int64_t k0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t k = k0 + r, j = j0 + tx;
    double v = 0.0;
    if (k < K && j < N) {
      v = X[k * ldx + j];
      if (row_exp) v = ldexp(v, row_exp[k]);
      v = ldexp(v, -col_exp[j]);
    }
    int8_t d[OZ_S];
    digits8(v, d);
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) t8[s][tx][r] = d[s];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t j = j0 + r, k = k0 + tx;
    const int64_t nt = j / BNmax;
    const int jj = int(j - nt * BNmax);
    const int bnt = BNmax;
    if (j < Np && jj < bnt && k < KTB * 32) {
      const int64_t tile = int64_t(bnt) * 32;
      int8_t* dst = img + nt * KTB * OZ_S * int64_t(BNmax) * 32 + (k / 32) * OZ_S * tile +
                    img_k32(jj, int(k % 32));
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) dst[s * tile] = t8[s][r][tx];
    }
  }
}

// ---------------------------------------------------------------------------
// the pass kernel

template <bool TRANS>
__global__ void __launch_bounds__(OTHREADS, 1)
ozaki_gemm_kernel(const int8_t* __restrict__ imgA, const int8_t* __restrict__ imgB, int64_t KTA,
                  int64_t KTB, int M, int N, int BNmax, int64_t k_per_split, int64_t K,
                  const int32_t* __restrict__ row_exp, const int32_t* __restrict__ col_exp,
                  double* __restrict__ C, int64_t ldc, int64_t cstride, int dbg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // uniform tile width (a narrower last tile -- 64 + 48 for l = 110 -- measured
  // no faster: the UMMA count per stage, not N, sets the time)
  const int n0 = blockIdx.x * BNmax;
  const int BN = BNmax;
  const int b_plane = BN * OBK;
  const int stage_bytes = A_STAGE + OZ_S * b_plane;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + OST * (A_STAGE + OZ_S * BNmax * OBK));
  uint64_t* empty = full + OST;
  uint64_t* acc_full = empty + OST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // N tile fastest in launch order: the CTAs sharing an A tile run together (L2 reuse)
  const int m0 = blockIdx.y * OBM;
  const int64_t kbeg = int64_t(blockIdx.z) * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int nk = int((kend - kbeg + OBK - 1) / OBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < OST; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t tmem_cols = 32;
  while (tmem_cols < uint32_t(OZ_ND * BN)) tmem_cols <<= 1;   // power of two, <= 512
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % OST;
        const uint32_t ph = uint32_t(kt / OST) & 1u;
        const int kc = int(kbeg + int64_t(kt) * OBK);
        mb_wait(&empty[s], ph ^ 1u);
        unsigned char* st = base + s * stage_bytes;
        if (dbg == 2) {   // development: no loads (MMA throughput alone)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
          continue;
        }
        mb_expect(&full[s], uint32_t(stage_bytes));
        // stage images: A tile (m0 / 128, kc / 32), B tile (n0 / BN, kc / 32)
        bulk_g2s(st, imgA + ((m0 / OZB) * KTA + kc / 32) * int64_t(A_STAGE), uint32_t(A_STAGE),
                 &full[s]);
        bulk_g2s(st + A_STAGE, imgB + (n0 / BNmax) * KTB * int64_t(OZ_S * BNmax * OBK) +
                                   (kc / 32) * int64_t(OZ_S * b_plane),
                 uint32_t(OZ_S * b_plane), &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::i8: D = s32 (c_format 2), A/B signed int8 (format 1), A MN-major for A^T
      const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((TRANS ? 1u : 0u) << 15) |
                              (uint32_t(OBM >> 4) << 24);
      // X planes t = 1..8 are consecutive BN-row blocks of one K-major operand,
      // and the accumulators of diagonals d = 2..9 consecutive BN-column blocks
      // of TMEM: for A plane sa, the products with planes t = t0 .. t0+np-1
      // land in diagonals sa+t0 .. sa+t0+np-1 -- ONE UMMA with N = np * BN.
      // 12 UMMAs per stage instead of 36: each UMMA re-reads its A plane from
      // shared memory, which bounded the 36-product version (~90 clk each).
      const int cmax = 256 / BN;
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % OST;
        const uint32_t ph = uint32_t(kt / OST) & 1u;
        mb_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const unsigned char* st = base + s * stage_bytes;
#pragma unroll
        for (int sa = 1; sa <= (dbg == 1 ? 0 : OZ_S); ++sa) {   // dbg 1: no MMA (loads alone)
          const uint64_t da = TRANS ? desc_mn_sw128(st + (sa - 1) * A_PLANE)
                                    : desc_k_sw32(st + (sa - 1) * A_PLANE);
          const int tmax = (OZ_ND + 1) - sa;   // t <= 9 - sa
          for (int t0 = 1; t0 <= tmax; t0 += cmax) {
            const int np = min(cmax, tmax - t0 + 1);
            const uint32_t idesc = idesc0 | (uint32_t((np * BN) >> 3) << 17);
            umma_i8(tmem + uint32_t((sa + t0 - 2) * BN),
                    da, desc_k_sw32(st + A_STAGE + (t0 - 1) * b_plane), idesc,
                    (kt > 0 || sa > 1) ? 1u : 0u);
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    mb_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp - 4;   // TMEM lane quarter: rows q*32 .. q*32+31
    const int row = m0 + q * 32 + lane;
    const int re = (row_exp && row < M) ? row_exp[row] : 0;
    double* wbuf = reinterpret_cast<double*>(base) + q * (32 * 33);   // ring is idle now
    double* cbase = C + int64_t(blockIdx.z) * cstride;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      double acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll 1
      for (int d = 9; d >= 2; --d) {   // smallest weights first
        uint32_t v[32];
        const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t((d - 2) * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const double w = ldexp(1.0, -(12 + 7 * (d - 2)) + re);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = fma(double(int32_t(v[j])), w, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) wbuf[lane * 33 + j] = acc[j];
      __syncwarp();
      const int col = n0 + c0 + lane;
      const int ce = col < N ? col_exp[col] : 0;
      for (int rr = 0; rr < 32; ++rr) {
        const int r = m0 + q * 32 + rr;
        if (r < M && col < N) cbase[int64_t(r) * ldc + col] = ldexp(wbuf[rr * 33 + lane], ce);
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_cols));
  }
}

// ---------------------------------------------------------------------------
// 2-SM variant (tcgen05.mma.cta_group::2): a CTA pair computes 256 rows x 56
// columns, one UMMA (issued by the even CTA) covering both SMs' 128-row A
// tiles.  The B operand of a cta_group::2 UMMA with N columns is split: the
// first N/2 rows come from the leader's shared memory, the last N/2 from the
// peer's, at the same address.  Each UMMA here has N = 112 = two X planes, so
// the peer keeps its X planes shifted by one slot: leader slot p = plane p+1,
// peer slot p = plane p+2.  For A plane s the planes t = 1..9-s go in pairs
// (t, t+1), t odd, at slot t-1 (D columns of diagonals s+t, s+t+1); an odd
// count's last pair reaches diagonal 10, kept in a 10th accumulator (9 x 56 =
// 504 TMEM columns) as an extra, correct high-order term -- no zero halves,
// and l = 110 pads to 112 columns, not 128.  20 UMMAs of 256 x 112 x 32 per
// stage.  Stage readiness of the peer's copies is relayed to the leader by a
// remote mbarrier arrive; the leader's commits multicast to both CTAs' "empty"
// and "accumulator full" barriers.
constexpr int B2_SLOTS = 8;
constexpr int BN2 = 56;
constexpr int ND2 = 9;                           // diagonals d = 2..10
constexpr int B2_STAGE = B2_SLOTS * BN2 * OBK;   // 14 KB
constexpr int ST2 = 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mb_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// arrive (release, cluster scope) on the barrier at the same offset in CTA `cta`
__device__ __forceinline__ void mb_arrive_remote(uint64_t* b, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(su32(b)),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ void umma2_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          su32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

template <bool TRANS>
__global__ void __launch_bounds__(OTHREADS, 1)
ozaki_gemm2_kernel(const int8_t* __restrict__ imgA, const int8_t* __restrict__ imgB, int64_t KTA,
                   int64_t KTB, int nt, int M, int N, int64_t k_per_split, int64_t K,
                   const int32_t* __restrict__ row_exp, const int32_t* __restrict__ col_exp,
                   double* __restrict__ C, int64_t ldc, int64_t cstride) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int stage_bytes = A_STAGE + B2_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + ST2 * stage_bytes);
  uint64_t* peer_full = full + ST2;
  uint64_t* empty = peer_full + ST2;
  uint64_t* acc_full = empty + ST2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int q = int(blockIdx.x >> 1);
  const int ntile = q % nt, pair = q / nt;
  const int m0 = (2 * pair + int(rank)) * OBM, n0 = ntile * BN2;
  const int64_t kbeg = int64_t(blockIdx.z) * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int nk = int((kend - kbeg + OBK - 1) / OBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST2; ++s) {
      mb_init(&full[s], 1);
      mb_init(&peer_full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  if (warp >= 4) {
    // the d = 10 accumulator is only ever accumulated into: zero it (each
    // epilogue warp its 32 lanes) before the pair's first UMMA
    const uint32_t base10 = tmem + (uint32_t((warp - 4) * 32) << 16) + uint32_t((ND2 - 1) * BN2);
#pragma unroll
    for (int c = 0; c < BN2; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       base10 + uint32_t(c)),
                   "r"(0u)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();   // both CTAs' barriers and TMEM (zeroed d = 10) ready before cross-CTA traffic
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (warp == 0) {
    if (lane == 0) {
      const int8_t* bsrc = imgB + (int64_t(ntile) * KTB * 2 + rank) * int64_t(B2_STAGE);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % ST2;
        const uint32_t ph = uint32_t(kt / ST2) & 1u;
        const int kc = int(kbeg + int64_t(kt) * OBK);
        mb_wait(&empty[s], ph ^ 1u);
        mb_expect(&full[s], uint32_t(stage_bytes));
        unsigned char* st = base + s * stage_bytes;
        bulk_g2s(st, imgA + ((m0 / OZB) * KTA + kc / 32) * int64_t(A_STAGE), uint32_t(A_STAGE),
                 &full[s]);
        bulk_g2s(st + A_STAGE, bsrc + int64_t(kc / 32) * 2 * B2_STAGE, uint32_t(B2_STAGE),
                 &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      if (rank != 0) {
        // peer: relay "my stage landed" to the leader
        for (int kt = 0; kt < nk; ++kt) {
          const int s = kt % ST2;
          mb_wait(&full[s], uint32_t(kt / ST2) & 1u);
          mb_arrive_remote(&peer_full[s], 0);
        }
      } else {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((TRANS ? 1u : 0u) << 15) |
                               (uint32_t((2 * BN2) >> 3) << 17) | (uint32_t(256 >> 4) << 24);
        for (int kt = 0; kt < nk; ++kt) {
          const int s = kt % ST2;
          const uint32_t ph = uint32_t(kt / ST2) & 1u;
          mb_wait(&full[s], ph);
          mb_wait_cluster(&peer_full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const unsigned char* st = base + s * stage_bytes;
          const unsigned char* bs = st + A_STAGE;
#pragma unroll
          for (int sa = 1; sa <= OZ_S; ++sa) {
            const uint64_t da = TRANS ? desc_mn_sw128(st + (sa - 1) * A_PLANE)
                                      : desc_k_sw32(st + (sa - 1) * A_PLANE);
            const int tmax = (OZ_ND + 1) - sa;
            // sa = 1 at the first stage writes diagonals 2..9 (d = 10 is pre-zeroed)
            const uint32_t acc = (kt > 0 || sa > 1) ? 1u : 0u;
            for (int t = 1; t <= tmax; t += 2)   // slot t-1: {plane t | plane t + 1}
              umma2_i8(tmem + uint32_t((sa + t - 2) * BN2), da,
                       desc_k_sw32(bs + (t - 1) * BN2 * OBK), idesc, acc);
          }
          umma2_commit_both(&empty[s]);
        }
        umma2_commit_both(acc_full);
      }
    }
  } else if (warp >= 4) {
    mb_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int qq = warp - 4;
    const int row = m0 + qq * 32 + lane;
    const int re = (row_exp && row < M) ? row_exp[row] : 0;
    double* wbuf = reinterpret_cast<double*>(base) + qq * (32 * 33);
    double* cbase = C + int64_t(blockIdx.z) * cstride;
    for (int c0 = 0; c0 < BN2; c0 += 32) {
      double acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll 1
      for (int d = ND2 + 1; d >= 2; --d) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (uint32_t(qq * 32) << 16) + uint32_t((d - 2) * BN2 + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const double w = ldexp(1.0, -(12 + 7 * (d - 2)) + re);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = fma(double(int32_t(v[j])), w, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) wbuf[lane * 33 + j] = acc[j];
      __syncwarp();
      const int col = n0 + c0 + lane;
      const bool cok = c0 + lane < BN2 && col < N;   // columns past the tile belong to the next diagonal
      const int ce = cok ? col_exp[col] : 0;
      for (int rr = 0; rr < 32; ++rr) {
        const int r = m0 + qq * 32 + rr;
        if (r < M && cok) cbase[int64_t(r) * ldc + col] = ldexp(wbuf[rr * 33 + lane], ce);
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();   // the peer's smem / TMEM stay alive until the pair is done
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// X' digits into the 2-SM B images: tile (nt, kt) holds two variants
// (leader, peer) of 8 slots x 56 rows x 32 B: leader slot p = plane p + 1,
// peer slot p = plane p + 2 (slot 7 zero).  Block: 32 k x 32
// j through shared memory; a thread then owns one row j and 4 consecutive k
// (one 4-byte word of a 16-byte chunk in every slot, the zero slots included,
// so the image needs no separate clearing).
__global__ void oz_slice_b2_kernel(int64_t K, int64_t N, int64_t Np, int64_t KTB,
                                   const double* __restrict__ X, int64_t ldx,
                                   const int32_t* __restrict__ row_exp,
                                   const int32_t* __restrict__ col_exp, int8_t* __restrict__ img) {
  __shared__ __align__(16) int8_t t8[OZ_S][32][36];
  const int64_t k0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    const int64_t k = k0 + r, j = j0 + tx;
    double v = 0.0;
    if (k < K && j < N) {
      v = X[k * ldx + j];
      if (row_exp) v = ldexp(v, row_exp[k]);
      v = ldexp(v, -col_exp[j]);
    }
    int8_t d[OZ_S];
    digits8(v, d);
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) t8[s][tx][r] = d[s];
  }
  __syncthreads();
  const int t = ty * 32 + tx;           // 256 threads: (row jj, k group kg)
  const int jj = t >> 3, kg = t & 7;
  const int64_t j = j0 + jj;
  if (j < Np && k0 < KTB * 32) {
    const int64_t nt = j / BN2;
    int8_t* tile = img + ((nt * KTB + k0 / 32) * 2) * int64_t(B2_STAGE);
    const int off = img_k32(int(j % BN2), 4 * kg);
    uint32_t w[OZ_S];
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) w[s] = *reinterpret_cast<const uint32_t*>(&t8[s][jj][4 * kg]);
    *reinterpret_cast<uint32_t*>(tile + B2_STAGE + 7 * BN2 * OBK + off) = 0u;        // peer slot 7
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) {
      *reinterpret_cast<uint32_t*>(tile + s * BN2 * OBK + off) = w[s];               // leader: plane s+1
      if (s >= 1)   // peer: plane s+1 at slot s-1
        *reinterpret_cast<uint32_t*>(tile + B2_STAGE + (s - 1) * BN2 * OBK + off) = w[s];
    }
  }
}

int oz_dbg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LR_OZ_DEBUG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

}  // namespace

// the two digit-plane images of A (see oz_slice_a_kernel): planes holds
// 16 * MP * NP bytes (imgN, then imgT), ldp = NP (n rounded up to 128).
// Rows [i0, i1) only (i0 a multiple of 128, i1 = m finishes the padding):
// the streamed upload prepares each chunk as it lands.
void ozaki_prepare_rows(Handle* h, int64_t m, int64_t n, int64_t i0, int64_t i1, const double* A,
                        int64_t lda, int8_t* planes, int64_t ldp, int32_t* row_exp,
                        int32_t* wide_rows) {
  LR_REQUIRE(ldp >= n && ldp % OZP == 0, LR_EINVAL,
             "ozaki_prepare: ldp must be n rounded up to a multiple of 256");
  LR_REQUIRE(i0 >= 0 && i0 % OZB == 0 && i1 > i0 && i1 <= m, LR_EINVAL,
             "ozaki_prepare: row range must start at a multiple of 128");
  const int64_t MP = ceil_div(m, OZP) * OZP;
  const int64_t iend = (i1 == m) ? MP : i1;
  LR_REQUIRE(iend % 32 == 0, LR_EINVAL, "ozaki_prepare: row range end must be a multiple of 32");
  const int blocks = h->sm_count * 8;
  oz_row_exp_kernel<<<blocks, 256, 0, h->stream>>>(i1, n, A, lda, row_exp, i0, wide_rows);
  LR_CHECK_LAUNCH();
  oz_slice_a_kernel<<<blocks, 256, 0, h->stream>>>(m, n, A, lda, row_exp, planes,
                                                   planes + OZ_S * MP * ldp, MP, ldp, i0, iend);
  LR_CHECK_LAUNCH();
}

void ozaki_prepare(Handle* h, int64_t m, int64_t n, const double* A, int64_t lda, int8_t* planes,
                   int64_t ldp, int32_t* row_exp, int32_t* wide_rows) {
  ozaki_prepare_rows(h, m, n, 0, m, A, lda, planes, ldp, row_exp, wide_rows);
}

namespace {
// LR_OZ_2SM=1 forces the CTA-pair kernel, =0 disables it; by default it runs
// for >= 8192 output rows (config 2: 0.530 / 0.540 ms vs 0.58 / 0.59 ms for
// A X / A^T Y; on a 4096-row A^T Y with K = 65536 it measured slower)
// ... and only where its 56-column tiles pad less than the single-CTA kernel's
// 64-column ones (l = 110: 112 vs 128 columns; at l = 128 the pair kernel's
// 3 x 56 measured 1.3 / 1.45 ms against 1.0 / 1.06 ms for 2 x 64).
bool oz_2sm(int64_t M, int64_t N) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LR_OZ_2SM");
    v = !e ? 2 : (e[0] == '1' ? 1 : 0);
  }
  return v == 1 || (v == 2 && M >= 8192 && ceil_div(N, 56) * 56 <= ceil_div(N, 64) * 64);
}

void ozaki_gemm_2sm(Handle* h, bool trans, int64_t M, int64_t N, int64_t K, const int8_t* imgA,
                    int64_t KTA, const int32_t* row_exp, const double* X, int64_t ldx,
                    const int32_t* rexp_b, const int32_t* col_exp, double* C, int64_t ldc) {
  const int64_t nt = ceil_div(N, BN2), Np = nt * BN2;
  const int64_t KTB = ceil_div(K, 32);
  int8_t* bimg = pool_alloc_t<int8_t>(h, size_t(nt) * KTB * 2 * B2_STAGE);
  {
    dim3 grid(unsigned(KTB), unsigned(ceil_div(Np, 32)));
    oz_slice_b2_kernel<<<grid, dim3(32, 8), 0, h->stream>>>(K, N, Np, KTB, X, ldx, rexp_b, col_exp,
                                                            bimg);
    LR_CHECK_LAUNCH();
  }
  const size_t smem = size_t(ST2) * (A_STAGE + B2_STAGE) + 1024 + 256;
  auto kern = trans ? ozaki_gemm2_kernel<true> : ozaki_gemm2_kernel<false>;
  static AttrOnce attr_once[2];
  attr_once[trans]([&] {
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  });
  const int64_t pairs = ceil_div(ceil_div(M, OBM), 2);
  int64_t want = choose_splits(h->sm_count, 2 * pairs * nt, K);
  want = std::max<int64_t>(want, ceil_div(K, OZ_KMAX));
  const int64_t kchunk = ceil_div(ceil_div(K, want), OBK) * OBK;
  const int64_t splits = ceil_div(K, kchunk);
  const int32_t* rexp_c = trans ? nullptr : row_exp;
  double* out = C;
  int64_t ldo = ldc, cstride = 0;
  if (splits > 1) {
    out = pool_alloc_t<double>(h, size_t(splits) * M * N);
    ldo = N;
    cstride = M * N;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(2 * pairs * nt), 1, unsigned(splits));
  cfg.blockDim = dim3(OTHREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 1;
  LR_CUDA(cudaLaunchKernelEx(&cfg, kern, imgA, static_cast<const int8_t*>(bimg), KTA, KTB, int(nt),
                             int(M), int(N), kchunk, K, rexp_c, col_exp, out, ldo, cstride));
  LR_CHECK_LAUNCH();
  if (splits > 1) splitk_reduce(h, M, N, int(splits), out, C, ldc);
}
}  // namespace

// C = A X (trans = false: A m x n, X n x N, C m x N) or C = A^T X (trans:
// X m x N, C n x N) from the prepared planes of A.
void ozaki_gemm(Handle* h, bool trans, int64_t m, int64_t n, int64_t N, const int8_t* planes,
                int64_t ldp, const int32_t* row_exp, const double* X, int64_t ldx, double* C,
                int64_t ldc) {
  const int64_t M = trans ? n : m;        // output rows
  const int64_t K = trans ? m : n;        // summation length
  if (M == 0 || N == 0) return;
  LR_REQUIRE(N <= 256, LR_EUNSUPPORTED, "ozaki_gemm: more than 256 columns");
  const int BN = N <= 32 ? 32 : 64;
  const int64_t nt = ceil_div(N, BN), Np = nt * BN;
  const int64_t KTB = ceil_div(K, 32);
  const int64_t MP = ceil_div(m, OZP) * OZP;
  // X' images and column exponents
  int8_t* bpl = pool_alloc_t<int8_t>(h, size_t(OZ_S) * Np * KTB * 32);
  unsigned long long* bits = pool_alloc_t<unsigned long long>(h, size_t(N));
  int32_t* col_exp = pool_alloc_t<int32_t>(h, size_t(N));
  LR_CUDA(cudaMemsetAsync(bits, 0, size_t(N) * sizeof(unsigned long long), h->stream));
  const int32_t* rexp_b = trans ? row_exp : nullptr;   // A^T Y: row scales fold into Y
  oz_col_max_kernel<<<unsigned(std::min<int64_t>(ceil_div(K, 64), int64_t(h->sm_count) * 4)),
                      dim3(32, 8), 0, h->stream>>>(K, N, X, ldx, rexp_b, bits);
  LR_CHECK_LAUNCH();
  oz_col_exp_kernel<<<1, 256, 0, h->stream>>>(N, bits, col_exp);
  LR_CHECK_LAUNCH();
  // A images: imgN tiles (m/128, n/32) for A X, imgT tiles (n/128, m/32) for A^T Y
  const int8_t* imgA = trans ? planes + OZ_S * MP * ldp : planes;
  const int64_t KTA = trans ? MP / 32 : ldp / 32;
  if (oz_2sm(M, N) && N > 32) {
    ozaki_gemm_2sm(h, trans, M, N, K, imgA, KTA, row_exp, X, ldx, rexp_b, col_exp, C, ldc);
    return;
  }
  {
    dim3 grid(unsigned(KTB), unsigned(ceil_div(Np, 32)));
    oz_slice_b_kernel<<<grid, dim3(32, 8), 0, h->stream>>>(K, N, Np, BN, KTB, X, ldx, rexp_b,
                                                           col_exp, bpl);
    LR_CHECK_LAUNCH();
  }
  const int stage_bytes = A_STAGE + OZ_S * BN * OBK;
  const size_t smem = size_t(OST) * stage_bytes + 1024 + 256;
  auto kern = trans ? ozaki_gemm_kernel<true> : ozaki_gemm_kernel<false>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t mt = ceil_div(M, OBM);
  int64_t want = choose_splits(h->sm_count, mt * nt, K);
  want = std::max<int64_t>(want, ceil_div(K, OZ_KMAX));
  const int64_t kchunk = ceil_div(ceil_div(K, want), OBK) * OBK;
  const int64_t splits = ceil_div(K, kchunk);
  dim3 grid{unsigned(nt), unsigned(mt), unsigned(splits)};
  const int32_t* rexp_c = trans ? nullptr : row_exp;
  if (splits == 1) {
    kern<<<grid, OTHREADS, smem, h->stream>>>(imgA, bpl, KTA, KTB, int(M), int(N), BN, kchunk, K, rexp_c,
                                              col_exp, C, ldc, 0, oz_dbg());
    LR_CHECK_LAUNCH();
    return;
  }
  double* part = pool_alloc_t<double>(h, size_t(splits) * M * N);
  kern<<<grid, OTHREADS, smem, h->stream>>>(imgA, bpl, KTA, KTB, int(M), int(N), BN, kchunk, K, rexp_c,
                                            col_exp, part, N, M * N, oz_dbg());
  LR_CHECK_LAUNCH();
  splitk_reduce(h, M, N, int(splits), part, C, ldc);
}

}  // namespace lr
