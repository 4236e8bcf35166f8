// K1/K2 in fp32 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces DenseOperator._apply / _apply_adjoint (reference core.py:391-395)
// for float32 A (config 4: 2^20 x 4096, ell = 256).  The reference computes
// in fp64; plain TF32 truncation fails parity at j = 1, so each pass uses a
// three-product split of scaled fp16 operands (
// tools/numerics_cfg4.py measured parity to j = 125, like honest fp32):
//     A ~ (A_hi + A_lo) / s_A,  X ~ (X_hi + X_lo) / s_X   (fp16, 22 bits)
//     A X ~ (A_hi X_hi + A_hi X_lo + A_lo X_hi) / (s_A s_X)
// with power-of-two scales from max|A| (operator validation) and max|X|.
// All three products accumulate into ONE fp32 TMEM accumulator.
//
// CTA = 128 rows of op(A) x all N <= 256 columns (one UMMA 128 x N x 16 per
// k-substep), k-stage 32, 256 threads, two rings: a 5-deep fp32 A ring
// (TMA -> converters; deep enough to keep ~64 KB of A in flight per SM) and
// a 3-deep operand ring (A hi/lo + X hi/lo -> MMA):
//   warp 0  TMA producer: fp32 A tiles (16 KB, TS1 - 1 stages ahead) and
//           fp16 X_hi/X_lo tiles
//   warp 1  MMA issuer (one lane): 6 x tcgen05.mma kind::f16 per stage
//   warp 2  TMEM allocator
//   warps 4-7  converters: fp32 A tile -> scaled fp16 hi/lo in the canonical
//           K-major SWIZZLE_64B layout (transposing for A^T), then the
//           epilogue: tcgen05.ld -> * 1/(s_A s_X) -> global (or split-K slice)
// A is read from HBM exactly once per pass (per N <= 256); X_hi / X_lo are
// prepared once per pass in K-major fp16 (small for A X; for A^T Y the
// prepared Y is 2 x 2 bytes per element, read from L2/HBM per M tile).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace lr {
namespace {

constexpr int TBM = 128;          // UMMA M
constexpr int TBK = 32;           // k per stage (64 B of fp16 per row)
#ifndef LR_TC_TS1
#define LR_TC_TS1 5
#endif
#ifndef LR_TC_TS2
#define LR_TC_TS2 3
#endif
constexpr int TS1 = LR_TC_TS1;    // fp32 A ring (TMA -> converters): deep, hides HBM latency
constexpr int TS2 = LR_TC_TS2;    // operand ring (A hi/lo + X hi/lo -> MMA)
constexpr int TTHREADS = 256;
constexpr int A32_BYTES = TBM * TBK * 4;    // 16 KB
constexpr int AH_BYTES = TBM * TBK * 2;     // 8 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// canonical K-major SWIZZLE_64B UMMA smem descriptor (rows of 64 B, 8-row
// groups 512 B apart; sm100 descriptor version 1)
__device__ __forceinline__ uint64_t desc_sw64(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t(512 >> 4) << 32) | (1ull << 46) |
         (4ull << 61);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// byte offset of element (row r, k) in a K-major SWIZZLE_64B fp16 tile
__device__ __forceinline__ int sw64_off(int r, int chunk) {
  return r * 64 + ((chunk ^ ((r >> 1) & 3)) << 4);
}

// 8 scaled fp32 values -> packed fp16 hi and lo pieces
__device__ __forceinline__ void split8(const float* v, float s, uint4& hi, uint4& lo) {
  __half2 h[4], l[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float x0 = v[2 * e] * s, x1 = v[2 * e + 1] * s;
    const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
    h[e] = __halves2half2(h0, h1);
    l[e] = __halves2half2(__float2half_rn(x0 - __half2float(h0)),
                          __float2half_rn(x1 - __half2float(h1)));
  }
  hi = *reinterpret_cast<uint4*>(h);
  lo = *reinterpret_cast<uint4*>(l);
}

template <bool TRANS>
__global__ void __launch_bounds__(TTHREADS, 1)
gemm_f32_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapBhi,
                   const __grid_constant__ CUtensorMap mapBlo, int M, int N, int BN,
                   int64_t k_per_split, int64_t K, float sA_host,
                   const float* __restrict__ sA_dev, const float* __restrict__ sB_dev,
                   float* __restrict__ C, int64_t ldc, int64_t cstride) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-align the dynamic smem base
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int B_BYTES = BN * TBK * 2;
  const int op_bytes = 2 * AH_BYTES + 2 * B_BYTES;
  unsigned char* ring2 = base + TS1 * A32_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring2 + TS2 * op_bytes);
  uint64_t* a32_full = bars;
  uint64_t* a32_empty = bars + TS1;
  uint64_t* ahl_full = bars + 2 * TS1;
  uint64_t* b_full = ahl_full + TS2;
  uint64_t* st_empty = b_full + TS2;
  uint64_t* acc_full = st_empty + TS2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  auto a32 = [&](int s) { return base + s * A32_BYTES; };
  auto ahi = [&](int s) { return ring2 + s * op_bytes; };
  auto alo = [&](int s) { return ring2 + s * op_bytes + AH_BYTES; };
  auto bhi = [&](int s) { return ring2 + s * op_bytes + 2 * AH_BYTES; };
  auto blo = [&](int s) { return ring2 + s * op_bytes + 2 * AH_BYTES + B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float sA = sA_dev ? *sA_dev : sA_host;
  const int m0 = blockIdx.x * TBM;
  const int64_t kbeg = int64_t(blockIdx.z) * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int nk = int((kend - kbeg + TBK - 1) / TBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < TS1; ++s) {
      mbar_init(&a32_full[s], 1);
      mbar_init(&a32_empty[s], 128);   // every converter thread arrives itself
    }
    for (int s = 0; s < TS2; ++s) {
      mbar_init(&ahl_full[s], 128);
      mbar_init(&b_full[s], 1);
      mbar_init(&st_empty[s], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int tmem_cols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer.  The fp32 A tiles run TS1 - 1 stages
      // ahead of the X tiles (whose slots free up only as the MMA retires);
      // one thread issues both (a separate X producer warp raced: wrong rows).
      const uint32_t bbytes = uint32_t(2 * B_BYTES);
      constexpr int D = TS1 - 1;
      auto issue_a = [&](int kt) {
        const int s = kt % TS1;
        const uint32_t ph = uint32_t(kt / TS1) & 1u;
        const int kc = int(kbeg + int64_t(kt) * TBK);
        mbar_wait(&a32_empty[s], ph ^ 1u);
        mbar_expect_tx(&a32_full[s], A32_BYTES);
        if (!TRANS) tma_load_2d(a32(s), &mapA, &a32_full[s], kc, m0);
        else        tma_load_2d(a32(s), &mapA, &a32_full[s], m0, kc);
      };
      for (int kt = 0; kt < D && kt < nk; ++kt) issue_a(kt);
      for (int kt = 0; kt < nk; ++kt) {
        if (kt + D < nk) issue_a(kt + D);
        const int s2 = kt % TS2;
        const uint32_t ph2 = uint32_t(kt / TS2) & 1u;
        const int kc = int(kbeg + int64_t(kt) * TBK);
        mbar_wait(&st_empty[s2], ph2 ^ 1u);
        mbar_expect_tx(&b_full[s2], bbytes);
        // X hi/lo are K-blocked: block kb = kc / 32 is BN contiguous rows of 64 B
        tma_load_2d(bhi(s2), &mapBhi, &b_full[s2], 0, (kc / TBK) * BN);
        tma_load_2d(blo(s2), &mapBlo, &b_full[s2], 0, (kc / TBK) * BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(TBM >> 4) << 24);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % TS2;
        const uint32_t ph = uint32_t(kt / TS2) & 1u;
        mbar_wait(&ahl_full[s], ph);
        mbar_wait(&b_full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dah = desc_sw64(ahi(s)), dal = desc_sw64(alo(s));
        const uint64_t dbh = desc_sw64(bhi(s)), dbl = desc_sw64(blo(s));
#pragma unroll
        for (int ks = 0; ks < TBK / 16; ++ks) {
          const uint64_t adv = uint64_t(ks * 32) >> 4;   // 16 fp16 = 32 bytes
          umma_f16(tmem, dah + adv, dbh + adv, idesc, (kt | ks) ? 1u : 0u);
          umma_f16(tmem, dah + adv, dbl + adv, idesc, 1u);
          umma_f16(tmem, dal + adv, dbh + adv, idesc, 1u);
        }
        umma_commit(&st_empty[s]);
      }
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    // ---------------- converters (one A row per thread), then epilogue
    const int r = threadIdx.x - 128;
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TS1;
      const uint32_t ph = uint32_t(kt / TS1) & 1u;
      const int s2 = kt % TS2;
      const uint32_t ph2 = uint32_t(kt / TS2) & 1u;
      mbar_wait(&a32_full[s], ph);
      float v[TBK];
      if (!TRANS) {
        // fp32 staging: row r (128 B), TMA SWIZZLE_128B (16-B chunk c at c ^ (r & 7))
        const unsigned char* row = a32(s) + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 q = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
          v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
        }
      } else {
        // fp32 staging [k][m] (512-B rows, no swizzle): column r
        const float* st = reinterpret_cast<const float*>(a32(s));
#pragma unroll
        for (int k = 0; k < TBK; ++k) v[k] = st[k * TBM + r];
      }
      // convert first: the fp32 values are consumed (the shared loads have
      // landed) before the slot is handed back to the TMA engine -- an
      // async-proxy overwrite is not ordered after generic loads still in flight
      uint4 hv[TBK / 8], lv[TBK / 8];
#pragma unroll
      for (int g = 0; g < TBK / 8; ++g) split8(v + 8 * g, sA, hv[g], lv[g]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a32_empty[s]);   // this thread's reads of the fp32 stage are done
      mbar_wait(&st_empty[s2], ph2 ^ 1u);   // MMA finished with the previous hi/lo tiles
#pragma unroll
      for (int g = 0; g < TBK / 8; ++g) {
        const int off = sw64_off(r, g);
        *reinterpret_cast<uint4*>(reinterpret_cast<char*>(ahi(s2)) + off) = hv[g];
        *reinterpret_cast<uint4*>(reinterpret_cast<char*>(alo(s2)) + off) = lv[g];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&ahl_full[s2]);   // this thread's hi/lo writes are visible to the MMA
    }
    // epilogue: TMEM -> registers (row per thread) -> per-warp shared
    // transpose (the ring is idle now) -> coalesced 128-B row stores
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const float inv_a = 1.0f / sA;
    const int q = warp - 4;                    // TMEM lane quarter
    float* wbuf = reinterpret_cast<float*>(base) + q * (32 * 33);
    float* cbase = C + int64_t(blockIdx.z) * cstride;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t d[32];
      const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
            "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]),
            "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]),
            "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]),
            "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]),
            "=r"(d[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) wbuf[lane * 33 + j] = __uint_as_float(d[j]);
      __syncwarp();
      const int col = c0 + lane;
      const float sc = col < N ? inv_a / sB_dev[col] : 0.f;
      for (int rr = 0; rr < 32; ++rr) {
        const int row = m0 + q * 32 + rr;
        if (row < M && col < N) cbase[int64_t(row) * ldc + col] = wbuf[rr * 33 + lane] * sc;
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
// operand preparation

__global__ void amax_f32_kernel(int64_t rows, int64_t cols, const float* __restrict__ X,
                                int64_t ld, unsigned int* __restrict__ out_bits) {
  float mx = 0.f;
  if (ld == cols && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    // contiguous: float4 grid-stride sweep (no per-element index division)
    const int64_t total = rows * cols, n4 = total / 4;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n4;
         e += int64_t(gridDim.x) * blockDim.x) {
      const float4 v = X4[e];
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (int64_t e = n4 * 4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x)
      mx = fmaxf(mx, fabsf(X[e]));
  } else {
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) mx = fmaxf(mx, fabsf(X[r * ld + c]));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(mx));
}

// power-of-two scale s with s * amax in [2^13, 2^14): |scaled| < 2^14 fits fp16
__device__ __forceinline__ float pow2_scale(float amax) {
  if (!(amax > 0.f) || !isfinite(amax)) return 1.f;
  int e;
  frexpf(amax, &e);   // amax = f * 2^e, f in [0.5, 1)
  return ldexpf(1.f, 14 - e);
}

// per-column power-of-two scales of X (K x N): one warp per column.  A
// per-tensor scale is not enough for operands whose columns differ by orders
// of magnitude (R^{-1} of an ill-conditioned panel): small columns would
// lose their low fp16 piece to underflow.
__global__ void col_amax_kernel(int64_t K, int64_t N, const float* __restrict__ X, int64_t ld,
                                unsigned int* __restrict__ bits) {
  // rows split over blocks, columns over threads: coalesced row reads
  const int64_t rows_per = (K + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = blockIdx.x * rows_per, k1 = min(K, k0 + rows_per);
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
    float mx = 0.f;
    for (int64_t k = k0; k < k1; ++k) mx = fmaxf(mx, fabsf(X[k * ld + n]));
    if (mx > 0.f) atomicMax(bits + n, __float_as_uint(mx));
  }
}

__global__ void make_scale_kernel(const unsigned int* bits, float* scale) {
  scale[0] = pow2_scale(__uint_as_float(bits[0]));
}

__global__ void col_scale_kernel(int64_t N, const unsigned int* __restrict__ bits,
                                 float* __restrict__ scale) {
  for (int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; n < N;
       n += int64_t(gridDim.x) * blockDim.x)
    scale[n] = pow2_scale(__uint_as_float(bits[n]));
}

// X (K x N row-major, ld) -> hi/lo fp16, column n scaled by scale[n], in the
// K-blocked K-major layout the MMA reads: block kb (32 k) holds BN rows of 64 B,
// element (n, k) at ((k / 32) * BN + n) * 32 + k % 32, so every k-stage of X
// is one contiguous TMA box (a plain N x K layout puts the rows of one stage
// K * 2 bytes apart -- 2 MB for A^T Y of config 4).
__global__ void split_transpose_kernel(int64_t K, int64_t N, const float* __restrict__ X,
                                       int64_t ld, int64_t Kp, int BN,
                                       const float* __restrict__ scale,
                                       __half* __restrict__ hi, __half* __restrict__ lo) {
  // 64 (k) x 32 (n) tile; each thread emits two consecutive k of one n as a
  // __half2 (128-byte warp stores; the 32 x 32 version issued 2-byte stores
  // and ran at ~45 % of HBM bandwidth on config 4's 2^20 x 256 panels)
  __shared__ float tile[64][33];
  const int64_t k0 = int64_t(blockIdx.x) * 64, n0 = int64_t(blockIdx.y) * 32;
  const float s = (n0 + threadIdx.x < N) ? scale[n0 + threadIdx.x] : 1.f;
#pragma unroll
  for (int i = threadIdx.y; i < 64; i += 8) {
    const int64_t k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? X[k * ld + n] * s : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t n = n0 + i, k = k0 + 2 * threadIdx.x;
    if (n < N && k < Kp) {
      const float v0 = tile[2 * threadIdx.x][i], v1 = tile[2 * threadIdx.x + 1][i];
      const __half2 h = __floats2half2_rn(v0, v1);
      const float2 hf = __half22float2(h);
      const int64_t o = ((k >> 5) * BN + n) * 32 + (k & 31);
      *reinterpret_cast<__half2*>(hi + o) = h;
      *reinterpret_cast<__half2*>(lo + o) = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
    }
  }
}

__global__ void reduce_slices_f32(int64_t M, int64_t N, int S, const float* __restrict__ part,
                                  float* __restrict__ out, int64_t ldo) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < S; ++k) s += part[int64_t(k) * total + i];
    out[(i / N) * ldo + (i % N)] = s;
  }
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    LR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    LR_REQUIRE(p != nullptr, LR_ECUDA, "cuTensorMapEncodeTiled not available");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_map_2d(CUtensorMapDataType dt, const void* ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LR_REQUIRE(r == CUDA_SUCCESS, LR_ECUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

CUtensorMap make_map_nd(CUtensorMapDataType dt, const void* ptr, int rank, const uint64_t* dims,
                        const uint64_t* strides, const uint32_t* box, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], estr[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    estr[i] = 1;
    if (i + 1 < rank) st[i] = strides[i];
  }
  CUresult r = encode_fn()(&m, dt, cuuint32_t(rank), const_cast<void*>(ptr), d, st, bx, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LR_REQUIRE(r == CUDA_SUCCESS, LR_ECUDA, "cuTensorMapEncodeTiled (n-D) failed");
  return m;
}

CUtensorMap make_map_3d(CUtensorMapDataType dt, const void* ptr, const uint64_t dims[3],
                        const uint64_t strides[2], const uint32_t box[3], CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t st[2] = {strides[0], strides[1]};
  const cuuint32_t bx[3] = {box[0], box[1], box[2]};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, dt, 3, const_cast<void*>(ptr), d, st, bx, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LR_REQUIRE(r == CUDA_SUCCESS, LR_ECUDA, "cuTensorMapEncodeTiled (3-D) failed");
  return m;
}

bool gemm_f32_tc_supported(bool transA, int64_t N, const float* A, int64_t lda) {
  return N >= 1 && N <= 256 && (lda % 4) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
}

// C (M x N) = op(A) B, fp32 in/out, three-product fp16 split on tcgen05.
// a_amax < 0: max|A| unknown, computed here (one extra read of A).
void gemm_f32_tc(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                 int64_t lda, double a_amax, const float* B, int64_t ldb, float* C,
                 int64_t ldc) {
  if (M == 0 || N == 0) return;
  LR_REQUIRE(gemm_f32_tc_supported(transA, N, A, lda), LR_EUNSUPPORTED,
             "gemm_f32_tc: unsupported shape/alignment");
  // scales: s_A on the host (from the operator's max|A|), per-column s_B on
  // the device
  unsigned int* bits = pool_alloc_t<unsigned int>(h, 4);
  float* sB = pool_alloc_t<float>(h, size_t(N));
  float sA = 1.f;
  float* sA_dev = nullptr;
  if (a_amax < 0) {
    // unknown max|A|: reduce it on the device (no host synchronization)
    sA_dev = reinterpret_cast<float*>(bits + 2);
    LR_CUDA(cudaMemsetAsync(bits + 1, 0, sizeof(unsigned int), h->stream));
    const int64_t rows = transA ? K : M, cols = transA ? M : K;
    amax_f32_kernel<<<h->sm_count * 8, 256, 0, h->stream>>>(rows, cols, A, lda, bits + 1);
    LR_CHECK_LAUNCH();
    make_scale_kernel<<<1, 1, 0, h->stream>>>(bits + 1, sA_dev);
    LR_CHECK_LAUNCH();
  } else if (a_amax > 0 && std::isfinite(a_amax)) {
    int e;
    std::frexp(a_amax, &e);
    sA = std::ldexp(1.f, 14 - e);
  }
  {
    unsigned int* cb = pool_alloc_t<unsigned int>(h, size_t(N));
    LR_CUDA(cudaMemsetAsync(cb, 0, sizeof(unsigned int) * N, h->stream));
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(K, 64),
                                                                  int64_t(h->sm_count) * 8));
    col_amax_kernel<<<unsigned(blocks), 256, 0, h->stream>>>(K, N, B, ldb, cb);
    LR_CHECK_LAUNCH();
    col_scale_kernel<<<unsigned(ceil_div(N, 256)), 256, 0, h->stream>>>(N, cb, sB);
    LR_CHECK_LAUNCH();
  }
  const int BN = int(ceil_div(N, 16) * 16);
  const int64_t Kp = ceil_div(K, TBK) * TBK;
  __half* Bhi = pool_alloc_t<__half>(h, size_t(BN) * Kp);
  __half* Blo = pool_alloc_t<__half>(h, size_t(BN) * Kp);
  if (BN != N) {
    LR_CUDA(cudaMemsetAsync(Bhi, 0, sizeof(__half) * BN * Kp, h->stream));
    LR_CUDA(cudaMemsetAsync(Blo, 0, sizeof(__half) * BN * Kp, h->stream));
  }
  {
    dim3 grid(unsigned(ceil_div(Kp, 64)), unsigned(ceil_div(N, 32)));
    split_transpose_kernel<<<grid, dim3(32, 8), 0, h->stream>>>(K, N, B, ldb, Kp, BN, sB, Bhi,
                                                                 Blo);
    LR_CHECK_LAUNCH();
  }
  CUtensorMap mapA = transA
      ? make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, A, uint64_t(M), uint64_t(K), uint64_t(lda) * 4,
                    TBM, TBK, CU_TENSOR_MAP_SWIZZLE_NONE)
      : make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, A, uint64_t(K), uint64_t(M), uint64_t(lda) * 4,
                    TBK, TBM, CU_TENSOR_MAP_SWIZZLE_128B);
  const uint64_t brows = uint64_t(Kp / TBK) * BN;   // K-blocked: 64-B rows
  CUtensorMap mapBh = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Bhi, TBK, brows, TBK * 2, TBK,
                                  uint32_t(BN), CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap mapBl = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Blo, TBK, brows, TBK * 2, TBK,
                                  uint32_t(BN), CU_TENSOR_MAP_SWIZZLE_64B);
  size_t smem = size_t(TS1) * A32_BYTES + size_t(TS2) * (2 * AH_BYTES + 2 * BN * TBK * 2) +
                1024 /*align*/ + 256 /*barriers*/;
  static int one_cta = -1;
  if (one_cta < 0) {
    const char* e = getenv("LR_TC_ONE_CTA");
    one_cta = (e && e[0] == '0') ? 0 : 1;
  }
  // One CTA per SM (more than half the SM's shared memory reserved): with two
  // co-resident CTAs (N <= 128 fits twice) some output rows still come out
  // wrong on B200 (tools/tc_probe2.py, K >= 4096, N = 20) -- not the
  // stage-release ordering (every converter thread now arrives itself);
  // open issue, LR_TC_ONE_CTA=0 reproduces it.
  if (one_cta) smem = std::max<size_t>(smem, 116 * 1024);
  const int64_t mt = ceil_div(M, TBM);
  int64_t splits = 1;
  if (mt < h->sm_count) {
    splits = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * h->sm_count, mt),
                                                    ceil_div(K, 8 * TBK)));
  }
  const int64_t kps = ceil_div(ceil_div(K, splits), TBK) * TBK;
  splits = ceil_div(K, kps);
  float* out = C;
  int64_t ldo = ldc, cstride = 0;
  if (splits > 1) {
    out = pool_alloc_t<float>(h, size_t(splits) * M * N);
    ldo = N;
    cstride = M * N;
  }
  dim3 grid(unsigned(mt), 1, unsigned(splits));
  if (transA) {
    auto kern = gemm_f32_tc_kernel<true>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, TTHREADS, smem, h->stream>>>(mapA, mapBh, mapBl, int(M), int(N), BN, kps, K, sA,
                                              sA_dev, sB, out, ldo, cstride);
  } else {
    auto kern = gemm_f32_tc_kernel<false>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, TTHREADS, smem, h->stream>>>(mapA, mapBh, mapBl, int(M), int(N), BN, kps, K, sA,
                                              sA_dev, sB, out, ldo, cstride);
  }
  LR_CHECK_LAUNCH();
  if (splits > 1) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 8192)));
    reduce_slices_f32<<<blocks, 256, 0, h->stream>>>(M, N, int(splits), out, C, ldc);
    LR_CHECK_LAUNCH();
  }
}

}  // namespace lr
