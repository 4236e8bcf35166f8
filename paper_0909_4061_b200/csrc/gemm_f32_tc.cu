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
#include <cstdio>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_common.cuh"
#include "tma.cuh"

namespace lr {
namespace {
using tc::mbar_arrive_cluster;
using tc::mbar_wait_cluster;
using tc::idesc_f16;
using tc::umma_f16_pair;
using tc::umma_commit_pair;
using tc::tmem_ld32;

constexpr int TBM = 128;          // UMMA M
constexpr int TBK = 32;           // k per stage (64 B of fp16 per row)
#ifndef LR_TC_DBG
#define LR_TC_DBG 0
#endif
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

// bulk tensor store smem -> global (bulk-group completion), and the waits
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map),
               "r"(c0), "r"(c1)
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
#if !(LR_TC_DBG & 1)   // timing experiment: hi*hi only (wrong results)
          umma_f16(tmem, dah + adv, dbl + adv, idesc, 1u);
          umma_f16(tmem, dal + adv, dbh + adv, idesc, 1u);
#endif
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
#if (LR_TC_DBG & 2)   // timing experiment: no conversion, no hi/lo writes
      mbar_arrive(&a32_empty[s]);
      mbar_wait(&st_empty[s2], ph2 ^ 1u);
      mbar_arrive(&ahl_full[s2]);
      continue;
#endif
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

// The same split, one 32-deep k-block per CTA iteration: the block's rows of
// X (32 x N fp32, contiguous when ld == N) are read with float4 loads into a
// [32][N] smem tile, and thread n writes the 64-byte hi and lo rows of
// output row n (4 x 16-byte stores; a warp writes 2 KB contiguous of each).
// Rows past K and columns N..BN-1 are written as zeros (no memset).  ~2x the
// bandwidth of split_transpose_kernel's 64 x 32 tiles on config 4's panels.
__global__ void __launch_bounds__(256)
split_kblock_kernel(int64_t K, int64_t N, const float* __restrict__ X, int64_t ld, int64_t Kp,
                    int BN, const float* __restrict__ scale, __half* __restrict__ hi,
                    __half* __restrict__ lo) {
  extern __shared__ float tile[];              // [32][BN + 1]
  const int64_t nkb = Kp / 32;
  const bool vec = (N % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  const int nq = BN / 4;                       // float4 per tile row
  const int per = (32 * nq + blockDim.x - 1) / blockDim.x;   // <= 8 (BN <= 256)
  // the next k-block's rows are loaded into registers while this one is
  // split and stored (one tile of loads in flight per thread)
  float4 buf[8];
  auto load = [&](int64_t kb) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + u * blockDim.x;
      buf[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u < per && e < 32 * nq) {
        const int r = e / nq, c = (e - r * nq) * 4;
        const int64_t k = kb * 32 + r;
        if (k < K && c < N) {
          if (vec) {
            buf[u] = __ldcs(reinterpret_cast<const float4*>(X + k * ld + c));
          } else {
            const float* xr = X + k * ld;
            buf[u].x = xr[c];
            buf[u].y = c + 1 < N ? xr[c + 1] : 0.f;
            buf[u].z = c + 2 < N ? xr[c + 2] : 0.f;
            buf[u].w = c + 3 < N ? xr[c + 3] : 0.f;
          }
        }
      }
    }
  };
  int64_t kb = blockIdx.x;
  if (kb < nkb) load(kb);
  for (; kb < nkb; kb += gridDim.x) {
    // tile row stride BN + 1: the column reads below (lane = (n, 8-k chunk))
    // hit 32 distinct banks
    const int TS = BN + 1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + u * blockDim.x;
      if (u < per && e < 32 * nq) {
        const int r = e / nq, c = (e - r * nq) * 4;
        float* t = tile + r * TS + c;
        t[0] = buf[u].x; t[1] = buf[u].y; t[2] = buf[u].z; t[3] = buf[u].w;
      }
    }
    __syncthreads();
    if (kb + gridDim.x < nkb) load(kb + gridDim.x);
    // 16-byte output chunk t = (n, q): k = 8q .. 8q + 7 of row n -- a warp
    // stores 512 contiguous bytes of hi and of lo
    for (int t = threadIdx.x; t < BN * 4; t += blockDim.x) {
      const int n = t >> 2, q = t & 3;
      const float sc = n < N ? scale[n] : 0.f;
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float v0 = tile[(8 * q + 2 * j) * TS + n] * sc;
        const float v1 = tile[(8 * q + 2 * j + 1) * TS + n] * sc;
        const __half2 h = __floats2half2_rn(v0, v1);
        const float2 hf = __half22float2(h);
        const __half2 l = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
        hw[j] = *reinterpret_cast<const uint32_t*>(&h);
        lw[j] = *reinterpret_cast<const uint32_t*>(&l);
      }
      reinterpret_cast<uint4*>(hi + (kb * BN + n) * 32)[q] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      reinterpret_cast<uint4*>(lo + (kb * BN + n) * 32)[q] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    __syncthreads();
  }
}

// X (K x N) -> the MMA's hi/lo operand layout (Kp = K rounded up to 32, BN >= N
// a multiple of 16); LR_SPLIT=tile keeps the 64 x 32 tile kernel
void split_operand(Handle* h, int64_t K, int64_t N, const float* X, int64_t ld, int64_t Kp,
                   int BN, const float* scale, __half* hi, __half* lo) {
  const char* e = getenv("LR_SPLIT");
  if (e && e[0] == 't') {
    if (BN != N) {
      LR_CUDA(cudaMemsetAsync(hi, 0, sizeof(__half) * BN * Kp, h->stream));
      LR_CUDA(cudaMemsetAsync(lo, 0, sizeof(__half) * BN * Kp, h->stream));
    }
    dim3 grid(unsigned(ceil_div(Kp, 64)), unsigned(ceil_div(N, 32)));
    split_transpose_kernel<<<grid, dim3(32, 8), 0, h->stream>>>(K, N, X, ld, Kp, BN, scale, hi,
                                                                 lo);
    LR_CHECK_LAUNCH();
    return;
  }
  const size_t smem = size_t(32) * (BN + 1) * sizeof(float);   // ~32 KB (BN <= 256)
  const int64_t nkb = Kp / 32;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(nkb, int64_t(h->sm_count) * 6)));
  split_kblock_kernel<<<grid, 256, smem, h->stream>>>(K, N, X, ld, Kp, BN, scale, hi, lo);
  LR_CHECK_LAUNCH();
}

// out (M x N, ldo) = sum over S slices of part (S x M x N), fixed order in
// fp64.  Each thread owns 4 consecutive elements (float4 loads) and keeps 8
// slice loads in flight (A^T Y at config 4 sums 256 slices of 4 MB: the
// one-element-per-thread version was latency-bound at ~0.8 ms).
__global__ void reduce_slices_f32(int64_t M, int64_t N, int S, const float* __restrict__ part,
                                  float* __restrict__ out, int64_t ldo) {
  const int64_t total = M * N;
  const bool vec = (total % 4) == 0 && (N % 4) == 0 &&
                   (reinterpret_cast<uintptr_t>(part) & 15) == 0;
  if (vec) {
    const int64_t t4 = total / 4;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < t4;
         q += int64_t(gridDim.x) * blockDim.x) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int k = 0;
      for (; k + 8 <= S; k += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = __ldcs(reinterpret_cast<const float4*>(part + int64_t(k + u) * total) + q);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s0 += double(v[u].x); s1 += double(v[u].y); s2 += double(v[u].z); s3 += double(v[u].w);
        }
      }
      for (; k < S; ++k) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(part + int64_t(k) * total) + q);
        s0 += double(v.x); s1 += double(v.y); s2 += double(v.z); s3 += double(v.w);
      }
      const int64_t i = q * 4, r = i / N, c = i % N;
      float* o = out + r * ldo + c;
      o[0] = float(s0); o[1] = float(s1); o[2] = float(s2); o[3] = float(s3);
    }
    return;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;     // fixed order, fp64
    for (int k = 0; k < S; ++k) s += double(part[int64_t(k) * total + i]);
    out[(i / N) * ldo + (i % N)] = float(s);
  }
}

// ---------------------------------------------------------------------------
// 256-row single-CTA pass kernel (deep-K passes over A, N <= 256).
//
// The round-1 kernel above (128 rows per CTA) streams the whole fp16 hi/lo
// X tile (2 x 2 bytes per element) out of L2 for every 128 rows of A: at
// config 4 the X stream is twice A's bytes, and with the conversion and 2/3
// of the UMMAs disabled the pass still took 4.6 ms (L2 -> SM traffic
// ~11 TB/s).  Here one CTA owns 256 rows of A -- two 128 x N TMEM
// accumulators (all 512 columns) sharing every X tile -- so the X stream per
// A byte halves without any cross-CTA handshake.
//   warp 0     TMA producer of the fp32 A tiles (256 rows x 32 k, one box)
//   warp 3     TMA producer of the X hi/lo tiles
//   warp 1     MMA issuer: 12 UMMAs (2 halves x 3 products x 2 k-steps)/stage
//   warp 2     TMEM owner
//   warps 4-11 converters (one A row each), then the epilogue (warps 4-7:
//              rows 0-127 from columns 0..N-1, warps 8-11: rows 128-255 from
//              columns 256..256+N-1 of TMEM)
constexpr int W_THREADS = 384;
constexpr int WBM = 256;
constexpr int W_A32 = WBM * TBK * 4;      // 32 KB
constexpr int W_AH = WBM * TBK * 2;       // 16 KB (one of hi / lo)
#ifndef LR_W_TS1
#define LR_W_TS1 3
#endif
#ifndef LR_W_TS2
#define LR_W_TS2 2
#endif
#ifndef LR_W_TS3
#define LR_W_TS3 2
#endif
constexpr int W_TS1 = LR_W_TS1;
constexpr int64_t W_KMAX = 4096;
#ifndef LR_W_PF
#define LR_W_PF 0      // measured: 0 / 3 / 6 / 12 stages ahead -> 5.50 / 5.67 / 5.71 / 6.47 ms
#endif
constexpr int W_PF = LR_W_PF;      // A stages prefetched into L2 ahead of the ring   // k-extent of one TMEM accumulator (see gemm_f32_m256)
constexpr int W_TS2 = LR_W_TS2;
constexpr int W_TS3 = LR_W_TS3;

template <bool TRANS>
__global__ void __launch_bounds__(W_THREADS, 1)
gemm_f32_m256_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapBhi,
                     const __grid_constant__ CUtensorMap mapBlo, int M, int N, int BN,
                     int64_t k_per_split, int64_t K, float sA_host,
                     const float* __restrict__ sA_dev, const float* __restrict__ sB_dev,
                     float* __restrict__ C, int64_t ldc, int64_t cstride) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int B_BYTES = BN * TBK * 2;
  const int B_SLOT = (2 * B_BYTES + 1023) & ~1023;
  unsigned char* ring2 = base + W_TS1 * W_A32;
  unsigned char* ring3 = ring2 + W_TS2 * 2 * W_AH;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring3 + W_TS3 * B_SLOT);
  uint64_t* a32_full = bars;
  uint64_t* a32_empty = a32_full + W_TS1;
  uint64_t* ahl_full = a32_empty + W_TS1;
  uint64_t* ahl_empty = ahl_full + W_TS2;
  uint64_t* b_full = ahl_empty + W_TS2;
  uint64_t* b_empty = b_full + W_TS3;
  uint64_t* acc_full = b_empty + W_TS3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  auto a32 = [&](int s) { return base + s * W_A32; };
  auto ahi = [&](int s) { return ring2 + s * 2 * W_AH; };
  auto alo = [&](int s) { return ring2 + s * 2 * W_AH + W_AH; };
  auto bhi = [&](int s) { return ring3 + s * B_SLOT; };
  auto blo = [&](int s) { return ring3 + s * B_SLOT + B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float sA = sA_dev ? *sA_dev : sA_host;
  const int m0 = blockIdx.x * WBM;
  const int64_t kbeg = int64_t(blockIdx.z) * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int nk = int((kend - kbeg + TBK - 1) / TBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_TS1; ++s) {
      mbar_init(&a32_full[s], 1);
      mbar_init(&a32_empty[s], 256);
    }
    for (int s = 0; s < W_TS2; ++s) {
      mbar_init(&ahl_full[s], 256);
      mbar_init(&ahl_empty[s], 1);
    }
    for (int s = 0; s < W_TS3; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // the fp32 ring holds only W_TS1 stages (32 KB each): A tiles further
      // ahead are prefetched into L2 so the ring's loads see L2, not HBM,
      // latency (the A stream needs ~40 GB/s per SM at the UMMA rate)
      auto prefetch = [&](int kt) {
        const int kc = int(kbeg + int64_t(kt) * TBK);
        if (!TRANS) tma_prefetch_2d(&mapA, kc, m0);
        else        tma_prefetch_2d(&mapA, m0, kc);
      };
      for (int kt = 0; kt < W_PF && kt < nk; ++kt) prefetch(kt);
      for (int kt = 0; kt < nk; ++kt) {
        if (W_PF > 0 && kt + W_PF < nk) prefetch(kt + W_PF);
        const int s = kt % W_TS1;
        mbar_wait(&a32_empty[s], (uint32_t(kt / W_TS1) & 1u) ^ 1u);
        mbar_expect_tx(&a32_full[s], W_A32);
        const int kc = int(kbeg + int64_t(kt) * TBK);
        if (!TRANS) tma_load_2d(a32(s), &mapA, &a32_full[s], kc, m0);
        else        tma_load_2d(a32(s), &mapA, &a32_full[s], m0, kc);
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % W_TS3;
        mbar_wait(&b_empty[s], (uint32_t(kt / W_TS3) & 1u) ^ 1u);
        mbar_expect_tx(&b_full[s], uint32_t(2 * B_BYTES));
        const int kc = int(kbeg + int64_t(kt) * TBK);
        tma_load_2d(bhi(s), &mapBhi, &b_full[s], 0, (kc / TBK) * BN);
        tma_load_2d(blo(s), &mapBlo, &b_full[s], 0, (kc / TBK) * BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(TBM >> 4) << 24);
      for (int kt = 0; kt < nk; ++kt) {
        const int s2 = kt % W_TS2, s3 = kt % W_TS3;
        mbar_wait(&ahl_full[s2], uint32_t(kt / W_TS2) & 1u);
        mbar_wait(&b_full[s3], uint32_t(kt / W_TS3) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dbh = desc_sw64(bhi(s3)), dbl = desc_sw64(blo(s3));
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint64_t dah = desc_sw64(ahi(s2) + half * (TBM * 64));
          const uint64_t dal = desc_sw64(alo(s2) + half * (TBM * 64));
          const uint32_t acc = tmem + uint32_t(half * 256);
#pragma unroll
          for (int ks = 0; ks < TBK / 16; ++ks) {
            const uint64_t adv = uint64_t(ks * 32) >> 4;
            umma_f16(acc, dah + adv, dbh + adv, idesc, (kt | ks) ? 1u : 0u);
#if !(LR_TC_DBG & 1)
            umma_f16(acc, dah + adv, dbl + adv, idesc, 1u);
            umma_f16(acc, dal + adv, dbh + adv, idesc, 1u);
#endif
          }
        }
        umma_commit(&ahl_empty[s2]);
        umma_commit(&b_empty[s3]);
      }
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    const int r = threadIdx.x - 128;           // A row within the 256-row tile
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % W_TS1;
      const int s2 = kt % W_TS2;
      mbar_wait(&a32_full[s], uint32_t(kt / W_TS1) & 1u);
#if (LR_TC_DBG & 2)
      mbar_arrive(&a32_empty[s]);
      mbar_wait(&ahl_empty[s2], (uint32_t(kt / W_TS2) & 1u) ^ 1u);
      mbar_arrive(&ahl_full[s2]);
      continue;
#endif
      float v[TBK];
      if (!TRANS) {
        const unsigned char* row = a32(s) + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 q = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
          v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
        }
      } else {
        const float* st = reinterpret_cast<const float*>(a32(s));
#pragma unroll
        for (int k = 0; k < TBK; ++k) v[k] = st[k * WBM + r];
      }
      uint4 hv[TBK / 8], lv[TBK / 8];
#pragma unroll
      for (int g = 0; g < TBK / 8; ++g) split8(v + 8 * g, sA, hv[g], lv[g]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a32_empty[s]);
      mbar_wait(&ahl_empty[s2], (uint32_t(kt / W_TS2) & 1u) ^ 1u);
#pragma unroll
      for (int g = 0; g < TBK / 8; ++g) {
        const int off = sw64_off(r, g);
        *reinterpret_cast<uint4*>(ahi(s2) + off) = hv[g];
        *reinterpret_cast<uint4*>(alo(s2) + off) = lv[g];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&ahl_full[s2]);
    }
    // epilogue: the rings are idle now; per-warp transpose buffers at base
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const float inv_a = 1.0f / sA;
    const int q = warp & 3;                     // TMEM lane quarter
    const int half = (warp - 4) >> 2;           // accumulator 0 / 1
    float* wbuf = reinterpret_cast<float*>(base) + (warp - 4) * (32 * 33);
    float* cbase = C + int64_t(blockIdx.z) * cstride;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t d[32];
      tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(half * 256 + c0), d);
#pragma unroll
      for (int j = 0; j < 32; ++j) wbuf[lane * 33 + j] = __uint_as_float(d[j]);
      __syncwarp();
      const int col = c0 + lane;
      const float sc = col < N ? inv_a / sB_dev[col] : 0.f;
#if !(LR_TC_DBG & 4)
      for (int rr = 0; rr < 32; ++rr) {
        const int row = m0 + half * TBM + q * 32 + rr;
        if (row < M && col < N) cbase[int64_t(row) * ldc + col] = wbuf[rr * 33 + lane] * sc;
      }
#endif
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair persistent pass kernel (default for N <= 256).
//
// Measured on the round-1 single-CTA kernel above at config 4 (2^20 x 4096,
// N = 256; tools/tc_pass_probe.py + LR_TC_DBG variants): 6.0 ms per A X
// pass, and still 4.6 ms with 1/3 of the UMMAs and no conversion at all --
// the pass was bound by L2 -> SM traffic, not by the tensor pipe: every
// 128-row CTA streams the whole fp16 hi/lo X (2 x 2 bytes per element, twice
// A's fp32 bytes per stage) out of L2.  Here two CTAs on a TPC form a pair
// (tcgen05.mma.cta_group::2, M = 256): each CTA converts its own 128 rows of
// A but loads only HALF of X's columns, so the L2 stream per A byte halves;
// the pair is persistent (one pair per TPC, static round-robin over the
// 256-row tiles / split-K units) with two TMEM accumulators, so the
// epilogue of one tile overlaps the main loop of the next.
//   warp 0      TMA producer of the fp32 A tiles
//   warp 3      TMA producer of this CTA's half of the X hi/lo tiles
//   warp 1      leader: MMA issuer (6 pair UMMAs of 256 x BN x 16 per
//               32-deep stage); peer: relays "stage ready" to the leader
//   warp 2      TMEM owner (2 x 256 columns, cta_group::2)
//   warps 4-7   converters (one A row per thread -> hi/lo fp16 K-major SW64)
//   warps 8-11  epilogue (TMEM -> x 1/(s_A s_X) -> smem transpose -> rows)
constexpr int P_THREADS = 384;
#ifndef LR_P_TS1
#define LR_P_TS1 5
#endif
#ifndef LR_P_SLEEP
#define LR_P_SLEEP 0
#endif
#ifndef LR_P_TS2
#define LR_P_TS2 3
#endif
#ifndef LR_P_TS3
#define LR_P_TS3 4
#endif
constexpr int P_STG_BYTES = 4 * 2 * 32 * 32 * 4;   // epilogue staging (>= 4 x 32 x 33 floats)
constexpr int P_TS1 = LR_P_TS1;   // fp32 A ring (TMA -> converters)
constexpr int P_TS2 = LR_P_TS2;   // A hi/lo ring (converters -> MMA)
constexpr int P_TS3 = LR_P_TS3;   // X-half hi/lo ring (TMA -> MMA)

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}

struct PairWork {
  int64_t units, mtiles, k_per_split, K;
  __device__ void unit(int64_t u, int64_t& tile, int64_t& split) const {
    tile = u % mtiles;
    split = u / mtiles;
  }
  __device__ int nk(int64_t split) const {
    const int64_t kb = split * k_per_split, ke = min(K, kb + k_per_split);
    return int((ke - kb + TBK - 1) / TBK);
  }
};

template <bool TRANS>
__global__ void __launch_bounds__(P_THREADS, 1)
gemm_f32_pair_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapBhi,
                     const __grid_constant__ CUtensorMap mapBlo,
                     const __grid_constant__ CUtensorMap mapC, bool tma_store, int M, int N,
                     int BN, PairWork w, float sA_host, const float* __restrict__ sA_dev,
                     const float* __restrict__ sB_dev, float* __restrict__ C, int64_t ldc,
                     int64_t cstride) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int HB = BN / 2;                      // X rows (output columns) per CTA
  const int HB_BYTES = HB * TBK * 2;
  const int HB_SLOT = (2 * HB_BYTES + 1023) & ~1023;
  unsigned char* ring2 = base + P_TS1 * A32_BYTES;                // A hi/lo
  unsigned char* ring3 = ring2 + P_TS2 * 2 * AH_BYTES;           // X half hi/lo
  // epilogue staging: per epilogue warp two 32 x 32 fp32 tiles (SW128, for the
  // bulk tensor stores), or the 32 x 33 transpose buffers of the row stores
  unsigned char* stg = ring3 + P_TS3 * HB_SLOT;                    // 4 x 8 KB
  float* ebuf = reinterpret_cast<float*>(stg);                     // 4 x 32 x 33 floats
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + P_STG_BYTES);
  uint64_t* a32_full = bars;
  uint64_t* a32_empty = a32_full + P_TS1;
  uint64_t* ahl_full = a32_empty + P_TS1;
  uint64_t* ahl_empty = ahl_full + P_TS2;
  uint64_t* b_full = ahl_empty + P_TS2;
  uint64_t* b_empty = b_full + P_TS3;
  uint64_t* peer_full = b_empty + P_TS3;      // [P_TS2] leader: peer's A hi/lo + X half ready
  uint64_t* acc_full = peer_full + P_TS2;     // [2]
  uint64_t* acc_empty = acc_full + 2;         // [2] (leader: 8 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  auto a32 = [&](int s) { return base + s * A32_BYTES; };
  auto ahi = [&](int s) { return ring2 + s * 2 * AH_BYTES; };
  auto alo = [&](int s) { return ring2 + s * 2 * AH_BYTES + AH_BYTES; };
  auto bhi = [&](int s) { return ring3 + s * HB_SLOT; };
  auto blo = [&](int s) { return ring3 + s * HB_SLOT + HB_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const float sA = sA_dev ? *sA_dev : sA_host;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_TS1; ++s) {
      mbar_init(&a32_full[s], 1);
      mbar_init(&a32_empty[s], 128);
    }
    for (int s = 0; s < P_TS2; ++s) {
      mbar_init(&ahl_full[s], 128);
      mbar_init(&ahl_empty[s], 1);
      mbar_init(&peer_full[s], 1);
    }
    for (int s = 0; s < P_TS3; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 3) {
    if (lane == 0) {
      // ---- TMA producers, one thread per stream (warp 0: fp32 A tiles into
      // the converters' ring; warp 3: this CTA's half of the X hi/lo tiles).
      // Separate threads: a single producer blocked on the A ring (which
      // drains only as fast as the converters) held back the X loads, so
      // every stage paid the L2 latency of its X tile.
      const bool is_a = warp == 0;
      int64_t g = 0;
      for (int64_t u = pair; u < w.units; u += npairs) {
        int64_t tile, sp;
        w.unit(u, tile, sp);
        const int nk = w.nk(sp);
        for (int kt = 0; kt < nk; ++kt, ++g) {
          const int kc = int(sp * w.k_per_split + int64_t(kt) * TBK);
          if (is_a) {
            const int s = int(g % P_TS1);
            mbar_wait(&a32_empty[s], (uint32_t(g / P_TS1) & 1u) ^ 1u);
            mbar_expect_tx(&a32_full[s], A32_BYTES);
            const int m0 = int(tile * 2 * TBM) + int(rank) * TBM;
            if (!TRANS) tma_load_2d(a32(s), &mapA, &a32_full[s], kc, m0);
            else        tma_load_2d(a32(s), &mapA, &a32_full[s], m0, kc);
          } else {
            const int s3 = int(g % P_TS3);
            mbar_wait(&b_empty[s3], (uint32_t(g / P_TS3) & 1u) ^ 1u);
            mbar_expect_tx(&b_full[s3], uint32_t(2 * HB_BYTES));
            const int brow = (kc / TBK) * BN + int(rank) * HB;
            tma_load_2d(bhi(s3), &mapBhi, &b_full[s3], 0, brow);
            tma_load_2d(blo(s3), &mapBlo, &b_full[s3], 0, brow);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int64_t g = 0;
      if (rank != 0) {
        // ---- peer: relay "my A hi/lo and X half are in place" to the leader
        for (int64_t u = pair; u < w.units; u += npairs) {
          int64_t t_, sp;
          w.unit(u, t_, sp);
          const int nk = w.nk(sp);
          for (int kt = 0; kt < nk; ++kt, ++g) {
            const int s2 = int(g % P_TS2), s3 = int(g % P_TS3);
            mbar_wait(&ahl_full[s2], uint32_t(g / P_TS2) & 1u);
            mbar_wait(&b_full[s3], uint32_t(g / P_TS3) & 1u);
            mbar_arrive_cluster(&peer_full[s2], 0);
          }
        }
      } else {
        // ---- leader: MMA issuer
        const uint32_t idesc = idesc_f16(256, BN);
        int64_t it = 0;
        for (int64_t u = pair; u < w.units; u += npairs, ++it) {
          int64_t t_, sp;
          w.unit(u, t_, sp);
          const int nk = w.nk(sp);
          const int b = int(it & 1);
          if (it >= 2) mbar_wait_cluster(&acc_empty[b], uint32_t((it >> 1) - 1) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t acc = tmem + uint32_t(b * 256);
          for (int kt = 0; kt < nk; ++kt, ++g) {
            const int s2 = int(g % P_TS2), s3 = int(g % P_TS3);
            const uint32_t ph = uint32_t(g / P_TS2) & 1u;
            mbar_wait(&ahl_full[s2], ph);
            mbar_wait(&b_full[s3], uint32_t(g / P_TS3) & 1u);
            mbar_wait_cluster(&peer_full[s2], ph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t dah = desc_sw64(ahi(s2)), dal = desc_sw64(alo(s2));
            const uint64_t dbh = desc_sw64(bhi(s3)), dbl = desc_sw64(blo(s3));
#pragma unroll
            for (int ks = 0; ks < TBK / 16; ++ks) {
              const uint64_t adv = uint64_t(ks * 32) >> 4;
              umma_f16_pair(acc, dah + adv, dbh + adv, idesc, (kt | ks) ? 1u : 0u);
#if !(LR_TC_DBG & 1)
              umma_f16_pair(acc, dah + adv, dbl + adv, idesc, 1u);
              umma_f16_pair(acc, dal + adv, dbh + adv, idesc, 1u);
#endif
            }
            umma_commit_pair(&ahl_empty[s2]);
            umma_commit_pair(&b_empty[s3]);
          }
          umma_commit_pair(&acc_full[b]);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---- converters: row r of this CTA's 128-row A tile
    const int r = threadIdx.x - 128;
    int64_t g = 0;
    for (int64_t u = pair; u < w.units; u += npairs) {
      int64_t t_, sp;
      w.unit(u, t_, sp);
      const int nk = w.nk(sp);
      for (int kt = 0; kt < nk; ++kt, ++g) {
        const int s = int(g % P_TS1);
        const uint32_t ph = uint32_t(g / P_TS1) & 1u;
        const int s2 = int(g % P_TS2);
        const uint32_t ph2 = uint32_t(g / P_TS2) & 1u;
        mbar_wait(&a32_full[s], ph);
#if (LR_TC_DBG & 2)   // timing experiment: no conversion, no hi/lo writes
        mbar_arrive(&a32_empty[s]);
        mbar_wait(&ahl_empty[s2], ph2 ^ 1u);
        mbar_arrive(&ahl_full[s2]);
        continue;
#endif
        float v[TBK];
        if (!TRANS) {
          const unsigned char* row = a32(s) + r * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
            v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
          }
        } else {
          const float* st = reinterpret_cast<const float*>(a32(s));
#pragma unroll
          for (int k = 0; k < TBK; ++k) v[k] = st[k * TBM + r];
        }
        uint4 hv[TBK / 8], lv[TBK / 8];
#pragma unroll
        for (int q = 0; q < TBK / 8; ++q) split8(v + 8 * q, sA, hv[q], lv[q]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&a32_empty[s]);
        mbar_wait(&ahl_empty[s2], ph2 ^ 1u);
#pragma unroll
        for (int q = 0; q < TBK / 8; ++q) {
          const int off = sw64_off(r, q);
          *reinterpret_cast<uint4*>(ahi(s2) + off) = hv[q];
          *reinterpret_cast<uint4*>(alo(s2) + off) = lv[q];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&ahl_full[s2]);
      }
    }
  } else if (warp >= 8) {
    // ---- epilogue: this CTA's 128 rows of the 256-row pair tile
    const int q = warp - 8;                  // TMEM lane quarter (warp % 4)
    float* wbuf = ebuf + q * (32 * 33);
    const float inv_a = 1.0f / sA;
    int64_t it = 0;
    int nst = 0;                             // bulk stores issued by this warp
    for (int64_t u = pair; u < w.units; u += npairs, ++it) {
      int64_t tile, sp;
      w.unit(u, tile, sp);
      const int b = int(it & 1);
#if LR_P_SLEEP
      // a whole tile's main loop passes before the accumulator is ready:
      // back off instead of spinning on the issue slots the converters use
      {
        const uint32_t par = uint32_t(it >> 1) & 1u;
        uint32_t done = 0;
        while (true) {
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
              "selp.u32 %0, 1, 0, p;\n}"
              : "=r"(done)
              : "r"(smem_u32(&acc_full[b])), "r"(par)
              : "memory");
          if (done) break;
          __nanosleep(256);
        }
      }
#else
      mbar_wait_cluster(&acc_full[b], uint32_t(it >> 1) & 1u);
#endif
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int64_t mrow0 = tile * 2 * TBM + int64_t(rank) * TBM + q * 32;
      float* cbase = C + sp * cstride;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t d[32];
        tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(b * 256 + c0), d);
        if (c0 + 32 >= BN) {
          // this warp's reads of buffer b are complete: hand it back
          asm volatile("tcgen05.fence::before_thread_sync;");
          if (lane == 0) {
            if (rank == 0) mbar_arrive(&acc_empty[b]);
            else           mbar_arrive_cluster(&acc_empty[b], 0);
          }
        }
        if (tma_store) {
          // lane = row: its 32 consecutive columns, scaled, into a SW128
          // staging tile (16-byte chunk c of row r at chunk c ^ (r & 7):
          // conflict-free quarter-warp stores), then one bulk tensor store of
          // the 32 x 32 tile (the per-row scalar stores below were ~0.33 ms
          // of the 1.3 ms m x 256 . 256 x 256 apply at config 4)
          unsigned char* sb = stg + q * 8192 + (nst & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();     // this buffer's store 2 chunks ago has read it
          __syncwarp();
          const int col = c0 + lane;
          const float scol = col < N ? inv_a / sB_dev[col] : 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float4 v;
            v.x = __uint_as_float(d[4 * c]) * __shfl_sync(0xffffffffu, scol, 4 * c);
            v.y = __uint_as_float(d[4 * c + 1]) * __shfl_sync(0xffffffffu, scol, 4 * c + 1);
            v.z = __uint_as_float(d[4 * c + 2]) * __shfl_sync(0xffffffffu, scol, 4 * c + 2);
            v.w = __uint_as_float(d[4 * c + 3]) * __shfl_sync(0xffffffffu, scol, 4 * c + 3);
            *reinterpret_cast<float4*>(sb + lane * 128 + ((c ^ (lane & 7)) << 4)) = v;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&mapC, sb, c0, int(mrow0));
            bulk_commit();
          }
          ++nst;
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) wbuf[lane * 33 + j] = __uint_as_float(d[j]);
        __syncwarp();
        const int col = c0 + lane;
        const float sc = col < N ? inv_a / sB_dev[col] : 0.f;
#if !(LR_TC_DBG & 4)
        for (int rr = 0; rr < 32; ++rr) {
          const int64_t row = mrow0 + rr;
          if (row < M && col < N) cbase[row * ldc + col] = wbuf[rr * 33 + lane] * sc;
        }
#endif
        __syncwarp();
      }
    }
    if (tma_store && lane == 0) bulk_wait_all();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
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

// LR_TC_PAIR=0 keeps the single-CTA kernel (round 1) for every pass
bool pair_enabled() {
  const char* e = getenv("LR_TC_PAIR");
  return !(e && e[0] == '0');
}

// units = 256-row tiles x split-K slices, spread round-robin over the
// persistent pairs: pick the split count that fills the pairs' rounds best
// (>= 97 % of the last round busy), preferring fewer slices
int64_t pair_splits(int64_t mtiles, int64_t npairs, int64_t K) {
  if (mtiles >= 4 * npairs) return 1;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(K / (16 * TBK), 64));
  int64_t best = 1;
  double best_eff = 0.0;
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t u = mtiles * sp;
    const int64_t rounds = ceil_div(u, npairs);
    const double eff = double(u) / double(rounds * npairs);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
    }
    if (eff >= 0.97 && rounds >= 2) return sp;
  }
  return best;
}

void gemm_f32_pair(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                   int64_t lda, float sA, const float* sA_dev, const float* sB, const float* B,
                   int64_t ldb, float* C, int64_t ldc) {
  const int BN = int(ceil_div(N, 32) * 32);          // two halves of multiples of 16
  const int64_t Kp = ceil_div(K, TBK) * TBK;
  __half* Bhi = pool_alloc_t<__half>(h, size_t(BN) * Kp);
  __half* Blo = pool_alloc_t<__half>(h, size_t(BN) * Kp);
  split_operand(h, K, N, B, ldb, Kp, BN, sB, Bhi, Blo);
  CUtensorMap mapA = transA
      ? make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, A, uint64_t(M), uint64_t(K), uint64_t(lda) * 4,
                    TBM, TBK, CU_TENSOR_MAP_SWIZZLE_NONE)
      : make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, A, uint64_t(K), uint64_t(M), uint64_t(lda) * 4,
                    TBK, TBM, CU_TENSOR_MAP_SWIZZLE_128B);
  const uint64_t brows = uint64_t(Kp / TBK) * BN;
  CUtensorMap mapBh = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Bhi, TBK, brows, TBK * 2, TBK,
                                  uint32_t(BN / 2), CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap mapBl = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Blo, TBK, brows, TBK * 2, TBK,
                                  uint32_t(BN / 2), CU_TENSOR_MAP_SWIZZLE_64B);
  const size_t hb_slot = (size_t(2) * (BN / 2) * TBK * 2 + 1023) & ~size_t(1023);
  const size_t smem = size_t(P_TS1) * A32_BYTES + size_t(P_TS2) * 2 * AH_BYTES +
                      size_t(P_TS3) * hb_slot + P_STG_BYTES + 1024 /*align*/ +
                      256 /*barriers*/;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(P_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto kern = transA ? gemm_f32_pair_kernel<true> : gemm_f32_pair_kernel<false>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  // a persistent grid must be co-resident: TPCs with a disabled SM cannot
  // host a pair, so ask the occupancy API how many pairs fit at once
  // (a grid of sm_count / 2 pairs would leave a few for a second wave)
  static int resident[16] = {0};
  const int dev = h->device >= 0 && h->device < 16 ? h->device : 0;
  if (!resident[dev]) {
    cfg.gridDim = dim3(unsigned(h->sm_count), 1, 1);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc < 1) {
      cudaGetLastError();
      nc = h->sm_count / 2;
    }
    resident[dev] = nc;
    if (getenv("LR_TC_INFO"))
      fprintf(stderr, "[lr] pair kernel: %d co-resident pairs (sm_count %d)\n", nc, h->sm_count);
  }
  const int64_t npairs_max = std::min<int64_t>(resident[dev], h->sm_count / 2);
  const int64_t mtiles = ceil_div(M, 2 * TBM);
  const int64_t splits0 = pair_splits(mtiles, npairs_max, K);
  const int64_t kps = ceil_div(ceil_div(K, splits0), TBK) * TBK;
  const int64_t splits = ceil_div(K, kps);
  PairWork w{mtiles * splits, mtiles, kps, K};
  const int64_t npairs = std::min<int64_t>(npairs_max, w.units);
  float* out = C;
  int64_t ldo = ldc, cstride = 0;
  if (splits > 1) {
    out = pool_alloc_t<float>(h, size_t(splits) * M * N);
    ldo = N;
    cstride = M * N;
  }
  cfg.gridDim = dim3(unsigned(2 * npairs), 1, 1);
  // bulk tensor stores of the epilogue: one output slice, 16-byte rows
  const bool tma_store = cstride == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                         (ldo % 4) == 0 && !getenv("LR_TC_ROWSTORE");
  CUtensorMap mapC = tma_store
      ? make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, uint64_t(N), uint64_t(M),
                    uint64_t(ldo) * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)
      : mapA;
  LR_CUDA(cudaLaunchKernelEx(&cfg, kern, mapA, mapBh, mapBl, mapC, tma_store, int(M), int(N), BN,
                             w, sA, sA_dev, sB, out, ldo, cstride));
  LR_CHECK_LAUNCH();
  if (splits > 1) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 8192)));
    reduce_slices_f32<<<blocks, 256, 0, h->stream>>>(M, N, int(splits), out, C, ldc);
    LR_CHECK_LAUNCH();
  }
}

// LR_TC_M256=0 keeps the 128-row kernel for the deep-K passes
bool m256_enabled() {
  const char* e = getenv("LR_TC_M256");
  return !(e && e[0] == '0');
}

int64_t wave_splits(int64_t mt, int sm_count, int64_t K) {
  if (mt >= sm_count) return 1;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(ceil_div(K, 8 * TBK), 64));
  const int64_t smin = std::min<int64_t>(smax, ceil_div(sm_count, mt));
  double best_eff = 0.0;
  int64_t best = smin;
  for (int64_t sp = smin; sp <= smax; ++sp) {
    const int64_t ctas = mt * sp;
    const double eff = double(ctas) / double(ceil_div(ctas, sm_count) * sm_count);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
    }
    if (eff >= 0.97) break;
  }
  return best;
}

void gemm_f32_m256(Handle* h, bool transA, int64_t M, int64_t N, int64_t K, const float* A,
                   int64_t lda, float sA, const float* sA_dev, const float* sB, int BN,
                   int64_t Kp, const __half* Bhi, const __half* Blo, float* C, int64_t ldc) {
  CUtensorMap mapA = transA
      ? make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, A, uint64_t(M), uint64_t(K), uint64_t(lda) * 4,
                    WBM, TBK, CU_TENSOR_MAP_SWIZZLE_NONE)
      : make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, A, uint64_t(K), uint64_t(M), uint64_t(lda) * 4,
                    TBK, WBM, CU_TENSOR_MAP_SWIZZLE_128B);
  const uint64_t brows = uint64_t(Kp / TBK) * BN;
  CUtensorMap mapBh = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Bhi, TBK, brows, TBK * 2, TBK,
                                  uint32_t(BN), CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap mapBl = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Blo, TBK, brows, TBK * 2, TBK,
                                  uint32_t(BN), CU_TENSOR_MAP_SWIZZLE_64B);
  const size_t b_slot = (size_t(2) * BN * TBK * 2 + 1023) & ~size_t(1023);
  const size_t smem = size_t(W_TS1) * W_A32 + size_t(W_TS2) * 2 * W_AH + size_t(W_TS3) * b_slot +
                      1024 /*align*/ + 256 /*barriers*/;
  const int64_t mt = ceil_div(M, WBM);
  // the tensor cores' fp32 accumulation truncates: each of the 6 UMMAs per
  // 32-deep stage shrinks |acc| by ~2^-25 on average, so the relative bias
  // grows with the k-extent one accumulator covers.  Cap it at 4096 (the
  // A X pass's own depth at config 4): A^T Y with K = m = 2^20 is split 256
  // ways (measured at 65536 rows: top sigma 1.7e-5 relative with ~3.6k-row
  // slices, vs 2e-8 for the round-to-nearest FFMA path)
  const int64_t splits0 = std::max(wave_splits(mt, h->sm_count, K), ceil_div(K, W_KMAX));
  const int64_t kps = ceil_div(ceil_div(K, splits0), TBK) * TBK;
  const int64_t splits = ceil_div(K, kps);
  float* out = C;
  int64_t ldo = ldc, cstride = 0;
  if (splits > 1) {
    out = pool_alloc_t<float>(h, size_t(splits) * M * N);
    ldo = N;
    cstride = M * N;
  }
  dim3 grid(unsigned(mt), 1, unsigned(splits));
  auto kern = transA ? gemm_f32_m256_kernel<true> : gemm_f32_m256_kernel<false>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<grid, W_THREADS, smem, h->stream>>>(mapA, mapBh, mapBl, int(M), int(N), BN, kps, K, sA,
                                             sA_dev, sB, out, ldo, cstride);
  LR_CHECK_LAUNCH();
  if (splits > 1) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M * N, 256), 8192)));
    reduce_slices_f32<<<blocks, 256, 0, h->stream>>>(M, N, int(splits), out, C, ldc);
    LR_CHECK_LAUNCH();
  }
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
  if (a_amax < 0 && h->amax_bits_hint) {
    // max|A| already reduced on the device by the caller's previous kernel
    sA_dev = reinterpret_cast<float*>(bits + 2);
    make_scale_kernel<<<1, 1, 0, h->stream>>>(h->amax_bits_hint, sA_dev);
    LR_CHECK_LAUNCH();
  } else if (a_amax < 0) {
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
  // the CTA-pair persistent kernel wins where the single-CTA kernel pays
  // per-tile prologue / epilogue on short K (the m x 256 . 256 x 256 panel
  // products: 1.1 vs 1.7 ms at config 4); on the deep-K passes over A its
  // per-stage pair handshake measured ~1 us (7.0 vs 6.0 ms per A X pass),
  // so those stay on the single-CTA kernel
  const char* pe = getenv("LR_TC_PAIR");
  const bool force_pair = pe && pe[0] == '1';
  if (pair_enabled() && (h->sm_count % 2) == 0 && (force_pair || K <= 1024)) {
    gemm_f32_pair(h, transA, M, N, K, A, lda, sA, sA_dev, sB, B, ldb, C, ldc);
    return;
  }
  const int BN = int(ceil_div(N, 16) * 16);
  const int64_t Kp = ceil_div(K, TBK) * TBK;
  __half* Bhi = pool_alloc_t<__half>(h, size_t(BN) * Kp);
  __half* Blo = pool_alloc_t<__half>(h, size_t(BN) * Kp);
  split_operand(h, K, N, B, ldb, Kp, BN, sB, Bhi, Blo);
  if (m256_enabled() && M >= 8 * 256) {
    gemm_f32_m256(h, transA, M, N, K, A, lda, sA, sA_dev, sB, BN, Kp, Bhi, Blo, C, ldc);
    return;
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
    // one CTA per SM: choose the split count so the CTAs fill whole waves
    // (A^T Y at config 4: 32 tiles x 10 splits = 2.16 waves ran at 72 %)
    const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(ceil_div(K, 8 * TBK), 64));
    const int64_t smin = std::min<int64_t>(smax, ceil_div(h->sm_count, mt));
    double best_eff = 0.0;
    splits = smin;
    for (int64_t sp = smin; sp <= smax; ++sp) {
      const int64_t ctas = mt * sp;
      const int64_t waves = ceil_div(ctas, h->sm_count);
      const double eff = double(ctas) / double(waves * h->sm_count);
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        splits = sp;
      }
      if (eff >= 0.97) break;
    }
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
