// K3 Gram of an fp32 panel on the 5th-generation tensor cores:
//     G (ell x ell, fp64) = Y^T Y,   Y m x ell fp32 (ell <= 256), m >> ell.
//
// Used for the SECOND CholeskyQR pass of an fp32 panel (orth_fast_impl):
// there Y = Q1 is already orthonormal to ~kappa^2 u64, so G = I + E needs
// fp32-level accuracy only (its error becomes the final loss of
// orthogonality, ~1e-7, the rounding level of the fp32 Q that is stored).
// The first pass's Gram of the ill-conditioned sample matrix stays exact
// (fp32 products in fp64 on DMMA, gemm_f64_tma.cu).  On the DMMA pipe this
// Gram of a 2^20 x 256 panel took ~2.9 ms (config 4, profiles/round1);
// here it is one read of Y (1 GiB: ~0.17 ms at HBM rate).
//
// Arithmetic: Y is scaled by a power of two s (entries must satisfy
// |y| s < 2^15, else status bit 1 sends the caller to the exact path) and
// split into fp16 hi + lo (22 bits); Y^T Y ~ hi^T hi + hi^T lo + lo^T hi,
// fp32 accumulation in TMEM over one CTA's row block (<= ~7k rows), the
// per-CTA partials summed in fp64 in a fixed order (deterministic).  The
// diagonal is taken from exact fp64 sums of squares accumulated by the
// converter threads (see gram_tc_reduce: the tensor-core accumulation
// truncates, which biases all-positive sums).
//
// CTA (one per SM, a contiguous block of rows): each 32-row stage of Y is
// TMA-loaded as fp32, converted by 4 warps into K-major SWIZZLE_64B hi/lo
// planes whose "rows" are the ell columns of Y (the k dimension is the 32
// panel rows), and the same planes serve as A (columns 0-127 / 128-255) and
// B: upper block row 0 is one M=128 x N=W product, block row 1 (W > 128) an
// M=128 x N=W-128 product on the diagonal block and right of it -- the
// lower-left block of the symmetric G is never computed.
//   warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM owner,
//   warps 4-7 converters, then the epilogue (TMEM -> fp32 partial tile).
#include "common.cuh"
#include "tc_common.cuh"
#include "tma.cuh"

namespace lr {
namespace {

using namespace tc;

constexpr int GK = 32;                 // panel rows per stage (two UMMA K = 16 steps)
constexpr int GS1 = 3;                 // fp32 ring
constexpr int GS2 = 2;                 // hi/lo operand ring
constexpr int GTHREADS = 256;

__global__ void __launch_bounds__(GTHREADS, 1)
gram_tc_kernel(const __grid_constant__ CUtensorMap mapY, int64_t m, int W, int64_t rows_per_cta,
               float scale, float* __restrict__ part, double* __restrict__ diagp,
               int32_t* __restrict__ status) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int R = W > 128 ? 256 : 128;             // operand rows (zero padded)
  const int F32_BYTES = GK * W * 4;
  const int PLANE = R * 64;                       // one K-major SW64 plane (32 k)
  const int F32_SLOT = (F32_BYTES + 1023) & ~1023;
  unsigned char* ring2 = base + GS1 * F32_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring2 + GS2 * 2 * PLANE);
  uint64_t* f_full = bars;
  uint64_t* f_empty = bars + GS1;
  uint64_t* hl_full = bars + 2 * GS1;
  uint64_t* hl_empty = hl_full + GS2;
  uint64_t* acc_full = hl_empty + GS2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  auto f32 = [&](int s) { return base + s * F32_SLOT; };
  auto hi = [&](int s) { return ring2 + s * 2 * PLANE; };
  auto lo = [&](int s) { return ring2 + s * 2 * PLANE + PLANE; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(m, r0 + rows_per_cta);
  const int nk = int((r1 - r0 + GK - 1) / GK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < GS1; ++s) {
      mbar_init(&f_full[s], 1);
      mbar_init(&f_empty[s], 128);
    }
    for (int s = 0; s < GS2; ++s) {
      mbar_init(&hl_full[s], 128);
      mbar_init(&hl_empty[s], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t tmem_cols = W > 128 ? 512 : (W <= 32 ? 32 : W <= 64 ? 64 : 128);
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
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % GS1;
        mbar_wait(&f_empty[s], (uint32_t(kt / GS1) & 1u) ^ 1u);
        mbar_expect_tx(&f_full[s], uint32_t(F32_BYTES));
        tma_load_2d(f32(s), &mapY, &f_full[s], 0, int(r0 + int64_t(kt) * GK));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id0 = idesc_f16(128, W);
      const uint32_t id1 = W > 128 ? idesc_f16(128, W - 128) : 0u;
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % GS2;
        mbar_wait(&hl_full[s], uint32_t(kt / GS2) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dh = desc_sw64(hi(s)), dl = desc_sw64(lo(s));
        const uint64_t up = uint64_t(128 * 64) >> 4;   // rows 128.. of a plane
#pragma unroll
        for (int ks = 0; ks < GK / 16; ++ks) {
          const uint64_t adv = uint64_t(ks * 32) >> 4;
          const uint32_t acc = (kt | ks) ? 1u : 0u;
          umma_f16(tmem, dh + adv, dh + adv, id0, acc);
          umma_f16(tmem, dh + adv, dl + adv, id0, 1u);
          umma_f16(tmem, dl + adv, dh + adv, id0, 1u);
          if (W > 128) {
            umma_f16(tmem + 256, dh + up + adv, dh + up + adv, id1, acc);
            umma_f16(tmem + 256, dh + up + adv, dl + up + adv, id1, 1u);
            umma_f16(tmem + 256, dl + up + adv, dh + up + adv, id1, 1u);
          }
        }
        umma_commit(&hl_empty[s]);
      }
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    const int t = threadIdx.x - 128;
    bool big = false;
    double dd[2] = {0.0, 0.0};     // exact diagonal: fp64 sums of squares
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % GS1;
      const int s2 = kt % GS2;
      mbar_wait(&f_full[s], uint32_t(kt / GS1) & 1u);
      const float* st = reinterpret_cast<const float*>(f32(s));
      uint4 hv[2][GK / 8], lv[2][GK / 8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = t + 128 * h;
        float v[GK];
#pragma unroll
        for (int k = 0; k < GK; ++k) {
          v[k] = c < W ? st[k * W + c] : 0.f;
          big |= !(fabsf(v[k]) * scale < 32768.f);
          dd[h] = fma(double(v[k]), double(v[k]), dd[h]);
        }
#pragma unroll
        for (int g = 0; g < GK / 8; ++g) split8(v + 8 * g, scale, hv[h][g], lv[h][g]);
      }
      // the fp32 stage is consumed: release it to the TMA engine (proxy
      // fence: generic loads before the async-proxy refill)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&f_empty[s]);
      mbar_wait(&hl_empty[s2], (uint32_t(kt / GS2) & 1u) ^ 1u);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = t + 128 * h;
        if (c < R) {
#pragma unroll
          for (int g = 0; g < GK / 8; ++g) {
            const int off = sw64_off(c, g);
            *reinterpret_cast<uint4*>(hi(s2) + off) = hv[h][g];
            *reinterpret_cast<uint4*>(lo(s2) + off) = lv[h][g];
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&hl_full[s2]);
    }
    if (big && status) atomicOr(status, 1);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (t + 128 * h < W) diagp[int64_t(blockIdx.x) * W + t + 128 * h] = dd[h];
    // epilogue: fp32 partial G of this CTA's rows (upper blocks only)
    float* P = part + int64_t(blockIdx.x) * W * W;
    const int q = warp - 4;
    if (nk > 0) {
      mbar_wait(acc_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    const int i0 = q * 32 + lane;                    // block row 0: G row i0
    for (int c0 = 0; c0 < W; c0 += 32) {
      uint32_t d[32];
      if (nk > 0) tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(c0), d);
      if (i0 < W) {
        float4* dst = reinterpret_cast<float4*>(P + int64_t(i0) * W + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (c0 + 4 * j < W)   // W is a multiple of 16: whole float4 groups
          dst[j] = nk > 0 ? make_float4(__uint_as_float(d[4 * j]), __uint_as_float(d[4 * j + 1]),
                                        __uint_as_float(d[4 * j + 2]), __uint_as_float(d[4 * j + 3]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (W > 128) {
      const int i1 = 128 + q * 32 + lane;              // block row 1: G row i1, cols 128..
      for (int c0 = 0; c0 < W - 128; c0 += 32) {
        uint32_t d[32];
        if (nk > 0) tmem_ld32(tmem + (uint32_t(q * 32) << 16) + 256u + uint32_t(c0), d);
        if (i1 < W) {
          float4* dst = reinterpret_cast<float4*>(P + int64_t(i1) * W + 128 + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (128 + c0 + 4 * j < W)
            dst[j] = nk > 0 ? make_float4(__uint_as_float(d[4 * j]), __uint_as_float(d[4 * j + 1]),
                                          __uint_as_float(d[4 * j + 2]),
                                          __uint_as_float(d[4 * j + 3]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_cols));
  }
}

// G[i][j] = G[j][i] = inv * sum_c part[c][i][j] (j > i), fixed order in fp64;
// the diagonal from the exact fp64 sums of squares.  (The tensor cores'
// fp32 accumulation truncates: on the all-positive diagonal sums that is a
// bias of ~2^-25 per accumulation step -- measured 2e-6 relative for
// 338-row blocks -- while the off-diagonal sums, of either sign and ~1e-3
// of the diagonal here, keep absolute errors ~1e-8.)
__global__ void gram_tc_reduce(int ell, int W, int nparts, const float* __restrict__ part,
                               const double* __restrict__ diagp, double inv,
                               double* __restrict__ G, int64_t ldg) {
  const int64_t total = int64_t(ell) * ell;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e / ell), j = int(e % ell);
    if (j < i) continue;
    double acc = 0.0;
    if (i == j) {
      for (int c = 0; c < nparts; ++c) acc += diagp[int64_t(c) * W + i];
      G[int64_t(i) * ldg + i] = acc;
      continue;
    }
    for (int c = 0; c < nparts; ++c) acc += double(part[(int64_t(c) * W + i) * W + j]);
    acc *= inv;
    G[int64_t(i) * ldg + j] = acc;
    G[int64_t(j) * ldg + i] = acc;
  }
}

}  // namespace

bool gram_tc_supported(int64_t m, int64_t ell, const float* Y, int64_t ldy) {
  const char* e = getenv("LR_GRAM_TC");
  const bool off = e && e[0] == '0';
  return !off && ell >= 1 && ell <= 256 && m >= 4096 && (ldy % 4) == 0 &&
         (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
}

void gram_tc_f32(Handle* h, int64_t m, int64_t ell, const float* Y, int64_t ldy, double* G,
                 int log2_scale, int32_t* status) {
  LR_REQUIRE(gram_tc_supported(m, ell, Y, ldy), LR_EUNSUPPORTED, "gram_tc: unsupported shape");
  const int W = int(ceil_div(ell, 16) * 16);
  const int64_t stages = ceil_div(m, GK);
  const int64_t per = ceil_div(stages, h->sm_count);          // stages per CTA
  const int64_t rows_per_cta = per * GK;
  const int grid = int(ceil_div(m, rows_per_cta));
  float* part = pool_alloc_t<float>(h, size_t(grid) * W * W);
  double* diagp = pool_alloc_t<double>(h, size_t(grid) * W);
  const CUtensorMap map = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, Y, uint64_t(ell),
                                      uint64_t(m), uint64_t(ldy) * 4, uint32_t(W), GK,
                                      CU_TENSOR_MAP_SWIZZLE_NONE);
  const int R = W > 128 ? 256 : 128;
  const size_t f32_slot = (size_t(GK) * W * 4 + 1023) & ~size_t(1023);
  const size_t smem = GS1 * f32_slot + size_t(GS2) * 2 * R * 64 + 1024 + 256;
  LR_CUDA(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem)));
  const float scale = std::ldexp(1.0f, log2_scale);
  gram_tc_kernel<<<grid, GTHREADS, smem, h->stream>>>(map, m, W, rows_per_cta, scale, part,
                                                      diagp, status);
  LR_CHECK_LAUNCH();
  const int blocks = int(std::min<int64_t>(ceil_div(ell * ell, 256), 1024));
  gram_tc_reduce<<<blocks, 256, 0, h->stream>>>(int(ell), W, grid, part, diagp,
                                                std::ldexp(1.0, -2 * log2_scale), G, ell);
  LR_CHECK_LAUNCH();
}

}  // namespace lr
