// K6: CSR SpMM for the sparse operator of config 5 (no reference code path
// exists for sparse A -- SURVEY.md §8c; this is the MatVecOperator plug-in
// the survey prescribes, core.py:343-380).
//
// Y (m x ell) (+)= S . X with S in CSR (int64 row pointers, int32 column
// indices, fp64 values) and X (n x ell) row-major.  One warp per row: the
// warp streams the row's nonzeros (coalesced), broadcasts (col, val) by
// shuffle, and each lane accumulates ell/32 columns of the gathered X rows
// (each gather is a contiguous 8*ell-byte row of X).  The transpose product
// uses the CSR of S^T (built once by the operator), so no atomics are needed
// and the result is deterministic.
#include <cstdlib>

#include "common.cuh"

namespace lr {
namespace {

template <int CPL>   // columns per lane (ell <= 32 * CPL)
__global__ void __launch_bounds__(256)
csr_spmm_kernel(int64_t m, int ell, const int64_t* __restrict__ rowptr,
                const int32_t* __restrict__ colidx, const double* __restrict__ vals,
                const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy,
                bool accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m;
       row += warps) {
    double acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    for (int64_t base = b; base < e; base += 32) {
      const int64_t idx = base + lane;
      int32_t cl = 0;
      double vl = 0.0;
      if (idx < e) {
        cl = colidx[idx];
        vl = vals[idx];
      }
      const int cnt = int(min(int64_t(32), e - base));
      for (int k = 0; k < cnt; ++k) {
        const int32_t col = __shfl_sync(0xffffffffu, cl, k);
        const double v = __shfl_sync(0xffffffffu, vl, k);
        const double* xr = X + int64_t(col) * ldx;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int j = c * 32 + lane;
          if (j < ell) acc[c] = fma(v, __ldg(xr + j), acc[c]);
        }
      }
    }
    double* yr = Y + row * ldy;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = c * 32 + lane;
      if (j < ell) yr[j] = accumulate ? yr[j] + acc[c] : acc[c];
    }
  }
}

// Narrow X (ell <= 64): a half-warp per nonzero, each lane gathering CPL
// doubles of the X row, two nonzeros per step and two steps in flight --
// four independent X-row gathers per warp instead of one (the one-warp-per-
// nonzero kernel left HBM ~50 % busy on config 5: latency, not bandwidth).
template <int CPL>   // columns per lane, ell <= 16 * CPL
__global__ void __launch_bounds__(256)
csr_spmm_half_kernel(int64_t m, int ell, const int64_t* __restrict__ rowptr,
                     const int32_t* __restrict__ colidx, const double* __restrict__ vals,
                     const double* __restrict__ X, int64_t ldx, double* __restrict__ Y,
                     int64_t ldy, bool accumulate) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m;
       row += warps) {
    double acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    for (int64_t base = b; base < e; base += 32) {
      const int64_t idx = base + lane;
      int32_t cl = 0;
      double vl = 0.0;
      if (idx < e) {
        cl = colidx[idx];
        vl = vals[idx];
      }
      const int cnt = int(min(int64_t(32), e - base));
      for (int k = 0; k < cnt; k += 4) {
        // nonzeros k + half and k + 2 + half (zero-weight padding past cnt)
        const int k0 = k + half, k1 = k + 2 + half;
        const int32_t c0 = __shfl_sync(0xffffffffu, cl, k0 & 31);
        const double s0 = __shfl_sync(0xffffffffu, vl, k0 & 31);
        const double v0 = k0 < cnt ? s0 : 0.0;
        const int32_t c1 = __shfl_sync(0xffffffffu, cl, k1 & 31);
        const double s1 = __shfl_sync(0xffffffffu, vl, k1 & 31);
        const double v1 = k1 < cnt ? s1 : 0.0;
        const double* x0 = X + int64_t(k0 < cnt ? c0 : 0) * ldx;
        const double* x1 = X + int64_t(k1 < cnt ? c1 : 0) * ldx;
        double g0[CPL], g1[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int j = c * 16 + hl;
          g0[c] = (j < ell && k0 < cnt) ? __ldg(x0 + j) : 0.0;
          g1[c] = (j < ell && k1 < cnt) ? __ldg(x1 + j) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = fma(v1, g1[c], fma(v0, g0[c], acc[c]));
      }
    }
    // the two half-warps hold partial sums of the same columns
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 16);
    if (half == 0) {
      double* yr = Y + row * ldy;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int j = c * 16 + hl;
        if (j < ell) yr[j] = accumulate ? yr[j] + acc[c] : acc[c];
      }
    }
  }
}

}  // namespace

void csr_spmm_f64(Handle* h, int64_t m, int64_t ell, const int64_t* rowptr,
                  const int32_t* colidx, const double* vals, const double* X, int64_t ldx,
                  double* Y, int64_t ldy, bool accumulate) {
  if (m == 0 || ell == 0) return;
  LR_REQUIRE(ell <= 256, LR_EUNSUPPORTED, "csr_spmm: ell > 256 not built");
  const int blocks = int(std::min<int64_t>(ceil_div(m, 8), int64_t(h->sm_count) * 16));
  static int old = -1;
  if (old < 0) {
    const char* e = getenv("LR_SPMM");
    old = (e && e[0] == 'w') ? 1 : 0;   // LR_SPMM=warp: one warp per nonzero
  }
  if (!old && ell <= 64) {
    const int c16 = int(ceil_div(ell, 16));
    switch (c16) {
      case 1: csr_spmm_half_kernel<1><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
      case 2: csr_spmm_half_kernel<2><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
      case 3: csr_spmm_half_kernel<3><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
      default: csr_spmm_half_kernel<4><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
    }
    LR_CHECK_LAUNCH();
    return;
  }
  const int cpl = int(ceil_div(ell, 32));
  switch (cpl) {
    case 1: csr_spmm_kernel<1><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
    case 2: csr_spmm_kernel<2><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
    case 3:
    case 4: csr_spmm_kernel<4><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
    default: csr_spmm_kernel<8><<<blocks, 256, 0, h->stream>>>(m, int(ell), rowptr, colidx, vals, X, ldx, Y, ldy, accumulate); break;
  }
  LR_CHECK_LAUNCH();
}

}  // namespace lr
