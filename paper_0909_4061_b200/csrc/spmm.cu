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
#include <cstdio>
#include <cstdlib>
#include <cstring>

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

// ---- column slices (opt-in, LR_SPMM=slice4|slice8) --------------------------
//
// With X (n x ell fp64) larger than L2 every gathered X row comes from HBM:
// config 5 (n = 2^21, ell = 48: X = 805 MB) moves 13.7 GB per product for
// 3.1 GB of compulsory traffic (nnz random rows of 384 B each).  This path
// copies X into slice-major panels Xs[s] (n x W, contiguous: 64 MB for W = 4,
// one 32-byte sector per gathered row) and runs the product slice by slice,
// Y[:, W s : W s + W] = S Xs[s], so the gathers can hit an L2-resident slice
// while the CSR arrays are streamed once per slice.  It is measured slower
// than the default (numbers below) and kept opt-in as the record of that
// experiment; results equal the default kernels' to rounding (tests).

// Xs[s][i][c] = X[i][W s + c] (zero past ell)
template <int W>
__global__ void __launch_bounds__(256)
repack_slices_kernel(int64_t n, int ell, int ns, const double* __restrict__ X, int64_t ldx,
                     double* __restrict__ Xs) {
  const int64_t total = n * int64_t(ns) * W;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    // e enumerates the source row-major (i, j) with j < ns W: coalesced reads
    const int64_t i = e / (int64_t(ns) * W);
    const int j = int(e - i * int64_t(ns) * W);
    const int s = j / W, c = j - s * W;
    Xs[(int64_t(s) * n + i) * W + c] = j < ell ? X[i * ldx + j] : 0.0;
  }
}

// A group of W lanes owns one row (a warp: 32 / W consecutive rows); lane c
// of the group accumulates column c of the slice over the row's nonzeros in
// CSR order (deterministic).  U nonzeros per step: U (col, val) loads, then U
// independent gathers -- ~32 U / W sector requests in flight per warp, the
// memory-level parallelism a one-row-per-warp loop lacks.
template <int W, int U>
__global__ void __launch_bounds__(256)
csr_spmm_slice_kernel(int64_t m, const int64_t* __restrict__ rowptr,
                      const int32_t* __restrict__ colidx, const double* __restrict__ vals,
                      const double* __restrict__ Xs, double* __restrict__ Y, int64_t ldy,
                      int ncols, bool accumulate) {
  const int c = threadIdx.x % W;
  const int64_t groups = int64_t(gridDim.x) * (blockDim.x / W);
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x / W) + threadIdx.x / W; row < m;
       row += groups) {
    const int64_t b = __ldg(rowptr + row), e = __ldg(rowptr + row + 1);
    double acc = 0.0;
    for (int64_t k = b; k < e; k += U) {
      int32_t col[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // clamped index (k < e): every load is in bounds, no predicated
        // loads; the nonzeros past the row's end get weight 0
        const int64_t q = min(k + u, e - 1);
        col[u] = __ldcs(colidx + q);
        v[u] = k + u < e ? __ldcs(vals + q) : 0.0;
      }
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = __ldg(Xs + int64_t(col[u]) * W + c);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = fma(v[u], x[u], acc);
    }
    if (c < ncols) {
      double* yr = Y + row * ldy + c;
      *yr = accumulate ? *yr + acc : acc;
    }
  }
}

// LR_SPMM: "warp" = one warp per nonzero; "slice4" / "slice8" = the column-
// slice path with W = 4 / 8.  Default: the half-warp row-major kernel.
// Measured at config 5 (n = 2^21, ell = 48, 33.5 M nonzeros, one B200):
// half-warp 3.14 ms per product (13.7 GB of DRAM traffic, 4.35 TB/s), slice8
// 4.75 ms, slice4 6.61 ms -- re-streaming the CSR arrays once per slice and
// 32-byte L2 gathers cost more than the HBM gathers of whole 384-byte X rows
// they replace, so the slices stay opt-in.
#ifndef LR_SPMM_U
#define LR_SPMM_U 8
#endif

int spmm_mode() {   // read per call: tests switch paths with the environment
  const char* e = getenv("LR_SPMM");
  if (!e) return 0;
  if (e[0] == 'w') return 1;
  if (e[0] == 'h') return 2;
  if (!strcmp(e, "slice4")) return 4;
  if (!strcmp(e, "slice8")) return 8;
  return 0;
}

template <int W>
void spmm_slices(Handle* h, int64_t m, int64_t n, int64_t ell, const int64_t* rowptr,
                 const int32_t* colidx, const double* vals, const double* X, int64_t ldx,
                 double* Y, int64_t ldy, bool accumulate) {
  const int ns = int(ceil_div(ell, W));
  double* Xs = pool_alloc_t<double>(h, size_t(ns) * n * W);
  const int rb = int(std::min<int64_t>(ceil_div(n * ns * W, 256), int64_t(h->sm_count) * 32));
  repack_slices_kernel<W><<<rb, 256, 0, h->stream>>>(n, int(ell), ns, X, ldx, Xs);
  LR_CHECK_LAUNCH();
  const int blocks = int(std::min<int64_t>(ceil_div(m, 256 / W), int64_t(h->sm_count) * 8));
  for (int s = 0; s < ns; ++s) {
    const int nc = int(std::min<int64_t>(W, ell - int64_t(s) * W));
    csr_spmm_slice_kernel<W, LR_SPMM_U><<<blocks, 256, 0, h->stream>>>(
        m, rowptr, colidx, vals, Xs + size_t(s) * n * W, Y + int64_t(s) * W, ldy, nc, accumulate);
    LR_CHECK_LAUNCH();
  }
}

}  // namespace

void csr_spmm_f64(Handle* h, int64_t m, int64_t n, int64_t ell, const int64_t* rowptr,
                  const int32_t* colidx, const double* vals, const double* X, int64_t ldx,
                  double* Y, int64_t ldy, bool accumulate) {
  if (m == 0 || ell == 0) return;
  LR_REQUIRE(ell <= 256, LR_EUNSUPPORTED, "csr_spmm: ell > 256 not built");
  const int blocks = int(std::min<int64_t>(ceil_div(m, 8), int64_t(h->sm_count) * 16));
  const int mode = spmm_mode();
  if (mode == 8) {
    spmm_slices<8>(h, m, n, ell, rowptr, colidx, vals, X, ldx, Y, ldy, accumulate);
    return;
  }
  if (mode == 4) {
    spmm_slices<4>(h, m, n, ell, rowptr, colidx, vals, X, ldx, Y, ldy, accumulate);
    return;
  }
  const bool old = mode == 1;   // LR_SPMM=warp: one warp per nonzero
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
