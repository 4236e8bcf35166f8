// K3 core, register-tiled variant for ell <= 128 (the default there):
// Cholesky with column deletion of a Gram matrix + the inverse of the kept
// triangle, same contract and arithmetic as chol_drop_kernel (chol.cu) --
// the rank decision of orthonormalize_double_gs, reference core.py:84-115.
//
// The earlier kernel kept the matrix in shared memory and had every warp walk
// rows of the trailing matrix each step: ~7k warp-instructions per column,
// instruction-issue bound (ncu: 56 % issue-busy, 180 us at ell = 110).  Here
// the upper triangle lives in registers as 4x4 tiles, one thread per upper
// tile (ell = 128: 528 threads).  Step j: the owners of row j publish it to a
// double-buffered shared row (one barrier per step), every thread reads the
// pivot and its 4 + 4 row entries and updates its 16 elements.  The scaled R
// rows go to a transposed copy Rt (shared memory when it fits), from which
// the inverse X = R~^{-1} is formed column by column, one warp per column,
// the column held in registers (4 rows per lane) and x_k broadcast with a
// shuffle -- no CTA barriers in the solve.
#include <cstdlib>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int TS = 4;       // tile size
constexpr int MAXN = 128;   // 4 rows per lane in the solve

template <int ITER>
__device__ __forceinline__ double rsqrt_newton(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < ITER; ++i) y = y * fma(-0.5 * x, y * y, 1.5);
  return y;
}

// shared-memory header (row buffers, pivots, compaction), 16-byte rounded
__host__ __device__ constexpr size_t head_bytes(int n, size_t esz) {
  return (size_t(2 * n) * esz + size_t(3 * n) * sizeof(double) + size_t(n) * sizeof(int) + 15) &
         ~size_t(15);
}

template <typename T>
__device__ __forceinline__ T sel4(const T (&v)[4], int i) {
  return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
}

template <typename T, bool RT_SMEM, int MAXT>
__global__ void __launch_bounds__(MAXT, 1)   // MAXT >= 32 * ceil(tiles / 32)
chol_tiled_kernel(int n, const T* __restrict__ G, int64_t ldg, double drop_tol, double unres_rel,
                  double shift_coef, T* __restrict__ P, T* __restrict__ Rout,
                  int32_t* __restrict__ info, T* __restrict__ gRt, int32_t* status,
                  const double* __restrict__ trace_dev, const T* __restrict__ diag_src,
                  int64_t diag_stride, bool compact, const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  // Block calls (chol_blocked below): trace_dev supplies the trace of the
  // whole Gram (drop threshold and shift), diag_src its original diagonal for
  // this block (the unresolved-pivot test), and compact = false writes P
  // uncompacted (column c of X in column c, zero for dropped c).
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* rowbuf = reinterpret_cast<T*>(smem_raw);            // [2][n]
  double* d0 = reinterpret_cast<double*>(rowbuf + 2 * n);  // shifted diagonal
  double* rd = d0 + n;                                    // R diagonal (0 = dropped)
  double* ri = rd + n;                                    // 1 / R diagonal (0 = dropped)
  int* pos = reinterpret_cast<int*>(ri + n);              // compact index or -1
  T* Rt = RT_SMEM ? reinterpret_cast<T*>(smem_raw + head_bytes(n, sizeof(T))) : gRt;

  __shared__ double s_trace;
  __shared__ int s_unres, s_bad, s_rank;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int nt = (n + TS - 1) / TS;
  const int ntiles = nt * (nt + 1) / 2;

  // my tile (ti <= tj)
  int ti = 0, rem = tid;
  while (ti < nt && rem >= nt - ti) { rem -= nt - ti; ++ti; }
  const bool owner = tid < ntiles;
  const int tj = ti + rem;
  const int r0 = TS * ti, c0 = TS * tj;

  if (warp == 0) {
    double tr = 0.0;
    if (!trace_dev)
      for (int i = lane; i < n; i += 32) tr += S::re(G[size_t(i) * ldg + i]);
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, m);
    if (lane == 0) { s_trace = trace_dev ? *trace_dev : tr; s_unres = 0; s_bad = 0; }
  }
  __syncthreads();
  const double trace = s_trace;
  const double thr2 = drop_tol * drop_tol * trace;
  const double shift = shift_coef * trace;

  T w[TS][TS];
#pragma unroll
  for (int a = 0; a < TS; ++a)
#pragma unroll
    for (int b = 0; b < TS; ++b) {
      const int i = r0 + a, k = c0 + b;
      T v = S::zero();
      if (owner && i < n && k < n && k >= i) v = G[size_t(i) * ldg + k];
      if (owner && i == k && i < n) {
        v = S::make(S::re(v) + shift, 0.0);
        d0[i] = diag_src ? S::re(diag_src[size_t(i) * diag_stride]) + shift : S::re(v);
      }
      w[a][b] = v;
    }

  // right-looking factorization, one barrier per column
  for (int j = 0; j < n; ++j) {
    T* rb = rowbuf + (j & 1) * n;
    if (owner && ti == j / TS) {
      const int a = j % TS;
#pragma unroll
      for (int aa = 0; aa < TS; ++aa) {
        if (aa != a) continue;
#pragma unroll
        for (int b = 0; b < TS; ++b) {
          const int k = c0 + b;
          if (k >= j && k < n) rb[k] = w[aa][b];
        }
      }
    }
    __syncthreads();
    const double d = S::re(rb[j]);
    const bool fin = isfinite(d);
    const bool keep = fin && d > thr2 && d > 0.0;
    const double iv = keep ? rsqrt_newton<2>(d) : 0.0;
    if (tid == 0) {
      rd[j] = keep ? d * iv : 0.0;
      ri[j] = iv;
      if (keep && d <= unres_rel * d0[j]) s_unres += 1;
      if (!fin) s_bad += 1;
    }
    // R row j (scaled), transposed: Rt[k*n + j] = R_jk, k > j (0 if dropped)
    if (owner && ti == j / TS) {
#pragma unroll
      for (int b = 0; b < TS; ++b) {
        const int k = c0 + b;
        if (k > j && k < n) Rt[size_t(k) * n + j] = S::scale(rb[k], iv);
      }
    }
    if (keep && owner && c0 + TS - 1 > j) {
      const double invd = iv * iv;
      T fr[TS], rc[TS];
#pragma unroll
      for (int a = 0; a < TS; ++a) {
        const int i = r0 + a;
        fr[a] = (i > j && i < n) ? S::scale(S::conj(rb[i]), invd) : S::zero();
      }
#pragma unroll
      for (int b = 0; b < TS; ++b) {
        const int k = c0 + b;
        rc[b] = (k > j && k < n) ? rb[k] : S::zero();
      }
#pragma unroll
      for (int a = 0; a < TS; ++a)
#pragma unroll
        for (int b = 0; b < TS; ++b) w[a][b] = S::sub(w[a][b], S::mul(fr[a], rc[b]));
    }
  }
  __syncthreads();

  // compaction of the kept pivots
  if (warp == 0) {
    int base = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool k = j < n && rd[j] > 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      if (j < n) pos[j] = k ? base + __popc(bal & ((1u << lane) - 1u)) : -1;
      base += __popc(bal);
    }
    if (lane == 0) s_rank = base;
  }
  __syncthreads();
  const int rank = s_rank;
  // R output (kept rows/cols only) and P cleared
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, k = e - i * n;
    T r = S::zero();
    if (pos[i] >= 0 && pos[k] >= 0) {
      if (k > i) r = Rt[size_t(k) * n + i];
      else if (k == i) r = S::make(rd[i], 0.0);
    }
    Rout[e] = r;
    P[e] = S::zero();
  }
  // R~ has the identity in dropped rows/cols: zero R entries touching them
  if (rank < n) {
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int k = e / n, i = e - k * n;   // Rt[k][i] = R_ik, i < k
      if (i < k && (pos[i] < 0 || pos[k] < 0)) Rt[e] = S::zero();
    }
  }
  __syncthreads();

  // X = R~^{-1}, one warp per column c, x in registers (row lane + 32 r)
  for (int c = n - 1 - warp; c >= 0; c -= nwarps) {
    if (pos[c] < 0) continue;
    T x[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) x[r] = (lane + 32 * r == c) ? S::one() : S::zero();
    for (int k = c; k >= 1; --k) {
      const double inv = ri[k];
      const T xk = S::scale(S::shfl_idx(sel4(x, k >> 5), k & 31), inv);
      if (inv != 0.0) {
        const T* rk = Rt + size_t(k) * n;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = lane + 32 * r;
          if (i < k) x[r] = S::sub(x[r], S::mul(rk[i], xk));
        }
      }
    }
    const int pc = compact ? pos[c] : c;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      if (i <= c) {
        const double inv = ri[i];
        if (inv != 0.0) P[size_t(i) * n + pc] = S::scale(x[r], inv);
      }
    }
  }
  if (tid == 0) {
    info[0] = rank;
    info[1] = s_unres;
    info[2] = s_bad;
    if (status) {
      const int bits = (s_unres ? 1 : 0) | (rank < n ? 2 : 0) | (s_bad ? 4 : 0);
      if (bits) atomicOr(status, bits);
    }
  }
}

template <typename T>
void launch(Handle* h, int n, const T* G, int64_t ldg, double drop_tol, double unres_rel,
            double shift_coef, T* P, T* R, int32_t* info, const double* trace_dev = nullptr,
            const T* diag_src = nullptr, int64_t diag_stride = 0, bool compact = true) {
  const int nt = (n + TS - 1) / TS;
  const int threads = ((nt * (nt + 1) / 2 + 31) / 32) * 32;
  const size_t head = head_bytes(n, sizeof(T));
  const size_t rt = size_t(n) * n * sizeof(T);
  const bool in_smem = head + rt <= 200 * 1024;
  // the register budget is 64K / threads: complex tiles (32 doubles) fit
  // without spills up to 320 threads (ell <= 96)
  T* gRt = in_smem ? nullptr : pool_alloc_t<T>(h, size_t(n) * n);
  const size_t smem = in_smem ? head + rt : head;
  auto go = [&](auto kern) {
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<1, threads, smem, h->stream>>>(n, G, ldg, drop_tol, unres_rel, shift_coef, P, R, info,
                                          gRt, h->status, trace_dev, diag_src, diag_stride,
                                          compact, h->gate);
  };
  if (threads <= 320) {
    if (in_smem) go(chol_tiled_kernel<T, true, 320>);
    else go(chol_tiled_kernel<T, false, 320>);
  } else {
    if (in_smem) go(chol_tiled_kernel<T, true, 544>);
    else go(chol_tiled_kernel<T, false, 544>);
  }
  LR_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// 128 < ell <= 256: one level of 2 x 2 blocking around the tiled kernel.
//   G = [G11 G12; G12^H G22] (+ shift on the diagonal),  R11 = chol(G11),
//   R12 = R~11^{-H} G12 (rows of dropped block-1 pivots zero),
//   S = G22 - R12^H R12,  R22 = chol(S),
//   X = R~^{-1} = [X11, -X11 R12 X22; 0, X22]  (R12 columns of dropped block-2
//   pivots zeroed: R~ has the identity there).
// The pivots, drop and unresolved decisions are those of the unblocked
// factorization (same Schur complements, thresholds from the whole G).

template <typename T>
__global__ void trace_kernel(int n, const T* __restrict__ G, double* __restrict__ tr) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += Sc<T>::re(G[size_t(i) * n + i]);
  for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    *tr = t;
  }
}

// S = G22 - T (n2 x n2; G22 inside G with ld n, T dense)
template <typename T>
__global__ void schur_kernel(int n2, const T* __restrict__ G22, int64_t ldg,
                             const T* __restrict__ Tm, T* __restrict__ Sout) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n2 * n2; e += gridDim.x * blockDim.x) {
    const int i = e / n2, k = e - i * n2;
    Sout[e] = Sc<T>::sub(G22[size_t(i) * ldg + k], Tm[e]);
  }
}

// zero the columns of R12 (n1 x n2) whose block-2 pivot was dropped
template <typename T>
__global__ void mask_cols_kernel(int n1, int n2, T* __restrict__ R12, const T* __restrict__ R22) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n1 * n2; e += gridDim.x * blockDim.x) {
    const int c = e % n2;
    if (Sc<T>::re(R22[size_t(c) * n2 + c]) == 0.0) R12[e] = Sc<T>::zero();
  }
}

// assemble P (compacted), R and info from the blocks (n <= 256).  Grid-wide:
// every CTA derives the kept-pivot positions itself (pos / kidx in shared
// memory) and gathers its share of R and P -- P column q holds kept column
// kidx[q], so no scatter (and no ordering between CTAs) is needed.  The
// former single-CTA version took 83 us at n = 256 (config 4, 8 per step).
template <typename T>
__global__ void assemble_kernel(int n, int n1, const T* __restrict__ X11, const T* __restrict__ X12n,
                                const T* __restrict__ X22, const T* __restrict__ R11,
                                const T* __restrict__ R12, const T* __restrict__ R22,
                                const int32_t* __restrict__ info1,
                                const int32_t* __restrict__ info2, T* __restrict__ P,
                                T* __restrict__ Rout, int32_t* __restrict__ info,
                                const int32_t* __restrict__ gate) {
  using S = Sc<T>;
  // gated off: the near-identity factor is already in P / Rout / info (the
  // block factorizations returned at once; the block products in between ran
  // on scratch nobody reads)
  if (gate && *gate == 0) return;
  const int n2 = n - n1;
  __shared__ int pos[256];
  __shared__ int kidx[256];
  __shared__ int s_rank;
  const int tid = threadIdx.x, lane = tid & 31;
  auto rdiag = [&](int j) {
    return j < n1 ? S::re(R11[size_t(j) * n1 + j]) : S::re(R22[size_t(j - n1) * n2 + (j - n1)]);
  };
  if (tid < 32) {
    int base = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool k = j < n && rdiag(j) > 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      const int p = base + __popc(bal & ((1u << lane) - 1u));
      if (j < n) {
        pos[j] = k ? p : -1;
        if (k) kidx[p] = j;
      }
      base += __popc(bal);
    }
    if (lane == 0) s_rank = base;
  }
  __syncthreads();
  const int rank = s_rank;
  auto rblk = [&](int i, int c) -> T {
    if (i < n1 && c < n1) return R11[size_t(i) * n1 + c];
    if (i < n1) return R12[size_t(i) * n2 + (c - n1)];
    if (c >= n1) return R22[size_t(i - n1) * n2 + (c - n1)];
    return S::zero();
  };
  auto xblk = [&](int i, int c) -> T {
    if (i < n1 && c < n1) return X11[size_t(i) * n1 + c];
    if (i < n1) return S::scale(X12n[size_t(i) * n2 + (c - n1)], -1.0);
    if (c >= n1) return X22[size_t(i - n1) * n2 + (c - n1)];
    return S::zero();
  };
  for (int e = blockIdx.x * blockDim.x + tid; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e / n, c = e - i * n;
    Rout[e] = (pos[i] < 0 || pos[c] < 0) ? S::zero() : rblk(i, c);
    P[e] = c < rank ? xblk(i, kidx[c]) : S::zero();
  }
  if (blockIdx.x == 0 && tid == 0) {
    info[0] = rank;
    info[1] = info1[1] + info2[1];
    info[2] = info1[2] + info2[2];
  }
}

// the 2 x 2 driver's block factorizations: the panel kernel when selected
template <typename T>
void block_chol(Handle* h, int n, const T* G, int64_t ldg, double drop_tol, double unres_rel,
                double shift_coef, T* P, T* R, int32_t* info, const double* trace_dev,
                const T* diag_src, int64_t diag_stride) {
  if (chol_mode() == 0) {
    if constexpr (sizeof(T) == 8)
      chol_panel_f64(h, n, G, ldg, drop_tol, unres_rel, shift_coef, P, R, info, trace_dev,
                     diag_src, diag_stride, false);
    else
      chol_panel_c128(h, n, G, ldg, drop_tol, unres_rel, shift_coef, P, R, info, trace_dev,
                      diag_src, diag_stride, false);
    return;
  }
  launch<T>(h, n, G, ldg, drop_tol, unres_rel, shift_coef, P, R, info, trace_dev, diag_src,
            diag_stride, false);
}

template <typename T>
void chol_blocked(Handle* h, int dtype, int n, const T* G, double drop_tol, double unres_rel,
                  double shift_coef, T* P, T* R, int32_t* info) {
  const int n1 = MAXN, n2 = n - n1;
  double* tr = pool_alloc_t<double>(h, 1);
  int32_t* inf = pool_alloc_t<int32_t>(h, 8);
  T* X11 = pool_alloc_t<T>(h, size_t(n1) * n1);
  T* R11 = pool_alloc_t<T>(h, size_t(n1) * n1);
  T* X22 = pool_alloc_t<T>(h, size_t(n2) * n2);
  T* R22 = pool_alloc_t<T>(h, size_t(n2) * n2);
  T* R12 = pool_alloc_t<T>(h, size_t(n1) * n2);
  T* Tm = pool_alloc_t<T>(h, size_t(n2) * n2);
  T* Sm = pool_alloc_t<T>(h, size_t(n2) * n2);
  T* T1 = pool_alloc_t<T>(h, size_t(n1) * n2);
  T* X12 = pool_alloc_t<T>(h, size_t(n1) * n2);
  trace_kernel<T><<<1, 256, 0, h->stream>>>(n, G, tr);
  LR_CHECK_LAUNCH();
  block_chol<T>(h, n1, G, n, drop_tol, unres_rel, shift_coef, X11, R11, inf, tr, nullptr, 0);
  // R12 = X11^H G12
  gemm_any(h, dtype, true, true, n1, n2, n1, X11, n1, G + n1, n, R12, n2);
  // S = G22 - R12^H R12
  gemm_any(h, dtype, true, true, n2, n2, n1, R12, n2, R12, n2, Tm, n2);
  schur_kernel<T><<<64, 256, 0, h->stream>>>(n2, G + size_t(n1) * n + n1, n, Tm, Sm);
  LR_CHECK_LAUNCH();
  block_chol<T>(h, n2, Sm, n2, drop_tol, unres_rel, shift_coef, X22, R22, inf + 4, tr,
                G + size_t(n1) * n + n1, n + 1);
  mask_cols_kernel<T><<<64, 256, 0, h->stream>>>(n1, n2, R12, R22);
  LR_CHECK_LAUNCH();
  // X12 = -(X11 R12) X22 (sign applied in the assembly)
  gemm_any(h, dtype, false, false, n1, n2, n1, X11, n1, R12, n2, T1, n2);
  gemm_any(h, dtype, false, false, n1, n2, n2, T1, n2, X22, n2, X12, n2);
  assemble_kernel<T><<<64, 256, 0, h->stream>>>(n, n1, X11, X12, X22, R11, R12, R22, inf,
                                                 inf + 4, P, R, info, h->gate);
  LR_CHECK_LAUNCH();
}

}  // namespace

bool chol_blocked_supported(int64_t n) { return n > MAXN && n <= 2 * MAXN; }

void chol_blocked_f64(Handle* h, int64_t n, const double* G, double drop_tol, double unres_rel,
                      double shift_coef, double* P, double* R, int32_t* info) {
  chol_blocked<double>(h, LR_F64, int(n), G, drop_tol, unres_rel, shift_coef, P, R, info);
}

void chol_blocked_c128(Handle* h, int64_t n, const double2* G, double drop_tol, double unres_rel,
                       double shift_coef, double2* P, double2* R, int32_t* info) {
  chol_blocked<double2>(h, LR_C128, int(n), G, drop_tol, unres_rel, shift_coef, P, R, info);
}

// ---------------------------------------------------------------------------
namespace {

// Second CholeskyQR pass: G = Q1^H Q1 = I + E with E tiny when the first
// pass succeeded.  Then R = I + N, N = triu(E, 1) + diag(Re E) / 2, gives
// R^H R = I + E + O(E^2) and P = R^{-1} = I - N + O(E^2), so
// (Q1 P)^H (Q1 P) = I + O(E^2): for max|E| <= 1e-8 the first-order factor is
// as good as the exact one in double precision, with no sequential
// dependency.  One CTA checks max|E|, writes the first-order P / R / info
// and clears *gate; otherwise it sets *gate and the exact kernel (launched
// right behind it, gated) runs.
// Two grid-wide kernels (one CTA moved 4 n^2 elements through a single SM:
// 61 us at n = 256): the check ORs "not near-identity" into *gate (zeroed by
// the caller), the write runs only when the gate stayed clear.
template <typename T>
__global__ void near_identity_check(int n, const T* __restrict__ G, int32_t* __restrict__ gate,
                                    double thr) {
  using S = Sc<T>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int bad = 0;
  for (int i = blockIdx.x * nw + warp; i < n; i += gridDim.x * nw) {
    const T* row = G + size_t(i) * n;
#pragma unroll 8
    for (int k = lane; k < n; k += 32) {
      const T g = row[k];
      const double dev = (i == k) ? fabs(S::re(g) - 1.0) + fabs(S::abs2(g) - S::re(g) * S::re(g))
                                  : sqrt(S::abs2(g));
      if (!(dev <= thr)) bad = 1;   // also catches NaN
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(gate, 1);
}

template <typename T>
__global__ void near_identity_write(int n, const T* __restrict__ G, T* __restrict__ P,
                                    T* __restrict__ Rout, int32_t* __restrict__ info,
                                    const int32_t* __restrict__ gate) {
  using S = Sc<T>;
  if (*gate != 0) return;   // the exact kernels behind this one run instead
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = blockIdx.x * nw + warp; i < n; i += gridDim.x * nw) {
    const size_t ro = size_t(i) * n;
#pragma unroll 8
    for (int k = lane; k < n; k += 32) {
      T nv = S::zero();
      if (k > i) nv = G[ro + k];
      else if (k == i) nv = S::make(0.5 * (S::re(G[ro + k]) - 1.0), 0.0);
      Rout[ro + k] = (k == i) ? S::add(S::one(), nv) : nv;
      P[ro + k] = (k == i) ? S::sub(S::one(), nv) : S::scale(nv, -1.0);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = n;
    info[1] = 0;
    info[2] = 0;
  }
}

template <typename T>
void launch_near_identity(Handle* h, int n, const T* G, T* P, T* R, int32_t* info, int32_t* gate,
                          double thr) {
  LR_CUDA(cudaMemsetAsync(gate, 0, sizeof(int32_t), h->stream));
  const int blocks = (n + 7) / 8;   // 8 warps per CTA, one row per warp
  near_identity_check<T><<<blocks, 256, 0, h->stream>>>(n, G, gate, thr);
  LR_CHECK_LAUNCH();
  near_identity_write<T><<<blocks, 256, 0, h->stream>>>(n, G, P, R, info, gate);
  LR_CHECK_LAUNCH();
}

}  // namespace

void chol_near_identity(Handle* h, int dtype, int64_t n, const void* G, double drop_tol,
                        double unres_rel, void* P, void* R, int32_t* info, double thr) {
  const bool cplx = dtype == LR_C64 || dtype == LR_C128;
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("LR_CHOL_NEARID");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  if (!mode || (n > MAXN && !chol_panel_supported(n, cplx) && !chol_blocked_supported(n))) {
    if (cplx) chol_drop_c128(h, n, static_cast<const double2*>(G), drop_tol, unres_rel, 0.0,
                             static_cast<double2*>(P), static_cast<double2*>(R), info);
    else chol_drop_f64(h, n, static_cast<const double*>(G), drop_tol, unres_rel, 0.0,
                       static_cast<double*>(P), static_cast<double*>(R), info);
    return;
  }
  int32_t* gate = pool_alloc_t<int32_t>(h, 1);
  if (cplx)
    launch_near_identity<double2>(h, int(n), static_cast<const double2*>(G),
                                  static_cast<double2*>(P), static_cast<double2*>(R), info, gate,
                                  thr);
  else
    launch_near_identity<double>(h, int(n), static_cast<const double*>(G),
                                 static_cast<double*>(P), static_cast<double*>(R), info, gate, thr);
  const int32_t* saved = h->gate;
  h->gate = gate;
  try {
    if (cplx) chol_drop_c128(h, n, static_cast<const double2*>(G), drop_tol, unres_rel, 0.0,
                             static_cast<double2*>(P), static_cast<double2*>(R), info);
    else chol_drop_f64(h, n, static_cast<const double*>(G), drop_tol, unres_rel, 0.0,
                       static_cast<double*>(P), static_cast<double*>(R), info);
  } catch (...) {
    h->gate = saved;
    throw;
  }
  h->gate = saved;
}

// Measured on B200 (tools/small_probe.py, CUDA-graph timed): the tiled
// kernel wins from ell ~ 80 (real: 133 vs 178 us at 110, 163 vs 380 us at
// 128) and for complex above 64 (336 vs 443 us at 120); below that the
// 1024-thread shared-memory kernel is faster.
bool chol_tiled_supported(int64_t n, bool cplx) {
  const int mode = chol_mode();   // LR_CHOL: panel (default) | tiled | smem
  if (n < 1 || n > MAXN || mode == 1) return false;
  return mode == 2 || n >= (cplx ? 65 : 80);
}

void chol_tiled_f64(Handle* h, int64_t n, const double* G, double drop_tol, double unres_rel,
                    double shift_coef, double* P, double* R, int32_t* info) {
  launch<double>(h, int(n), G, n, drop_tol, unres_rel, shift_coef, P, R, info);
}

void chol_tiled_c128(Handle* h, int64_t n, const double2* G, double drop_tol, double unres_rel,
                     double shift_coef, double2* P, double2* R, int32_t* info) {
  launch<double2>(h, int(n), G, n, drop_tol, unres_rel, shift_coef, P, R, info);
}

}  // namespace lr
