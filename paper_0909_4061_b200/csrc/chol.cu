// K3 core: Cholesky with column deletion of an ell x ell Gram matrix, and
// the inverse of the kept triangle (single CTA, fp64 / complex128).
//
// This is the rank decision of orthonormalize_double_gs (reference
// core.py:84-115) restated for a Gram-based QR: for Y = [y_1..y_ell],
// G = Y^H Y = R^H R, the Cholesky pivot d_j = G_jj - sum_{i<j, i kept} |r_ij|^2
// equals ||y_j - P_{kept<j} y_j||^2, the squared residual the reference
// compares with tol * ||Y||_F.  A dropped column is excluded from every later
// projection (its row of R is skipped), exactly like the reference skipping
// it in the basis.  ||Y||_F^2 = trace(G).
//
// The kernel is latency-bound (one SM, ell^3/3 flops), so it is written for
// short critical paths: one n x n row-major buffer in shared memory (LDS/STS
// via a template specialisation; global scratch only for very large ell),
// 32 warps, ONE barrier per column.  Every thread reads the pivot itself and
// forms 1/sqrt(d) with rsqrt (no divides on the critical path); the trailing
// update uses the unscaled pivot row times 1/d and the scaling of row j is
// deferred to step j+1.  The inverse X = R~^{-1} (R~ = R with dropped
// rows/cols replaced by the identity) is formed column by column, one warp
// per column (independent back substitutions, no CTA barriers), into the
// lower triangle (X^T), then scattered into P with the kept columns
// compacted.
//
// Outputs: P (ell x ell): Q = Y . P[:, :rank] has orthonormal columns;
// R (ell x ell) the factor restricted to kept rows/cols;
// info = {rank, unresolved pivots, bad (non-finite) pivots}.
#include <cstdlib>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {


// 1/sqrt(d) to full double precision (MUFU seed + two Newton steps)
__device__ __forceinline__ double rsqrt_full(double d) { return rsqrt(d); }

// largest n whose n x n working matrix (+ per-column vectors) fits the
// 227 KB opt-in shared memory of one CTA
template <typename T>
constexpr int smem_maxn() { return sizeof(T) == 8 ? 168 : 118; }

template <typename T, bool SMEM, int CHOL_THREADS>
__global__ void __launch_bounds__(CHOL_THREADS, 1)
chol_drop_kernel(int n, const T* __restrict__ G, double drop_tol, double unres_rel,
                 double shift_coef, T* __restrict__ P, T* __restrict__ Rout,
                 int32_t* __restrict__ info, T* gW, int32_t* status,
                 const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* __restrict__ W;
  unsigned char* tail;
  if constexpr (SMEM) {
    W = reinterpret_cast<T*>(smem_raw);
    tail = reinterpret_cast<unsigned char*>(W + size_t(n) * n);
  } else {
    W = gW;
    tail = smem_raw;
  }
  double* d0 = reinterpret_cast<double*>(tail);         // original (shifted) pivots
  double* rd = d0 + n;                                  // R diagonal (0 = dropped)
  double* ri = rd + n;                                  // 1 / R diagonal
  int* pos = reinterpret_cast<int*>(ri + n);            // compact index or -1
  int* kidx = pos + n;                                  // compact -> original

  constexpr int NW = CHOL_THREADS / 32;
  constexpr int SMEM_MAXN = smem_maxn<T>();
  __shared__ double s_red[NW];
  __shared__ int s_unres, s_bad, s_rank;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // 1. load the upper triangle, trace
  double tr = 0.0;
  for (int i = warp; i < n; i += NW) {
    for (int j = i + lane; j < n; j += 32) {
      const T g = G[size_t(i) * n + j];
      W[i * n + j] = g;
      if (j == i) tr += S::re(g);
    }
  }
  for (int m = 16; m > 0; m >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, m);
  if (lane == 0) s_red[warp] = tr;
  if (tid == 0) { s_unres = 0; s_bad = 0; }
  __syncthreads();
  double trace = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) trace += s_red[w];
  const double thr2 = drop_tol * drop_tol * trace;
  const double shift = shift_coef * trace;
  for (int i = tid; i < n; i += CHOL_THREADS) {
    const double d = S::re(W[i * n + i]) + shift;
    W[i * n + i] = S::make(d, 0.0);
    d0[i] = d;
  }
  __syncthreads();

  // 2. right-looking factorization, one barrier per column
  for (int j = 0; j <= n; ++j) {
    if (j > 0) {   // deferred scaling of row j-1
      const int p = j - 1;
      const double inv = ri[p];
      T* rowp = W + p * n;
      for (int c = p + 1 + tid; c < n; c += CHOL_THREADS) rowp[c] = S::scale(rowp[c], inv);
    }
    if (j == n) break;
    const double d = S::re(W[j * n + j]);
    const bool fin = isfinite(d);
    const bool keep = fin && d > thr2 && d > 0.0;
    if (keep) {
      const double iv = rsqrt_full(d);       // 1 / r_jj
      const double invd = iv * iv;           // 1 / d
      if (tid == 0) {
        rd[j] = d * iv;
        ri[j] = iv;
        if (d <= unres_rel * d0[j]) s_unres += 1;
      }
      const T* rowj = W + j * n;
      if constexpr (SMEM) {
        // n <= SMEM_MAXN: every lane issues all its loads of a row before any
        // store, so the shared-memory latencies overlap (the store/load
        // aliasing otherwise serializes the row)
        constexpr int MAXC = (SMEM_MAXN + 31) / 32;
        for (int a = j + 1 + warp; a < n; a += NW) {
          const T f = S::scale(S::conj(rowj[a]), invd);
          T* rowa = W + a * n;
          T rj[MAXC], ra[MAXC];
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int b = a + lane + 32 * q;
            if (b < n) { rj[q] = rowj[b]; ra[q] = rowa[b]; }
          }
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int b = a + lane + 32 * q;
            if (b < n) rowa[b] = S::sub(ra[q], S::mul(f, rj[q]));
          }
        }
      } else {
        for (int a = j + 1 + warp; a < n; a += NW) {
          const T f = S::scale(S::conj(rowj[a]), invd);
          T* rowa = W + a * n;
          for (int b = a + lane; b < n; b += 32) rowa[b] = S::sub(rowa[b], S::mul(f, rowj[b]));
        }
      }
    } else if (tid == 0) {
      if (!fin) s_bad += 1;
      rd[j] = 0.0;
      ri[j] = 0.0;   // deferred scaling zeroes the row
    }
    __syncthreads();
  }

  // 3. compaction; zero R entries in rows/columns of dropped pivots
  if (warp == 0) {
    int base = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool k = j < n && rd[j] > 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      const int pj = base + __popc(bal & ((1u << lane) - 1u));
      if (j < n) pos[j] = k ? pj : -1;
      if (k) kidx[pj] = j;
      base += __popc(bal);
    }
    if (lane == 0) s_rank = base;
  }
  __syncthreads();
  const int rank = s_rank;
  if (rank < n) {
    for (int e = tid; e < n * n; e += CHOL_THREADS) {
      const int i = e / n, c = e - (e / n) * n;
      if (c > i && (pos[i] < 0 || pos[c] < 0)) W[e] = S::zero();
    }
  }
  // X initialised to the identity in the lower triangle (X[i][c] at W[c][i])
  for (int e = tid; e < n * n; e += CHOL_THREADS) {
    const int c = e / n, i = e - (e / n) * n;
    if (i <= c) W[e] = (i == c) ? S::one() : S::zero();
  }
  __syncthreads();

  // 4. X = R~^{-1}: the columns are independent triangular solves, so each
  // warp back-substitutes whole columns on its own (column c in row c of the
  // lower triangle, X[i][c] at W[c*n+i]) with only warp-level syncs; the
  // 1/r_kk scaling of each entry is applied once at the end.
  for (int c = n - 1 - warp; c >= 0; c -= NW) {
    T* xc = W + c * n;
    for (int k = c; k >= 1; --k) {
      const double inv = ri[k];
      if (inv != 0.0) {
        // x_i -= R[i][k] * x_k / r_kk   for i < k
        const T xk = S::scale(xc[k], inv);
        for (int i = lane; i < k; i += 32) xc[i] = S::sub(xc[i], S::mul(W[i * n + k], xk));
      }
      __syncwarp();
    }
    for (int i = lane; i <= c; i += 32) {
      const double inv = ri[i];
      if (inv != 0.0) xc[i] = S::scale(xc[i], inv);
    }
  }
  __syncthreads();

  // 5. outputs
  for (int e = tid; e < n * n; e += CHOL_THREADS) {
    const int i = e / n, j = e - (e / n) * n;
    T r = S::zero();
    if (pos[i] >= 0 && pos[j] >= 0) {
      if (j > i) r = W[e];
      else if (j == i) r = S::make(rd[i], 0.0);
    }
    Rout[e] = r;
    // P[i][c'] = X[i][c] with c' = pos[c] (gathered by destination)
    T pv = S::zero();
    if (pos[i] >= 0 && j < rank) {
      const int c = kidx[j];
      if (i <= c) pv = W[c * n + i];
    }
    P[e] = pv;
  }
  if (tid == 0) {
    info[0] = rank;
    info[1] = s_unres;
    info[2] = s_bad;
    if (status) {
      // speculative-path flags: 1 unresolved pivot, 2 column dropped, 4 non-finite
      const int bits = (s_unres ? 1 : 0) | (rank < n ? 2 : 0) | (s_bad ? 4 : 0);
      if (bits) atomicOr(status, bits);
    }
  }
}

template <typename T>
void launch_chol(Handle* h, int64_t ell, const T* G, double drop_tol, double unres_rel,
                 double shift_coef, T* P, T* R, int32_t* info) {
  LR_REQUIRE(ell >= 1 && ell <= 4096, LR_EINVAL, "chol_drop: ell out of range [1, 4096]");
  const int n = int(ell);
  const size_t tail = size_t(n) * (3 * sizeof(double) + 2 * sizeof(int));
  const size_t full = size_t(n) * n * sizeof(T) + tail;
  int max_smem = 0;
  LR_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  const bool in_smem = full <= size_t(max_smem) - 1024 && n <= smem_maxn<T>();
  // few warps: the kernel is latency-bound and per-column overhead is paid
  // by every warp, so small problems run fastest on 4 warps
  if (in_smem) {
    static int forced = -1;
    if (forced < 0) {
      const char* e = getenv("LR_CHOL_THREADS");
      forced = e ? atoi(e) : 0;
    }
    const int nt = forced ? forced : 1024;
    auto launch = [&](auto kern, int threads) {
      LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(full)));
      kern<<<1, threads, full, h->stream>>>(n, G, drop_tol, unres_rel, shift_coef, P, R, info,
                                            nullptr, h->status, h->gate);
    };
    if (nt <= 128) launch(chol_drop_kernel<T, true, 128>, 128);
    else if (nt <= 256) launch(chol_drop_kernel<T, true, 256>, 256);
    else if (nt <= 512) launch(chol_drop_kernel<T, true, 512>, 512);
    else launch(chol_drop_kernel<T, true, 1024>, 1024);
  } else {
    T* gW = pool_alloc_t<T>(h, size_t(n) * n);
    auto kern = chol_drop_kernel<T, false, 512>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tail)));
    kern<<<1, 512, tail, h->stream>>>(n, G, drop_tol, unres_rel, shift_coef, P, R, info, gW,
                                      h->status, h->gate);
  }
  LR_CHECK_LAUNCH();
}

}  // namespace

void chol_drop_f64(Handle* h, int64_t ell, const double* G, double drop_tol, double unres_rel,
                   double shift_coef, double* P, double* R, int32_t* info) {
  LR_REQUIRE(ell >= 1 && ell <= 4096, LR_EINVAL, "chol_drop: ell out of range [1, 4096]");
  if (chol_panel_supported(ell, false)) {
    chol_panel_f64(h, ell, G, ell, drop_tol, unres_rel, shift_coef, P, R, info, nullptr, nullptr,
                   0, true);
    return;
  }
  if (chol_tiled_supported(ell, false)) {
    chol_tiled_f64(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
    return;
  }
  if (chol_blocked_supported(ell)) {
    chol_blocked_f64(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
    return;
  }
  launch_chol<double>(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
}

void chol_drop_c128(Handle* h, int64_t ell, const double2* G, double drop_tol,
                    double unres_rel, double shift_coef, double2* P, double2* R,
                    int32_t* info) {
  LR_REQUIRE(ell >= 1 && ell <= 4096, LR_EINVAL, "chol_drop: ell out of range [1, 4096]");
  if (chol_panel_supported(ell, true)) {
    chol_panel_c128(h, ell, G, ell, drop_tol, unres_rel, shift_coef, P, R, info, nullptr,
                    nullptr, 0, true);
    return;
  }
  if (chol_tiled_supported(ell, true)) {
    chol_tiled_c128(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
    return;
  }
  if (chol_blocked_supported(ell)) {
    chol_blocked_c128(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
    return;
  }
  launch_chol<double2>(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
}

}  // namespace lr
