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
// Outputs: P (ell x ell): Q = Y . P[:, :rank] has orthonormal columns,
// P[kept_i][c] = (R_SS^{-1})[i][c];  R (ell x ell) the factor restricted to
// kept rows/cols; info = {rank, unresolved pivots, bad pivots}.
#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int CHOL_THREADS = 1024;

__device__ __forceinline__ int up_idx(int i, int j, int n) {
  // packed upper triangle, row-major: row i holds columns i..n-1
  return i * n - (i * (i - 1)) / 2 + (j - i);
}

template <typename T>
__device__ __forceinline__ bool finite_sc(T v);
template <>
__device__ __forceinline__ bool finite_sc<double>(double v) { return isfinite(v); }
template <>
__device__ __forceinline__ bool finite_sc<double2>(double2 v) {
  return isfinite(v.x) && isfinite(v.y);
}

template <typename T>
__global__ void __launch_bounds__(CHOL_THREADS, 1)
chol_drop_kernel(int n, const T* __restrict__ G, double drop_tol, double unres_rel,
                 double shift_coef, T* __restrict__ P, T* __restrict__ Rout,
                 int32_t* __restrict__ info, T* gW, bool w_in_smem) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int np = n * (n + 1) / 2;
  T* W;
  T* X;
  unsigned char* tail;
  if (w_in_smem) {
    W = reinterpret_cast<T*>(smem_raw);
    X = W + np;
    tail = reinterpret_cast<unsigned char*>(X + np);
  } else {
    W = gW;
    X = gW + np;
    tail = smem_raw;
  }
  double* d0 = reinterpret_cast<double*>(tail);         // original pivots (shifted)
  int* pos = reinterpret_cast<int*>(d0 + n);            // compact index or -1
  int* kidx = pos + n;                                  // compact -> original

  __shared__ double s_red[32];
  __shared__ double s_thr2, s_shift, s_rjj;
  __shared__ int s_keep, s_unres, s_bad, s_rank;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;

  // 1. load upper triangle, trace
  double tr = 0.0;
  for (int i = warp; i < n; i += nwarps) {
    for (int j = i + lane; j < n; j += 32) {
      T g = G[int64_t(i) * n + j];
      W[up_idx(i, j, n)] = g;
      if (j == i) tr += S::re(g);
    }
  }
  for (int m = 16; m > 0; m >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, m);
  if (lane == 0) s_red[warp] = tr;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < nwarps; ++w) t += s_red[w];
    s_thr2 = drop_tol * drop_tol * t;
    s_shift = shift_coef * t;
    s_unres = 0;
    s_bad = 0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    T w = W[up_idx(i, i, n)];
    double d = S::re(w) + s_shift;
    W[up_idx(i, i, n)] = S::make(d, 0.0);
    d0[i] = d;
  }
  __syncthreads();

  // 2. right-looking factorization with deletion
  for (int j = 0; j < n; ++j) {
    if (tid == 0) {
      const double d = S::re(W[up_idx(j, j, n)]);
      int keep = 0;
      double r = 0.0;
      if (!isfinite(d)) {
        s_bad += 1;
      } else if (d > s_thr2 && d > 0.0) {
        keep = 1;
        r = sqrt(d);
        if (d <= unres_rel * d0[j]) s_unres += 1;
      }
      s_keep = keep;
      s_rjj = r;
    }
    __syncthreads();
    const int keep = s_keep;
    const double rjj = s_rjj;
    if (keep) {
      const double inv = 1.0 / rjj;
      for (int i = j + 1 + tid; i < n; i += blockDim.x)
        W[up_idx(j, i, n)] = S::scale(W[up_idx(j, i, n)], inv);
      if (tid == 0) W[up_idx(j, j, n)] = S::make(rjj, 0.0);
    } else {
      for (int i = j + tid; i < n; i += blockDim.x) W[up_idx(j, i, n)] = S::zero();
    }
    __syncthreads();
    if (keep) {
      for (int a = j + 1 + warp; a < n; a += nwarps) {
        const T rja = S::conj(W[up_idx(j, a, n)]);
        for (int b = a + lane; b < n; b += 32) {
          const int ib = up_idx(a, b, n);
          W[ib] = S::sub(W[ib], S::mul(rja, W[up_idx(j, b, n)]));
        }
      }
    }
    __syncthreads();
  }

  // 3. compaction of kept columns
  if (tid == 0) {
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const bool k = S::re(W[up_idx(j, j, n)]) > 0.0;
      pos[j] = k ? r : -1;
      if (k) kidx[r++] = j;
    }
    s_rank = r;
  }
  __syncthreads();
  const int rank = s_rank;

  // 4. X = R_SS^{-1} (upper, rank x rank, packed with dimension rank)
  for (int c = warp; c < rank; c += nwarps) {
    const int oc = kidx[c];
    const double rcc = S::re(W[up_idx(oc, oc, n)]);
    if (lane == 0) X[up_idx(c, c, rank)] = S::make(1.0 / rcc, 0.0);
    __syncwarp();
    for (int i = c - 1; i >= 0; --i) {
      const int oi = kidx[i];
      T acc = S::zero();
      for (int k = i + 1 + lane; k <= c; k += 32)
        acc = S::add(acc, S::mul(W[up_idx(oi, kidx[k], n)], X[up_idx(k, c, rank)]));
      acc = warp_sum(acc);
      if (lane == 0) {
        const double rii = S::re(W[up_idx(oi, oi, n)]);
        X[up_idx(i, c, rank)] = S::scale(acc, -1.0 / rii);
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // 5. outputs
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    // P: row i (original column of Y), column j (compact basis index)
    T p = S::zero();
    const int pi = pos[i];
    if (pi >= 0 && j < rank && pi <= j) p = X[up_idx(pi, j, rank)];
    P[e] = p;
    T r = S::zero();
    if (j >= i && pos[i] >= 0 && pos[j] >= 0) r = W[up_idx(i, j, n)];
    Rout[e] = r;
  }
  if (tid == 0) {
    info[0] = rank;
    info[1] = s_unres;
    info[2] = s_bad;
  }
}

template <typename T>
void launch_chol(Handle* h, int64_t ell, const T* G, double drop_tol, double unres_rel,
                 double shift_coef, T* P, T* R, int32_t* info) {
  LR_REQUIRE(ell >= 1 && ell <= 2048, LR_EINVAL, "chol_drop: ell out of range [1, 2048]");
  const int n = int(ell);
  const size_t np = size_t(n) * (n + 1) / 2;
  const size_t tail = size_t(n) * (sizeof(double) + 2 * sizeof(int));
  const size_t full = 2 * np * sizeof(T) + tail;
  int max_smem = 0;
  LR_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  const size_t limit = size_t(max_smem) - 4096;   // static shared + slack
  bool in_smem = full <= limit;
  T* gW = nullptr;
  size_t dyn = full;
  if (!in_smem) {
    gW = pool_alloc_t<T>(h, 2 * np);
    dyn = tail;
  }
  auto kern = chol_drop_kernel<T>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn)));
  kern<<<1, CHOL_THREADS, dyn, h->stream>>>(n, G, drop_tol, unres_rel, shift_coef, P, R, info,
                                            gW, in_smem);
  LR_CHECK_LAUNCH();
}

}  // namespace

void chol_drop_f64(Handle* h, int64_t ell, const double* G, double drop_tol, double unres_rel,
                   double shift_coef, double* P, double* R, int32_t* info) {
  launch_chol<double>(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
}

void chol_drop_c128(Handle* h, int64_t ell, const double2* G, double drop_tol,
                    double unres_rel, double shift_coef, double2* P, double2* R,
                    int32_t* info) {
  launch_chol<double2>(h, ell, G, drop_tol, unres_rel, shift_coef, P, R, info);
}

}  // namespace lr
