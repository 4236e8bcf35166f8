// Row interpolative decomposition on the device (reference factor.py:198-258:
// _column_id / row_id, and the Businger-Golub pivoted QR of core.py:133-186
// they start from), the skeleton step of svd_via_row_extraction
// (factor.py:267-281).
//
// row_id(M, k) is the column ID of B = M^H (k x m): B P = Q [R11 R12] by
// column-pivoted Householder QR -- at step j the column of largest remaining
// norm ||B[j:, c]|| (ties to the lowest position) is swapped to position j
// and reflected -- then T = R11^{-1} R12 with the reference's truncated back
// substitution (rows with |r_ii| <= 1e-12 max|r_ii| give zero), and
// X (m x k) = M-rows: X[J] = I, X[free] = T^H.  Here column c of B is kept as
// row c of a device work matrix W (m x k), so a step is one sweep over the
// rows: apply the previous reflector, re-evaluate the remaining norm exactly
// (the reference recomputes norms, it does not downdate) and reduce the
// arg-max per block; a single-block kernel picks the pivot, swaps positions
// and forms the next reflector.  No host synchronization inside the k steps.
// mode 1 ("forced"): the pivot order is given (the Gu-Eisenstat refinement's
// recomputation, np.linalg.qr(B[:, order]) in the reference).
#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int RT = 256;   // threads per block

template <typename T>
__device__ __forceinline__ T conj_t(T a) { return Sc<T>::conj(a); }

// step j: rows with pos >= j - 1 take reflector j - 1 (v stored at
// vbuf[(j-1) k ...], entries r >= j - 1); rows with pos >= j report their
// remaining squared norm sum_{r >= j} |W[i][r]|^2 for the arg-max
template <typename T>
__global__ void __launch_bounds__(RT) pqr_step_kernel(int64_t m, int kc, int k, int j,
                                                      T* __restrict__ W,
                                                      const T* __restrict__ vbuf,
                                                      const int32_t* __restrict__ vvalid,
                                                      const int32_t* __restrict__ pos_of,
                                                      double* __restrict__ cand_norm,
                                                      int64_t* __restrict__ cand_pos) {
  using S = Sc<T>;
  __shared__ double sn[RT];
  __shared__ int64_t sp[RT];
  double best = -1.0;
  int64_t bestp = INT64_MAX;
  const bool apply = j > 0 && vvalid[j - 1];
  const T* v = vbuf + int64_t(j > 0 ? j - 1 : 0) * kc;
  for (int64_t i = blockIdx.x * int64_t(RT) + threadIdx.x; i < m; i += int64_t(gridDim.x) * RT) {
    const int64_t p = pos_of[i];
    if (p < j - 1) continue;
    T* w = W + i * kc;
    if (apply) {
      T s = S::zero();
      for (int r = j - 1; r < kc; ++r) s = S::add(s, S::cmul(v[r], w[r]));   // v^H w
      for (int r = j - 1; r < kc; ++r) w[r] = S::sub(w[r], S::scale(S::mul(v[r], s), 2.0));
    }
    if (p >= j && j < k) {
      double nr = 0.0;
      for (int r = j; r < kc; ++r) nr += S::abs2(w[r]);
      if (nr > best || (nr == best && p < bestp)) {
        best = nr;
        bestp = p;
      }
    }
  }
  sn[threadIdx.x] = best;
  sp[threadIdx.x] = bestp;
  __syncthreads();
  for (int o = RT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double a = sn[threadIdx.x + o];
      const int64_t ap = sp[threadIdx.x + o];
      if (a > sn[threadIdx.x] || (a == sn[threadIdx.x] && ap < sp[threadIdx.x])) {
        sn[threadIdx.x] = a;
        sp[threadIdx.x] = ap;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cand_norm[blockIdx.x] = sn[0];
    cand_pos[blockIdx.x] = sp[0];
  }
}

// pick the pivot (largest norm, lowest position; mode 1: the given order),
// swap it to position j, and form reflector j from its entries r >= j:
// v = x + ph ||x|| e_1, normalized (core.py:157-168)
template <typename T>
__global__ void __launch_bounds__(RT) pqr_pivot_kernel(int64_t m, int kc, int j, int nblocks,
                                                       int forced, const double* cand_norm,
                                                       const int64_t* cand_pos, T* __restrict__ W,
                                                       T* __restrict__ vbuf,
                                                       int32_t* __restrict__ vvalid,
                                                       int32_t* __restrict__ pos_of,
                                                       int32_t* __restrict__ orig_at) {
  using S = Sc<T>;
  __shared__ double red[RT];
  __shared__ int64_t piv_s;
  if (threadIdx.x == 0) {
    int64_t piv = j;
    if (!forced) {
      double best = -1.0;
      int64_t bp = INT64_MAX;
      for (int b = 0; b < nblocks; ++b)
        if (cand_norm[b] > best || (cand_norm[b] == best && cand_pos[b] < bp)) {
          best = cand_norm[b];
          bp = cand_pos[b];
        }
      piv = bp;
    }
    // swap positions j and piv
    const int32_t a = orig_at[j], p = orig_at[piv];
    orig_at[j] = p;
    orig_at[piv] = a;
    pos_of[p] = j;
    pos_of[a] = int32_t(piv);
    piv_s = p;
  }
  __syncthreads();
  T* x = W + piv_s * kc;
  double part = 0.0;
  for (int r = j + threadIdx.x; r < kc; r += RT) part += S::abs2(x[r]);
  red[threadIdx.x] = part;
  __syncthreads();
  for (int o = RT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double xnorm = sqrt(red[0]);
  __syncthreads();
  T* v = vbuf + int64_t(j) * kc;
  if (!(xnorm > 0.0)) {
    if (threadIdx.x == 0) vvalid[j] = 0;
    return;
  }
  const T x0 = x[j];
  const double a0 = sqrt(S::abs2(x0));
  const T ph = a0 > 0.0 ? S::scale(x0, 1.0 / a0) : S::one();
  // ||v||^2 = ||x||^2 + 2 xnorm |x0| + xnorm^2
  const double vn2 = 2.0 * xnorm * xnorm + 2.0 * xnorm * a0;
  const double inv = vn2 > 0.0 ? 1.0 / sqrt(vn2) : 0.0;
  for (int r = threadIdx.x; r < kc; r += RT) {
    T e = r < j ? S::zero() : x[r];
    if (r == j) e = S::add(e, S::scale(ph, xnorm));
    v[r] = S::scale(e, inv);
  }
  if (threadIdx.x == 0) vvalid[j] = vn2 > 0.0 ? 1 : 0;
}

// R11 (k x k, row-major, upper): R11[r][t] = W[orig_at[t]][r] * conj(ph_r)
// with ph_r the phase of the diagonal (core.py:177-180); also the phases
template <typename T>
__global__ void pqr_r11_kernel(int kc, int k, const T* __restrict__ W,
                               const int32_t* __restrict__ orig_at, T* __restrict__ R11,
                               T* __restrict__ ph) {
  using S = Sc<T>;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int r = e / k, t = e % k;
    const T d = W[int64_t(orig_at[r]) * kc + r];
    const double ad = sqrt(S::abs2(d));
    const T p = ad > 0.0 ? S::scale(d, 1.0 / ad) : S::one();
    if (t == 0) ph[r] = p;
    R11[e] = t >= r ? S::cmul(p, W[int64_t(orig_at[t]) * kc + r]) : S::zero();
  }
}

// Rinv = R11^{-1} with the reference's truncation (solve_triangular_trunc,
// core.py:275-294, applied to the identity: the solve is linear in the
// right-hand side, so T = Rinv R12).  One thread per column of the identity.
template <typename T>
__global__ void trunc_inverse_kernel(int k, const T* __restrict__ R, T* __restrict__ Rinv,
                                     double trunc_tol) {
  using S = Sc<T>;
  __shared__ double dmax;
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int i = 0; i < k; ++i) mx = fmax(mx, sqrt(S::abs2(R[i * k + i])));
    dmax = mx;
  }
  __syncthreads();
  const double cutoff = trunc_tol * dmax;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    for (int i = k - 1; i >= 0; --i) {
      const T dii = R[i * k + i];
      if (!(sqrt(S::abs2(dii)) > cutoff)) {
        Rinv[i * k + c] = S::zero();
        continue;
      }
      T acc = i == c ? S::one() : S::zero();
      for (int l = i + 1; l < k; ++l) acc = S::sub(acc, S::mul(R[i * k + l], Rinv[l * k + c]));
      // acc / dii
      const double den = S::abs2(dii);
      Rinv[i * k + c] = S::scale(S::mul(acc, conj_t(dii)), 1.0 / den);
    }
  }
}

// X (m x k): X[i] = (Rinv R12_i)^H for free rows, e_t for the skeleton row at
// position t; R12_i[r] = conj(ph_r) W[i][r].  tmax[0] = max |X_free| (the
// refinement test, factor.py:222); the arg-max position is reduced by the
// caller (host) only when tmax exceeds the bound.
template <typename T>
__global__ void rowid_x_kernel(int64_t m, int kc, int k, const T* __restrict__ W,
                               const T* __restrict__ Rinv,
                               const T* __restrict__ ph, const int32_t* __restrict__ pos_of,
                               T* __restrict__ X, int64_t ldx, unsigned long long* tmax_bits) {
  using S = Sc<T>;
  double local = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * k;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / k;
    const int c = int(e % k);
    const int p = pos_of[i];
    T out;
    if (p < k) {
      out = p == c ? S::one() : S::zero();
    } else {
      T acc = S::zero();
      const T* w = W + i * kc;
      for (int r = 0; r < k; ++r) acc = S::add(acc, S::mul(Rinv[c * k + r], S::cmul(ph[r], w[r])));
      out = conj_t(acc);
      local = fmax(local, sqrt(S::abs2(out)));
    }
    X[i * ldx + c] = out;
  }
  for (int o = 16; o > 0; o >>= 1) local = fmax(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0 && local > 0.0)
    atomicMax(tmax_bits, static_cast<unsigned long long>(__double_as_longlong(local)));
}

template <typename T>
__global__ void conj_copy_rows(int64_t m, int kc, const T* __restrict__ M, int64_t ldm,
                               T* __restrict__ W) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * kc;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / kc;
    const int c = int(e % kc);
    W[e] = conj_t(M[i * ldm + c]);
  }
}

__global__ void iota_kernel(int64_t m, int32_t* pos_of, int32_t* orig_at, const int32_t* order) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t o = order ? order[i] : int32_t(i);
    orig_at[i] = o;
    pos_of[o] = int32_t(i);
  }
}

template <typename T>
void row_id_impl(Handle* h, int64_t m, int kc, int k, const T* M, int64_t ldm, int32_t* perm,
                 int forced, T* X, int64_t ldx, double* tmax_dev) {
  T* W = pool_alloc_t<T>(h, size_t(m) * kc);
  T* vbuf = pool_alloc_t<T>(h, size_t(k) * kc);
  int32_t* vvalid = pool_alloc_t<int32_t>(h, size_t(k));
  int32_t* pos_of = pool_alloc_t<int32_t>(h, size_t(m));
  int32_t* order_in = forced ? pool_alloc_t<int32_t>(h, size_t(m)) : nullptr;
  const int nb = int(std::min<int64_t>(ceil_div(m, RT), int64_t(h->sm_count) * 4));
  double* cn = pool_alloc_t<double>(h, size_t(nb));
  int64_t* cp = pool_alloc_t<int64_t>(h, size_t(nb));
  T* R11 = pool_alloc_t<T>(h, size_t(k) * k);
  T* Rinv = pool_alloc_t<T>(h, size_t(k) * k);
  T* ph = pool_alloc_t<T>(h, size_t(k));
  conj_copy_rows<T><<<int(std::min<int64_t>(ceil_div(m * kc, 256), 8192)), 256, 0, h->stream>>>(
      m, kc, M, ldm, W);
  LR_CHECK_LAUNCH();
  if (forced) LR_CUDA(cudaMemcpyAsync(order_in, perm, sizeof(int32_t) * m,
                                      cudaMemcpyDeviceToDevice, h->stream));
  iota_kernel<<<int(std::min<int64_t>(ceil_div(m, 256), 4096)), 256, 0, h->stream>>>(
      m, pos_of, perm, order_in);
  LR_CHECK_LAUNCH();
  for (int j = 0; j <= k; ++j) {
    pqr_step_kernel<T><<<nb, RT, 0, h->stream>>>(m, kc, k, j, W, vbuf, vvalid, pos_of, cn, cp);
    LR_CHECK_LAUNCH();
    if (j == k) break;
    pqr_pivot_kernel<T><<<1, RT, 0, h->stream>>>(m, kc, j, nb, forced, cn, cp, W, vbuf, vvalid,
                                                 pos_of, perm);
    LR_CHECK_LAUNCH();
  }
  pqr_r11_kernel<T><<<int(ceil_div(int64_t(k) * k, 256)), 256, 0, h->stream>>>(kc, k, W, perm,
                                                                              R11, ph);
  LR_CHECK_LAUNCH();
  trunc_inverse_kernel<T><<<1, 256, 0, h->stream>>>(k, R11, Rinv, 1e-12);
  LR_CHECK_LAUNCH();
  LR_CUDA(cudaMemsetAsync(tmax_dev, 0, sizeof(double), h->stream));
  rowid_x_kernel<T><<<int(std::min<int64_t>(ceil_div(m * k, 256), 8192)), 256, 0, h->stream>>>(
      m, kc, k, W, Rinv, ph, pos_of, X, ldx, reinterpret_cast<unsigned long long*>(tmax_dev));
  LR_CHECK_LAUNCH();
}

}  // namespace

void row_id(Handle* h, int dtype, int64_t m, int64_t kc, int64_t k, const void* M, int64_t ldm,
            int32_t* perm, int forced, void* X, int64_t ldx, double* tmax_dev) {
  LR_REQUIRE(k >= 1 && k <= m && k <= kc && kc <= 1024, LR_EINVAL,
             "row_id: need 1 <= k <= min(m, ncols) and ncols <= 1024");
  if (dtype == LR_F64)
    row_id_impl<double>(h, m, int(kc), int(k), static_cast<const double*>(M), ldm, perm, forced,
                        static_cast<double*>(X), ldx, tmax_dev);
  else if (dtype == LR_C128)
    row_id_impl<double2>(h, m, int(kc), int(k), static_cast<const double2*>(M), ldm, perm, forced,
                         static_cast<double2*>(X), ldx, tmax_dev);
  else
    throw Error{LR_EINVAL, "row_id: float64 / complex128"};
}

}  // namespace lr
