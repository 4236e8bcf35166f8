// Stage-B Hermitian helpers (reference factor.py:168-335, core.py:233-272):
// the small Hermitian eigendecomposition of direct_eig_hermitian /
// eig_nystrom is computed as the SVD of a shifted positive-definite matrix
// by the K4 small-SVD kernels:
//   H = (B + B^H) / 2 + s I,  s = 2 ||sym(B)||_F  (all eigenvalues of H lie in
//   [s - ||.||_2, s + ||.||_2] subset [||.||_F, 3 ||.||_F]: SPD, kappa <= 3)
// so H = U diag(sigma) U^H with lambda = sigma - s.  The absolute accuracy
// is O(u ||B||), that of LAPACK eigh (the reference's small_eig_hermitian).
#include <cstdlib>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int HT = 1024;

template <typename T>
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// H = sym(B) + shift I; out[0] = shift, out[1] = ||sym(B)||_2 estimate
// (power iteration, power_iters steps) when power_iters > 0.
template <typename T>
__global__ void __launch_bounds__(HT) herm_prep_kernel(int n, const T* __restrict__ B, int64_t ldb,
                                                       T* __restrict__ H, double shift_mult,
                                                       int power_iters, double* __restrict__ out) {
  using S = Sc<T>;
  __shared__ double red[32];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* x = reinterpret_cast<T*>(smem_raw);   // [n] power-iteration vector
  T* y = x + n;
  double fro = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, k = e - i * n;
    const T a = B[size_t(i) * ldb + k], b = B[size_t(k) * ldb + i];
    const T v = S::scale(S::add(a, S::conj(b)), 0.5);
    H[e] = v;
    fro += S::abs2(v);
  }
  fro = sqrt(block_sum<T>(fro, red));
  double shift = 0.0;
  if (shift_mult > 0.0) shift = fro > 0.0 ? shift_mult * fro : 1.0;
  __syncthreads();   // H complete (every thread reads rows below)
  if (power_iters > 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      x[i] = S::make(rsqrt(double(n)) * (1.0 + 0.25 * sin(1.7 * i + 0.3)), 0.0);
    __syncthreads();
    double nrm = 0.0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int it = 0; it < power_iters; ++it) {
      double part = 0.0;
      for (int r = w; r < n; r += nw) {
        T acc = S::zero();
        for (int c = lane; c < n; c += 32) acc = S::add(acc, S::mul(H[size_t(r) * n + c], x[c]));
        acc = warp_sum(acc);
        if (lane == 0) y[r] = acc;
        part += lane == 0 ? S::abs2(acc) : 0.0;
      }
      nrm = sqrt(block_sum<T>(part, red));
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = S::scale(y[i], inv);
      __syncthreads();
    }
    if (threadIdx.x == 0) out[1] = nrm;
  }
  if (shift != 0.0)
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      H[size_t(i) * n + i] = S::add(H[size_t(i) * n + i], S::make(shift, 0.0));
  if (threadIdx.x == 0) out[0] = shift;
}

// lambda_i = sigma_i - shift, ordered by descending |lambda| (ties: descending
// lambda, then index) as the reference's np.lexsort((-lam, -|lam|));
// column i of U goes to column rank(i) of V.
template <typename T>
__global__ void __launch_bounds__(HT) eig_finish_kernel(int n, const double* __restrict__ sig,
                                                        const double* __restrict__ shift,
                                                        const T* __restrict__ U,
                                                        double* __restrict__ lam,
                                                        T* __restrict__ V) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* l = reinterpret_cast<double*>(smem_raw);
  int* rk = reinterpret_cast<int*>(l + n);
  const double s = *shift;
  for (int i = threadIdx.x; i < n; i += blockDim.x) l[i] = sig[i] - s;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(l[i]), li = l[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double b = fabs(l[j]);
      r += (b > a) || (b == a && (l[j] > li || (l[j] == li && j < i)));
    }
    rk[i] = r;
    lam[r] = li;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int row = e / n, c = e - row * n;
    V[size_t(row) * n + rk[c]] = U[e];
  }
}

}  // namespace

void herm_prep(Handle* h, int dtype_wide, int64_t n, const void* B, int64_t ldb, void* H,
               double shift_mult, int power_iters, double* out2) {
  const size_t smem = size_t(2 * n) * (dtype_wide == LR_C128 ? 16 : 8);
  if (dtype_wide == LR_C128)
    herm_prep_kernel<double2><<<1, HT, smem, h->stream>>>(
        int(n), static_cast<const double2*>(B), ldb, static_cast<double2*>(H), shift_mult,
        power_iters, out2);
  else
    herm_prep_kernel<double><<<1, HT, smem, h->stream>>>(
        int(n), static_cast<const double*>(B), ldb, static_cast<double*>(H), shift_mult,
        power_iters, out2);
  LR_CHECK_LAUNCH();
}

void eig_finish(Handle* h, int dtype_wide, int64_t n, const double* S, const double* shift,
                const void* U, double* lam, void* V) {
  const size_t smem = size_t(n) * (sizeof(double) + sizeof(int));
  if (dtype_wide == LR_C128)
    eig_finish_kernel<double2><<<1, HT, smem, h->stream>>>(
        int(n), S, shift, static_cast<const double2*>(U), lam, static_cast<double2*>(V));
  else
    eig_finish_kernel<double><<<1, HT, smem, h->stream>>>(
        int(n), S, shift, static_cast<const double*>(U), lam, static_cast<double*>(V));
  LR_CHECK_LAUNCH();
}

}  // namespace lr
