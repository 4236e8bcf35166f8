// K4: one-sided (Hestenes) Jacobi SVD of a small square matrix, one CTA.
//
// Used by the small SVD of direct_svd (reference core.py:199-230,
// factor.py:163-165): B^H = Q2 R2 (CholeskyQR), then R2 = W diag(S) J^H by
// orthogonalizing the columns of R2 with plane rotations: R2 J = W diag(S).
// Then B = J diag(S) (Q2 W)^H, i.e. U_B = J and V_B = Q2 W.  One-sided Jacobi
// is used instead of bidiagonalization because it is accurate in a relative
// sense for the graded triangular factors CholeskyQR produces and maps onto
// warp-parallel column pairs (round-robin ordering, n/2 pairs per round).
//
// Outputs follow the reference conventions: S descending, and the first
// entry of each J column with |j| > 1e-10 max|j| made real positive (the W
// column absorbs the same phase, core.py:221-229).
#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int JAC_THREADS = 1024;

template <typename T>
__global__ void __launch_bounds__(JAC_THREADS, 1)
jacobi_kernel(int rows, int n, const T* __restrict__ M, T* __restrict__ Wout,
              double* __restrict__ Sout, T* __restrict__ Jout, int32_t* __restrict__ info, T* gbuf,
              bool in_smem, double tol, int max_sweeps) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Mc;
  T* Jc;
  unsigned char* tail;
  if (in_smem) {
    Mc = reinterpret_cast<T*>(smem_raw);
    Jc = Mc + size_t(rows) * n;
    tail = reinterpret_cast<unsigned char*>(Jc + size_t(n) * n);
  } else {
    Mc = gbuf;
    Jc = gbuf + size_t(rows) * n;
    tail = smem_raw;
  }
  double* sig = reinterpret_cast<double*>(tail);
  int* order = reinterpret_cast<int*>(sig + n);   // order[o] = source column

  __shared__ int s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;

  // column-major working copies
  for (int64_t e = tid; e < int64_t(rows) * n; e += blockDim.x) {
    const int i = int(e / n), j = int(e % n);
    Mc[size_t(j) * rows + i] = M[e];
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    Jc[size_t(j) * n + i] = (i == j) ? S::one() : S::zero();
  }
  __syncthreads();

  const int np2 = n + (n & 1);
  const int rounds = np2 - 1, pairs = np2 / 2;
  int sweep = 0;
  bool converged = (n == 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < rounds; ++r) {
      for (int k = warp; k < pairs; k += nwarps) {
        const int ia = k, ib = np2 - 1 - k;
        int p = (ia == 0) ? 0 : 1 + (ia - 1 + r) % rounds;
        int q = (ib == 0) ? 0 : 1 + (ib - 1 + r) % rounds;
        if (p > q) { const int t = p; p = q; q = t; }
        if (q >= n) continue;
        T* mp = Mc + size_t(p) * rows;
        T* mq = Mc + size_t(q) * rows;
        double a = 0.0, b = 0.0;
        T gmm = S::zero();
        for (int i = lane; i < rows; i += 32) {
          const T x = mp[i], y = mq[i];
          a += S::abs2(x);
          b += S::abs2(y);
          gmm = S::add(gmm, S::cmul(x, y));
        }
        a = warp_sum(a);
        b = warp_sum(b);
        gmm = warp_sum(gmm);
        const double ag = sqrt(S::abs2(gmm));
        if (!(ag > tol * sqrt(a * b)) || ag == 0.0) continue;
        const double zeta = (b - a) / (2.0 * ag);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        const T e = S::scale(gmm, 1.0 / ag);        // phase of gamma
        const T se = S::scale(e, s);                 // s e
        const T sec = S::conj(se);                   // s conj(e)
        for (int i = lane; i < rows; i += 32) {
          const T x = mp[i], y = mq[i];
          mp[i] = S::sub(S::scale(x, c), S::mul(sec, y));
          mq[i] = S::add(S::mul(se, x), S::scale(y, c));
        }
        T* jp = Jc + size_t(p) * n;
        T* jq = Jc + size_t(q) * n;
        for (int i = lane; i < n; i += 32) {
          const T x = jp[i], y = jq[i];
          jp[i] = S::sub(S::scale(x, c), S::mul(sec, y));
          jq[i] = S::add(S::mul(se, x), S::scale(y, c));
        }
        if (lane == 0) s_rot = 1;
      }
      __syncthreads();
    }
    converged = (s_rot == 0);
    __syncthreads();
  }

  // singular values, descending order (ties by index)
  for (int j = warp; j < n; j += nwarps) {
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) a += S::abs2(Mc[size_t(j) * rows + i]);
    a = warp_sum(a);
    if (lane == 0) sig[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) {
    int rk = 0;
    const double sj = sig[j];
    for (int i = 0; i < n; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
    order[rk] = j;
  }
  __syncthreads();

  // outputs with the reference sign convention, one warp per output column
  for (int o = warp; o < n; o += nwarps) {
    const int j = order[o];
    const T* jc = Jc + size_t(j) * n;
    const T* mc = Mc + size_t(j) * rows;
    double mx = 0.0;
    for (int i = lane; i < n; i += 32) mx = fmax(mx, sqrt(S::abs2(jc[i])));
    for (int m = 16; m > 0; m >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    // first index with |j_i| > 1e-10 * max
    int first = n;
    for (int base = 0; base < n && first == n; base += 32) {
      const int i = base + lane;
      const bool hit = (i < n) && (sqrt(S::abs2(jc[i])) > 1e-10 * mx);
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (bal) first = base + __ffs(bal) - 1;
    }
    T ph = S::one();
    if (first < n) {
      const T z = jc[first];
      ph = S::conj(S::scale(z, 1.0 / sqrt(S::abs2(z))));  // conj(phase)
    }
    const double sj = sig[j];
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    for (int i = lane; i < n; i += 32) Jout[size_t(i) * n + o] = S::mul(jc[i], ph);
    for (int i = lane; i < rows; i += 32)
      Wout[size_t(i) * n + o] = S::mul(S::scale(mc[i], inv), ph);
    if (lane == 0) Sout[o] = sj;
  }
  if (tid == 0) info[0] = converged ? sweep : -sweep;
}

template <typename T>
void launch_jacobi(Handle* h, int64_t rows64, int64_t n64, const T* M, T* W, double* S, T* J,
                   int32_t* info) {
  LR_REQUIRE(n64 >= 1 && n64 <= 4096 && rows64 >= n64 && rows64 < (int64_t(1) << 31),
             LR_EINVAL, "jacobi_svd: need 1 <= cols <= 4096 and rows >= cols");
  const int n = int(n64), rows = int(rows64);
  const size_t tail = size_t(n) * (sizeof(double) + sizeof(int));
  const size_t full = (size_t(rows) + n) * n * sizeof(T) + tail;
  int max_smem = 0;
  LR_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  const bool in_smem = full <= size_t(max_smem) - 1024;
  T* gbuf = nullptr;
  size_t dyn = full;
  if (!in_smem) {
    gbuf = pool_alloc_t<T>(h, (size_t(rows) + n) * n);
    dyn = tail;
  }
  auto kern = jacobi_kernel<T>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn)));
  kern<<<1, JAC_THREADS, dyn, h->stream>>>(rows, n, M, W, S, J, info, gbuf, in_smem, 1e-15, 80);
  LR_CHECK_LAUNCH();
}

}  // namespace

void jacobi_svd_f64(Handle* h, int64_t rows, int64_t n, const double* M, double* W, double* S,
                    double* J, int32_t* info) {
  launch_jacobi<double>(h, rows, n, M, W, S, J, info);
}

void jacobi_svd_c128(Handle* h, int64_t rows, int64_t n, const double2* M, double2* W,
                     double* S, double2* J, int32_t* info) {
  launch_jacobi<double2>(h, rows, n, M, W, S, J, info);
}

}  // namespace lr
