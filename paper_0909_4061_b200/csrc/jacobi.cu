// K4: one-sided (Hestenes) Jacobi SVD of a small matrix, one CTA.
//
// Used by the small SVD of direct_svd (reference core.py:199-230,
// factor.py:163-165): B^H = Q2 R2 (CholeskyQR), then R2 = W diag(S) J^H by
// orthogonalizing the columns of R2 with plane rotations: R2 J = W diag(S).
// Then B = J diag(S) (Q2 W)^H, i.e. U_B = J and V_B = Q2 W.  One-sided Jacobi
// is used instead of bidiagonalization because it is accurate in a relative
// sense for the graded triangular factors CholeskyQR produces and maps onto
// parallel column pairs (round-robin ordering, n/2 pairs per round).
//
// Parallel layout: each pair of a round is owned by a group of GS lanes
// (GS = 8..32, chosen so all n/2 pairs of a round run at once); the three
// dot products are reduced with xor-shuffles inside the group; one barrier
// per round.  Columns are stored contiguously (column-major working copies)
// so a group's loads are conflict-free.
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
__device__ __forceinline__ T group_sum(T v, int gs) {
  for (int m = gs >> 1; m > 0; m >>= 1) v = Sc<T>::add(v, Sc<T>::shfl_xor(v, m));
  return v;
}

template <typename T, bool SMEM>
__global__ void __launch_bounds__(JAC_THREADS, 1)
jacobi_kernel(int rows, int n, const T* __restrict__ M, T* __restrict__ Wout,
              double* __restrict__ Sout, T* __restrict__ Jout, int32_t* __restrict__ info, T* gbuf,
              double tol, int max_sweeps, int gs, int32_t* status) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* __restrict__ Mc;
  T* __restrict__ Jc;
  unsigned char* tail;
  if constexpr (SMEM) {
    Mc = reinterpret_cast<T*>(smem_raw);
    Jc = Mc + size_t(rows) * n;
    tail = reinterpret_cast<unsigned char*>(Jc + size_t(n) * n);
  } else {
    Mc = gbuf;
    Jc = gbuf + size_t(rows) * n;
    tail = smem_raw;
  }
  const int np2 = n + (n & 1);
  const int pairs = np2 / 2;
  T* pgm = reinterpret_cast<T*>(tail);                // pairs: m_p^H m_q, then s e
  double* sig = reinterpret_cast<double*>(pgm + pairs);  // n
  double* pa = sig + n;                               // pairs: ||m_p||^2
  double* pb = pa + pairs;                            // pairs: ||m_q||^2
  double* pc = pb + pairs;                            // pairs: c (0 = no rotation)
  int* order = reinterpret_cast<int*>(pc + pairs);    // n: order[o] = source column

  __shared__ int s_rot[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int glane = tid % gs, group = tid / gs, ngroups = blockDim.x / gs;

  // column-major working copies
  for (int64_t e = tid; e < int64_t(rows) * n; e += blockDim.x) {
    const int i = int(e / n), j = int(e % n);
    Mc[size_t(j) * rows + i] = M[e];
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    Jc[size_t(j) * n + i] = (i == j) ? S::one() : S::zero();
  }
  if (tid == 0) { s_rot[0] = 0; s_rot[1] = 0; }
  __syncthreads();

  const int rounds = np2 - 1;
  const int iters = (pairs + ngroups - 1) / ngroups;
  int sweep = 0;
  bool converged = (n == 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    const int flag = sweep & 1;   // double-buffered "rotated" flag
    for (int r = 0; r < rounds; ++r) {
      // phase 1: the three inner products of every pair (one group per pair)
      for (int it = 0; it < iters; ++it) {
        const int k = group + it * ngroups;
        int p = -1, q = -1;
        if (k < pairs) {
          const int ia = k, ib = np2 - 1 - k;
          p = (ia == 0) ? 0 : 1 + (ia - 1 + r) % rounds;
          q = (ib == 0) ? 0 : 1 + (ib - 1 + r) % rounds;
          if (p > q) { const int t = p; p = q; q = t; }
          if (q >= n) p = q = -1;
        }
        double a = 0.0, b = 0.0;
        T gmm = S::zero();
        if (p >= 0) {
          const T* mp = Mc + size_t(p) * rows;
          const T* mq = Mc + size_t(q) * rows;
          for (int i = glane; i < rows; i += gs) {
            const T x = mp[i], y = mq[i];
            a += S::abs2(x);
            b += S::abs2(y);
            gmm = S::add(gmm, S::cmul(x, y));
          }
        }
        a = group_sum(a, gs);
        b = group_sum(b, gs);
        gmm = group_sum(gmm, gs);
        if (k < pairs && glane == 0) {
          pa[k] = (p >= 0) ? a : -1.0;
          pb[k] = b;
          pgm[k] = gmm;
        }
      }
      __syncthreads();
      // phase 2: rotation parameters, one pair per lane of the first warps
      for (int k = tid; k < pairs; k += blockDim.x) {
        const double a = pa[k], b = pb[k];
        const T gmm = pgm[k];
        const double g2 = S::abs2(gmm);
        double c = 0.0;
        T se = S::zero();
        if (a >= 0.0 && g2 > 0.0 && g2 > tol * tol * a * b) {
          const double iag = rsqrt(g2);                 // 1 / |gamma|
          const double zeta = 0.5 * (b - a) * iag;
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = rsqrt(1.0 + t * t);
          se = S::scale(gmm, c * t * iag);              // s * phase(gamma)
          s_rot[flag] = 1;
        }
        pc[k] = c;
        pgm[k] = se;
      }
      __syncthreads();
      // phase 3: apply the rotations to the columns of M and J
      for (int it = 0; it < iters; ++it) {
        const int k = group + it * ngroups;
        if (k >= pairs) continue;
        const double c = pc[k];
        if (c == 0.0) continue;
        const int ia = k, ib = np2 - 1 - k;
        int p = (ia == 0) ? 0 : 1 + (ia - 1 + r) % rounds;
        int q = (ib == 0) ? 0 : 1 + (ib - 1 + r) % rounds;
        if (p > q) { const int t = p; p = q; q = t; }
        const T se = pgm[k];
        const T sec = S::conj(se);
        T* mp = Mc + size_t(p) * rows;
        T* mq = Mc + size_t(q) * rows;
        for (int i = glane; i < rows; i += gs) {
          const T x = mp[i], y = mq[i];
          mp[i] = S::sub(S::scale(x, c), S::mul(sec, y));
          mq[i] = S::add(S::mul(se, x), S::scale(y, c));
        }
        T* jp = Jc + size_t(p) * n;
        T* jq = Jc + size_t(q) * n;
        for (int i = glane; i < n; i += gs) {
          const T x = jp[i], y = jq[i];
          jp[i] = S::sub(S::scale(x, c), S::mul(sec, y));
          jq[i] = S::add(S::mul(se, x), S::scale(y, c));
        }
      }
      __syncthreads();
    }
    converged = (s_rot[flag] == 0);
    __syncthreads();
    if (tid == 0) s_rot[flag] = 0;   // re-arm this buffer for sweep + 2
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
  if (tid == 0) {
    info[0] = converged ? sweep : -sweep;
    if (!converged && status) atomicOr(status, 8);   // speculative-path flag
  }
}

template <typename T>
void launch_jacobi(Handle* h, int64_t rows64, int64_t n64, const T* M, T* W, double* S, T* J,
                   int32_t* info) {
  LR_REQUIRE(n64 >= 1 && n64 <= 4096 && rows64 >= n64 && rows64 < (int64_t(1) << 31),
             LR_EINVAL, "jacobi_svd: need 1 <= cols <= 4096 and rows >= cols");
  const int n = int(n64), rows = int(rows64);
  const int pairs = (n + (n & 1)) / 2;
  const size_t tail = size_t(n) * (sizeof(double) + sizeof(int)) +
                      size_t(pairs) * (3 * sizeof(double) + sizeof(T)) + 64;
  const size_t full = (size_t(rows) + n) * n * sizeof(T) + tail;
  int max_smem = 0;
  LR_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  const bool in_smem = full <= size_t(max_smem) - 1024;
  // lanes per pair: all pairs of a round in flight, 8..32 lanes each
  int gs = 32;
  while (gs > 8 && pairs * gs > JAC_THREADS) gs >>= 1;
  while (gs > 8 && gs / 2 >= rows) gs >>= 1;
  const double tol = 4e-15;
  if (in_smem) {
    auto kern = jacobi_kernel<T, true>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(full)));
    kern<<<1, JAC_THREADS, full, h->stream>>>(rows, n, M, W, S, J, info, nullptr, tol, 60, gs,
                                              h->status);
  } else {
    T* gbuf = pool_alloc_t<T>(h, (size_t(rows) + n) * n);
    auto kern = jacobi_kernel<T, false>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tail)));
    kern<<<1, JAC_THREADS, tail, h->stream>>>(rows, n, M, W, S, J, info, gbuf, tol, 60, gs,
                                              h->status);
  }
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
