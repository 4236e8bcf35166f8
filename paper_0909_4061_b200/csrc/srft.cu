// K5: SRFT sketch Y = scale * (A o d) F R and the unitary row DFT.
//
// Replaces srft_apply -> dft -> _fft_pow2 (reference sketch.py:306-320,
// 179-200, 129-148): for each row a_i of A (length n, a power of two),
//   y_i[t] = scale * n^{-1/2} * sum_k a_ik d_k exp(-2 pi i k picks_t / n).
// One CTA per row: the row is loaded once from HBM (coalesced), multiplied
// by d and stored into shared memory in bit-reversed order, transformed by
// an in-place radix-2 DIT FFT in shared memory, and only the ell picked bins
// are written back (the sketch is HBM-read-bound: one pass over A, ell/n of
// it written).  Twiddles come from sincospi of exact dyadic arguments.
#include <cstdlib>

#include "common.cuh"

namespace lr {
namespace {

template <typename C>
struct Cx;
template <>
struct Cx<float2> {
  using R = float;
  __device__ static float2 mul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __device__ static float2 tw(int k, int span) {  // exp(-2 pi i k / span)
    float s, c;
    sincospif(-2.0f * float(k) / float(span), &s, &c);
    return make_float2(c, s);
  }
  __device__ static float2 add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
  __device__ static float2 sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
  __device__ static float2 scl(float2 a, double s) { return make_float2(a.x * float(s), a.y * float(s)); }
};
template <>
struct Cx<double2> {
  using R = double;
  __device__ static double2 mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __device__ static double2 tw(int k, int span) {
    double s, c;
    sincospi(-2.0 * double(k) / double(span), &s, &c);
    return make_double2(c, s);
  }
  __device__ static double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
  __device__ static double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
  __device__ static double2 scl(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
};

__device__ __forceinline__ int bitrev(int x, int bits) { return int(__brev(unsigned(x)) >> (32 - bits)); }

// In-place radix-2 DIT FFT of buf (bit-reversed input) in shared memory.
template <typename C>
__device__ void fft_smem(C* buf, int n, int bits) {
  for (int span = 2; span <= n; span <<= 1) {
    const int half = span >> 1;
    for (int b = threadIdx.x; b < (n >> 1); b += blockDim.x) {
      const int grp = b / half, k = b % half;
      const int i0 = grp * span + k, i1 = i0 + half;
      const C w = Cx<C>::tw(k, span);
      const C t = Cx<C>::mul(buf[i1], w);
      const C u = buf[i0];
      buf[i0] = Cx<C>::add(u, t);
      buf[i1] = Cx<C>::sub(u, t);
    }
    __syncthreads();
  }
}

template <typename C>
__global__ void srft_kernel(int64_t m, int n, int bits, int ell, const C* A,
                            int64_t lda, const C* __restrict__ d, const int32_t* __restrict__ picks,
                            double scale, C* Y, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const double s = scale * rsqrt(double(n));
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    const C* a = A + row * lda;
    for (int k = threadIdx.x; k < n; k += blockDim.x)
      buf[bitrev(k, bits)] = d ? Cx<C>::mul(a[k], d[k]) : a[k];
    __syncthreads();
    fft_smem(buf, n, bits);
    for (int t = threadIdx.x; t < ell; t += blockDim.x) {
      const int p = picks ? picks[t] : t;
      Y[row * ldy + t] = Cx<C>::scl(buf[p], s);
    }
    __syncthreads();
  }
}

template <typename C>
void launch_srft(Handle* h, int64_t m, int64_t n, int64_t ell, const C* A, int64_t lda,
                 const C* d, const int32_t* picks, double scale, C* Y, int64_t ldy) {
  const size_t smem = size_t(n) * sizeof(C);
  int max_smem = 0;
  LR_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  LR_REQUIRE(smem <= size_t(max_smem), LR_EUNSUPPORTED,
             "srft: row length exceeds the shared-memory FFT size");
  int bits = 0;
  while ((int64_t(1) << bits) < n) ++bits;
  auto kern = srft_kernel<C>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int blocks = int(std::min<int64_t>(m, int64_t(h->sm_count) * 8));
  if (blocks == 0) return;
  kern<<<blocks, 512, smem, h->stream>>>(m, int(n), bits, int(ell), A, lda, d, picks, scale, Y,
                                         ldy);
  LR_CHECK_LAUNCH();
}

}  // namespace

namespace {

// The SRFT restricted to its ell picked bins is the n x ell matrix
//   X[k, t] = scale n^{-1/2} d_k exp(-2 pi i k picks_t / n),
// so Y = A X is one more pass over A -- for ANY n (the FFT kernel needs a
// power of two; the reference uses Bluestein there, sketch.py:155-176, which
// is the same linear map).  Entries in fp64 from the exact residue
// (k picks_t) mod n.  d == nullptr: d = 1; picks == nullptr: picks_t = t.
template <typename C>
__global__ void srft_matrix_kernel(int64_t n, int64_t ell, const C* __restrict__ d,
                                   const int32_t* __restrict__ picks, double scale,
                                   C* __restrict__ X) {
  const double sn = scale / sqrt(double(n));
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * ell;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = e / ell, t = e - k * ell;
    const int64_t p = picks ? int64_t(picks[t]) : t;
    const int64_t r = (k * p) % n;
    double sv, cv;
    sincospi(-2.0 * double(r) / double(n), &sv, &cv);
    const double dr = d ? double(d[k].x) : 1.0, di = d ? double(d[k].y) : 0.0;
    using R = decltype(X[0].x);
    X[e] = C{R(sn * (dr * cv - di * sv)), R(sn * (dr * sv + di * cv))};
  }
}

// Y (m x ell) = A (m x n) X with X the picked, D-scaled DFT columns.
template <typename C>
void srft_gemm(Handle* h, int64_t m, int64_t n, int64_t ell, const C* A, int64_t lda,
               const C* d, const int32_t* picks, double scale, C* Y, int64_t ldy,
               double a_amax) {
  C* X = pool_alloc_t<C>(h, size_t(n) * ell);
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n * ell, 256), 8192)));
  srft_matrix_kernel<C><<<blocks, 256, 0, h->stream>>>(n, ell, d, picks, scale, X);
  LR_CHECK_LAUNCH();
  if constexpr (sizeof(C) == 8)
    gemm_c64_hint(h, false, false, m, ell, n, A, lda, a_amax, X, ell, Y, ldy);
  else
    gemm_c128(h, false, false, m, ell, n, A, lda, X, ell, Y, ldy);
}

bool pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

// ---- Givens-chain SRFT (reference sketch.py:221-337) -----------------------
// Omega = D'' Theta' D' Theta D F R with Theta = P G_0 ... G_{n-2} acting on
// row vectors (x -> x P: x[:, perm]; G_i rotates columns (i, i+1) by
// [[c, s], [-s, c]]).  Its ell picked columns are built right to left on the
// device -- X = D F_R, then X <- G_0 ... G_{n-2} X, X <- P X, X <- D' X, ... --
// after which Y = A X is one pass over A.

// X <- G_0 G_1 ... G_{n-2} X (G_{n-2} applied first): one thread per column,
// the carried row i is the only state between consecutive rotations.
__global__ void givens_rows_kernel(int64_t n, int64_t ell, const double* __restrict__ thetas,
                                   double2* __restrict__ X) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= ell || n < 2) return;
  double2 hi = X[(n - 1) * ell + t];              // row i+1, updated in place
  for (int64_t i = n - 2; i >= 0; --i) {
    const double2 lo = X[i * ell + t];
    double sv, cv;
    sincos(thetas[i], &sv, &cv);
    // (G_i X)[i] = c x_i + s x_{i+1};  (G_i X)[i+1] = -s x_i + c x_{i+1}
    const double2 ni = make_double2(cv * lo.x + sv * hi.x, cv * lo.y + sv * hi.y);
    const double2 nh = make_double2(-sv * lo.x + cv * hi.x, -sv * lo.y + cv * hi.y);
    X[(i + 1) * ell + t] = nh;
    hi = ni;
  }
  X[t] = hi;
}

// Y[perm[j], :] = d[perm[j]] * X[j, :]   (P X, then the diagonal D)
__global__ void permute_scale_rows(int64_t n, int64_t ell, const int32_t* __restrict__ perm,
                                   const double2* __restrict__ d, const double2* __restrict__ X,
                                   double2* __restrict__ Y) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * ell;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / ell, t = e - j * ell;
    const int64_t r = perm[j];
    const double2 x = X[e], w = d[r];
    Y[r * ell + t] = make_double2(w.x * x.x - w.y * x.y, w.x * x.y + w.y * x.x);
  }
}

__global__ void to_c64(int64_t count, const double2* __restrict__ X, float2* __restrict__ Y) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count;
       e += int64_t(gridDim.x) * blockDim.x)
    Y[e] = make_float2(float(X[e].x), float(X[e].y));
}

}  // namespace

void gsrft_matrix(Handle* h, int dtype, int64_t n, int64_t ell, const double2* d_outer,
                  const int32_t* perm_outer, const double* thetas_outer, const double2* d_mid,
                  const int32_t* perm_inner, const double* thetas_inner, const double2* d_inner,
                  const int32_t* picks, double scale, void* Xout) {
  const size_t cnt = size_t(n) * ell;
  double2* X = pool_alloc_t<double2>(h, cnt);
  double2* T = pool_alloc_t<double2>(h, cnt);
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(int64_t(cnt), 256), 8192)));
  const int cb = int(ceil_div(ell, 128));
  srft_matrix_kernel<double2><<<blocks, 256, 0, h->stream>>>(n, ell, d_inner, picks, scale, X);
  LR_CHECK_LAUNCH();
  givens_rows_kernel<<<cb, 128, 0, h->stream>>>(n, ell, thetas_inner, X);
  LR_CHECK_LAUNCH();
  permute_scale_rows<<<blocks, 256, 0, h->stream>>>(n, ell, perm_inner, d_mid, X, T);
  LR_CHECK_LAUNCH();
  givens_rows_kernel<<<cb, 128, 0, h->stream>>>(n, ell, thetas_outer, T);
  LR_CHECK_LAUNCH();
  double2* out = dtype == LR_C128 ? static_cast<double2*>(Xout) : X;
  permute_scale_rows<<<blocks, 256, 0, h->stream>>>(n, ell, perm_outer, d_outer, T, out);
  LR_CHECK_LAUNCH();
  if (dtype == LR_C64) {
    to_c64<<<blocks, 256, 0, h->stream>>>(int64_t(cnt), X, static_cast<float2*>(Xout));
    LR_CHECK_LAUNCH();
  }
}

// complex64 SRFT: for ell <= 128 as a pass over A on the tcgen05 tensor
// cores (Y = A X with the picked DFT columns, three-product split, the same
// kernel as the Gaussian passes: ~0.15 ms for config 3 against ~1.7 ms for the
// shared-memory FFT of all n bins, of which ell/n are kept); larger ell or
// LR_SRFT=fft use the radix-2 FFT kernel, non-power-of-two n always the GEMM.
// a_amax < 0: unknown (computed).
void srft_c64(Handle* h, int64_t m, int64_t n, int64_t ell, const float2* A, int64_t lda,
              const float2* d, const int32_t* picks, float scale, float2* Y, int64_t ldy,
              double a_amax) {
  static int fft_only = -1;
  if (fft_only < 0) {
    const char* e = getenv("LR_SRFT");
    fft_only = (e && e[0] == 'f') ? 1 : 0;
  }
  if (!pow2(n) ||
      (!fft_only && ell <= 128 && h->f32_mode == LR_F32_SPLIT3 && m >= 1024)) {
    srft_gemm<float2>(h, m, n, ell, A, lda, d, picks, double(scale), Y, ldy, a_amax);
    return;
  }
  launch_srft<float2>(h, m, n, ell, A, lda, d, picks, double(scale), Y, ldy);
}

void srft_c128(Handle* h, int64_t m, int64_t n, int64_t ell, const double2* A, int64_t lda,
               const double2* d, const int32_t* picks, double scale, double2* Y, int64_t ldy) {
  if (!pow2(n)) {
    srft_gemm<double2>(h, m, n, ell, A, lda, d, picks, scale, Y, ldy, -1.0);
    return;
  }
  launch_srft<double2>(h, m, n, ell, A, lda, d, picks, scale, Y, ldy);
}

void dft_rows(Handle* h, int dtype, int64_t rows, int64_t n, void* X, int64_t ldx) {
  // unitary DFT of every row, in place: picks = identity, d = 1, scale = 1
  if (!pow2(n)) {   // dense DFT matrix product (any n), through a scratch copy
    const size_t es = dtype == LR_C64 ? sizeof(float2) : sizeof(double2);
    void* T = pool_alloc(h, size_t(rows) * n * es);
    if (dtype == LR_C64)
      srft_gemm<float2>(h, rows, n, n, static_cast<const float2*>(X), ldx, nullptr, nullptr, 1.0,
                        static_cast<float2*>(T), n, -1.0);
    else
      srft_gemm<double2>(h, rows, n, n, static_cast<const double2*>(X), ldx, nullptr, nullptr,
                         1.0, static_cast<double2*>(T), n, -1.0);
    LR_CUDA(cudaMemcpy2DAsync(X, ldx * es, T, n * es, n * es, rows, cudaMemcpyDeviceToDevice,
                              h->stream));
    return;
  }
  if (dtype == LR_C64)
    launch_srft<float2>(h, rows, n, n, static_cast<const float2*>(X), ldx, nullptr, nullptr, 1.0,
                        static_cast<float2*>(X), ldx);
  else
    launch_srft<double2>(h, rows, n, n, static_cast<const double2*>(X), ldx, nullptr, nullptr,
                         1.0, static_cast<double2*>(X), ldx);
}

}  // namespace lr
