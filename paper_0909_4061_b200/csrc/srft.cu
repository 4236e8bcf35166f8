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

// ---- radix-16 Stockham FFT (default for power-of-two n) ----------------------
// The radix-2 kernel above makes log2(n) passes through shared memory with a
// barrier each and computes every twiddle with sincospi (config 3: ~1.7 ms,
// ~5 % of the HBM bound).  Here each thread keeps 16 points in registers:
// n = 16^p * r is transformed in p radix-16 passes plus one radix-r pass
// (8192 = 16^3 * 2: 4 passes, 4 barriers), twiddles come from a table
// W[k] = exp(-2 pi i k / n) built once per n (L1-resident), and the pass
// structure is Stockham's autosort (natural-order output, no bit reversal):
//   pass (R, Ns): for j < n/R: v_r = x[j + r n/R] * W^{(j mod Ns) r n/(Ns R)},
//                 v = DFT_R(v), x'[(j/Ns) Ns R + j mod Ns + r Ns] = v_r.
// The first pass reads the row of A straight from HBM (coalesced) times d;
// the last writes its result to shared memory, from which the ell picked bins
// are gathered.  Shared memory is padded one element in 16 (stride-16
// stores of the first pass would otherwise hit one bank).

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) { return Cx<C>::mul(a, b); }
template <typename C>
__device__ __forceinline__ C cadd(C a, C b) { return Cx<C>::add(a, b); }
template <typename C>
__device__ __forceinline__ C csub(C a, C b) { return Cx<C>::sub(a, b); }
// a * (-i)
template <typename C>
__device__ __forceinline__ C mul_mi(C a) { C r; r.x = a.y; r.y = -a.x; return r; }

template <typename C>
__device__ __forceinline__ void dft2(C& a, C& b) {
  const C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
// in-place 4-point DFT (W4 = -i): natural order in and out
template <typename C>
__device__ __forceinline__ void dft4(C& x0, C& x1, C& x2, C& x3) {
  const C s02 = cadd(x0, x2), d02 = csub(x0, x2);
  const C s13 = cadd(x1, x3), d13 = mul_mi(csub(x1, x3));
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, d13);
  x3 = csub(d02, d13);
}

template <typename C>
__device__ __forceinline__ C w16(int m) {   // exp(-2 pi i m / 16)
  using R = typename Cx<C>::R;
  constexpr double c16[16] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
                              0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
                              -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977,
                              0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674};
  C w;
  w.x = R(c16[m & 15]);
  w.y = R(-c16[(m + 12) & 15]);   // -sin(2 pi m / 16) = -cos(2 pi (m - 4) / 16)
  return w;
}

// DFT of size R in registers, natural order in and out (R = 2, 4, 8, 16)
template <typename C, int R>
__device__ __forceinline__ void dft_reg(C (&v)[R]) {
  if constexpr (R == 2) {
    dft2(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    // 8 = 2 x 4: columns n2 = 0, 1 of x[2 n1 + n2]
    C a[4] = {v[0], v[2], v[4], v[6]}, b[4] = {v[1], v[3], v[5], v[7]};
    dft4(a[0], a[1], a[2], a[3]);
    dft4(b[0], b[1], b[2], b[3]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      const C t = cmul(b[k1], w16<C>(2 * k1));     // W8^k1
      v[k1] = cadd(a[k1], t);
      v[k1 + 4] = csub(a[k1], t);
    }
  } else {
    // 16 = 4 x 4: X[k1 + 4 k2] = sum_n2 W16^(n2 k1) W4^(n2 k2) DFT4_n1(x[4 n1 + n2])[k1]
    C a[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      a[n2][0] = v[n2];
      a[n2][1] = v[4 + n2];
      a[n2][2] = v[8 + n2];
      a[n2][3] = v[12 + n2];
      dft4(a[n2][0], a[n2][1], a[n2][2], a[n2][3]);
#pragma unroll
      for (int k1 = 1; k1 < 4; ++k1)
        if (n2) a[n2][k1] = cmul(a[n2][k1], w16<C>(n2 * k1));
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      C b0 = a[0][k1], b1 = a[1][k1], b2 = a[2][k1], b3 = a[3][k1];
      dft4(b0, b1, b2, b3);
      v[k1] = b0;
      v[k1 + 4] = b1;
      v[k1 + 8] = b2;
      v[k1 + 12] = b3;
    }
  }
}

// one Stockham pass of radix R over the padded shared-memory row; each of the
// n/16 threads owns 16/R butterfly groups (16 registers).  FIRST: inputs from
// the global row a times d.  Ns = 2^ls; the twiddles W^(jm r), r = 1..R-1, are
// powers of one table entry (one table read per group; the error of the
// 15-fold product is ~15 ulp of the working precision).
template <typename C, int R, bool FIRST>
__device__ __forceinline__ void stockham_pass(C* buf, int n, int ls, const C* __restrict__ tw,
                                              const C* a, const C* __restrict__ d) {
  constexpr int G = 16 / R;
  constexpr int LR = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
  const int nr = n / R;
  const int Ns = 1 << ls;
  C v[G][R];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = threadIdx.x + g * blockDim.x;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int idx = j + r * nr;
      if constexpr (FIRST) v[g][r] = d ? cmul(__ldg(a + idx), __ldg(d + idx)) : __ldg(a + idx);
      else                 v[g][r] = buf[pad16(idx)];
    }
    if (ls > 0) {
      const int jm = j & (Ns - 1);
      // W_{Ns R}^jm = W_n^(jm n / (Ns R)); n / (Ns R) = n >> (ls + LR)
      const C w = tw[jm * (n >> (ls + LR))];
      C wr = w;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        v[g][r] = cmul(v[g][r], wr);
        if (r + 1 < R) wr = cmul(wr, w);
      }
    }
    dft_reg<C, R>(v[g]);
  }
  __syncthreads();   // every load of this pass precedes the stores (in place)
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = threadIdx.x + g * blockDim.x;
    const int jm = j & (Ns - 1);
    const int base = ((j >> ls) << (ls + LR)) + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pad16(base + (r << ls))] = v[g][r];
  }
  __syncthreads();
}

template <typename C>
__global__ void __launch_bounds__(sizeof(C) == 8 ? 1024 : 512) srft16_kernel(int64_t m, int n, int p16, int rlast,
                                                      int ell, const C* A, int64_t lda,
                                                      const C* __restrict__ d,
                                                      const int32_t* __restrict__ picks,
                                                      const C* __restrict__ tw, double scale,
                                                      C* Y, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const double s = scale * rsqrt(double(n));
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    const C* a = A + row * lda;
    int ls = 0;
    for (int q = 0; q < p16; ++q, ls += 4) {
      if (q == 0) stockham_pass<C, 16, true>(buf, n, ls, tw, a, d);
      else        stockham_pass<C, 16, false>(buf, n, ls, tw, a, d);
    }
    const bool first = p16 == 0;
    switch (rlast) {
      case 2: first ? stockham_pass<C, 2, true>(buf, n, ls, tw, a, d)
                    : stockham_pass<C, 2, false>(buf, n, ls, tw, a, d); break;
      case 4: first ? stockham_pass<C, 4, true>(buf, n, ls, tw, a, d)
                    : stockham_pass<C, 4, false>(buf, n, ls, tw, a, d); break;
      case 8: first ? stockham_pass<C, 8, true>(buf, n, ls, tw, a, d)
                    : stockham_pass<C, 8, false>(buf, n, ls, tw, a, d); break;
      default: break;
    }
    for (int t = threadIdx.x; t < ell; t += blockDim.x) {
      const int pk = picks ? picks[t] : t;
      Y[row * ldy + t] = Cx<C>::scl(buf[pad16(pk)], s);
    }
    __syncthreads();
  }
}

template <typename C>
__global__ void twiddle_table_kernel(int n, C* __restrict__ tw) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double sv, cv;
    sincospi(-2.0 * double(k) / double(n), &sv, &cv);
    using R = typename Cx<C>::R;
    C w;
    w.x = R(cv);
    w.y = R(sv);
    tw[k] = w;
  }
}

bool srft16_ok(int64_t n, size_t elem) {
  if (n < 256 || (n & (n - 1)) != 0 || n / 16 > (elem == 8 ? 1024 : 512)) return false;
  return size_t(n + n / 16) * elem <= 200 * 1024;
}

template <typename C>
void launch_srft16(Handle* h, int64_t m, int64_t n, int64_t ell, const C* A, int64_t lda,
                   const C* d, const int32_t* picks, double scale, C* Y, int64_t ldy) {
  int bits = 0;
  while ((int64_t(1) << bits) < n) ++bits;
  const int p16 = bits / 4, rlast = 1 << (bits % 4);
  C* tw = pool_alloc_t<C>(h, size_t(n));
  twiddle_table_kernel<C><<<int(ceil_div(n, 256)), 256, 0, h->stream>>>(int(n), tw);
  LR_CHECK_LAUNCH();
  const size_t smem = size_t(n + n / 16) * sizeof(C);
  auto kern = srft16_kernel<C>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int threads = int(n / 16);
  int per_sm = 1;
  LR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  const int blocks = int(std::min<int64_t>(m, int64_t(h->sm_count) * std::max(per_sm, 1)));
  if (blocks == 0) return;
  kern<<<blocks, threads, smem, h->stream>>>(m, int(n), p16, rlast == 1 ? 0 : rlast, int(ell), A,
                                             lda, d, picks, tw, scale, Y, ldy);
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
  // LR_SRFT=gemm: the dense picked-DFT-columns pass on the tensor cores
  // (O(m n ell)); LR_SRFT=radix2: the radix-2 kernel; default radix-16 FFT
  const char* e = getenv("LR_SRFT");
  const bool gemm_mode = e && e[0] == 'g';
  const bool r2_mode = e && e[0] == 'r';
  if (!pow2(n) || (gemm_mode && ell <= 128 && h->f32_mode == LR_F32_SPLIT3 && m >= 1024)) {
    srft_gemm<float2>(h, m, n, ell, A, lda, d, picks, double(scale), Y, ldy, a_amax);
    return;
  }
  if (!r2_mode && srft16_ok(n, sizeof(float2))) {
    launch_srft16<float2>(h, m, n, ell, A, lda, d, picks, double(scale), Y, ldy);
    return;
  }
  if (size_t(n) * sizeof(float2) > 200 * 1024) {   // row too long for shared memory
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
  const char* e = getenv("LR_SRFT");
  if (!(e && e[0] == 'r') && srft16_ok(n, sizeof(double2))) {
    launch_srft16<double2>(h, m, n, ell, A, lda, d, picks, scale, Y, ldy);
    return;
  }
  if (size_t(n) * sizeof(double2) > 200 * 1024) {   // row too long for shared memory
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
  const char* e = getenv("LR_SRFT");
  const bool r2 = e && e[0] == 'r';
  if (dtype == LR_C64) {
    if (!r2 && srft16_ok(n, sizeof(float2)))
      launch_srft16<float2>(h, rows, n, n, static_cast<const float2*>(X), ldx, nullptr, nullptr,
                            1.0, static_cast<float2*>(X), ldx);
    else
      launch_srft<float2>(h, rows, n, n, static_cast<const float2*>(X), ldx, nullptr, nullptr, 1.0,
                          static_cast<float2*>(X), ldx);
  } else {
    if (!r2 && srft16_ok(n, sizeof(double2)))
      launch_srft16<double2>(h, rows, n, n, static_cast<const double2*>(X), ldx, nullptr, nullptr,
                             1.0, static_cast<double2*>(X), ldx);
    else
      launch_srft<double2>(h, rows, n, n, static_cast<const double2*>(X), ldx, nullptr, nullptr,
                           1.0, static_cast<double2*>(X), ldx);
  }
}

}  // namespace lr
