// Small HBM-bound helper kernels: estimator tail, input validation,
// casts/adjoints, triangular products.
#include <type_traits>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

template <typename T>
__device__ __forceinline__ double abs2_any(T v);
template <>
__device__ __forceinline__ double abs2_any<float>(float v) { return double(v) * double(v); }
template <>
__device__ __forceinline__ double abs2_any<double>(double v) { return v * v; }
template <>
__device__ __forceinline__ double abs2_any<float2>(float2 v) {
  return double(v.x) * double(v.x) + double(v.y) * double(v.y);
}
template <>
__device__ __forceinline__ double abs2_any<double2>(double2 v) { return v.x * v.x + v.y * v.y; }

// Column sums of squares, stage 1: block b reduces rows [b*rows_per, ...)
// into part[b][j] (deterministic two-level reduction, no atomics).
template <typename T>
__global__ void colsq_stage1(int64_t m, int r, const T* __restrict__ Z, int64_t ldz,
                             int64_t rows_per, double* __restrict__ part) {
  extern __shared__ double sh[];   // blockDim.y x r
  const int64_t r0 = int64_t(blockIdx.x) * rows_per;
  const int64_t r1 = min(m, r0 + rows_per);
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double acc = 0.0;
    for (int64_t i = r0 + threadIdx.y; i < r1; i += blockDim.y) acc += abs2_any(Z[i * ldz + j]);
    sh[threadIdx.y * r + j] = acc;
  }
  __syncthreads();
  if (threadIdx.y == 0) {
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
      double acc = 0.0;
      for (int y = 0; y < int(blockDim.y); ++y) acc += sh[y * r + j];
      part[int64_t(blockIdx.x) * r + j] = acc;
    }
  }
}

__global__ void colsq_stage2(int nb, int r, const double* __restrict__ part,
                             double* __restrict__ out) {
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += part[int64_t(b) * r + j];
    out[j] = acc;
  }
}

__global__ void estimate_finish_kernel(int r, const double* __restrict__ sumsq, double alpha,
                                       double* __restrict__ est) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double mx = 0.0;
    for (int j = 0; j < r; ++j) mx = fmax(mx, sumsq[j]);
    // alpha * sqrt(2/pi) * max_i ||z_i||  (reference rangefinder.py:82)
    est[0] = alpha * sqrt(2.0 / 3.14159265358979323846) * sqrt(mx);
  }
}

template <typename T>
__device__ __forceinline__ bool isfin(T v);
template <>
__device__ __forceinline__ bool isfin<float>(float v) { return isfinite(v); }
template <>
__device__ __forceinline__ bool isfin<double>(double v) { return isfinite(v); }
template <>
__device__ __forceinline__ bool isfin<float2>(float2 v) { return isfinite(v.x) && isfinite(v.y); }
template <>
__device__ __forceinline__ bool isfin<double2>(double2 v) { return isfinite(v.x) && isfinite(v.y); }

template <typename T>
__device__ __forceinline__ double absmax_part(T v);
template <>
__device__ __forceinline__ double absmax_part<float>(float v) { return fabs(double(v)); }
template <>
__device__ __forceinline__ double absmax_part<double>(double v) { return fabs(v); }
template <>
__device__ __forceinline__ double absmax_part<float2>(float2 v) {
  return fmax(fabs(double(v.x)), fabs(double(v.y)));
}
template <>
__device__ __forceinline__ double absmax_part<double2>(double2 v) {
  return fmax(fabs(v.x), fabs(v.y));
}

// as_matrix validation (reference core.py:44-49) + max |a| (real/imag parts)
template <typename T>
__global__ void check_finite_kernel(int64_t m, int64_t n, const T* __restrict__ A, int64_t lda,
                                    unsigned long long* __restrict__ bad,
                                    unsigned long long* __restrict__ amax_bits) {
  unsigned long long nb = 0;
  double mx = 0.0;
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const T v = A[(e / n) * lda + (e % n)];
    if (!isfin(v)) ++nb;
    else mx = fmax(mx, absmax_part(v));
  }
  for (int o = 16; o > 0; o >>= 1) {
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (nb) atomicAdd(bad, nb);
    // non-negative doubles order like their bit patterns
    atomicMax(amax_bits, static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
}

__global__ void finish_check(const unsigned long long* bad, const unsigned long long* bits,
                             int64_t* nonfinite, double* amax) {
  nonfinite[0] = int64_t(bad[0]);
  amax[0] = __longlong_as_double(static_cast<long long>(bits[0]));
}

template <typename TS, typename TD>
__device__ __forceinline__ TD conv(TS v, bool cj);
template <> __device__ __forceinline__ double conv<float, double>(float v, bool) { return double(v); }
template <> __device__ __forceinline__ float conv<double, float>(double v, bool) { return float(v); }
template <> __device__ __forceinline__ double conv<double, double>(double v, bool) { return v; }
template <> __device__ __forceinline__ float conv<float, float>(float v, bool) { return v; }
template <> __device__ __forceinline__ double2 conv<float2, double2>(float2 v, bool cj) {
  return make_double2(v.x, cj ? -double(v.y) : double(v.y));
}
template <> __device__ __forceinline__ float2 conv<double2, float2>(double2 v, bool cj) {
  return make_float2(float(v.x), float(cj ? -v.y : v.y));
}
template <> __device__ __forceinline__ double2 conv<double2, double2>(double2 v, bool cj) {
  return make_double2(v.x, cj ? -v.y : v.y);
}
template <> __device__ __forceinline__ float2 conv<float2, float2>(float2 v, bool cj) {
  return make_float2(v.x, cj ? -v.y : v.y);
}

template <> __device__ __forceinline__ double2 conv<double, double2>(double v, bool) {
  return make_double2(v, 0.0);
}
template <> __device__ __forceinline__ float2 conv<float, float2>(float v, bool) {
  return make_float2(v, 0.f);
}
template <> __device__ __forceinline__ double2 conv<float, double2>(float v, bool) {
  return make_double2(double(v), 0.0);
}

// dst (rows x cols) = src, or dst = src^H when ct (src is cols x rows)
template <typename TS, typename TD>
__global__ void cast_copy_kernel(int64_t rows, int64_t cols, const TS* __restrict__ src,
                                 int64_t lds, TD* __restrict__ dst, int64_t ldd, bool ct) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    const TS v = ct ? src[j * lds + i] : src[i * lds + j];
    dst[i * ldd + j] = conv<TS, TD>(v, ct);
  }
}

// R = R2 . R1 for upper-triangular n x n (row-major, dense storage)
template <typename T>
__global__ void trmm_upper_kernel(int n, const T* __restrict__ R2, const T* __restrict__ R1,
                                  T* __restrict__ R) {
  using S = Sc<T>;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e / n, j = e % n;
    T acc = S::zero();
    for (int k = i; k <= j; ++k) acc = S::add(acc, S::mul(R2[i * n + k], R1[k * n + j]));
    R[e] = (j >= i) ? acc : S::zero();
  }
}

template <typename T>
__global__ void axpy_sub_kernel(int64_t rows, int64_t cols, const T* __restrict__ Tm, int64_t ldt,
                                T* __restrict__ Z, int64_t ldz) {
  using S = Sc<T>;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    Z[i * ldz + j] = S::sub(Z[i * ldz + j], Tm[i * ldt + j]);
  }
}
template <>
__global__ void axpy_sub_kernel<float>(int64_t rows, int64_t cols, const float* __restrict__ Tm,
                                       int64_t ldt, float* __restrict__ Z, int64_t ldz) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    Z[i * ldz + j] -= Tm[i * ldt + j];
  }
}
template <>
__global__ void axpy_sub_kernel<float2>(int64_t rows, int64_t cols, const float2* __restrict__ Tm,
                                        int64_t ldt, float2* __restrict__ Z, int64_t ldz) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    float2 z = Z[i * ldz + j];
    const float2 t = Tm[i * ldt + j];
    z.x -= t.x;
    z.y -= t.y;
    Z[i * ldz + j] = z;
  }
}

template <typename T>
__global__ void scale_col_kernel(int64_t rows, const T* __restrict__ src, int64_t lds, double inv,
                                 T* __restrict__ dst, int64_t ldd) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T v = src[i * lds];
    T o;
    if constexpr (sizeof(T) == 4) o = T(double(v) * inv);
    else if constexpr (sizeof(T) == 8 && std::is_same<T, double>::value) o = v * inv;
    else if constexpr (std::is_same<T, float2>::value) o = make_float2(float(v.x * inv), float(v.y * inv));
    else o = make_double2(v.x * inv, v.y * inv);
    dst[i * ldd] = o;
  }
}

template <typename T>
void launch_colsq(Handle* h, int64_t m, int64_t r, const T* Z, int64_t ldz, double* out) {
  const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(h->sm_count * 2, ceil_div(m, 256)));
  const int64_t rows_per = ceil_div(m, nb);
  double* part = pool_alloc_t<double>(h, size_t(nb) * r);
  dim3 blk(32, 8);
  const size_t sh = size_t(8) * r * sizeof(double);
  LR_REQUIRE(sh <= 48 * 1024, LR_EINVAL, "col_sumsq: too many columns");
  colsq_stage1<T><<<unsigned(nb), blk, sh, h->stream>>>(m, int(r), Z, ldz, rows_per, part);
  LR_CHECK_LAUNCH();
  colsq_stage2<<<1, 256, 0, h->stream>>>(int(nb), int(r), part, out);
  LR_CHECK_LAUNCH();
}

template <typename TS, typename TD>
void launch_cast(Handle* h, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                 int64_t cols, bool ct) {
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * cols, 256),
                                                                int64_t(h->sm_count) * 16)));
  cast_copy_kernel<TS, TD><<<blocks, 256, 0, h->stream>>>(
      rows, cols, static_cast<const TS*>(src), lds, static_cast<TD*>(dst), ldd, ct);
  LR_CHECK_LAUNCH();
}

}  // namespace

void col_sumsq(Handle* h, int dtype, int64_t m, int64_t r, const void* Z, int64_t ldz,
               double* out) {
  switch (dtype) {
    case LR_F32: launch_colsq(h, m, r, static_cast<const float*>(Z), ldz, out); break;
    case LR_F64: launch_colsq(h, m, r, static_cast<const double*>(Z), ldz, out); break;
    case LR_C64: launch_colsq(h, m, r, static_cast<const float2*>(Z), ldz, out); break;
    case LR_C128: launch_colsq(h, m, r, static_cast<const double2*>(Z), ldz, out); break;
    default: throw Error{LR_EINVAL, "col_sumsq: bad dtype"};
  }
}

void estimate_finish(Handle* h, int64_t r, const double* sumsq, double alpha, double* est) {
  estimate_finish_kernel<<<1, 32, 0, h->stream>>>(int(r), sumsq, alpha, est);
  LR_CHECK_LAUNCH();
}

void check_finite(Handle* h, int dtype, int64_t m, int64_t n, const void* A, int64_t lda,
                  int64_t* nonfinite, double* amax) {
  unsigned long long* buf = pool_alloc_t<unsigned long long>(h, 2);
  LR_CUDA(cudaMemsetAsync(buf, 0, 2 * sizeof(unsigned long long), h->stream));
  const int blocks = h->sm_count * 8;
  switch (dtype) {
    case LR_F32:
      check_finite_kernel<<<blocks, 256, 0, h->stream>>>(m, n, static_cast<const float*>(A), lda,
                                                         buf, buf + 1);
      break;
    case LR_F64:
      check_finite_kernel<<<blocks, 256, 0, h->stream>>>(m, n, static_cast<const double*>(A), lda,
                                                         buf, buf + 1);
      break;
    case LR_C64:
      check_finite_kernel<<<blocks, 256, 0, h->stream>>>(m, n, static_cast<const float2*>(A), lda,
                                                         buf, buf + 1);
      break;
    case LR_C128:
      check_finite_kernel<<<blocks, 256, 0, h->stream>>>(m, n, static_cast<const double2*>(A),
                                                         lda, buf, buf + 1);
      break;
    default: throw Error{LR_EINVAL, "check_finite: bad dtype"};
  }
  LR_CHECK_LAUNCH();
  finish_check<<<1, 1, 0, h->stream>>>(buf, buf + 1, nonfinite, amax);
  LR_CHECK_LAUNCH();
}

void cast_copy(Handle* h, int sd, const void* src, int64_t lds, int dd, void* dst, int64_t ldd,
               int64_t rows, int64_t cols, bool ct) {
  if (rows == 0 || cols == 0) return;
  if (sd == LR_F32 && dd == LR_F64) return launch_cast<float, double>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_F64 && dd == LR_F32) return launch_cast<double, float>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_F64 && dd == LR_F64) return launch_cast<double, double>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_F32 && dd == LR_F32) return launch_cast<float, float>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_C64 && dd == LR_C128) return launch_cast<float2, double2>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_C128 && dd == LR_C64) return launch_cast<double2, float2>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_C128 && dd == LR_C128) return launch_cast<double2, double2>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_C64 && dd == LR_C64) return launch_cast<float2, float2>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_F64 && dd == LR_C128) return launch_cast<double, double2>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_F32 && dd == LR_C64) return launch_cast<float, float2>(h, src, lds, dst, ldd, rows, cols, ct);
  if (sd == LR_F32 && dd == LR_C128) return launch_cast<float, double2>(h, src, lds, dst, ldd, rows, cols, ct);
  throw Error{LR_EINVAL, "cast_copy: unsupported dtype pair"};
}

// Z (rows x cols) += T, fp64 / complex128 (row-block accumulation of the
// one-pass sketch, reference io.py:381 "Yt += block* Omega_t[rows]")
template <typename T>
__global__ void axpy_add_kernel(int64_t rows, int64_t cols, const T* __restrict__ Tm, int64_t ldt,
                                T* __restrict__ Z, int64_t ldz) {
  using S = Sc<T>;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    Z[i * ldz + j] = S::add(Z[i * ldz + j], Tm[i * ldt + j]);
  }
}

// C_ij <- C_ij / (d2_i + d1_j) (zero where the denominator is not positive
// beyond roundoff): the diagonalized Sylvester normal equations of the
// one-pass least-squares problem (see factor.svd_one_pass_general)
template <typename T>
__global__ void sylvester_div_kernel(int64_t k, int64_t kt, T* __restrict__ C, int64_t ldc,
                                     const double* __restrict__ d2, const double* __restrict__ d1,
                                     double floor) {
  using S = Sc<T>;
  const int64_t total = k * kt;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / kt, j = e % kt;
    const double den = d2[i] + d1[j];
    C[i * ldc + j] = den > floor ? S::scale(C[i * ldc + j], 1.0 / den) : S::zero();
  }
}

void axpy_add(Handle* h, int dtype, int64_t rows, int64_t cols, const void* Tm, int64_t ldt,
              void* Z, int64_t ldz) {
  if (rows == 0 || cols == 0) return;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * cols, 256),
                                                                int64_t(h->sm_count) * 16)));
  switch (dtype) {
    case LR_F64: axpy_add_kernel<double><<<blocks, 256, 0, h->stream>>>(rows, cols, static_cast<const double*>(Tm), ldt, static_cast<double*>(Z), ldz); break;
    case LR_C128: axpy_add_kernel<double2><<<blocks, 256, 0, h->stream>>>(rows, cols, static_cast<const double2*>(Tm), ldt, static_cast<double2*>(Z), ldz); break;
    default: throw Error{LR_EINVAL, "axpy_add: fp64 / complex128 only"};
  }
  LR_CHECK_LAUNCH();
}

void sylvester_div(Handle* h, int dtype, int64_t k, int64_t kt, void* C, int64_t ldc,
                   const double* d2, const double* d1, double floor) {
  if (k == 0 || kt == 0) return;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(k * kt, 256), 1024)));
  switch (dtype) {
    case LR_F64: sylvester_div_kernel<double><<<blocks, 256, 0, h->stream>>>(k, kt, static_cast<double*>(C), ldc, d2, d1, floor); break;
    case LR_C128: sylvester_div_kernel<double2><<<blocks, 256, 0, h->stream>>>(k, kt, static_cast<double2*>(C), ldc, d2, d1, floor); break;
    default: throw Error{LR_EINVAL, "sylvester_div: fp64 / complex128 only"};
  }
  LR_CHECK_LAUNCH();
}

void axpy_sub(Handle* h, int dtype, int64_t rows, int64_t cols, const void* Tm, int64_t ldt,
              void* Z, int64_t ldz) {
  if (rows == 0 || cols == 0) return;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * cols, 256),
                                                                int64_t(h->sm_count) * 16)));
  switch (dtype) {
    case LR_F32: axpy_sub_kernel<float><<<blocks, 256, 0, h->stream>>>(rows, cols, static_cast<const float*>(Tm), ldt, static_cast<float*>(Z), ldz); break;
    case LR_F64: axpy_sub_kernel<double><<<blocks, 256, 0, h->stream>>>(rows, cols, static_cast<const double*>(Tm), ldt, static_cast<double*>(Z), ldz); break;
    case LR_C64: axpy_sub_kernel<float2><<<blocks, 256, 0, h->stream>>>(rows, cols, static_cast<const float2*>(Tm), ldt, static_cast<float2*>(Z), ldz); break;
    case LR_C128: axpy_sub_kernel<double2><<<blocks, 256, 0, h->stream>>>(rows, cols, static_cast<const double2*>(Tm), ldt, static_cast<double2*>(Z), ldz); break;
    default: throw Error{LR_EINVAL, "axpy_sub: bad dtype"};
  }
  LR_CHECK_LAUNCH();
}

void scale_col(Handle* h, int dtype, int64_t rows, const void* src, int64_t lds, double inv,
               void* dst, int64_t ldd) {
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 256), 4096)));
  switch (dtype) {
    case LR_F32: scale_col_kernel<float><<<blocks, 256, 0, h->stream>>>(rows, static_cast<const float*>(src), lds, inv, static_cast<float*>(dst), ldd); break;
    case LR_F64: scale_col_kernel<double><<<blocks, 256, 0, h->stream>>>(rows, static_cast<const double*>(src), lds, inv, static_cast<double*>(dst), ldd); break;
    case LR_C64: scale_col_kernel<float2><<<blocks, 256, 0, h->stream>>>(rows, static_cast<const float2*>(src), lds, inv, static_cast<float2*>(dst), ldd); break;
    case LR_C128: scale_col_kernel<double2><<<blocks, 256, 0, h->stream>>>(rows, static_cast<const double2*>(src), lds, inv, static_cast<double2*>(dst), ldd); break;
    default: throw Error{LR_EINVAL, "scale_col: bad dtype"};
  }
  LR_CHECK_LAUNCH();
}

namespace {
template <typename T>
__device__ __forceinline__ double cabs_any(T v) { return sqrt(abs2_any(v)); }

template <typename T>
__device__ __forceinline__ T phase_conj_mul(T v, T ph);
template <> __device__ __forceinline__ float phase_conj_mul<float>(float v, float ph) { return v * ph; }
template <> __device__ __forceinline__ double phase_conj_mul<double>(double v, double ph) { return v * ph; }
template <> __device__ __forceinline__ float2 phase_conj_mul<float2>(float2 v, float2 p) {
  return make_float2(v.x * p.x - v.y * p.y, v.x * p.y + v.y * p.x);
}
template <> __device__ __forceinline__ double2 phase_conj_mul<double2>(double2 v, double2 p) {
  return make_double2(v.x * p.x - v.y * p.y, v.x * p.y + v.y * p.x);
}
template <typename T> __device__ __forceinline__ T make_ph(T z, double inv_abs);
template <> __device__ __forceinline__ float make_ph<float>(float z, double) { return z >= 0.f ? 1.f : -1.f; }
template <> __device__ __forceinline__ double make_ph<double>(double z, double) { return z >= 0.0 ? 1.0 : -1.0; }
template <> __device__ __forceinline__ float2 make_ph<float2>(float2 z, double ia) {
  return make_float2(float(z.x * ia), float(-z.y * ia));
}
template <> __device__ __forceinline__ double2 make_ph<double2>(double2 z, double ia) {
  return make_double2(z.x * ia, -z.y * ia);
}

// one warp per column (reference core.py:221-229)
template <typename T>
__global__ void sign_fix_kernel(int64_t rows, int64_t vrows, int64_t cols, T* U, int64_t ldu, T* V,
                                int64_t ldv) {
  const int lane = threadIdx.x & 31;
  const int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= cols) return;
  double mx = 0.0;
  for (int64_t i = lane; i < rows; i += 32) mx = fmax(mx, cabs_any(U[i * ldu + j]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int64_t first = -1;
  for (int64_t base = 0; base < rows && first < 0; base += 32) {
    const int64_t i = base + lane;
    const bool hit = i < rows && cabs_any(U[i * ldu + j]) > 1e-10 * mx;
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (b) first = base + __ffs(b) - 1;
  }
  if (first < 0) return;
  const T z = U[first * ldu + j];
  const T ph = make_ph(z, 1.0 / cabs_any(z));   // conj(z/|z|)
  for (int64_t i = lane; i < rows; i += 32) U[i * ldu + j] = phase_conj_mul(U[i * ldu + j], ph);
  for (int64_t i = lane; i < vrows; i += 32) V[i * ldv + j] = phase_conj_mul(V[i * ldv + j], ph);
}

template <typename T>
__global__ void max_imag_kernel(int64_t m, int64_t n, const T* __restrict__ Y, int64_t ldy,
                                unsigned long long* bits) {
  double mx = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * n;
       e += int64_t(gridDim.x) * blockDim.x)
    mx = fmax(mx, fabs(double(Y[(e / n) * ldy + (e % n)].y)));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(bits, static_cast<unsigned long long>(__double_as_longlong(mx)));
}

__global__ void bits_to_double(const unsigned long long* bits, double* out) {
  out[0] = __longlong_as_double(static_cast<long long>(bits[0]));
}
}  // namespace

void sign_fix(Handle* h, int dtype, int64_t rows, int64_t vrows, int64_t cols, void* U,
              int64_t ldu, void* V, int64_t ldv) {
  if (cols == 0) return;
  const int blocks = int(ceil_div(cols, 8));
  switch (dtype) {
    case LR_F32: sign_fix_kernel<float><<<blocks, 256, 0, h->stream>>>(rows, vrows, cols, static_cast<float*>(U), ldu, static_cast<float*>(V), ldv); break;
    case LR_F64: sign_fix_kernel<double><<<blocks, 256, 0, h->stream>>>(rows, vrows, cols, static_cast<double*>(U), ldu, static_cast<double*>(V), ldv); break;
    case LR_C64: sign_fix_kernel<float2><<<blocks, 256, 0, h->stream>>>(rows, vrows, cols, static_cast<float2*>(U), ldu, static_cast<float2*>(V), ldv); break;
    case LR_C128: sign_fix_kernel<double2><<<blocks, 256, 0, h->stream>>>(rows, vrows, cols, static_cast<double2*>(U), ldu, static_cast<double2*>(V), ldv); break;
    default: throw Error{LR_EINVAL, "sign_fix: bad dtype"};
  }
  LR_CHECK_LAUNCH();
}

void max_abs_imag(Handle* h, int dtype, int64_t m, int64_t n, const void* Y, int64_t ldy,
                  double* out) {
  unsigned long long* bits = pool_alloc_t<unsigned long long>(h, 1);
  LR_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long), h->stream));
  const int blocks = h->sm_count * 4;
  if (dtype == LR_C64)
    max_imag_kernel<float2><<<blocks, 256, 0, h->stream>>>(m, n, static_cast<const float2*>(Y), ldy, bits);
  else if (dtype == LR_C128)
    max_imag_kernel<double2><<<blocks, 256, 0, h->stream>>>(m, n, static_cast<const double2*>(Y), ldy, bits);
  else
    throw Error{LR_EINVAL, "max_abs_imag: complex dtypes only"};
  LR_CHECK_LAUNCH();
  bits_to_double<<<1, 1, 0, h->stream>>>(bits, out);
  LR_CHECK_LAUNCH();
}

namespace {
template <typename T>
__global__ void ns_coef_kernel(int n, T* G) {
  using S = Sc<T>;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e / n, j = e % n;
    T v = S::scale(G[e], -0.5);
    if (i == j) v = S::add(v, S::make(1.5, 0.0));
    G[e] = v;
  }
}
}  // namespace

void ns_coef(Handle* h, int dtype_wide, int64_t n, void* G) {
  const int blocks = int(std::max<int64_t>(1, ceil_div(n * n, 256)));
  if (dtype_wide == LR_C128)
    ns_coef_kernel<double2><<<blocks, 256, 0, h->stream>>>(int(n), static_cast<double2*>(G));
  else
    ns_coef_kernel<double><<<blocks, 256, 0, h->stream>>>(int(n), static_cast<double*>(G));
  LR_CHECK_LAUNCH();
}

void trmm_upper(Handle* h, int dtype, int64_t n, const void* R2, const void* R1, void* R) {
  const int blocks = int(std::max<int64_t>(1, ceil_div(n * n, 256)));
  if (dtype == LR_F64 || dtype == LR_F32) {
    trmm_upper_kernel<double><<<blocks, 256, 0, h->stream>>>(
        int(n), static_cast<const double*>(R2), static_cast<const double*>(R1),
        static_cast<double*>(R));
  } else {
    trmm_upper_kernel<double2><<<blocks, 256, 0, h->stream>>>(
        int(n), static_cast<const double2*>(R2), static_cast<const double2*>(R1),
        static_cast<double2*>(R));
  }
  LR_CHECK_LAUNCH();
}

}  // namespace lr
