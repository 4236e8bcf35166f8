// Real / complex scalar helpers shared by the small dense kernels.
#pragma once
#include <cuda_runtime.h>

namespace lr {

template <typename T>
struct Sc;

template <>
struct Sc<double> {
  using R = double;
  static constexpr bool cplx = false;
  __host__ __device__ static double zero() { return 0.0; }
  __host__ __device__ static double one() { return 1.0; }
  __host__ __device__ static double re(double a) { return a; }
  __host__ __device__ static double conj(double a) { return a; }
  __host__ __device__ static double mul(double a, double b) { return a * b; }
  __host__ __device__ static double cmul(double a, double b) { return a * b; }  // conj(a)*b
  __host__ __device__ static double add(double a, double b) { return a + b; }
  __host__ __device__ static double sub(double a, double b) { return a - b; }
  __host__ __device__ static double scale(double a, double s) { return a * s; }
  __host__ __device__ static double abs2(double a) { return a * a; }
  __host__ __device__ static double make(double r, double) { return r; }
  __device__ static double shfl_xor(double a, int m) { return __shfl_xor_sync(0xffffffffu, a, m); }
  __device__ static double shfl_idx(double a, int src) { return __shfl_sync(0xffffffffu, a, src); }
  __device__ static double div_re(double a, double r) { return a / r; }
};

template <>
struct Sc<double2> {
  using R = double;
  static constexpr bool cplx = true;
  __host__ __device__ static double2 zero() { return make_double2(0.0, 0.0); }
  __host__ __device__ static double2 one() { return make_double2(1.0, 0.0); }
  __host__ __device__ static double re(double2 a) { return a.x; }
  __host__ __device__ static double2 conj(double2 a) { return make_double2(a.x, -a.y); }
  __host__ __device__ static double2 mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __host__ __device__ static double2 cmul(double2 a, double2 b) {  // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
  }
  __host__ __device__ static double2 add(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
  }
  __host__ __device__ static double2 sub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
  }
  __host__ __device__ static double2 scale(double2 a, double s) {
    return make_double2(a.x * s, a.y * s);
  }
  __host__ __device__ static double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
  __host__ __device__ static double2 make(double r, double i) { return make_double2(r, i); }
  __device__ static double2 shfl_xor(double2 a, int m) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m));
  }
  __device__ static double2 shfl_idx(double2 a, int src) {
    return make_double2(__shfl_sync(0xffffffffu, a.x, src), __shfl_sync(0xffffffffu, a.y, src));
  }
  __device__ static double2 div_re(double2 a, double r) { return make_double2(a.x / r, a.y / r); }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = Sc<T>::add(v, Sc<T>::shfl_xor(v, m));
  return v;
}

}  // namespace lr
