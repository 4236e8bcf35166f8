// K4 (fast path): register-resident one-sided Jacobi for square n <= 128.
//
// The small SVD of direct_svd (reference core.py:199-230) factors the
// triangular R of B^H = Q2 R (CholeskyQR) as R J = M (orthogonal columns,
// M = W diag(S)).  This kernel keeps the columns of M in registers: each
// round-robin slot is a group of GS lanes holding two columns (EPL rows per
// lane), so the inner products and the rotation touch no memory; between
// rounds the columns rotate one slot through shared memory.  The rotation
// angles are computed once per pair by one lane each (not redundantly by
// every lane of every group), with the tangent formed in fp32 -- any angle
// gives an exactly orthogonal rotation (c = rsqrt(1 + t^2), s = c t in fp64),
// the angle accuracy only sets the convergence rate -- and the test
// |m_p^H m_q| <= tol sqrt(|m_p|^2 |m_q|^2) evaluated in fp64.
//
// The rotations are not accumulated: J = R^{-1} M is formed afterwards with
// one GEMM (R^{-1} is the product of the CholeskyQR passes' inverses) and
// re-orthonormalized by one CholeskyQR pass, which halves the per-round
// work and register footprint.  svd_finalize sorts, applies the reference
// sign convention (core.py:221-229) and normalizes W.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

template <typename T, int GS>
__device__ __forceinline__ T gsum(T v) {
#pragma unroll
  for (int m = GS >> 1; m > 0; m >>= 1) v = Sc<T>::add(v, Sc<T>::shfl_xor(v, m));
  return v;
}

__device__ __forceinline__ double ldsd(const double* p) { return *p; }

template <typename T, int GS, int EPL>
__global__ void __launch_bounds__(1024, 1)
jacobi_reg_kernel(int n, const T* __restrict__ R, T* __restrict__ Mout, double* __restrict__ sig,
                  int32_t* __restrict__ info, double tol, int max_sweeps, int32_t* status) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int np2 = n + (n & 1);
  const int pairs = np2 / 2;
  const int rows = n;
  // exchange buffer: two columns per slot (double buffered by role)
  T* xbuf = reinterpret_cast<T*>(smem_raw);                    // np2 * rows
  T* pg = xbuf + size_t(np2) * rows;                           // pairs: gamma, then s e
  double* pa = reinterpret_cast<double*>(pg + pairs);          // pairs
  double* pb = pa + pairs;                                     // pairs
  double* pc = pb + pairs;                                     // pairs: c (0 = none)
  int* cid = reinterpret_cast<int*>(pc + pairs);               // np2: column id per position

  __shared__ int s_rot[2];
  const int tid = threadIdx.x;
  const int g = tid / GS, gl = tid % GS;
  const bool active = g < pairs;

  // initial placement: slot g holds columns g (top) and np2-1-g (bot)
  int ctop = g, cbot = np2 - 1 - g;
  T xa[EPL], xb[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const int i = gl + GS * e;
    xa[e] = (active && i < rows && ctop < n) ? R[size_t(i) * n + ctop] : S::zero();
    xb[e] = (active && i < rows && cbot < n) ? R[size_t(i) * n + cbot] : S::zero();
  }
  if (tid == 0) { s_rot[0] = 0; s_rot[1] = 0; }
  __syncthreads();

  const int rounds = np2 - 1;
  int sweep = 0;
  bool converged = (n == 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    const int flag = sweep & 1;
    for (int r = 0; r < rounds; ++r) {
      // inner products in registers
      double a = 0.0, b = 0.0;
      T gm = S::zero();
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        a += S::abs2(xa[e]);
        b += S::abs2(xb[e]);
        gm = S::add(gm, S::cmul(xa[e], xb[e]));
      }
      a = gsum<double, GS>(a);
      b = gsum<double, GS>(b);
      gm = gsum<T, GS>(gm);
      const bool real_pair = active && ctop < n && cbot < n;
      if (active && gl == 0) {
        pa[g] = real_pair ? a : -1.0;
        pb[g] = b;
        pg[g] = gm;
      }
      __syncthreads();
      // rotation parameters: one lane per pair
      for (int k = tid; k < pairs; k += blockDim.x) {
        const double aa = pa[k], bb = pb[k];
        const T gg = pg[k];
        const double g2 = S::abs2(gg);
        double c = 0.0;
        T se = S::zero();
        if (aa >= 0.0 && g2 > 0.0 && g2 > tol * tol * aa * bb) {
          const double iag = rsqrt(g2);                        // 1/|gamma|
          const float zeta = float(0.5 * (bb - aa) * iag);
          const float tf = copysignf(1.0f, zeta) / (fabsf(zeta) + sqrtf(1.0f + zeta * zeta));
          const double t = double(tf);
          c = rsqrt(1.0 + t * t);
          se = S::scale(gg, c * t * iag);                      // s * phase(gamma)
          s_rot[flag] = 1;
        }
        pc[k] = c;
        pg[k] = se;
      }
      __syncthreads();
      // apply
      if (active) {
        const double c = pc[g];
        if (c != 0.0) {
          const T se = pg[g];
          const T sec = S::conj(se);
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            const T x = xa[e], y = xb[e];
            xa[e] = S::sub(S::scale(x, c), S::mul(sec, y));
            xb[e] = S::add(S::mul(se, x), S::scale(y, c));
          }
        }
      }
      // rotate slots: top'[0] = top[0]; top'[1] = bot[0]; top'[g] = top[g-1];
      // bot'[g] = bot[g+1]; bot'[pairs-1] = top[pairs-1]
      // position index in xbuf: tops at 0..pairs-1, bots at pairs..np2-1 (by slot)
      if (active) {
        int dt = -1, db = -1;   // destination position of my top / bot column
        if (g >= 1) dt = (g + 1 < pairs) ? (g + 1) : (pairs + pairs - 1);
        db = (g >= 1) ? (pairs + g - 1) : 1;
        if (g == 0) dt = -1;   // top of slot 0 stays
        if (dt >= 0) {
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            const int i = gl + GS * e;
            if (i < rows) xbuf[size_t(dt) * rows + i] = xa[e];
          }
          if (gl == 0) cid[dt] = ctop;
        }
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int i = gl + GS * e;
          if (i < rows) xbuf[size_t(db) * rows + i] = xb[e];
        }
        if (gl == 0) cid[db] = cbot;
      }
      __syncthreads();
      if (active) {
        if (g >= 1) {
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            const int i = gl + GS * e;
            xa[e] = i < rows ? xbuf[size_t(g) * rows + i] : S::zero();
          }
          ctop = cid[g];
        }
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int i = gl + GS * e;
          xb[e] = i < rows ? xbuf[size_t(pairs + g) * rows + i] : S::zero();
        }
        cbot = cid[pairs + g];
      }
      // (the next write to xbuf / pa happens after the next barrier)
    }
    __syncthreads();
    converged = (s_rot[flag] == 0);
    __syncthreads();
    if (tid == 0) s_rot[flag] = 0;
  }

  // write M_final (row-major, column = original column id) and norms
  if (active) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const int i = gl + GS * e;
      a += S::abs2(xa[e]);
      b += S::abs2(xb[e]);
      if (i < rows) {
        if (ctop < n) Mout[size_t(i) * n + ctop] = xa[e];
        if (cbot < n) Mout[size_t(i) * n + cbot] = xb[e];
      }
    }
    a = gsum<double, GS>(a);
    b = gsum<double, GS>(b);
    if (gl == 0) {
      if (ctop < n) sig[ctop] = sqrt(a);
      if (cbot < n) sig[cbot] = sqrt(b);
    }
  }
  if (tid == 0) {
    info[0] = converged ? sweep : -sweep;
    if (!converged && status) atomicOr(status, 8);
  }
}

// sort by sigma (desc, ties by index), sign-fix J's columns (reference
// core.py:221-229), W = M / sigma with the same phase.  Grid-wide: every CTA
// ranks the singular values itself (n^2 comparisons) and takes 8 output
// columns, one per warp (one CTA streamed four n x n matrices through a
// single SM with column-strided reads: 217 us at n = 256).
// swap: U = M / sigma (sign-fixed) and W = J (same phase) -- the Jacobi on R^H
// variant, where the orthogonal-columns factor M gives the left vectors.
template <typename T>
__global__ void svd_finalize_kernel(int n, const T* __restrict__ Jun, const T* __restrict__ Mun,
                                    const double* __restrict__ sig, T* __restrict__ U,
                                    double* __restrict__ S_out, T* __restrict__ Wout,
                                    bool swap) {
  using S = Sc<T>;
  extern __shared__ int order[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int j = tid; j < n; j += blockDim.x) {
    int rk = 0;
    const double sj = sig[j];
    for (int i = 0; i < n; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
    order[rk] = j;
  }
  __syncthreads();
  if (swap) {   // the sign convention applies to U = M / sigma: use M's columns
    const T* t = Jun;
    Jun = Mun;
    Mun = t;
  }
  for (int o = blockIdx.x * nw + warp; o < n; o += gridDim.x * nw) {
    const int j = order[o];
    double mx = 0.0;
    for (int i = lane; i < n; i += 32) mx = fmax(mx, sqrt(S::abs2(Jun[size_t(i) * n + j])));
    for (int m = 16; m > 0; m >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    int first = n;
    for (int base = 0; base < n && first == n; base += 32) {
      const int i = base + lane;
      const bool hit = (i < n) && (sqrt(S::abs2(Jun[size_t(i) * n + j])) > 1e-10 * mx);
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (bal) first = base + __ffs(bal) - 1;
    }
    T ph = S::one();
    if (first < n) {
      const T z = Jun[size_t(first) * n + j];
      ph = S::conj(S::scale(z, 1.0 / sqrt(S::abs2(z))));
    }
    const double sj = sig[j];
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    for (int i = lane; i < n; i += 32) {
      if (!swap) {
        U[size_t(i) * n + o] = S::mul(Jun[size_t(i) * n + j], ph);
        Wout[size_t(i) * n + o] = S::mul(S::scale(Mun[size_t(i) * n + j], inv), ph);
      } else {   // Jun holds M here: U = M / sigma, W = J
        U[size_t(i) * n + o] = S::mul(S::scale(Jun[size_t(i) * n + j], inv), ph);
        Wout[size_t(i) * n + o] = S::mul(Mun[size_t(i) * n + j], ph);
      }
    }
    if (lane == 0) S_out[o] = sj;
  }
}

template <typename T, int GS, int EPL>
void launch_reg(Handle* h, int n, const T* R, T* Mout, double* sig, int32_t* info) {
  const int np2 = n + (n & 1), pairs = np2 / 2;
  const size_t smem = size_t(np2) * n * sizeof(T) + size_t(pairs) * (sizeof(T) + 3 * sizeof(double)) +
                      size_t(np2) * sizeof(int) + 64;
  auto kern = jacobi_reg_kernel<T, GS, EPL>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int threads = ((pairs * GS + 31) / 32) * 32;
  kern<<<1, threads, smem, h->stream>>>(n, R, Mout, sig, info, 4e-15, 60, h->status);
  LR_CHECK_LAUNCH();
}

}  // namespace

// LR_DEBUG_JACOBI=1: report the sweep count of every register-resident
// Jacobi launch on stderr (synchronizes; development only)
void debug_sweeps(Handle* h, const int32_t* info, int64_t n, const char* kind) {
  static int dbg = -1;
  if (dbg < 0) dbg = getenv("LR_DEBUG_JACOBI") ? 1 : 0;
  if (!dbg) return;
  int32_t v = 0;
  LR_CUDA(cudaMemcpyAsync(&v, info, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
  LR_CUDA(cudaStreamSynchronize(h->stream));
  fprintf(stderr, "[lr] jacobi %s n=%lld sweeps=%d\n", kind, (long long)n, v);
}

bool jacobi_reg_supported(int64_t n, bool cplx) {
  // register-resident: one CTA up to 128 real / 64 complex, a DSMEM cluster
  // (jacobi_blk.cu) up to 256 real / 128 complex
  return n >= 2 && n <= (jacobi_blk_enabled() ? (cplx ? 128 : 256) : (cplx ? 64 : 128));
}

void jacobi_reg_f64(Handle* h, int64_t n, const double* R, double* Mout, double* sig,
                    int32_t* info) {
  if (jacobi_blk_enabled()) {
    jacobi_blk_f64(h, n, R, Mout, sig, info);
    debug_sweeps(h, info, n, "blk");
    return;
  }
  if (n <= 32) launch_reg<double, 32, 1>(h, int(n), R, Mout, sig, info);
  else if (n <= 64) launch_reg<double, 32, 2>(h, int(n), R, Mout, sig, info);
  else launch_reg<double, 16, 8>(h, int(n), R, Mout, sig, info);
  debug_sweeps(h, info, n, "round");
}

void jacobi_reg_c128(Handle* h, int64_t n, const double2* R, double2* Mout, double* sig,
                     int32_t* info) {
  if (jacobi_blk_enabled()) {
    jacobi_blk_c128(h, n, R, Mout, sig, info);
    debug_sweeps(h, info, n, "blk");
    return;
  }
  if (n <= 32) launch_reg<double2, 32, 1>(h, int(n), R, Mout, sig, info);
  else launch_reg<double2, 32, 2>(h, int(n), R, Mout, sig, info);
  debug_sweeps(h, info, n, "round");
}

void svd_finalize(Handle* h, int dtype_wide, int64_t n, const void* Jun, const void* Mun,
                  const double* sig, void* U, double* S, void* W, bool swap) {
  const size_t smem = size_t(n) * sizeof(int);
  if (dtype_wide == LR_C128)
    svd_finalize_kernel<double2><<<unsigned(ceil_div(n, 8)), 256, smem, h->stream>>>(
        int(n), static_cast<const double2*>(Jun), static_cast<const double2*>(Mun), sig,
        static_cast<double2*>(U), S, static_cast<double2*>(W), swap);
  else
    svd_finalize_kernel<double><<<unsigned(ceil_div(n, 8)), 256, smem, h->stream>>>(
        int(n), static_cast<const double*>(Jun), static_cast<const double*>(Mun), sig,
        static_cast<double*>(U), S, static_cast<double*>(W), swap);
  LR_CHECK_LAUNCH();
}

}  // namespace lr
