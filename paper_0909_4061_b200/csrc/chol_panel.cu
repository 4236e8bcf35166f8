// K3 core, panel-blocked variant (default for ell <= 200 real / 140 complex):
// Cholesky with column deletion of a Gram matrix + the inverse of the kept
// triangle, same contract and arithmetic decisions as chol_drop_kernel
// (chol.cu) -- the rank decision of orthonormalize_double_gs, reference
// core.py:84-115.
//
// The unblocked kernels pay one CTA barrier AND a rank-1 update of the whole
// trailing matrix per column (chol_tiled: ~2500 cycles per column, issue
// bound).  Here the factorization is right-looking over panels of NB = 16
// rows, the packed upper triangle resident in shared memory:
//   (a) one warp factors the 16 x 16 diagonal block (warp barriers only),
//   (b) every thread forward-substitutes one column of the panel rows
//       (R12 = R11^{-H} G12),
//   (c) the trailing matrix takes one rank-16 update, register-blocked
//       micro-tiles (4 x 4 real, 2 x 4 complex).
// Three CTA barriers per panel instead of sixteen.  The inverse X = R~^{-1}
// (R~: dropped rows/cols replaced by the identity) is formed in place by
// blocks: every warp inverts diagonal blocks, then block column J is
// X[:J, J] = -X[:J, :J] (R[:J, J] X_JJ), two barriers per block column.
//
// Pivot decisions are those of the unblocked algorithm: pivot j is the
// Schur complement G_jj - sum_{i<j kept} |r_ij|^2, compared with
// drop_tol^2 trace(G) (drop) and unres_rel * G_jj (unresolved); a dropped
// pivot leaves a zero row of R and takes no part in later updates.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int NB = 16;     // panel width
constexpr int NT = 512;    // threads per CTA
constexpr int NW = NT / 32;
constexpr int TBS = NB + 2;   // row stride of the inverse's T buffer (bank spread)

// fp64 1/sqrt: MUFU seed + ITER Newton steps (2 give full precision)
template <int ITER>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < ITER; ++i) y = y * fma(-0.5 * x, y * y, 1.5);
  return y;
}

template <int ITER>
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < ITER; ++i) y = y * fma(-x, y, 2.0);
  return y;
}

template <typename T>
constexpr int panel_maxn() { return sizeof(T) == 8 ? 200 : 140; }

// packed upper triangle: row i holds columns i..n-1
__device__ __forceinline__ int poff(int n, int i) { return i * n - (i * (i - 1)) / 2; }

template <typename T>
__host__ __device__ constexpr int tile_i() { return sizeof(T) == 8 ? 4 : 2; }

template <typename T>
size_t panel_smem_bytes(int n) {
  return size_t(n) * (n + 1) / 2 * sizeof(T)       // W
         + size_t(n) * TBS * sizeof(T)             // T buffer (inverse)
         + size_t(n) * 4 * sizeof(double)          // d0, rd, ri, rti
         + size_t(n) * 2 * sizeof(int) + 64;       // pos, kidx
}

template <typename T>
__global__ void __launch_bounds__(NT, 1)
chol_panel_kernel(int n, const T* __restrict__ G, int64_t ldg, double drop_tol, double unres_rel,
                  double shift_coef, T* __restrict__ P, T* __restrict__ Rout,
                  int32_t* __restrict__ info, int32_t* status, const double* __restrict__ trace_dev,
                  const T* __restrict__ diag_src, int64_t diag_stride, bool compact,
                  const int32_t* __restrict__ gate, double psd_neg, long long* prof) {
  if (gate && *gate == 0) return;
  using S = Sc<T>;
  int np = 0;   // LR_CHOL_PROF: phase timestamps of thread 0
#define PROF_MARK() \
  do { if (prof && threadIdx.x == 0 && np < 64) prof[np++] = clock64(); } while (0)
  PROF_MARK();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* W = reinterpret_cast<T*>(smem_raw);
  T* Tb = W + size_t(n) * (n + 1) / 2;
  double* d0 = reinterpret_cast<double*>(Tb + size_t(n) * TBS);
  double* rd = d0 + n;
  double* ri = rd + n;
  double* rti = ri + n;
  int* pos = reinterpret_cast<int*>(rti + n);
  int* kidx = pos + n;
  __shared__ double s_trace;
  __shared__ int s_unres, s_bad, s_rank, s_npsd;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto at = [&](int i, int k) -> T& { return W[poff(n, i) + (k - i)]; };

  // ---- load the upper triangle, trace, shift ----
  if (warp == 0) {
    double tr = 0.0;
    if (!trace_dev)
      for (int i = lane; i < n; i += 32) tr += S::re(G[size_t(i) * ldg + i]);
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, m);
    if (lane == 0) { s_trace = trace_dev ? *trace_dev : tr; s_unres = 0; s_bad = 0; }
  }
  __syncthreads();
  const double trace = s_trace;
  const double thr2 = drop_tol * drop_tol * trace;
  const double shift = shift_coef * trace;
  // elements of the upper triangle: UL loads in flight per thread, the row
  // index from a float quotient corrected by one step (no integer division)
  {
    constexpr int UL = 8;
    const float inv_n = 1.0f / float(n);
    for (int e0 = tid; e0 < n * n; e0 += UL * NT) {
      T v[UL];
      int ii[UL], kk[UL];
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * NT;
        int i = int(float(e) * inv_n);
        i -= (i * n > e) ? 1 : 0;
        i += ((i + 1) * n <= e) ? 1 : 0;
        ii[u] = i;
        kk[u] = e - i * n;
        v[u] = (e < n * n && kk[u] >= i) ? G[size_t(i) * ldg + kk[u]] : S::zero();
      }
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int i = ii[u], k = kk[u];
        if (e0 + u * NT < n * n && k >= i) {
          T x = v[u];
          if (k == i) {
            x = S::make(S::re(x) + shift, 0.0);
            d0[i] = diag_src ? S::re(diag_src[size_t(i) * diag_stride]) + shift : S::re(x);
          }
          W[poff(n, i) + (k - i)] = x;
        }
      }
    }
  }
  __syncthreads();

  // ---- right-looking panel factorization ----
  int my_unres = 0, my_bad = 0, my_npsd = 0;   // warp 0, lane 0
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int nb = min(NB, n - j0), j1 = j0 + nb;
    // (a) diagonal block, one warp, in registers: lane l holds column
    // b = l & 15 of rows 8h..8h+7 (h = l >> 4).  Step s broadcasts the pivot
    // row with shuffles; updates use the unscaled pivot row times 1/d.
    if (warp == 0) {
      const int b = lane & 15, h = lane >> 4;
      T w[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int a = 8 * h + r;
        w[r] = (a < nb && b < nb && b >= a) ? at(j0 + a, j0 + b) : S::zero();
      }
      PROF_MARK();
      double myd = 0.0;   // lane s keeps pivot s (no branches in the chain)
#pragma unroll 1
      for (int hs = 0; hs < 2; ++hs) {        // pivot rows 8 hs .. 8 hs + 7
        const int src = 16 * hs;
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) {
          const int s = 8 * hs + s2;   // s >= nb: zero pivot row, no update
          {
            const T ps = S::shfl_idx(w[s2], src + b);              // W(s, b)
            const double d = S::re(S::shfl_idx(w[s2], src + s));   // W(s, s)
            T t[8];
#pragma unroll
            for (int r = 0; r < 8; ++r)   // conj(W(s, a)) W(s, b), off the 1/d chain
              t[r] = S::mul(S::conj(S::shfl_idx(w[s2], src + 8 * h + r)), ps);
            const bool keep = isfinite(d) && d > thr2 && d > 0.0;
            const double invd = keep ? 1.0 / d : 0.0;
            myd = (lane == s) ? d : myd;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int a = 8 * h + r;
              if (a > s && b >= a) w[r] = S::sub(w[r], S::scale(t[r], invd));
            }
          }
        }
      }
      if (lane < nb) {
        const int j = j0 + lane;
        const bool fin = isfinite(myd);
        const bool keep = fin && myd > thr2 && myd > 0.0;
        const double r = keep ? sqrt(myd) : 0.0;
        rd[j] = r;
        ri[j] = keep ? 1.0 / r : 0.0;
        const unsigned msk = (1u << nb) - 1u;   // lanes 0 .. nb-1 (nb <= 16)
        const unsigned un = __ballot_sync(msk, keep && myd <= unres_rel * d0[j]);
        const unsigned bd = __ballot_sync(msk, !fin);
        // PSD mode (cholesky of the reference, core.py:249-272): pivots below
        // -psd_neg are a NotPSDError; those in [-psd_neg, 0] are clamped (dropped)
        const unsigned ng = __ballot_sync(msk, psd_neg >= 0.0 && myd < -psd_neg);
        if (lane == 0) { my_unres += __popc(un); my_bad += __popc(bd); my_npsd += __popc(ng); }
      }
      __syncwarp();
      PROF_MARK();
      // R rows of the block: R_ab = W_ab / R_aa (zero row for a dropped pivot)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int a = 8 * h + r;
        if (a < nb && b < nb && b >= a)
          at(j0 + a, j0 + b) = (b == a) ? S::make(rd[j0 + a], 0.0) : S::scale(w[r], ri[j0 + a]);
      }
    }
    __syncthreads();
    PROF_MARK();
    if (j1 >= n) break;
    // (b) panel rows right of the block: R12 = R11^{-H} G12, one column per thread
    for (int k = j1 + tid; k < n; k += NT) {
      T x[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) x[u] = u < nb ? at(j0 + u, k) : S::zero();
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        if (s < nb) {
          const T xs = S::scale(x[s], ri[j0 + s]);
          x[s] = xs;
#pragma unroll
          for (int u = s + 1; u < NB; ++u)
            if (u < nb) x[u] = S::sub(x[u], S::mul(S::conj(at(j0 + s, j0 + u)), xs));
        }
      }
#pragma unroll
      for (int u = 0; u < NB; ++u)
        if (u < nb) at(j0 + u, k) = x[u];
    }
    __syncthreads();
    PROF_MARK();
    // (c) trailing update W(i, k) -= sum_s conj(R(s, i)) R(s, k), j1 <= i <= k.
    // Warp tiles of (4 TI) x 32: lane (ly, lx) = (lane >> 3, lane & 7) owns
    // rows ly + 4a and columns lx + 8b -- the row loads are 8 consecutive
    // elements (one wavefront), the column loads 4 broadcasts.
    {
      constexpr int TI = tile_i<T>();
      const int m = n - j1;
      const int wr = 4 * TI;                  // rows per warp tile
      const int nti = (m + wr - 1) / wr, ntk = (m + 31) / 32;
      const int ly = lane >> 3, lx = lane & 7;
      for (int e = warp; e < nti * ntk; e += NW) {
        const int ti = e / ntk, tk = e - ti * ntk;
        const int i0 = j1 + ti * wr, k0 = j1 + tk * 32;
        if (k0 + 31 < i0) continue;           // entirely below the diagonal
        T acc[TI][4];
#pragma unroll
        for (int a = 0; a < TI; ++a)
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) acc[a][bb] = S::zero();
        const T* row = W + poff(n, j0) - j0;  // row[c] = R(r, c), c >= r
        for (int s = 0; s < nb; ++s) {
          T av[TI], bv[4];
#pragma unroll
          for (int a = 0; a < TI; ++a) {
            const int i = i0 + ly + 4 * a;
            av[a] = i < n ? S::conj(row[i]) : S::zero();
          }
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int k = k0 + lx + 8 * bb;
            bv[bb] = k < n ? row[k] : S::zero();
          }
#pragma unroll
          for (int a = 0; a < TI; ++a)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) acc[a][bb] = S::add(acc[a][bb], S::mul(av[a], bv[bb]));
          row += n - (j0 + s) - 1;            // next row: poff(r + 1) - (r + 1)
        }
#pragma unroll
        for (int a = 0; a < TI; ++a) {
          const int i = i0 + ly + 4 * a;
          if (i < n) {
            T* rowi = W + poff(n, i) - i;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
              const int k = k0 + lx + 8 * bb;
              if (k < n && k >= i) rowi[k] = S::sub(rowi[k], acc[a][bb]);
            }
          }
        }
      }
    }
    PROF_MARK();
    __syncthreads();
  }

  PROF_MARK();
  // ---- compaction of the kept pivots ----
  if (warp == 0) {
    if (lane == 0) { s_unres = my_unres; s_bad = my_bad; s_npsd = my_npsd; }
    int base = 0;
    for (int jj = 0; jj < n; jj += 32) {
      const int j = jj + lane;
      const bool k = j < n && rd[j] > 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      const int p = base + __popc(bal & ((1u << lane) - 1u));
      if (j < n) {
        pos[j] = k ? p : -1;
        if (k) kidx[p] = j;
        rti[j] = k ? ri[j] : 1.0;
      }
      base += __popc(bal);
    }
    if (lane == 0) s_rank = base;
  }
  __syncthreads();
  const int rank = s_rank;

  // ---- R output (kept rows/cols), then R~ in place ----
  {
    const float inv_n = 1.0f / float(n);
#pragma unroll 4
    for (int e = tid; e < n * n; e += NT) {
      int i = int(float(e) * inv_n);
      i -= (i * n > e) ? 1 : 0;
      i += ((i + 1) * n <= e) ? 1 : 0;
      const int k = e - i * n;
      Rout[e] = (k >= i && pos[i] >= 0 && pos[k] >= 0) ? W[poff(n, i) + (k - i)] : S::zero();
    }
  }
  __syncthreads();
  if (rank < n) {
    for (int i = warp; i < n; i += NW) {
      T* rowi = W + poff(n, i) - i;
      for (int k = i + lane; k < n; k += 32)   // column k dropped: identity column
        if (pos[k] < 0) rowi[k] = (i == k) ? S::one() : S::zero();
    }
    __syncthreads();
  }
  PROF_MARK();

  // ---- X = R~^{-1} in place: diagonal blocks (one warp each) ----
  const int nbk = (n + NB - 1) / NB;
  for (int J = warp; J < nbk; J += NW) {
    const int j0 = J * NB, nb = min(NB, n - j0);
    const int c = lane;
    T x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) x[i] = (i == c) ? S::one() : S::zero();
#pragma unroll
    for (int k = NB - 1; k >= 0; --k) {
      if (k <= c && c < nb) {
        const T xk = S::scale(x[k], rti[j0 + k]);
        x[k] = xk;
#pragma unroll
        for (int i = 0; i < k; ++i) x[i] = S::sub(x[i], S::mul(at(j0 + i, j0 + k), xk));
      }
    }
    __syncwarp();
    if (c < nb) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
        if (i <= c) at(j0 + i, j0 + c) = x[i];
    }
  }
  __syncthreads();
  PROF_MARK();
  // ---- block columns: X[:j0, J] = -X[:j0, :j0] (R[:j0, J] X_JJ) ----
  // Register-blocked: a thread owns RB consecutive rows x 4 consecutive
  // columns (RB = 4 real, 2 complex), row pointers hoisted -- the per-element
  // version was instruction-issue bound (~35 instructions per 4 FMAs).
  {
    constexpr int RB = sizeof(T) == 8 ? 4 : 2;
    for (int J = 1; J < nbk; ++J) {
      const int j0 = J * NB, nb = min(NB, n - j0);
      const int nq = (nb + 3) / 4, nr = (j0 + RB - 1) / RB;
      // T = R[:j0, J] X_JJ  (X_JJ upper: entry (k, c) nonzero for k <= c)
      for (int e = tid; e < nr * nq; e += NT) {
        const int rq = e / nq, c0 = 4 * (e - rq * nq);
        const int i0 = RB * rq;
        const T* rr[RB];
#pragma unroll
        for (int a = 0; a < RB; ++a) {
          const int i = min(i0 + a, j0 - 1);
          rr[a] = W + poff(n, i) - i + j0;          // rr[a][k] = R(i, j0 + k)
        }
        T acc[RB][4];
#pragma unroll
        for (int a = 0; a < RB; ++a)
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[a][t] = S::zero();
        const int kmax = min(c0 + 3, nb - 1);
        for (int k = 0; k <= kmax; ++k) {
          const T* xk = W + poff(n, j0 + k) - (j0 + k) + j0;   // xk[c] = X_JJ(k, c)
          T xv[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) xv[t] = (c0 + t >= k && c0 + t < nb) ? xk[c0 + t] : S::zero();
#pragma unroll
          for (int a = 0; a < RB; ++a) {
            const T r = rr[a][k];
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[a][t] = S::add(acc[a][t], S::mul(r, xv[t]));
          }
        }
#pragma unroll
        for (int a = 0; a < RB; ++a)
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (i0 + a < j0) Tb[(i0 + a) * TBS + c0 + t] = acc[a][t];
      }
      __syncthreads();
      // X(i, j0 + c) = -sum_{k >= i} X(i, k) T(k, c): the k-sum of each
      // RB x 4 output block is split over KS consecutive lanes (interleaved
      // k) and reduced with shuffles (one thread per block ran chains of up
      // to j0 dependent steps with most of the CTA idle)
      {
        constexpr int KS = 4;
        const int tot = nr * nq * KS;
        for (int eb = warp * 32; eb < tot; eb += NT) {
          const int e = eb + lane;
          const bool valid = e < tot;
          const int sub = e & (KS - 1);
          const int gi = valid ? e / KS : 0;
          const int rq = gi / nq, c0 = 4 * (gi - rq * nq);
          const int i0 = RB * rq;
          const T* xr[RB];
#pragma unroll
          for (int a = 0; a < RB; ++a) {
            const int i = min(i0 + a, j0 - 1);
            xr[a] = W + poff(n, i) - i;                // xr[a][k] = X(i, k), k >= i
          }
          T acc[RB][4];
#pragma unroll
          for (int a = 0; a < RB; ++a)
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[a][t] = S::zero();
          if (valid && sub == 0) {
            // the first RB - 1 columns k are inside the row block's triangle
#pragma unroll
            for (int kk = 0; kk < RB - 1; ++kk) {
              const int k = i0 + kk;
              if (k < j0) {
                const T* tb = Tb + k * TBS + c0;
#pragma unroll
                for (int a = 0; a < RB; ++a) {
                  if (a <= kk) {
                    const T x = xr[a][k];
#pragma unroll
                    for (int t = 0; t < 4; ++t) acc[a][t] = S::add(acc[a][t], S::mul(x, tb[t]));
                  }
                }
              }
            }
          }
          const int kend = valid ? j0 : 0;
#pragma unroll 2
          for (int k = i0 + RB - 1 + sub; k < kend; k += KS) {
            const T* tb = Tb + k * TBS + c0;
            T tv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) tv[t] = tb[t];
#pragma unroll
            for (int a = 0; a < RB; ++a) {
              const T x = xr[a][k];
#pragma unroll
              for (int t = 0; t < 4; ++t) acc[a][t] = S::add(acc[a][t], S::mul(x, tv[t]));
            }
          }
#pragma unroll
          for (int a = 0; a < RB; ++a)
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
              for (int o = 1; o < KS; o <<= 1) acc[a][t] = S::add(acc[a][t], S::shfl_xor(acc[a][t], o));
          if (valid && sub == 0) {
#pragma unroll
            for (int a = 0; a < RB; ++a) {
              if (i0 + a < j0) {
                T* row = W + poff(n, i0 + a) - (i0 + a) + j0;
#pragma unroll
                for (int t = 0; t < 4; ++t)
                  if (c0 + t < nb) row[c0 + t] = S::scale(acc[a][t], -1.0);
              }
            }
          }
        }
      }
      __syncthreads();
    }
  }

  PROF_MARK();
  // ---- P: kept columns (compacted or in place), zero elsewhere ----
  {
    const float inv_n = 1.0f / float(n);
#pragma unroll 4
    for (int e = tid; e < n * n; e += NT) {
      int i = int(float(e) * inv_n);
      i -= (i * n > e) ? 1 : 0;
      i += ((i + 1) * n <= e) ? 1 : 0;
      const int q = e - i * n;
      const int c = compact ? (q < rank ? kidx[q] : -1) : (pos[q] >= 0 ? q : -1);
      P[e] = (pos[i] >= 0 && c >= i) ? W[poff(n, i) + (c - i)] : S::zero();
    }
  }
  __syncthreads();
  PROF_MARK();
  if (prof && tid == 0) prof[63] = np;
#undef PROF_MARK
  if (tid == 0) {
    info[0] = rank;
    info[1] = s_unres;
    info[2] = s_bad;
    if (psd_neg >= 0.0) info[3] = s_npsd;
    if (status) {
      const int bits = (s_unres ? 1 : 0) | (rank < n ? 2 : 0) | (s_bad ? 4 : 0);
      if (bits) atomicOr(status, bits);
    }
  }
}

template <typename T>
void launch_panel(Handle* h, int n, const T* G, int64_t ldg, double drop_tol, double unres_rel,
                  double shift_coef, T* P, T* R, int32_t* info, const double* trace_dev,
                  const T* diag_src, int64_t diag_stride, bool compact, double psd_neg) {
  const size_t smem = panel_smem_bytes<T>(n);
  auto kern = chol_panel_kernel<T>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  static int prof_on = -1;
  if (prof_on < 0) prof_on = getenv("LR_CHOL_PROF") ? 1 : 0;
  long long* prof = prof_on ? pool_alloc_t<long long>(h, 64) : nullptr;
  kern<<<1, NT, smem, h->stream>>>(n, G, ldg, drop_tol, unres_rel, shift_coef, P, R, info,
                                   h->status, trace_dev, diag_src, diag_stride, compact, h->gate,
                                   psd_neg, prof);
  LR_CHECK_LAUNCH();
  if (prof) {   // development only: synchronizes
    long long hp[64];
    LR_CUDA(cudaMemcpyAsync(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost, h->stream));
    LR_CUDA(cudaStreamSynchronize(h->stream));
    fprintf(stderr, "[lr] chol_panel n=%d cycles:", n);
    for (int i = 1; i < int(hp[63]); ++i) fprintf(stderr, " %lld", hp[i] - hp[i - 1]);
    fprintf(stderr, " | total %lld\n", hp[int(hp[63]) - 1] - hp[0]);
  }
}

}  // namespace

// LR_CHOL=panel (default) | tiled | smem selects the Cholesky kernel family
int chol_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("LR_CHOL");
    mode = !e ? 0 : (e[0] == 's' ? 1 : e[0] == 't' ? 2 : 0);
  }
  return mode;
}

bool chol_panel_supported(int64_t n, bool cplx) {
  return chol_mode() == 0 && n >= 1 && n <= (cplx ? panel_maxn<double2>() : panel_maxn<double>());
}

void chol_panel_f64(Handle* h, int64_t n, const double* G, int64_t ldg, double drop_tol,
                    double unres_rel, double shift_coef, double* P, double* R, int32_t* info,
                    const double* trace_dev, const double* diag_src, int64_t diag_stride,
                    bool compact, double psd_neg) {
  launch_panel<double>(h, int(n), G, ldg, drop_tol, unres_rel, shift_coef, P, R, info,
                       trace_dev, diag_src, diag_stride, compact, psd_neg);
}

void chol_panel_c128(Handle* h, int64_t n, const double2* G, int64_t ldg, double drop_tol,
                     double unres_rel, double shift_coef, double2* P, double2* R, int32_t* info,
                     const double* trace_dev, const double2* diag_src, int64_t diag_stride,
                     bool compact, double psd_neg) {
  launch_panel<double2>(h, int(n), G, ldg, drop_tol, unres_rel, shift_coef, P, R, info,
                        trace_dev, diag_src, diag_stride, compact, psd_neg);
}

}  // namespace lr
