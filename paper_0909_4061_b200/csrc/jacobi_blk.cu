// K4 fast path, block variant: register-resident BLOCK one-sided Jacobi for
// square n <= 128 (real) / 64 (complex), the small SVD of direct_svd
// (reference core.py:199-230) on the CholeskyQR factor R of B^H.
//
// Same contract as jacobi_reg_kernel (R J = M with orthogonal columns, M and
// the column norms written unsorted; J is formed afterwards as R^{-1} M), but
// organised to move less data: the columns are grouped in blocks of BW = 4,
// each warp holds two blocks (8 columns, rows spread over the lanes: row
// lane + 32 r), and one "round" orthogonalizes all 16 cross pairs of the two
// blocks in 4 sub-rounds of 4 disjoint pairs -- inner products reduced with
// warp butterflies, the rotation computed redundantly by every lane in fp64,
// applied in registers.  Blocks then move one slot of the round-robin
// tournament through shared memory, so a sweep is nb-1 rounds (nb = n/4
// blocks) instead of n-1, and moves the matrix nb-1 times instead of n-1.
// The 6 intra-block pairs of each block are done once per sweep.  Every
// pair is visited once per sweep, so the cyclic-Jacobi convergence theory
// applies; the test is |m_p^H m_q| <= tol ||m_p|| ||m_q|| as before.
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int BW = 4;        // columns per block
// Early exit: once every rotation of a sweep had |m_p^H m_q| <= 1e-9
// ||m_p|| ||m_q||, the sweep's own rotations leave off-diagonal terms of
// order 1e-18 / (relative gap) (quadratic convergence of cyclic Jacobi), far
// below the test tolerance -- the confirming sweep that would find nothing
// to rotate is skipped.  sigma = ||m_j|| is second-order in the remaining
// off-diagonal terms.
constexpr double kTQ2 = 1e-18;
constexpr int WC = 2 * BW;   // columns held by one warp

// call-free fp64 rsqrt / reciprocal (MUFU approximation + Newton steps):
// the libdevice versions branch to out-of-line slow paths whose calling
// convention spills the register-resident columns.  Inputs are positive and
// normal here.
// ITER Newton steps: the ~2^-23 MUFU seed doubles its bits per step, so 2
// steps give full double precision and 0-1 steps suffice where only the
// convergence rate depends on the value.
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

// Rotation that zeroes m_p^H m_q: x_p' = c x_p - conj(se) x_q,
// x_q' = se x_p + c x_q with se = s e^{i arg g}; the squared column norms
// then change by -/+ t |g| (tg).  Branch-free: a pair that needs no rotation
// gets the exact identity (c = 1, se = 0, tg = 0), so the four pairs of a
// sub-round are computed and applied without divergent control flow.  Only
// c (and the phase of g, complex case) must be accurate to keep the rotation
// orthogonal; t only sets the convergence rate.
template <typename T>
__device__ __forceinline__ bool rot_params(double a, double b, T g, double tol, double& c, T& se,
                                           double& tg) {
  using S = Sc<T>;
  const double g2 = S::abs2(g);
  const bool rot = a > 0.0 && b > 0.0 && g2 > tol * tol * a * b;
  const double g2s = rot ? g2 : 1.0;
  double iag;
  if constexpr (S::cplx) iag = rsqrt_nr<2>(g2s);   // phase g / |g| must be unit
  else iag = rsqrt_nr<1>(g2s);
  const double ag = g2s * iag;
  const double zeta = 0.5 * (b - a) * iag;
  const double az = fmin(fabs(zeta), 1e150);
  const double q = fma(az, az, 1.0);
  const double t = copysign(rcp_nr<1>(az + q * rsqrt_nr<1>(q)), zeta);
  const double cc = rsqrt_nr<2>(fma(t, t, 1.0));
  c = rot ? cc : 1.0;
  if constexpr (S::cplx) se = rot ? S::scale(g, cc * t * iag) : S::zero();
  else se = rot ? (g < 0.0 ? -cc * t : cc * t) : 0.0;   // s sign(g)
  tg = rot ? t * ag : 0.0;
  return rot;
}

template <typename T, int R>
__device__ __forceinline__ double col_norm2(const T (&v)[R]) {
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) s += Sc<T>::abs2(v[r]);
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  return s;
}

// The four disjoint pairs (P_k, Q_k) of a sub-round cover the warp's 8
// columns.  Inner products: 4R multiply-adds per lane, then a reduce-scatter
// butterfly (6 shuffle levels instead of 4 x 5) that leaves pair k's sum in
// lanes 8k..8k+7; lane 8k alone forms pair k's rotation (one rotation per
// pair instead of one per lane), and (c, se) are broadcast back.  Squared
// column norms live one per lane (lane c < WC holds column c's) and are
// updated analytically (a' = a - t|g|, b' = b + t|g|), recomputed exactly
// when a shrinks by more than 10x (cancellation) and once per sweep.
template <int P0, int Q0, int P1, int Q1, int P2, int Q2, int P3, int Q3>
struct Pairs {
  __device__ static constexpr int p(int k) { return k == 0 ? P0 : k == 1 ? P1 : k == 2 ? P2 : P3; }
  __device__ static constexpr int q(int k) { return k == 0 ? Q0 : k == 1 ? Q1 : k == 2 ? Q2 : Q3; }
  // pair containing column c, and whether c is its first member
  __device__ static constexpr int of(int c) {
    return (c == P0 || c == Q0) ? 0 : (c == P1 || c == Q1) ? 1 : (c == P2 || c == Q2) ? 2 : 3;
  }
  __device__ static constexpr bool first(int c) { return c == P0 || c == P1 || c == P2 || c == P3; }
  // lane-dependent lookups as shifts of compile-time packed tables (the
  // select chains of p()/q()/of() on runtime indices cost ~10% of a subround)
  static constexpr unsigned PT = unsigned(P0) | unsigned(P1) << 4 | unsigned(P2) << 8 | unsigned(P3) << 12;
  static constexpr unsigned QT = unsigned(Q0) | unsigned(Q1) << 4 | unsigned(Q2) << 8 | unsigned(Q3) << 12;
  __device__ static constexpr unsigned of_tab() {
    unsigned t = 0;
    for (int c = 0; c < 8; ++c) t |= unsigned(of(c)) << (2 * c);
    return t;
  }
  __device__ static constexpr unsigned first_tab() {
    unsigned t = 0;
    for (int c = 0; c < 8; ++c) t |= (first(c) ? 1u : 0u) << c;
    return t;
  }
  __device__ static __forceinline__ int p_rt(int k) { return int((PT >> (4 * k)) & 15u); }
  __device__ static __forceinline__ int q_rt(int k) { return int((QT >> (4 * k)) & 15u); }
  __device__ static __forceinline__ int of_rt(int c) { return int((of_tab() >> (2 * c)) & 3u); }
  __device__ static __forceinline__ bool first_rt(int c) { return (first_tab() >> c) & 1u; }
};

template <typename T, int R, int P0, int Q0, int P1, int Q1, int P2, int Q2, int P3, int Q3>
__device__ __forceinline__ void subround(T (&x)[WC][R], double& nrmv, int lane, double tol,
                                         int& did) {
  using S = Sc<T>;
  using PR = Pairs<P0, Q0, P1, Q1, P2, Q2, P3, Q3>;
  T g[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    g[k] = S::zero();
#pragma unroll
    for (int r = 0; r < R; ++r) g[k] = S::add(g[k], S::cmul(x[PR::p(k)][r], x[PR::q(k)][r]));
  }
  // reduce-scatter: after the xor-16 level lanes with bit 4 clear keep pairs
  // {0,1}, set keep {2,3}; after xor-8 bit 3 picks one; then plain butterfly
  const bool b4 = lane & 16, b3 = lane & 8;
  T k0 = b4 ? g[2] : g[0], k1 = b4 ? g[3] : g[1];
  k0 = S::add(k0, S::shfl_xor(b4 ? g[0] : g[2], 16));
  k1 = S::add(k1, S::shfl_xor(b4 ? g[1] : g[3], 16));
  T v = S::add(b3 ? k1 : k0, S::shfl_xor(b3 ? k0 : k1, 8));
  v = S::add(v, S::shfl_xor(v, 4));
  v = S::add(v, S::shfl_xor(v, 2));
  v = S::add(v, S::shfl_xor(v, 1));
  const int kk = (lane >> 3) & 3;   // = 2 b4 + b3: the pair whose sum this lane holds
  const double a = __shfl_sync(0xffffffffu, nrmv, PR::p_rt(kk));
  const double b = __shfl_sync(0xffffffffu, nrmv, PR::q_rt(kk));
  double c, tg;
  T se;
  const bool rot = rot_params(a, b, v, tol, c, se, tg);
  // bit 1: a rotation above the quadratic-phase threshold (see kTQ2)
  did |= (rot ? 1 : 0) | ((rot && S::abs2(v) > kTQ2 * a * b) ? 2 : 0);
  const double an = a - tg, bn = b + tg;
  // apply the four rotations (identity for pairs below the threshold)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double ck = __shfl_sync(0xffffffffu, c, 8 * k);
    const T sek = S::shfl_idx(se, 8 * k);
    const T sec = S::conj(sek);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const T xp = x[PR::p(k)][r], xq = x[PR::q(k)][r];
      x[PR::p(k)][r] = S::sub(S::scale(xp, ck), S::mul(sec, xq));
      x[PR::q(k)][r] = S::add(S::mul(sek, xp), S::scale(xq, ck));
    }
  }
  // new norms: lane c < WC fetches its column's from lane 8 * pair(c)
  const int lc = lane & (WC - 1);
  const int src = 8 * PR::of_rt(lc);
  const double na = __shfl_sync(0xffffffffu, an, src);
  const double nb = __shfl_sync(0xffffffffu, bn, src);
  if (lane < WC) nrmv = PR::first_rt(lc) ? na : nb;
  // cancellation guard (rare, warp-uniform)
  const unsigned need = __ballot_sync(0xffffffffu, (lane & 7) == 0 && rot && an < 0.1 * a);
  if (need) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (need & (1u << (8 * k))) {
        const double e = col_norm2<T, R>(x[PR::p(k)]);
        if (lane == PR::p(k)) nrmv = e;
      }
    }
  }
}

template <typename T, int R, int MAXT>
__global__ void __launch_bounds__(MAXT, 1)   // MAXT = 32 * (blocks / 2)
jacobi_blk_kernel(int n, const T* __restrict__ Rin, T* __restrict__ Mout, double* __restrict__ sig,
                  int32_t* __restrict__ info, double tol, int max_sweeps, int32_t* status) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb = (n + BW - 1) / BW;
  const int nbp = nb + (nb & 1);
  const int P = nbp / 2;
  constexpr int ROWS = 32 * R;
  T* xbuf = reinterpret_cast<T*>(smem_raw);                               // [2P][BW][ROWS]
  double* nbuf = reinterpret_cast<double*>(xbuf + size_t(2 * P) * BW * ROWS);  // norms moved
  int* bid = reinterpret_cast<int*>(nbuf + 2 * P * BW);                       // block id per position

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int btop = w, bbot = nbp - 1 - w;
  T x[WC][R];
#pragma unroll
  for (int c = 0; c < WC; ++c) {
    const int col = (c < BW ? btop : bbot) * BW + (c & (BW - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = lane + 32 * r;
      x[c][r] = (row < n && col < n) ? Rin[size_t(row) * n + col] : S::zero();
    }
  }

  double nrmv = 0.0;   // lane c < WC: squared norm of column c
  int sweep = 0;
  bool converged = (n <= 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    int did = 0;
#pragma unroll
    for (int c = 0; c < WC; ++c) {
      const double v = col_norm2<T, R>(x[c]);
      if (lane == c) nrmv = v;
    }
    // intra-block pairs of both blocks (once per sweep)
    subround<T, R, 0, 1, 2, 3, 4, 5, 6, 7>(x, nrmv, lane, tol, did);
    subround<T, R, 0, 2, 1, 3, 4, 6, 5, 7>(x, nrmv, lane, tol, did);
    subround<T, R, 0, 3, 1, 2, 4, 7, 5, 6>(x, nrmv, lane, tol, did);
    for (int rd = 0; rd < nbp - 1; ++rd) {
      // the 16 cross pairs (a, BW + ((a + s) mod BW)), s = 0..3
      subround<T, R, 0, 4, 1, 5, 2, 6, 3, 7>(x, nrmv, lane, tol, did);
      subround<T, R, 0, 5, 1, 6, 2, 7, 3, 4>(x, nrmv, lane, tol, did);
      subround<T, R, 0, 6, 1, 7, 2, 4, 3, 5>(x, nrmv, lane, tol, did);
      subround<T, R, 0, 7, 1, 4, 2, 5, 3, 6>(x, nrmv, lane, tol, did);
      if (nbp > 2) {
        // tournament move: top'[0] = top[0], top'[1] = bot[0], top'[g] = top[g-1],
        // bot'[g] = bot[g+1], bot'[P-1] = top[P-1]; positions: tops 0..P-1, bots P..2P-1
        __syncthreads();   // everyone has read the previous move
        const int dt = (w == 0) ? -1 : (w + 1 < P ? w + 1 : 2 * P - 1);
        const int db = (w >= 1) ? P + w - 1 : 1;
        if (dt >= 0) {
#pragma unroll
          for (int c = 0; c < BW; ++c)
#pragma unroll
            for (int r = 0; r < R; ++r) xbuf[(size_t(dt) * BW + c) * ROWS + lane + 32 * r] = x[c][r];
          if (lane < BW) nbuf[dt * BW + lane] = nrmv;
          if (lane == 0) bid[dt] = btop;
        }
#pragma unroll
        for (int c = 0; c < BW; ++c)
#pragma unroll
          for (int r = 0; r < R; ++r)
            xbuf[(size_t(db) * BW + c) * ROWS + lane + 32 * r] = x[BW + c][r];
        if (lane >= BW && lane < WC) nbuf[db * BW + lane - BW] = nrmv;
        if (lane == 0) bid[db] = bbot;
        __syncthreads();
        if (w >= 1) {
#pragma unroll
          for (int c = 0; c < BW; ++c)
#pragma unroll
            for (int r = 0; r < R; ++r) x[c][r] = xbuf[(size_t(w) * BW + c) * ROWS + lane + 32 * r];
          btop = bid[w];
          if (lane < BW) nrmv = nbuf[w * BW + lane];
        }
#pragma unroll
        for (int c = 0; c < BW; ++c)
#pragma unroll
          for (int r = 0; r < R; ++r)
            x[BW + c][r] = xbuf[(size_t(P + w) * BW + c) * ROWS + lane + 32 * r];
        bbot = bid[P + w];
        if (lane >= BW && lane < WC) nrmv = nbuf[(P + w) * BW + lane - BW];
      }
    }
    converged = !__syncthreads_or(did & 2);
  }

  // M (row-major, column = original column id) and the column norms
#pragma unroll
  for (int c = 0; c < WC; ++c) {
    const int col = (c < BW ? btop : bbot) * BW + (c & (BW - 1));
    double nrm = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = lane + 32 * r;
      nrm += S::abs2(x[c][r]);
      if (row < n && col < n) Mout[size_t(row) * n + col] = x[c][r];
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, m);
    if (lane == 0 && col < n) sig[col] = sqrt(nrm);
  }
  if (threadIdx.x == 0) {
    info[0] = converged ? sweep : -sweep;
    if (!converged && status) atomicOr(status, 8);
  }
}

template <typename T, int R, int MAXT>
void launch_blk(Handle* h, int n, const T* Rin, T* Mout, double* sig, int32_t* info) {
  const int nb = (n + BW - 1) / BW, nbp = nb + (nb & 1), P = nbp / 2;
  const size_t smem = size_t(2 * P) * BW * 32 * R * sizeof(T) +
                      size_t(2 * P) * (BW * sizeof(double) + sizeof(int));
  auto kern = jacobi_blk_kernel<T, R, MAXT>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<1, P * 32, smem, h->stream>>>(n, Rin, Mout, sig, info, 4e-15, 60, h->status);
  LR_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// Cluster variant for the columns that do not fit one SM's register file
// (real 128 < n <= 256, complex 64 < n <= 128): the same block tournament
// over a thread-block cluster of CL CTAs x WPC warps.  Tournament position
// pos (tops 0..P-1, bottoms P..2P-1) lives in the shared memory of the CTA
// owning warp (pos mod P); moved blocks are written straight into the
// owner's slot through distributed shared memory (DSMEM) and two cluster
// barriers per round order the writes and reads.  256 threads per CTA leave
// 255 registers per thread for the 8 x R column block.
template <typename T, int R, int CL, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1)
jacobi_cl_kernel(int n, const T* __restrict__ Rin, T* __restrict__ Mout, double* __restrict__ sig,
                 int32_t* __restrict__ info, double tol, int max_sweeps, int32_t* status) {
  namespace cg = cooperative_groups;
  using S = Sc<T>;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int ROWS = 32 * R;
  constexpr int SLOTS = 2 * WPC;
  T* xbuf = reinterpret_cast<T*>(smem_raw);                                 // [SLOTS][BW][ROWS]
  double* nbuf = reinterpret_cast<double*>(xbuf + size_t(SLOTS) * BW * ROWS);  // [SLOTS][BW]
  int* bid = reinterpret_cast<int*>(nbuf + SLOTS * BW);                        // [SLOTS]
  int* cflag = bid + SLOTS;                                                    // [2][CL]

  const int nb = (n + BW - 1) / BW;
  const int nbp = nb + (nb & 1);
  const int P = nbp / 2;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int rank = int(cluster.block_rank());
  const int w = rank * WPC + wl;       // tournament slot of this warp
  const bool active = w < P;
  // position -> (owner CTA, local slot)
  auto owner = [&](int pos) { return (pos < P ? pos : pos - P) / WPC; };
  auto lslot = [&](int pos) { return (pos < P ? 0 : WPC) + (pos < P ? pos : pos - P) % WPC; };

  int btop = w, bbot = nbp - 1 - w;
  T x[WC][R];
#pragma unroll
  for (int c = 0; c < WC; ++c) {
    const int col = (c < BW ? btop : bbot) * BW + (c & (BW - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = lane + 32 * r;
      x[c][r] = (active && row < n && col < n) ? Rin[size_t(row) * n + col] : S::zero();
    }
  }

  double nrmv = 0.0;
  int sweep = 0;
  bool converged = (n <= 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    int did = 0;
    if (active) {
#pragma unroll
      for (int c = 0; c < WC; ++c) {
        const double v = col_norm2<T, R>(x[c]);
        if (lane == c) nrmv = v;
      }
      subround<T, R, 0, 1, 2, 3, 4, 5, 6, 7>(x, nrmv, lane, tol, did);
      subround<T, R, 0, 2, 1, 3, 4, 6, 5, 7>(x, nrmv, lane, tol, did);
      subround<T, R, 0, 3, 1, 2, 4, 7, 5, 6>(x, nrmv, lane, tol, did);
    }
    for (int rd = 0; rd < nbp - 1; ++rd) {
#ifndef LR_JAC_NOSUB     // development: time the exchange alone
      if (active) {
        subround<T, R, 0, 4, 1, 5, 2, 6, 3, 7>(x, nrmv, lane, tol, did);
        subround<T, R, 0, 5, 1, 6, 2, 7, 3, 4>(x, nrmv, lane, tol, did);
        subround<T, R, 0, 6, 1, 7, 2, 4, 3, 5>(x, nrmv, lane, tol, did);
        subround<T, R, 0, 7, 1, 4, 2, 5, 3, 6>(x, nrmv, lane, tol, did);
      }
#endif
#ifdef LR_JAC_NOXCHG     // development: time the rotations alone
      continue;
#endif
      cluster.sync();   // every slot has been read
      if (active) {
        const int dt = (w == 0) ? -1 : (w + 1 < P ? w + 1 : 2 * P - 1);
        const int db = (w >= 1) ? P + w - 1 : 1;
        if (dt >= 0) {
          const int o = owner(dt), ls = lslot(dt);
          T* xb = cluster.map_shared_rank(xbuf, o) + size_t(ls) * BW * ROWS;
#pragma unroll
          for (int c = 0; c < BW; ++c)
#pragma unroll
            for (int r = 0; r < R; ++r) xb[c * ROWS + lane + 32 * r] = x[c][r];
          if (lane < BW) cluster.map_shared_rank(nbuf, o)[ls * BW + lane] = nrmv;
          if (lane == 0) cluster.map_shared_rank(bid, o)[ls] = btop;
        }
        const int o = owner(db), ls = lslot(db);
        T* xb = cluster.map_shared_rank(xbuf, o) + size_t(ls) * BW * ROWS;
#pragma unroll
        for (int c = 0; c < BW; ++c)
#pragma unroll
          for (int r = 0; r < R; ++r) xb[c * ROWS + lane + 32 * r] = x[BW + c][r];
        if (lane >= BW && lane < WC) cluster.map_shared_rank(nbuf, o)[ls * BW + lane - BW] = nrmv;
        if (lane == 0) cluster.map_shared_rank(bid, o)[ls] = bbot;
      }
      cluster.sync();   // the moves have landed
      if (active) {
        if (w >= 1) {
          const T* xb = xbuf + size_t(lslot(w)) * BW * ROWS;
#pragma unroll
          for (int c = 0; c < BW; ++c)
#pragma unroll
            for (int r = 0; r < R; ++r) x[c][r] = xb[c * ROWS + lane + 32 * r];
          btop = bid[lslot(w)];
          if (lane < BW) nrmv = nbuf[lslot(w) * BW + lane];
        }
        const int lb = lslot(P + w);
        const T* xb = xbuf + size_t(lb) * BW * ROWS;
#pragma unroll
        for (int c = 0; c < BW; ++c)
#pragma unroll
          for (int r = 0; r < R; ++r) x[BW + c][r] = xb[c * ROWS + lane + 32 * r];
        bbot = bid[lb];
        if (lane >= BW && lane < WC) nrmv = nbuf[lb * BW + lane - BW];
      }
    }
    // cluster-wide "any rotation": per-CTA OR, gathered in rank 0
    const int any_cta = __syncthreads_or(did & 2);
    int* flags = cflag + (sweep & 1) * CL;
    if (threadIdx.x == 0) cluster.map_shared_rank(flags, 0)[rank] = any_cta;
    cluster.sync();
    int any = 0;
    const int* f0 = cluster.map_shared_rank(flags, 0);
#pragma unroll
    for (int c = 0; c < CL; ++c) any |= f0[c];
    converged = (any == 0);
  }

  if (active) {
#pragma unroll
    for (int c = 0; c < WC; ++c) {
      const int col = (c < BW ? btop : bbot) * BW + (c & (BW - 1));
      double nrm = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int row = lane + 32 * r;
        nrm += S::abs2(x[c][r]);
        if (row < n && col < n) Mout[size_t(row) * n + col] = x[c][r];
      }
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, m);
      if (lane == 0 && col < n) sig[col] = sqrt(nrm);
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    info[0] = converged ? sweep : -sweep;
    if (!converged && status) atomicOr(status, 8);
  }
  cluster.sync();   // keep every CTA's shared memory alive until all DSMEM reads are done
}

template <typename T, int R, int CL, int WPC>
void launch_cl(Handle* h, int n, const T* Rin, T* Mout, double* sig, int32_t* info) {
  constexpr int SLOTS = 2 * WPC;
  const size_t smem = size_t(SLOTS) * BW * 32 * R * sizeof(T) +
                      size_t(SLOTS) * (BW * sizeof(double) + sizeof(int)) + 2 * CL * sizeof(int);
  auto kern = jacobi_cl_kernel<T, R, CL, WPC>;
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL, 1, 1);
  cfg.blockDim = dim3(WPC * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LR_CUDA(cudaLaunchKernelEx(&cfg, kern, n, Rin, Mout, sig, info, 4e-15, 60, h->status));
  LR_CHECK_LAUNCH();
}

}  // namespace

bool jacobi_blk_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LR_JACOBI");
    v = (e && std::strcmp(e, "round") == 0) ? 0 : 1;
  }
  return v == 1;
}

// 96 < n <= 128 real: a 2-CTA cluster (255 registers per thread, no spills)
// instead of one 448/512-thread CTA (128 registers, spills); LR_JACOBI_CL=0
// selects the single CTA.
static bool cl_mid() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LR_JACOBI_CL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// CTAs of the cluster Jacobi (warps spread over more SMs: fewer warps per SM
// contending for the shuffle / FP64 pipes on the latency-bound subrounds).
// Measured (tools/small_probe.py, MIXED): real 110: 2 CTAs 1252 us, 4: 1050,
// 8: 1039; complex 120: 2416 / 1931 / 2058; real 256: 4 CTAs 4578 us, 8: 3622.
// LR_JACOBI_CLN overrides (2 | 4 | 8 | 16).
static int cln(int def) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LR_JACOBI_CLN");
    v = e ? atoi(e) : 0;
  }
  return v ? v : def;
}

void jacobi_blk_f64(Handle* h, int64_t n, const double* R, double* Mout, double* sig,
                    int32_t* info) {
  // thread count = 32 * ceil(ceil(n/4)/2): the register budget per thread is
  // 64K / threads, so the widest case of each row count gets its own bound
  if (n <= 32) launch_blk<double, 1, 128>(h, int(n), R, Mout, sig, info);
  else if (n <= 64) launch_blk<double, 2, 256>(h, int(n), R, Mout, sig, info);
  else if (n <= 80) launch_blk<double, 3, 320>(h, int(n), R, Mout, sig, info);
  else if (n <= 96) launch_blk<double, 3, 384>(h, int(n), R, Mout, sig, info);
  else if (n <= 128 && cl_mid() && cln(8) == 8) launch_cl<double, 4, 8, 2>(h, int(n), R, Mout, sig, info);
  else if (n <= 128 && cl_mid() && cln(8) == 4) launch_cl<double, 4, 4, 4>(h, int(n), R, Mout, sig, info);
  else if (n <= 128 && cl_mid()) launch_cl<double, 4, 2, 8>(h, int(n), R, Mout, sig, info);
  else if (n <= 112) launch_blk<double, 4, 448>(h, int(n), R, Mout, sig, info);
  else if (n <= 128) launch_blk<double, 4, 512>(h, int(n), R, Mout, sig, info);
  else if (cln(8) == 16) launch_cl<double, 8, 16, 2>(h, int(n), R, Mout, sig, info);
  else if (cln(8) == 8) launch_cl<double, 8, 8, 4>(h, int(n), R, Mout, sig, info);
  else launch_cl<double, 8, 4, 8>(h, int(n), R, Mout, sig, info);
}

void jacobi_blk_c128(Handle* h, int64_t n, const double2* R, double2* Mout, double* sig,
                     int32_t* info) {
  if (n <= 32) launch_blk<double2, 1, 128>(h, int(n), R, Mout, sig, info);
  else if (n <= 48) launch_blk<double2, 2, 192>(h, int(n), R, Mout, sig, info);
  else if (n <= 64) launch_blk<double2, 2, 256>(h, int(n), R, Mout, sig, info);
  else if (cln(4) == 8) launch_cl<double2, 4, 8, 2>(h, int(n), R, Mout, sig, info);
  else if (cln(4) == 4) launch_cl<double2, 4, 4, 4>(h, int(n), R, Mout, sig, info);
  else launch_cl<double2, 4, 2, 8>(h, int(n), R, Mout, sig, info);
}

}  // namespace lr
