// K3 core, blocked: Cholesky with column deletion + inverse, one CTA.
//
// Same contract as chol.cu (the rank decision of orthonormalize_double_gs,
// reference core.py:84-115, restated on the Gram matrix: the pivot of column
// j is the squared residual of y_j against the kept columns before it),
// organised in 32-column blocks so the CTA synchronizes O(ell/32) times
// instead of O(ell):
//   for each diagonal block k:
//     warp 0 factors the 32 x 32 block in registers (lane c owns column c,
//     pivots broadcast by shuffles, drop / unresolved decision per column)
//     and inverts it (D_k = R_kk^{-1}, back substitution per lane);
//     all warps form the panel R_k,> = D_k^H G_k,> and the trailing update
//     G_>,> -= R_k,>^H R_k,>;
//   X = R~^{-1} by block superdiagonals: X_kk = D_k,
//     X_ij = -D_i sum_{k=i+1..j} R_ik X_kj.
// Dropped columns get zero rows/columns in R and identity in R~, so they
// drop out of every later projection, as the reference skips them.
//
// Storage (padded size np = 32 * ceil(n / 32)): one np x np buffer W whose
// strict upper triangle holds R (G before factorization) and whose lower
// triangle including the diagonal holds X^T; the R diagonal lives in rd[];
// a 32 x np scratch TB holds panel / block-inverse temporaries.
#include "common.cuh"
#include "scalar.cuh"

namespace lr {
namespace {

constexpr int CB = 32;      // block size
constexpr int CBT = 256;    // threads (warp 0 keeps a 32-entry column in registers)

template <typename T, bool SMEM>
__global__ void __launch_bounds__(CBT, 1)
chol_blocked_kernel(int n, const T* __restrict__ G, double drop_tol, double unres_rel,
                    double shift_coef, T* __restrict__ P, T* __restrict__ Rout,
                    int32_t* __restrict__ info, T* gbuf, int32_t* status) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int np = ((n + CB - 1) / CB) * CB;
  const int nb = np / CB;
  T* __restrict__ W;
  T* __restrict__ TB;
  unsigned char* tail;
  if constexpr (SMEM) {
    W = reinterpret_cast<T*>(smem_raw);
    TB = W + size_t(np) * np;
    tail = reinterpret_cast<unsigned char*>(TB + size_t(CB) * np);
  } else {
    W = gbuf;
    TB = gbuf + size_t(np) * np;
    tail = smem_raw;
  }
  double* d0 = reinterpret_cast<double*>(tail);   // original (shifted) pivots
  double* rd = d0 + np;                           // R diagonal, 0 = dropped
  int* pos = reinterpret_cast<int*>(rd + np);     // compact index or -1
  int* kidx = pos + np;                           // compact -> original

  __shared__ double s_red[CBT / 32];
  __shared__ int s_unres, s_bad, s_rank;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#define WIJ(i, j) W[size_t(i) * np + (j)]
#define XIJ(i, j) W[size_t(j) * np + (i)]   /* X[i][j], i <= j, stored transposed */

  // 0. load the upper triangle of G, identity padding, trace
  double tr = 0.0;
  for (int e = tid; e < np * np; e += CBT) {
    const int i = e / np, j = e - i * np;
    T v = S::zero();
    if (j >= i) {
      if (i < n && j < n) {
        v = G[size_t(i) * n + j];
        if (i == j) tr += S::re(v);
      } else if (i == j) {
        v = S::one();
      }
    }
    W[e] = v;
  }
  for (int m = 16; m > 0; m >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, m);
  if (lane == 0) s_red[warp] = tr;
  if (tid == 0) { s_unres = 0; s_bad = 0; }
  __syncthreads();
  double trace = 0.0;
#pragma unroll
  for (int w = 0; w < CBT / 32; ++w) trace += s_red[w];
  const double thr2 = drop_tol * drop_tol * trace;
  const double shift = shift_coef * trace;
  for (int i = tid; i < np; i += CBT) {
    double d = 1.0;
    if (i < n) {
      d = S::re(WIJ(i, i)) + shift;
      WIJ(i, i) = S::make(d, 0.0);
    }
    d0[i] = d;
  }
  __syncthreads();

  for (int kb = 0; kb < nb; ++kb) {
    const int j0 = kb * CB;
    // (1) warp 0: factor and invert the diagonal block
    if (warp == 0) {
      T a[CB];   // lane c: column j0+c of R, rows j0..j0+c
#pragma unroll
      for (int i = 0; i < CB; ++i) a[i] = (i <= lane) ? WIJ(j0 + i, j0 + lane) : S::zero();
      int unres = 0, bad = 0;
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        const double d = __shfl_sync(0xffffffffu, S::re(a[k]), k);
        const bool pad = (j0 + k) >= n;
        const bool fin = isfinite(d);
        const bool keep = pad || (fin && d > thr2 && d > 0.0);
        bad += (!pad && !fin) ? 1 : 0;
        if (keep) {
          const double iv = rsqrt(d);
          unres += (!pad && d <= unres_rel * d0[j0 + k]) ? 1 : 0;
          const double rk = d * iv;
          if (lane == 0) rd[j0 + k] = rk;
          if (lane > k) a[k] = S::scale(a[k], iv);
          else if (lane == k) a[k] = S::make(rk, 0.0);
#pragma unroll
          for (int i = k + 1; i < CB; ++i) {
            const T rki = S::shfl_idx(a[k], i);
            if (lane >= i) a[i] = S::sub(a[i], S::mul(S::conj(rki), a[k]));
          }
        } else {
          if (lane == 0) rd[j0 + k] = 0.0;
          if (lane >= k) a[k] = S::zero();       // row k of R
          if (lane == k) {                       // column k of R (deletion)
#pragma unroll
            for (int i = 0; i < CB; ++i) a[i] = S::zero();
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CB; ++i)
        if (i < lane) WIJ(j0 + i, j0 + lane) = a[i];
      __syncwarp();
      // D = R~_kk^{-1}: lane c solves R~ d = e_c by back substitution
      T dcol[CB];
#pragma unroll
      for (int i = CB - 1; i >= 0; --i) {
        T acc = (i == lane) ? S::one() : S::zero();
#pragma unroll
        for (int k2 = i + 1; k2 < CB; ++k2)
          if (k2 <= lane) acc = S::sub(acc, S::mul(WIJ(j0 + i, j0 + k2), dcol[k2]));
        const double ri = rd[j0 + i];
        const double rii = ri > 0.0 ? ri : 1.0;   // R~: identity on drops
        dcol[i] = (i <= lane) ? S::div_re(acc, rii) : S::zero();
      }
#pragma unroll
      for (int i = 0; i < CB; ++i)
        if (i <= lane) XIJ(j0 + i, j0 + lane) = dcol[i];
      if (lane == 0) {
        atomicAdd(&s_unres, unres);
        atomicAdd(&s_bad, bad);
      }
    }
    __syncthreads();
    if (kb + 1 == nb) break;
    const int c0 = j0 + CB, nc = np - c0;
    // (2) panel R_k,> = D^H G_k,>  (rows of dropped pivots -> 0), into TB;
    //     4 x 4 register tiles (rows i, columns c)
    {
      const int tc = nc / 4;
      for (int t = tid; t < 8 * tc; t += CBT) {
        const int i0 = (t / tc) * 4, cc0 = c0 + (t % tc) * 4;
        T acc[4][4];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = S::zero();
        for (int k = 0; k <= i0 + 3; ++k) {
          T xa[4], gb[4];
#pragma unroll
          for (int p = 0; p < 4; ++p)
            xa[p] = (k <= i0 + p) ? S::conj(XIJ(j0 + k, j0 + i0 + p)) : S::zero();
#pragma unroll
          for (int q = 0; q < 4; ++q) gb[q] = WIJ(j0 + k, cc0 + q);
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] = S::add(acc[p][q], S::mul(xa[p], gb[q]));
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const bool dropped = rd[j0 + i0 + p] == 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            TB[size_t(i0 + p) * np + cc0 + q] = dropped ? S::zero() : acc[p][q];
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < CB * nc; e += CBT) {
      const int i = e / nc, c = c0 + (e - i * nc);
      WIJ(j0 + i, c) = TB[size_t(i) * np + c];
    }
    // (3) trailing update G_ab -= sum_i conj(R_ia) R_ib for c0 <= a <= b (4 x 4 tiles)
    {
      const int tn = nc / 4;
      for (int t = tid; t < tn * tn; t += CBT) {
        const int ta = t / tn, tb = t % tn;
        if (tb < ta) continue;
        const int a0 = c0 + ta * 4, b0 = c0 + tb * 4;
        T acc[4][4];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = S::zero();
#pragma unroll 4
        for (int i = 0; i < CB; ++i) {
          T ra[4], rb[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) ra[p] = S::conj(TB[size_t(i) * np + a0 + p]);
#pragma unroll
          for (int q = 0; q < 4; ++q) rb[q] = TB[size_t(i) * np + b0 + q];
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] = S::add(acc[p][q], S::mul(ra[p], rb[q]));
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (b0 + q >= a0 + p) WIJ(a0 + p, b0 + q) = S::sub(WIJ(a0 + p, b0 + q), acc[p][q]);
      }
    }
    __syncthreads();
  }

  // zero R entries in columns of dropped pivots (panels computed them)
  for (int e = tid; e < np * np; e += CBT) {
    const int i = e / np, c = e - i * np;
    if (c > i && rd[c] == 0.0) WIJ(i, c) = S::zero();
  }
  // compaction of kept columns
  if (warp == 0) {
    int base = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool k = j < n && rd[j] > 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      const int pj = base + __popc(bal & ((1u << lane) - 1u));
      if (j < n) pos[j] = k ? pj : -1;
      if (k) kidx[pj] = j;
      base += __popc(bal);
    }
    if (lane == 0) s_rank = base;
  }
  __syncthreads();

  // (4) off-diagonal blocks of X by superdiagonals (4 x 4 register tiles)
  for (int d = 1; d < nb; ++d) {
    const int nbl = nb - d;   // blocks (bi, bi + d)
    // T_ij = sum_{k=bi+1..bj} R_{bi,k} X_{k,bj}
    for (int t = tid; t < nbl * 64; t += CBT) {
      const int blk = t / 64, r0 = ((t % 64) / 8) * 4, q0 = (t % 8) * 4;
      const int bi = blk, bj = blk + d;
      const int r = bi * CB + r0, c = bj * CB + q0;
      T acc[4][4];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = S::zero();
      for (int k = (bi + 1) * CB; k <= c + 3; ++k) {
        T ra[4], xb[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) ra[p] = WIJ(r + p, k);
#pragma unroll
        for (int q = 0; q < 4; ++q) xb[q] = (k <= c + q) ? XIJ(k, c + q) : S::zero();
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = S::add(acc[p][q], S::mul(ra[p], xb[q]));
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) TB[size_t(blk) * CB * CB + (r0 + p) * CB + q0 + q] = acc[p][q];
    }
    __syncthreads();
    // X_ij = -D_i T_ij
    for (int t = tid; t < nbl * 64; t += CBT) {
      const int blk = t / 64, r0 = ((t % 64) / 8) * 4, q0 = (t % 8) * 4;
      const int bi = blk, bj = blk + d;
      const int r = bi * CB + r0, c = bj * CB + q0;
      T acc[4][4];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = S::zero();
      for (int k = r0; k < CB; ++k) {
        T da[4], tb[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) da[p] = (k >= r0 + p) ? XIJ(r + p, bi * CB + k) : S::zero();
#pragma unroll
        for (int q = 0; q < 4; ++q) tb[q] = TB[size_t(blk) * CB * CB + k * CB + q0 + q];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = S::add(acc[p][q], S::mul(da[p], tb[q]));
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) XIJ(r + p, c + q) = S::scale(acc[p][q], -1.0);
    }
    __syncthreads();
  }

  // (5) outputs
  const int rank = s_rank;
  for (int e = tid; e < n * n; e += CBT) {
    const int i = e / n, j = e - (e / n) * n;
    T r = S::zero();
    if (pos[i] >= 0 && pos[j] >= 0) {
      if (j > i) r = WIJ(i, j);
      else if (j == i) r = S::make(rd[i], 0.0);
    }
    Rout[e] = r;
    T pv = S::zero();
    if (pos[i] >= 0 && j < rank) {
      const int c = kidx[j];
      if (i <= c) pv = XIJ(i, c);
    }
    P[e] = pv;
  }
  if (tid == 0) {
    info[0] = rank;
    info[1] = s_unres;
    info[2] = s_bad;
    if (status) {
      const int bits = (s_unres ? 1 : 0) | (rank < n ? 2 : 0) | (s_bad ? 4 : 0);
      if (bits) atomicOr(status, bits);
    }
  }
#undef WIJ
#undef XIJ
}

}  // namespace

template <typename T>
bool chol_blocked_launch(Handle* h, int64_t ell, const T* G, double drop_tol, double unres_rel,
                         double shift_coef, T* P, T* R, int32_t* info) {
  const int n = int(ell);
  const int np = ((n + CB - 1) / CB) * CB;
  const size_t tail = size_t(np) * (2 * sizeof(double) + 2 * sizeof(int));
  const size_t bufs = (size_t(np) * np + size_t(CB) * np) * sizeof(T);
  int max_smem = 0;
  LR_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  if (bufs + tail <= size_t(max_smem) - 2048) {
    auto kern = chol_blocked_kernel<T, true>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(bufs + tail)));
    kern<<<1, CBT, bufs + tail, h->stream>>>(n, G, drop_tol, unres_rel, shift_coef, P, R, info,
                                             nullptr, h->status);
  } else {
    T* g = static_cast<T*>(pool_alloc(h, bufs));
    auto kern = chol_blocked_kernel<T, false>;
    LR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tail)));
    kern<<<1, CBT, tail, h->stream>>>(n, G, drop_tol, unres_rel, shift_coef, P, R, info, g,
                                      h->status);
  }
  LR_CHECK_LAUNCH();
  return true;
}

template bool chol_blocked_launch<double>(Handle*, int64_t, const double*, double, double, double,
                                          double*, double*, int32_t*);
template bool chol_blocked_launch<double2>(Handle*, int64_t, const double2*, double, double,
                                           double, double2*, double2*, int32_t*);

}  // namespace lr
