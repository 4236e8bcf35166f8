// K3 preconditioner for tall fp32 panels: a sparse-sign row sketch S Y of the
// m x ell sample panel (S: d x m, ZETA = 2 entries +-1 per column), one read of
// Y, exact fp64 accumulation.
//
// Why: orthonormalize_double_gs (reference core.py:84-115) of a panel with
// kappa(Y) ~ 1e6 (config 4) needs an R factor accurate to kappa^2 u -- an fp64
// Gram.  The exact Gram of an m x 256 fp32 panel costs m ell^2 DMMA flops
// (2.97 ms at m = 2^20).  The QR factor R0 of the SKETCH (d = 1024 rows, fp64)
// is a preconditioner instead: S is a subspace embedding of range(Y), so
// Q1 = Y R0^{-1} has kappa(Q1) <= ~3 whatever kappa(Y) was, and the second
// CholeskyQR pass on Q1 (tensor-core Gram, fp32-level accuracy suffices at
// kappa ~ 3) finishes the job.  R0 and R2 are upper triangular, so Q = Y
// (R2 R0)^{-1} is the same Gram-Schmidt basis as before up to roundoff.  The
// embedding is certified a posteriori: the second pass's Cholesky flags any
// pivot below 1e-3 of its diagonal (kappa(Q1)^2 > 1e3), which reruns the step
// on the exact path.
//
// Kernel: grid (ell / 16 column slices, row chunks).  A CTA keeps its d x 16
// slice of the sketch in shared memory as fp64 (128 KiB) and streams its rows:
// every half-warp takes one row per step (16 lanes = 16 columns, one 64-byte
// segment) and adds it, signed, to two bucket rows.  Half-warp w only ever
// touches buckets = w (mod 32), so no two half-warps race and no atomics are
// needed; within a half-warp the program order of one thread per column
// serializes updates of the same bucket.  The row's two buckets lie in
// different halves of the bucket range, so they never coincide.  The same
// pass reduces max|Y| (the scale of the tensor-core split that applies
// R0^{-1}), saving that kernel a read of Y.
#include "common.cuh"

namespace lr {
namespace {

constexpr int SK_W = 16;        // columns per slice
constexpr int SK_D = 1024;      // sketch rows
constexpr int SK_THREADS = 512;
constexpr int SK_HW = SK_THREADS / 16;            // half-warps (owner groups): 32
constexpr int SK_T = SK_D / 2 / SK_HW;            // buckets per owner per half: 16
constexpr int SK_U = 16;                          // rows in flight per half-warp

// murmur3's 32-bit finalizer: the bucket / sign bits of one row
__device__ __forceinline__ uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__global__ void __launch_bounds__(SK_THREADS, 1)
sketch_rows_kernel(int64_t m, int ell, const float* __restrict__ Y, int64_t ldy, uint64_t seed,
                   int64_t rows_per_chunk, double* __restrict__ part,
                   unsigned int* __restrict__ amax_bits) {
  extern __shared__ double acc[];   // [SK_D][SK_W]
  const int tid = threadIdx.x;
  for (int e = tid; e < SK_D * SK_W; e += SK_THREADS) acc[e] = 0.0;
  __syncthreads();
  const int hw = tid >> 4, c = tid & 15;
  const int col = blockIdx.x * SK_W + c;
  const bool col_ok = col < ell;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = min(m, r0 + rows_per_chunk);
  const float* yc = Y + (col_ok ? col : 0);
  float amax = 0.f;
  double* a0 = acc + hw * SK_W + c;                       // bucket hw + 32 t, lower half
  double* a1 = acc + (SK_D / 2 + hw) * SK_W + c;          // upper half
  // The first version computed a 64-bit hash per row in every lane: 48 warp
  // instructions per row step, issue-bound at 0.57 ms (ncu: issue active 67 %,
  // 408 M instructions).  Here lane c of a half-warp hashes row c of the batch
  // of SK_U = 16 rows and the packed result travels by one shuffle per row.
  static_assert(SK_U == 16, "one hashed row per lane of the half-warp");
  static_assert(SK_T == 16 && SK_HW * SK_W * 8 == 4096, "4-bit bucket fields, 4 KiB apart");
  const uint32_t seed_lo = uint32_t(seed), seed_hi = uint32_t(seed >> 32);
  const int src0 = threadIdx.x & 16;                      // first lane of my half-warp
  char* b0 = reinterpret_cast<char*>(a0);
  char* b1 = reinterpret_cast<char*>(a1);
  // (a lane past the last column streams column 0 into a slice column nobody
  // stores: no predicate in the loop, and max|Y| is unaffected)
  const int64_t stride = int64_t(SK_HW) * ldy;
  const float* p = yc + (r0 + hw) * ldy;
  for (int64_t base = r0; base < r1; base += int64_t(SK_HW) * SK_U, p += SK_U * stride) {
    float v[SK_U];
    if (base + int64_t(SK_HW) * SK_U <= r1) {
#pragma unroll
      for (int u = 0; u < SK_U; ++u) v[u] = __ldg(p + u * stride);
    } else {
#pragma unroll
      for (int u = 0; u < SK_U; ++u)
        v[u] = (base + int64_t(u) * SK_HW + hw < r1) ? __ldg(p + u * stride) : 0.f;
    }
    uint32_t mypk;
    {
      const int64_t r = base + int64_t(c) * SK_HW + hw;
      const uint32_t hsh = mix32((uint32_t(r) ^ seed_lo) + 0x9e3779b9u * (uint32_t(uint64_t(r) >> 32) ^ seed_hi));
      // bits 12..15: byte offset t0 << 12 of the lower bucket, bits 20..23: t1, bits 0 / 1: signs
      mypk = ((hsh & 15u) << 12) | (((hsh >> 4) & 15u) << 20) | ((hsh >> 8) & 3u);
    }
#pragma unroll
    for (int u = 0; u < SK_U; ++u) {
      const uint32_t pk = __shfl_sync(0xffffffffu, mypk, src0 | u);
      const double x = double(v[u]);
      const int hi = __double2hiint(x), lo = __double2loint(x);
      const double x0 = __hiloint2double(hi ^ int(pk << 31), lo);
      const double x1 = __hiloint2double(hi ^ int((pk << 30) & 0x80000000u), lo);
      amax = fmaxf(amax, fabsf(v[u]));
      double* p0 = reinterpret_cast<double*>(b0 + (pk & 0xf000u));
      double* p1 = reinterpret_cast<double*>(b1 + ((pk >> 8) & 0xf000u));
      const double s0 = *p0, s1 = *p1;   // distinct addresses: independent chains
      *p0 = s0 + x0;
      *p1 = s1 + x1;
    }
  }
  // max|Y| (NaN maps above every finite value so a non-finite panel is seen)
  unsigned int bits = __float_as_uint(amax);
  if (amax != amax) bits = 0x7fc00000u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, o));
  if ((tid & 31) == 0 && bits) atomicMax(amax_bits, bits);
  __syncthreads();
  // partial sketch of this chunk: part[chunk][d][ell]
  double* out = part + int64_t(blockIdx.y) * SK_D * ell;
  for (int e = tid; e < SK_D * SK_W; e += SK_THREADS) {
    const int b = e / SK_W, cc = e % SK_W;
    const int gc = blockIdx.x * SK_W + cc;
    if (gc < ell) out[int64_t(b) * ell + gc] = acc[e];
  }
}

__global__ void sketch_reduce_kernel(int64_t total, int chunks, const double* __restrict__ part,
                                     double scale, double* __restrict__ SY) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < chunks; ++k) s += part[int64_t(k) * total + i];
    SY[i] = s * scale;
  }
}

}  // namespace

int64_t sketch_rows_dim() { return SK_D; }

bool sketch_rows_supported(int64_t m, int64_t ell) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("LR_SKETCH_QR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  // worth it (and an embedding: d >= 4 ell) for tall panels only
  return on && ell >= 16 && ell <= SK_D / 4 && m >= 64 * SK_D;
}

// SY (SK_D x ell, fp64, ld ell) = S Y / sqrt(2), amax_bits = float bits of max|Y|.
// `seed` selects S (a sharded caller passes a different seed per rank: the
// sum of the ranks' sketches is then one sketch of the stacked panel).
void sketch_rows_f32(Handle* h, int64_t m, int64_t ell, const float* Y, int64_t ldy,
                     uint64_t seed, double* SY, unsigned int* amax_bits) {
  const int slices = int(ceil_div(ell, SK_W));
  int chunks = std::max(1, h->sm_count / slices);
  const int64_t step = int64_t(SK_HW) * SK_U;
  const int64_t rows_per_chunk = ceil_div(ceil_div(m, chunks), step) * step;
  chunks = int(ceil_div(m, rows_per_chunk));
  double* part = pool_alloc_t<double>(h, size_t(chunks) * SK_D * ell);
  LR_CUDA(cudaMemsetAsync(amax_bits, 0, sizeof(unsigned int), h->stream));
  static AttrOnce once;
  const size_t smem = size_t(SK_D) * SK_W * sizeof(double);
  once([&] {
    LR_CUDA(cudaFuncSetAttribute(sketch_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
  });
  sketch_rows_kernel<<<dim3(slices, chunks), SK_THREADS, smem, h->stream>>>(
      m, int(ell), Y, ldy, seed, rows_per_chunk, part, amax_bits);
  LR_CHECK_LAUNCH();
  const int64_t total = int64_t(SK_D) * ell;
  sketch_reduce_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, h->stream>>>(
      total, chunks, part, 0.70710678118654752440, SY);
  LR_CHECK_LAUNCH();
}

}  // namespace lr
