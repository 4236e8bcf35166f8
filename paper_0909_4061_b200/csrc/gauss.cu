// K0: the reference's Gaussian sketch Omega, generated on the GPU.
//
// The reference draws Omega with numpy's Generator(Philox(key)).
// standard_normal (reference sketch.py:32-42, 96-100; rangefinder.py:78 for
// the estimator probes): Philox4x64-10 (counter starting at 1, four uint64
// per block) feeding a 256-layer ziggurat.  On the host that costs ~30 ns
// per draw (26 ms for config 2's 8192 x 110 Omega, ~3 s for config 5's
// 2^21 x 48); here the same stream is produced on the device.
//
// The ziggurat consumes a variable number of uint64 per normal (99.3 % take
// one; the wedge takes two, the tail 1 + 2k), so the stream is not
// trivially parallel.  Three passes make it so:
//   A  every stream position t is evaluated as if an attempt started there:
//      value, #uint64 consumed c(t), whether it yields a normal;
//   B  "special" positions (c > 1 or rejected) are rare and only interact
//      within 64 positions; a special with no special in the 63 positions
//      before it is certainly an attempt start (a "head"), and one thread per
//      head walks its short cluster, marking the positions consumed as
//      continuation draws;
//   C  a prefix sum over {start and yields} assigns output indices.
// Tables: numpy's own ziggurat tables (ziggurat_tables.cuh, extracted and
// verified by tools/philox_ziggurat.py).  The tail/wedge use log1p/exp; the
// result equals numpy's stream bit for bit except possibly the last ulp of
// tail draws (|x| > 3.654) where CUDA's log1p could round differently from
// glibc's (tests/test_gpu_kernels.py counts mismatches).
#include "common.cuh"
#include "ziggurat_tables.cuh"

namespace lr {
namespace {

constexpr int MAXC = 64;   // max uint64 one attempt may consume (cap; flagged)
constexpr double ZIG_R = 3.6541528853610087963519472518;
constexpr double ZIG_INV_R = 0.27366123732975827203338247596;

struct PhiloxKey {
  uint64_t k0, k1;
};

__device__ __forceinline__ void philox4x64_10(uint64_t ctr0, PhiloxKey key, uint64_t (&out)[4]) {
  uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
  uint64_t k0 = key.k0, k1 = key.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0), lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c2), lo1 = 0xCA5A826395121157ULL * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// stream position t (0-based) = word t % 4 of block counter t / 4 + 1
__device__ __forceinline__ uint64_t raw_at(PhiloxKey key, int64_t t) {
  uint64_t o[4];
  philox4x64_10(uint64_t(t >> 2) + 1, key, o);
  const int w = int(t & 3);
  return w == 0 ? o[0] : w == 1 ? o[1] : w == 2 ? o[2] : o[3];
}

__device__ __forceinline__ double next_double(uint64_t u) {
  return double(u >> 11) * (1.0 / 9007199254740992.0);
}

// flags byte: bit7 yields a normal, bit6 continuation draw (set by pass B),
// bits0-5 draws consumed by an attempt starting here (0x3f without bit7 = cap overflow)
__device__ __forceinline__ bool is_special(uint8_t f) { return (f & 0x3f) != 1 || !(f & 0x80); }

// pass A: one thread per Philox block (4 positions), a warp per 128
// positions; besides value and flags it writes the bitmask of "special"
// positions (one uint32 per 32 positions) that pass B scans.  The ziggurat
// tables are indexed by random bytes: staged in shared memory (a __constant__
// lookup with 32 different addresses per warp serializes 32-fold).
__global__ void __launch_bounds__(256)
gauss_eval(PhiloxKey key, int64_t L, double* __restrict__ val, uint8_t* __restrict__ flags,
           uint32_t* __restrict__ smask) {
  __shared__ uint64_t ki[256];
  __shared__ double wi[256], fi[256];
  ki[threadIdx.x] = kZigKi[threadIdx.x];
  wi[threadIdx.x] = kZigWi[threadIdx.x];
  fi[threadIdx.x] = kZigFi[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t blocks = (L + 3) >> 2;
  const int64_t wstride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t bw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) - lane; bw < blocks;
       bw += wstride) {
    const int64_t b = bw + lane;
    uint32_t nib = 0;
    if (b < blocks) {
      uint64_t o[4];
      philox4x64_10(uint64_t(b) + 1, key, o);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int64_t t = b * 4 + w;
        if (t >= L) break;
        const uint64_t u = o[w];
        const int idx = int(u & 0xff);
        const uint64_t r = u >> 8;
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = double(rabs) * wi[idx];
        if (r & 1) x = -x;
        uint8_t f;
        if (rabs < ki[idx]) {
          f = 0x80 | 1;
        } else if (idx != 0) {
          const double nd = next_double(raw_at(key, t + 1));
          const bool yes = ((fi[idx - 1] - fi[idx]) * nd + fi[idx]) < exp(-0.5 * x * x);
          f = uint8_t((yes ? 0x80 : 0) | 2);
        } else {
          int64_t j = t + 1;
          int used = 1;
          f = 0x3f;   // overflow marker (c = 63, no yield) unless accepted within the cap
          while (used + 2 < MAXC) {
            const double xx = -ZIG_INV_R * log1p(-next_double(raw_at(key, j)));
            const double yy = -log1p(-next_double(raw_at(key, j + 1)));
            j += 2;
            used += 2;
            if (yy + yy > xx * xx) {
              x = ((rabs >> 8) & 1) ? -(ZIG_R + xx) : ZIG_R + xx;
              f = uint8_t(0x80 | used);
              break;
            }
          }
        }
        val[t] = x;
        flags[t] = f;
        if (is_special(f)) nib |= 1u << w;
      }
    }
    // lanes 8k..8k+7 hold positions 32k..32k+31 of this warp's 128
    uint32_t word = nib << (4 * (lane & 7));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    const int64_t wi32 = (bw >> 3) + (lane >> 3);   // (bw * 4) / 32 + k
    if ((lane & 7) == 0 && wi32 * 32 < L) smask[wi32] = word;
  }
}

__device__ __forceinline__ uint32_t mask_word(const uint32_t* smask, int64_t k, int64_t W) {
  return (k >= 0 && k < W) ? smask[k] : 0u;
}

// first special position in [p, min(p + 64, L)), or -1
__device__ __forceinline__ int64_t next_special(const uint32_t* smask, int64_t W, int64_t L,
                                                int64_t p) {
  const int64_t end = min(p + MAXC, L);
  for (int64_t q = p; q < end;) {
    const int64_t k = q >> 5;
    const uint32_t m = mask_word(smask, k, W) >> (q & 31);
    if (m) {
      const int64_t r = q + __ffs(m) - 1;
      return r < end ? r : -1;
    }
    q = (k + 1) << 5;
  }
  return -1;
}

// pass B: mark continuation draws (bit6 of flags) by walking from each head.
// One thread per 32 positions; a special position is a head iff the 63
// positions before it hold no special (read off the bitmask, not the bytes).
__global__ void gauss_fixup(int64_t L, uint8_t* __restrict__ flags,
                            const uint32_t* __restrict__ smask, int32_t* status) {
  const int64_t W = (L + 31) >> 5;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < W;
       k += int64_t(gridDim.x) * blockDim.x) {
    uint32_t m = smask[k];
    if (!m) continue;
    const uint64_t lo = (uint64_t(mask_word(smask, k - 1, W)) << 32) | mask_word(smask, k - 2, W);
    while (m) {
      const int i = __ffs(m) - 1;
      m &= m - 1;
      // bits of positions t-63 .. t-1 (t = 32k + i at bit 64 + i of m:lo)
      const uint64_t win =
          ((lo >> (i + 1)) | (uint64_t(smask[k]) << (63 - i))) & 0x7fffffffffffffffULL;
      if (win) continue;
      int64_t p = k * 32 + i;
      for (;;) {   // walk the cluster: p is always an attempt start here
        const uint8_t g = flags[p];
        const int c = g & 0x3f;
        if (c == 0x3f && !(g & 0x80)) {   // cap exceeded
          if (status) atomicOr(status, 16);
          break;
        }
        for (int j = 1; j < c && p + j < L; ++j) flags[p + j] |= 0x40;
        p += c;
        if (p >= L) break;
        p = next_special(smask, W, L, p);   // fast starts in between
        if (p < 0) break;
      }
    }
  }
}

__device__ __forceinline__ int keep_of(uint8_t f) { return ((f & 0x80) && !(f & 0x40)) ? 1 : 0; }

constexpr int SCAN_T = 512;
constexpr int SCAN_E = 8;                  // elements per thread
constexpr int SCAN_B = SCAN_T * SCAN_E;    // positions per block

__global__ void gauss_count(int64_t L, const uint8_t* __restrict__ flags, int32_t* __restrict__ bsum) {
  __shared__ int red[SCAN_T / 32];
  const int64_t base = int64_t(blockIdx.x) * SCAN_B;
  int c = 0;
  for (int e = 0; e < SCAN_E; ++e) {
    const int64_t t = base + int64_t(threadIdx.x) * SCAN_E + e;
    if (t < L) c += keep_of(flags[t]);
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < SCAN_T / 32; ++w) s += red[w];
    bsum[blockIdx.x] = s;
  }
}

// exclusive scan of the block sums (single CTA, sequential chunks)
__global__ void gauss_scan_bsum(int nb, int32_t* __restrict__ bsum, int64_t* __restrict__ boff,
                                int64_t count, int32_t* status) {
  __shared__ int64_t carry;
  __shared__ int64_t part[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const int64_t v = i < nb ? bsum[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t add = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < nb) boff[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0 && carry < count && status) atomicOr(status, 32);   // stream too short
}

template <typename TO>
__global__ void gauss_scatter(int64_t L, const double* __restrict__ val,
                              const uint8_t* __restrict__ flags, const int64_t* __restrict__ boff,
                              int64_t count, TO* __restrict__ out) {
  __shared__ int wsum[SCAN_T / 32];
  const int64_t base = int64_t(blockIdx.x) * SCAN_B + int64_t(threadIdx.x) * SCAN_E;
  int k[SCAN_E];
  int c = 0;
#pragma unroll
  for (int e = 0; e < SCAN_E; ++e) {
    const int64_t t = base + e;
    k[e] = t < L ? keep_of(flags[t]) : 0;
    c += k[e];
  }
  // block-exclusive scan of per-thread counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < SCAN_T / 32 ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane < SCAN_T / 32) wsum[lane] = v;
  }
  __syncthreads();
  int64_t pos = boff[blockIdx.x] + (warp ? wsum[warp - 1] : 0) + (incl - c);
#pragma unroll
  for (int e = 0; e < SCAN_E; ++e) {
    if (k[e]) {
      if (pos < count) out[pos] = TO(val[base + e]);
      ++pos;
    }
  }
}

}  // namespace

void gaussian_stream(Handle* h, uint64_t key_lo, uint64_t key_hi, int64_t count, int out_dtype,
                     void* out) {
  if (count <= 0) return;
  const int64_t L = count + count / 32 + 4096;
  double* val = pool_alloc_t<double>(h, size_t(L));
  uint8_t* flags = pool_alloc_t<uint8_t>(h, size_t(L));
  const int64_t nb = ceil_div(L, SCAN_B);
  int32_t* bsum = pool_alloc_t<int32_t>(h, size_t(nb));
  int64_t* boff = pool_alloc_t<int64_t>(h, size_t(nb));
  uint32_t* smask = pool_alloc_t<uint32_t>(h, size_t((L + 31) / 32));
  PhiloxKey key{key_lo, key_hi};
  const int grid = int(std::min<int64_t>(ceil_div(ceil_div(L, 4), 256), int64_t(h->sm_count) * 32));
  gauss_eval<<<grid, 256, 0, h->stream>>>(key, L, val, flags, smask);
  LR_CHECK_LAUNCH();
  const int grid2 = int(std::min<int64_t>(ceil_div(ceil_div(L, 32), 256), int64_t(h->sm_count) * 8));
  gauss_fixup<<<grid2, 256, 0, h->stream>>>(L, flags, smask, h->status);
  LR_CHECK_LAUNCH();
  gauss_count<<<unsigned(nb), SCAN_T, 0, h->stream>>>(L, flags, bsum);
  LR_CHECK_LAUNCH();
  gauss_scan_bsum<<<1, 1024, 0, h->stream>>>(int(nb), bsum, boff, count, h->status);
  LR_CHECK_LAUNCH();
  if (out_dtype == LR_F64)
    gauss_scatter<double><<<unsigned(nb), SCAN_T, 0, h->stream>>>(L, val, flags, boff, count,
                                                                   static_cast<double*>(out));
  else if (out_dtype == LR_F32)
    gauss_scatter<float><<<unsigned(nb), SCAN_T, 0, h->stream>>>(L, val, flags, boff, count,
                                                                  static_cast<float*>(out));
  else
    throw Error{LR_EINVAL, "gaussian: output dtype must be f32 or f64"};
  LR_CHECK_LAUNCH();
}

}  // namespace lr
