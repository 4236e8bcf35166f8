// Development microbenchmark: dependent-chain latencies on the B200 of the
// operations the latency-bound kernels (Cholesky, Jacobi) are built from.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dmul(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * b;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ffma(float* out, float a, float b, int n, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmaf(x, b, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_rsq(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, int n, long long* cyc) {
  __shared__ int buf[1024];
  buf[threadIdx.x] = (threadIdx.x + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = buf[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 16);
  cudaMalloc(&c, 64);
  long long h;
  const int n = 4096;
  auto rep = [&](const char* name, int div) {
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %.2f cycles/op\n", name, double(h) / n / div);
  };
  k_dfma<<<1, 32>>>(d, 1.0, 0.999, n, c); k_dfma<<<1, 32>>>(d, 1.0, 0.999, n, c); rep("DFMA chain (1 warp)", 1);
  k_dmul<<<1, 32>>>(d, 1.0, 0.999, n, c); k_dmul<<<1, 32>>>(d, 1.0, 0.999, n, c); rep("DMUL chain (1 warp)", 1);
  k_ffma<<<1, 32>>>((float*)d, 1.f, 0.999f, n, c); k_ffma<<<1, 32>>>((float*)d, 1.f, 0.999f, n, c); rep("FFMA chain (1 warp)", 1);
  k_rsq<<<1, 32>>>(d, 2.0, n, c); k_rsq<<<1, 32>>>(d, 2.0, n, c); rep("MUFU.RSQ64H + DADD", 1);
  k_shfl<<<1, 32>>>(d, 2.0, n, c); k_shfl<<<1, 32>>>(d, 2.0, n, c); rep("SHFL(f64) + DADD", 1);
  for (int t : {32, 128, 256, 512, 1024}) {
    k_bar<<<1, t>>>(d, n, c); k_bar<<<1, t>>>(d, n, c);
    char nm[64]; snprintf(nm, 64, "BAR.SYNC %d threads", t); rep(nm, 1);
  }
  k_lds<<<1, 32>>>(d, n, c); k_lds<<<1, 32>>>(d, n, c); rep("LDS pointer chase", 1);
  k_dfma<<<1, 512>>>(d, 1.0, 0.999, n, c); k_dfma<<<1, 512>>>(d, 1.0, 0.999, n, c); rep("DFMA chain (16 warps)", 1);
  return 0;
}
