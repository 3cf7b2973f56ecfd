// Latency microbenchmark: dependent chains of FP64 ops on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9, y = b;
  long long t0, t1;
  __shared__ double sm[1024];
  __shared__ long long tt[16];
  sm[threadIdx.x] = x;
  __syncthreads();
#define TIME(idx, body) \
  t0 = clock64(); for (int i = 0; i < n; ++i) { body; } t1 = clock64(); if (threadIdx.x == 0) cyc[idx] = (t1 - t0) / n;
  TIME(0, x = fma(x, y, 1e-3))
  TIME(1, x = x + y)
  TIME(2, x = x * y)
  TIME(3, x = 1.0 / x)
  TIME(4, x = sqrt(x) + 0.5)
  TIME(5, { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 0.5; })
  TIME(6, { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 0.5; })
  TIME(7, x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9)
  TIME(8, x = sm[(threadIdx.x + (int)x) & 1023] + 0.0)
  TIME(9, { float f = (float)x; f = fmaf(f, 1.0001f, 1e-3f); x = f; })
  TIME(10, { __syncthreads(); x += 1e-9; })
  TIME(11, x = fma(x, y, 1e-3); x = fma(x, y, 1e-3); x = fma(x, y, 1e-3); x = fma(x, y, 1e-3))
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  const char* names[] = {"dfma", "dadd", "dmul", "ddiv", "dsqrt+add", "rcp.approx.f64+add", "rsqrt.approx.f64+add",
                         "shfl.f64+add", "lds.f64+add", "f32 round trip", "syncthreads(256)", "4 dfma"};
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(o, c, 1.0000001, 0.9999999, 1000);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, c, 8 * 16, cudaMemcpyDeviceToHost);
    printf("threads %d\n", threads);
    for (int i = 0; i < 12; ++i) printf("  %-24s %lld cyc\n", names[i], h[i]);
  }
  return 0;
}
