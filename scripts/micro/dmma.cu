// DMMA (mma.sync.m8n8k4.f64) throughput / latency on one SM vs warps per CTA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8 * 1024 * 1024);
  cudaMalloc(&c, 8 * 4096);
  const int n = 2000;
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int ch : {1, 4, 8}) {
      long long h = 0;
      if (ch == 1) k<1><<<1, warps * 32>>>(o, c, 1.0, 1e-9, n);
      if (ch == 4) k<4><<<1, warps * 32>>>(o, c, 1.0, 1e-9, n);
      if (ch == 8) k<8><<<1, warps * 32>>>(o, c, 1.0, 1e-9, n);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      const double dmmas = double(n) * ch * warps;
      printf("warps %2d chains %d: %.2f cyc per DMMA per SM, %.1f flop/clk/SM, chain latency %.1f cyc\n",
             warps, ch, double(h) / dmmas, dmmas * 512.0 / double(h), double(h) / (double(n)));
    }
  }
  return 0;
}
