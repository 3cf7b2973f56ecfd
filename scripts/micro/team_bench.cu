// Micro-benchmark of the reduce kernel's trailing updates in isolation:
// 148 CTAs (one per SM), each owning a c2-shaped X (LP x NP = 768 x 368) and
// a fixed random panel V / T, run the QR-phase sequence of left updates
// (panels k0 = 0, 16, ..., rows [k0, 720)) and report cycles per slice.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -Iinclude -Ipaper_2605_16058_b200/csrc scripts/micro/team_bench.cu
//        paper_2605_16058_b200/libstarm.so -o scripts/micro/team_bench
#include <vector>
#include "svd_f64.cu"

namespace starm {
namespace {
template <int NT>
__global__ void __launch_bounds__(NT, 1) bench_left(double* Xall, int LP, int NP, int L, int mode,
                                                    long long* cyc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrSmemFixed& q = *reinterpret_cast<QrSmemFixed*>(smem_raw);
  const int prs = LP + 36;
  double* pan = reinterpret_cast<double*>(smem_raw + sizeof(QrSmemFixed));
  double* wbase = pan + BW * prs;
  double* X = Xall + size_t(blockIdx.x) * LP * NP;
  for (int i = threadIdx.x; i < BW * prs; i += NT) pan[i] = 1e-3 * ((i * 7919) % 1000) / 1000.0;
  for (int i = threadIdx.x; i < BW * 17; i += NT) q.t[i] = ((i % 17) >= (i / 17)) ? 0.5 : 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int k0 = 0; k0 + BW < NP; k0 += BW) {
    if (mode == 0) {
      team_left_update<NT>(q, wbase, pan, prs, X, LP, L, NP, k0, k0 + BW);
    } else if (mode == 1) {
      const int kc = (k0 / RCH) * RCH;
      trailing_update_w<NT, true>(q, wbase, pan, prs, X, LP, LP, NP, kc, k0 + BW);
    } else if (mode == 2) {
      team_right_update<NT>(q, wbase, pan, prs, X, LP, NP, NP, k0 + BW, k0 + BW);
    } else if (mode == 3) {
      panel_factor_any<NT>(q, pan, prs, k0, LP, X + k0 * LP, 1, LP, 0);
    } else if (mode == 4) {
      panel_factor_any<NT>(q, pan, prs, k0, NP, X + k0 * LP, 1, LP, 0);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
}  // namespace
}  // namespace starm

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  using namespace starm;
  const int LP = 768, NP = 368, L = 720, nblk = 148;
  double* X;
  long long* cyc;
  cudaMalloc(&X, size_t(nblk) * LP * NP * 8);
  {
    std::vector<double> h(size_t(LP) * NP);
    for (size_t i = 0; i < h.size(); ++i) h[i] = double((i * 2654435761ull) % 1000003) / 1000003.0 - 0.5;
    for (int b = 0; b < nblk; ++b) cudaMemcpy(X + size_t(b) * LP * NP, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&cyc, nblk * 8);
  const size_t smem = sizeof(QrSmemFixed) + size_t(BW) * (LP + 36) * 8 + size_t(TEAM_SMEM_DOUBLES) * 8;
  cudaFuncSetAttribute(bench_left<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const char* names[] = {"team left (QR phase)", "ring left (QR phase)", "team right (band)", "panel factor (QR phase)", "panel factor (band)"};
  for (int mode = 0; mode < 5; ++mode) {
    if (only >= 0 && mode != only) continue;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      bench_left<256><<<nblk, 256, smem>>>(X, LP, NP, L, mode, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      long long h[148];
      cudaMemcpy(h, cyc, nblk * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < nblk; ++i) avg += h[i];
      avg /= nblk;
      unsigned long long st[16];
      cudaMemcpyFromSymbol(st, g_stats, sizeof(st));
      cudaMemset(cyc, 0, 8);
      unsigned long long z[16] = {0};
      cudaMemcpyToSymbol(g_stats, z, sizeof(z));
      if (rep == 2) printf("   probe per CTA: acc %.3f M, reduce %.3f M, rest %.3f M\n", st[4] / 148e6, st[5] / 148e6, st[6] / 148e6);
      if (rep == 2) printf("%-24s %.3f ms  %.3f Mcycles per CTA  err=%s\n", names[mode], ms, avg / 1e6,
                           cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
