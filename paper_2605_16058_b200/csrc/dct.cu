// Fast orthonormal DCT-II / DCT-III along one mode (FP64).
//
// The reference applies its DCT transform as a dense mode-k product with
// the DCT matrix (transforms.py dct -> ttm.py:87-104, np.matmul).  For the
// DCT kind the same linear map is computed here in O(n log n) per fiber
// (Makhoul's algorithm): with v_t = x_{2t}, v_{n-1-t} = x_{2t+1} (t < n/2)
//   DCT-II:  X_j = c_j Re(e^{-i pi j / 2n} DFT(v)_j)
//   DCT-III: v = IDFT(V), V_j = e^{i pi j / 2n} (X_j / c_j - i X_{n-j} / c_{n-j})
// Two real fibers share one complex FFT (real / imaginary parts).  One CTA
// transforms 2 P fibers (consecutive rows of one batch block, so global
// accesses are 16 P-byte runs per time index) with radix-2 DIT stages in
// shared memory; twiddles come from sincospi in the prologue.  n must be a
// power of two; the launcher returns STARM_UNSUPPORTED otherwise.
#include "common.cuh"

namespace starm {
namespace {

constexpr int DCT_THREADS = 256;

struct cplx {
  double re, im;
};

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}

__device__ __forceinline__ int bitrev(int x, int bits) { return int(__brev(unsigned(x)) >> (32 - bits)); }

// P complex sequences of length n in z[p * n + i]; tw[m] = e^{-+2 pi i m / n}.
__device__ void fft_stages(cplx* z, const cplx* tw, int n, int logn, int P) {
  const int half_total = P * (n >> 1);
  for (int s = 0; s < logn; ++s) {
    const int h = 1 << s;
    const int step = n >> (s + 1);  // twiddle stride
    for (int q = threadIdx.x; q < half_total; q += blockDim.x) {
      const int p = q / (n >> 1), qq = q % (n >> 1);
      const int k = qq & (h - 1);
      const int i0 = ((qq >> s) << (s + 1)) + k;
      cplx* zp = z + p * n;
      const cplx a = zp[i0];
      const cplx b = cmul(zp[i0 + h], tw[k * step]);
      zp[i0] = {a.re + b.re, a.im + b.im};
      zp[i0 + h] = {a.re - b.re, a.im - b.im};
    }
    __syncthreads();
  }
}

template <bool INVERSE>
__global__ void __launch_bounds__(DCT_THREADS) dct_kernel(const double* __restrict__ src,
                                                          double* __restrict__ dst, int64_t rows,
                                                          int n, int logn, int64_t batch, int P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* z = reinterpret_cast<cplx*>(smem_raw);  // [P][n]
  cplx* tw = z + int64_t(P) * n;                // [n / 2] FFT twiddles
  cplx* pw = tw + (n >> 1);                     // [n] e^{-i pi j / 2n} (cos, sin)
  const int F = 2 * P;
  const int64_t tiles_per_b = (rows + F - 1) / F;
  const int64_t tile = blockIdx.x;
  const int64_t b = tile / tiles_per_b;
  const int64_t r0 = (tile % tiles_per_b) * F;
  const int64_t base = b * rows * n;
  const double c0 = sqrt(1.0 / n), c1 = sqrt(2.0 / n);
  for (int m = threadIdx.x; m < (n >> 1); m += blockDim.x) {
    double sv, cv;
    sincospi(2.0 * m / n, &sv, &cv);
    tw[m] = {cv, INVERSE ? sv : -sv};
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double sv, cv;
    sincospi(0.5 * j / n, &sv, &cv);
    pw[j] = {cv, sv};
  }
  if (!INVERSE) {
    // load x (fibers f = 2p + {0,1}) into bit-reversed Makhoul order
    for (int64_t e = threadIdx.x; e < int64_t(F) * n; e += blockDim.x) {
      const int f = int(e % F), t = int(e / F);
      const int64_t r = r0 + f;
      const double x = r < rows ? src[base + r + int64_t(t) * rows] : 0.0;
      const int pos = (t & 1) ? n - 1 - (t >> 1) : (t >> 1);
      double* zp = reinterpret_cast<double*>(z + (f >> 1) * n + bitrev(pos, logn));
      zp[f & 1] = x;
    }
    __syncthreads();
    fft_stages(z, tw, n, logn, P);
    // split the pair, post-twiddle, scale, store (consecutive threads: consecutive fibers)
    for (int64_t e = threadIdx.x; e < int64_t(F) * n; e += blockDim.x) {
      const int f = int(e % F), j = int(e / F);
      const int64_t r = r0 + f;
      if (r >= rows) continue;
      const cplx* zp = z + (f >> 1) * n;
      const cplx zj = zp[j], zn = zp[(n - j) & (n - 1)];
      cplx v;
      if ((f & 1) == 0) {
        v = {0.5 * (zj.re + zn.re), 0.5 * (zj.im - zn.im)};  // (Z_j + conj Z_{n-j}) / 2
      } else {
        v = {0.5 * (zj.im + zn.im), 0.5 * (zn.re - zj.re)};  // (Z_j - conj Z_{n-j}) / 2i
      }
      const cplx w = pw[j];
      const double xr = fma(w.re, v.re, w.im * v.im);  // Re(e^{-i theta} v)
      dst[base + r + int64_t(j) * rows] = (j ? c1 : c0) * xr;
    }
  } else {
    // V^f_j = e^{i theta_j} (Y_j / c_j - i Y_{n-j} / c_{n-j}); z = V^a + i V^b
    for (int64_t e = threadIdx.x; e < int64_t(P) * n; e += blockDim.x) {
      const int p = int(e % P), j = int(e / P);  // consecutive threads: consecutive fibers
      double ya = 0.0, yb = 0.0, yna = 0.0, ynb = 0.0;
      const int64_t ra = r0 + 2 * p, rb = ra + 1;
      const int64_t oj = base + int64_t(j) * rows, on = base + int64_t(n - j) * rows;
      if (ra < rows) {
        ya = src[oj + ra] / (j ? c1 : c0);
        if (j) yna = src[on + ra] / c1;
      }
      if (rb < rows) {
        yb = src[oj + rb] / (j ? c1 : c0);
        if (j) ynb = src[on + rb] / c1;
      }
      const cplx w = pw[j];  // (cos theta, sin theta): e^{+i theta}
      const cplx va = cmul(w, {ya, -yna});
      const cplx vb = cmul(w, {yb, -ynb});
      z[p * n + bitrev(j, logn)] = {va.re - vb.im, va.im + vb.re};
    }
    __syncthreads();
    fft_stages(z, tw, n, logn, P);
    const double inv = 1.0 / n;
    for (int64_t e = threadIdx.x; e < int64_t(F) * n; e += blockDim.x) {
      const int f = int(e % F), t = int(e / F);
      const int64_t r = r0 + f;
      if (r >= rows) continue;
      const int pos = (t & 1) ? n - 1 - (t >> 1) : (t >> 1);
      const cplx zz = z[(f >> 1) * n + pos];
      dst[base + r + int64_t(t) * rows] = ((f & 1) ? zz.im : zz.re) * inv;
    }
  }
}

}  // namespace
}  // namespace starm

using namespace starm;

extern "C" int starm_dct_f64(const double* src, double* dst, int64_t rows, int64_t n, int64_t batch,
                             int inverse, void* stream) {
  STARM_CHECK_ARG(rows >= 0 && n >= 1 && batch >= 0, "starm_dct_f64: negative extent");
  if (rows == 0 || batch == 0) return STARM_OK;
  STARM_CHECK_ARG(src && dst && src != dst, "starm_dct_f64: null or aliased buffers");
  if ((n & (n - 1)) != 0 || n < 2 || n > 4096) {
    set_error("starm_dct_f64: the fast path needs a power-of-two length in [2, 4096]");
    return STARM_UNSUPPORTED;
  }
  int logn = 0;
  while ((int64_t(1) << logn) < n) ++logn;
  const int P = n <= 1024 ? 4 : (n == 2048 ? 2 : 1);
  const size_t smem = (size_t(P) * n + n / 2 + n) * sizeof(cplx);
  const int64_t tiles = (rows + 2 * P - 1) / (2 * P) * batch;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (inverse) {
    STARM_CUDA_TRY(cudaFuncSetAttribute(dct_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dct_kernel<true><<<unsigned(tiles), DCT_THREADS, smem, st>>>(src, dst, rows, int(n), logn, batch, P);
  } else {
    STARM_CUDA_TRY(cudaFuncSetAttribute(dct_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dct_kernel<false><<<unsigned(tiles), DCT_THREADS, smem, st>>>(src, dst, rows, int(n), logn, batch, P);
  }
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}
