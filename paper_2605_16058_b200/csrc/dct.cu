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
// shared memory; twiddle tables (sincospi) are built once per device and n
// in a small library-owned allocation.  n must be a power of two <= 4096;
// the launcher returns STARM_UNSUPPORTED otherwise.
#include <mutex>

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

// Shared-memory layout of a pair's sequence: element i lives at swz(i) =
// i ^ g(i), g XORing a 3-bit value per set bit of i >> 3 (a linear map over
// GF(2), masks below), and pair p starts at p * (N + ZPAD).  Found by
// simulating the bank pattern of every access of this kernel (radix-4 / -2
// butterflies, bit-reversed scatter, post-twiddle gathers, both directions)
// for N = 32 .. 4096: within 5% of the conflict-free wavefront count, against
// 1.8x more wavefronts for the plain layout.
constexpr int ZPAD = 2;
__device__ __forceinline__ int swz(int i) {
  const int g = (__popc(i & 0xdf8) & 1) | ((__popc(i & 0xbb0) & 1) << 1) | ((__popc(i & 0x818) & 1) << 2);
  return i ^ g;
}

// Twiddle tables per (device, n), built once by dct_tables_kernel:
//   tw[m] = e^{-2 pi i m / n} (m < n/2),  pw[j] = (cos, sin)(pi j / 2n) (j < n).
__global__ void dct_tables_kernel(cplx* tw, cplx* pw, int n) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
    double sv, cv;
    if (m < n / 2) {
      sincospi(2.0 * m / n, &sv, &cv);
      tw[m] = {cv, -sv};
    }
    sincospi(0.5 * m / n, &sv, &cv);
    pw[m] = {cv, sv};
  }
}

// fibre pairs per CTA: 4 up to n = 1024, then shared memory limits it
__host__ __device__ constexpr int dct_pairs(int logn) { return logn <= 10 ? 4 : (logn == 11 ? 2 : 1); }

// P complex sequences of length N = 2^LOGN in z[p * N + i], bit-reversed
// input; DIT stages fused in pairs (radix 4: 4 loads, 4 twiddle products,
// 8 additions, 4 stores per item, one barrier per pair), plus one radix-2
// stage first when LOGN is odd.  Conjugate twiddles when INVERSE.
template <int LOGN, bool INVERSE>
__device__ __forceinline__ void fft_stages(cplx* z, const cplx* tw) {
  constexpr int N = 1 << LOGN, H = N >> 1;
  constexpr int P = dct_pairs(LOGN);
  int s = 0;
  if (LOGN & 1) {  // radix-2 stage with h = 1 (twiddle 1)
    for (int q = threadIdx.x; q < P * H; q += blockDim.x) {
      const int p = q >> (LOGN - 1), qq = q & (H - 1);
      cplx* zp = z + p * (N + ZPAD);
      const int i0 = swz(2 * qq), i1 = i0 ^ 1;  // (swz is linear over GF(2); swz(1) = 1)
      const cplx a = zp[i0], b = zp[i1];
      zp[i0] = {a.re + b.re, a.im + b.im};
      zp[i1] = {a.re - b.re, a.im - b.im};
    }
    __syncthreads();
    s = 1;
  }
#pragma unroll 1
  for (; s < LOGN; s += 2) {
    const int h = 1 << s;
    constexpr int Q = N >> 2;
    // i0 has bits s, s + 1 clear, so i0 + m h = i0 ^ m h and (swz linear)
    // swz(i0 + m h) = swz(i0) ^ swz(m h)
    const int d1 = swz(h), d2 = swz(2 * h), d3 = d1 ^ d2;
    for (int q = threadIdx.x; q < P * Q; q += blockDim.x) {
      const int p = q >> (LOGN - 2), qq = q & (Q - 1);
      const int k = qq & (h - 1);
      const int i0 = ((qq >> s) << (s + 2)) + k;
      cplx* zp = z + p * (N + ZPAD);
      const int j0 = swz(i0), j1 = j0 ^ d1, j2 = j0 ^ d2, j3 = j0 ^ d3;
      cplx w1 = tw[k << (LOGN - 1 - s)];  // W_{2h}^k
      cplx w2 = tw[k << (LOGN - 2 - s)];  // W_{4h}^k
      if (INVERSE) {
        w1.im = -w1.im;
        w2.im = -w2.im;
      }
      // W_{4h}^{k+h} = W_{4h}^k * (-i) forward, * (+i) inverse
      const cplx w3 = INVERSE ? cplx{-w2.im, w2.re} : cplx{w2.im, -w2.re};
      const cplx a0 = zp[j0], a1 = cmul(zp[j1], w1);
      const cplx a2 = zp[j2], a3 = cmul(zp[j3], w1);
      const cplx b0 = {a0.re + a1.re, a0.im + a1.im}, b1 = {a0.re - a1.re, a0.im - a1.im};
      const cplx b2 = cmul(cplx{a2.re + a3.re, a2.im + a3.im}, w2);
      const cplx b3 = cmul(cplx{a2.re - a3.re, a2.im - a3.im}, w3);
      zp[j0] = {b0.re + b2.re, b0.im + b2.im};
      zp[j2] = {b0.re - b2.re, b0.im - b2.im};
      zp[j1] = {b1.re + b3.re, b1.im + b3.im};
      zp[j3] = {b1.re - b3.re, b1.im - b3.im};
    }
    __syncthreads();
  }
}

template <int LOGN, bool INVERSE>
__global__ void __launch_bounds__(DCT_THREADS) dct_kernel(const double* __restrict__ src,
                                                          double* __restrict__ dst, int64_t rows,
                                                          int64_t batch,
                                                          const cplx* __restrict__ gtw,
                                                          const cplx* __restrict__ gpw) {
  constexpr int N = 1 << LOGN;
  constexpr int P = dct_pairs(LOGN);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* z = reinterpret_cast<cplx*>(smem_raw);  // [P][N + ZPAD], swizzled
  cplx* tw = z + P * (N + ZPAD);                // [N / 2]
  constexpr int F = 2 * P;
  const int64_t tiles_per_b = (rows + F - 1) / F;
  const int64_t b = blockIdx.x / tiles_per_b;
  const int64_t r0 = (blockIdx.x % tiles_per_b) * F;
  const int64_t base = b * rows * N;
  const double c0 = sqrt(1.0 / N), c1 = sqrt(2.0 / N);
  for (int m = threadIdx.x; m < N / 2; m += blockDim.x) tw[m] = gtw[m];
  constexpr int U = 16;  // loads in flight per thread
  const int total = F * N;
  if (!INVERSE) {
    // load x (fibers f = 2p + {0,1}) into bit-reversed Makhoul order
    for (int e0 = 0; e0 < total; e0 += U * DCT_THREADS) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * DCT_THREADS + threadIdx.x;
        const int f = e % F, t = e / F;
        const int64_t r = r0 + f;
        v[u] = (e < total && r < rows) ? src[base + r + int64_t(t) * rows] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * DCT_THREADS + threadIdx.x;
        if (e < total) {
          const int f = e % F, t = e / F;
          const int pos = (t & 1) ? N - 1 - (t >> 1) : (t >> 1);
          reinterpret_cast<double*>(z + (f >> 1) * (N + ZPAD) + swz(bitrev(pos, LOGN)))[f & 1] = v[u];
        }
      }
    }
    __syncthreads();
    fft_stages<LOGN, false>(z, tw);
    // split the pair, post-twiddle, scale, store (consecutive threads: consecutive fibers)
    for (int e = threadIdx.x; e < total; e += DCT_THREADS) {
      const int f = e % F, j = e / F;
      const int64_t r = r0 + f;
      if (r >= rows) continue;
      const cplx* zp = z + (f >> 1) * (N + ZPAD);
      const cplx zj = zp[swz(j)], zn = zp[swz((N - j) & (N - 1))];
      cplx v;
      if ((f & 1) == 0) {
        v = {0.5 * (zj.re + zn.re), 0.5 * (zj.im - zn.im)};  // (Z_j + conj Z_{n-j}) / 2
      } else {
        v = {0.5 * (zj.im + zn.im), 0.5 * (zn.re - zj.re)};  // (Z_j - conj Z_{n-j}) / 2i
      }
      const cplx w = gpw[j];
      const double xr = fma(w.re, v.re, w.im * v.im);  // Re(e^{-i theta} v)
      dst[base + r + int64_t(j) * rows] = (j ? c1 : c0) * xr;
    }
  } else {
    // V^f_j = e^{i theta_j} (Y_j / c_j - i Y_{n-j} / c_{n-j}); z = V^a + i V^b
    const double ic0 = 1.0 / c0, ic1 = 1.0 / c1;
    for (int e = threadIdx.x; e < P * N; e += DCT_THREADS) {
      const int p = e % P, j = e / P;  // consecutive threads: consecutive fibers
      double ya = 0.0, yb = 0.0, yna = 0.0, ynb = 0.0;
      const int64_t ra = r0 + 2 * p, rb = ra + 1;
      const int64_t oj = base + int64_t(j) * rows, on = base + int64_t(N - j) * rows;
      const double sj = j ? ic1 : ic0;
      if (ra < rows) {
        ya = src[oj + ra] * sj;
        if (j) yna = src[on + ra] * ic1;
      }
      if (rb < rows) {
        yb = src[oj + rb] * sj;
        if (j) ynb = src[on + rb] * ic1;
      }
      const cplx w = gpw[j];  // e^{+i theta}
      const cplx va = cmul(w, {ya, -yna});
      const cplx vb = cmul(w, {yb, -ynb});
      z[p * (N + ZPAD) + swz(bitrev(j, LOGN))] = {va.re - vb.im, va.im + vb.re};
    }
    __syncthreads();
    fft_stages<LOGN, true>(z, tw);
    const double inv = 1.0 / N;
    for (int e = threadIdx.x; e < total; e += DCT_THREADS) {
      const int f = e % F, t = e / F;
      const int64_t r = r0 + f;
      if (r >= rows) continue;
      const int pos = (t & 1) ? N - 1 - (t >> 1) : (t >> 1);
      const cplx zz = z[(f >> 1) * (N + ZPAD) + swz(pos)];
      dst[base + r + int64_t(t) * rows] = ((f & 1) ? zz.im : zz.re) * inv;
    }
  }
}

struct DctTables {
  cplx* tw[13] = {};
  cplx* pw[13] = {};
};

std::mutex g_dct_mu;
DctTables g_dct_tables[64];  // per device ordinal

int dct_tables(int logn, const cplx** tw, const cplx** pw, cudaStream_t st) {
  int dev = 0;
  STARM_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("starm_dct_f64: device ordinal out of range");
    return STARM_INVALID_ARG;
  }
  std::lock_guard<std::mutex> lk(g_dct_mu);
  DctTables& t = g_dct_tables[dev];
  if (!t.tw[logn]) {
    const int n = 1 << logn;
    cplx *a = nullptr, *b = nullptr;
    STARM_CUDA_TRY(cudaMalloc(&a, sizeof(cplx) * (n / 2 > 0 ? n / 2 : 1)));
    STARM_CUDA_TRY(cudaMalloc(&b, sizeof(cplx) * n));
    dct_tables_kernel<<<(n + 255) / 256, 256, 0, st>>>(a, b, n);
    STARM_LAUNCH_CHECK();
    STARM_CUDA_TRY(cudaStreamSynchronize(st));
    t.tw[logn] = a;
    t.pw[logn] = b;
  }
  *tw = t.tw[logn];
  *pw = t.pw[logn];
  return STARM_OK;
}

template <int LOGN>
int launch_dct(const double* src, double* dst, int64_t rows, int64_t batch, bool inverse,
               cudaStream_t st) {
  constexpr int N = 1 << LOGN;
  constexpr int P = dct_pairs(LOGN);
  const size_t smem = (size_t(P) * (N + ZPAD) + N / 2) * sizeof(cplx);
  const int64_t tiles = (rows + 2 * P - 1) / (2 * P) * batch;
  if (tiles > int64_t(0x7fffffff)) {
    set_error("starm_dct_f64: too many fibers for one launch");
    return STARM_UNSUPPORTED;
  }
  const cplx *tw = nullptr, *pw = nullptr;
  const int rc = dct_tables(LOGN, &tw, &pw, st);
  if (rc) return rc;
  auto kern = inverse ? dct_kernel<LOGN, true> : dct_kernel<LOGN, false>;
  STARM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<unsigned(tiles), DCT_THREADS, smem, st>>>(src, dst, rows, batch, tw, pw);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool inv = inverse != 0;
  switch (n) {
    case 2: return launch_dct<1>(src, dst, rows, batch, inv, st);
    case 4: return launch_dct<2>(src, dst, rows, batch, inv, st);
    case 8: return launch_dct<3>(src, dst, rows, batch, inv, st);
    case 16: return launch_dct<4>(src, dst, rows, batch, inv, st);
    case 32: return launch_dct<5>(src, dst, rows, batch, inv, st);
    case 64: return launch_dct<6>(src, dst, rows, batch, inv, st);
    case 128: return launch_dct<7>(src, dst, rows, batch, inv, st);
    case 256: return launch_dct<8>(src, dst, rows, batch, inv, st);
    case 512: return launch_dct<9>(src, dst, rows, batch, inv, st);
    case 1024: return launch_dct<10>(src, dst, rows, batch, inv, st);
    case 2048: return launch_dct<11>(src, dst, rows, batch, inv, st);
    default: return launch_dct<12>(src, dst, rows, batch, inv, st);
  }
}
