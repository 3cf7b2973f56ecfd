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
// accesses are 16 P-byte runs per time index).  n = 1024 (config c2) runs
// the four-step register FFT of dct1024_kernel; other lengths run radix-4
// DIT stages in shared memory (dct_kernel).  Twiddle tables (sincospi) are
// built once per device and n in a small library-owned allocation.  n must
// be a power of two <= 4096; the launcher returns STARM_UNSUPPORTED
// otherwise.
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include <cuda_bf16.h>

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
      // the loop never runs for LOGN = 1 (odd LOGN enters it at s = 1); the
      // guard keeps that instantiation's shift count non-negative
      const int p = q >> (LOGN >= 2 ? LOGN - 2 : 0), qq = q & (Q - 1);
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
                                                          int64_t pitch, int64_t batch,
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
        v[u] = (e < total && r < rows) ? src[base + r + int64_t(t) * pitch] : 0.0;
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
      dst[base + r + int64_t(j) * pitch] = (j ? c1 : c0) * xr;
    }
  } else {
    // V^f_j = e^{i theta_j} (Y_j / c_j - i Y_{n-j} / c_{n-j}); z = V^a + i V^b
    const double ic0 = 1.0 / c0, ic1 = 1.0 / c1;
    for (int e = threadIdx.x; e < P * N; e += DCT_THREADS) {
      const int p = e % P, j = e / P;  // consecutive threads: consecutive fibers
      double ya = 0.0, yb = 0.0, yna = 0.0, ynb = 0.0;
      const int64_t ra = r0 + 2 * p, rb = ra + 1;
      const int64_t oj = base + int64_t(j) * pitch, on = base + int64_t(N - j) * pitch;
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
      dst[base + r + int64_t(t) * pitch] = ((f & 1) ? zz.im : zz.re) * inv;
    }
  }
}

// ---------------------------------------------------------------------------
// Forward DCT-II for n = 1024 with register-resident FFT passes.
//
// The pair sequence z (length N = 32 x 32) is transformed by the four-step
// factorisation: lane t1 of the pair's warp holds z[t1 + 32 t2] (t2 < 32) and
// does a 32-point DFT over t2 in registers, multiplies by W_N^{t1 k1}, the
// warp transposes through its own shared-memory chunks, and lane k1 does the
// second 32-point DFT, ending with Z[k1 + 32 k2].  The Makhoul post-twiddle
// needs Z[N - j], which sits in lane (32 - k1) mod 32: one shuffle per value.
// Shared memory is touched 3 times per element (load, transpose, output)
// instead of once per radix-4 stage, and only the load and the store need a
// CTA barrier.  Layout: 16-byte chunk (fibre pair s, time t) at ck(t, s);
// every access pattern below is bank-conflict free (simulated).
constexpr int D32_WARPS = 4;  // fibre pairs per CTA (8 fibres: 64-byte runs per time index)
constexpr int D32_N = 1024;
constexpr int D32_CHUNKS = 4 * D32_N + D32_N / 2;

__constant__ double c_w32[16][2] = {  // W_32^e = (cos, -sin)(2 pi e / 32)
    {1.0, -0.0},
    {0.9807852804032304, -0.19509032201612825},
    {0.9238795325112867, -0.3826834323650898},
    {0.8314696123025452, -0.5555702330196022},
    {0.7071067811865476, -0.7071067811865475},
    {0.5555702330196023, -0.8314696123025452},
    {0.38268343236508984, -0.9238795325112867},
    {0.19509032201612833, -0.9807852804032304},
    {6.123233995736766e-17, -1.0},
    {-0.1950903220161282, -0.9807852804032304},
    {-0.3826834323650897, -0.9238795325112867},
    {-0.555570233019602, -0.8314696123025455},
    {-0.7071067811865475, -0.7071067811865476},
    {-0.8314696123025453, -0.5555702330196022},
    {-0.9238795325112867, -0.3826834323650899},
    {-0.9807852804032304, -0.1950903220161286},
};

__constant__ double c_pw32[32][2] = {  // (cos, sin)(pi 32 k2 / 2N): post-twiddle of j = 32 k2
    {1.0, 0.0},
    {0.9987954562051724, 0.049067674327418015},
    {0.9951847266721969, 0.0980171403295606},
    {0.989176509964781, 0.14673047445536175},
    {0.9807852804032304, 0.19509032201612825},
    {0.970031253194544, 0.24298017990326387},
    {0.9569403357322088, 0.29028467725446233},
    {0.9415440651830208, 0.33688985339222005},
    {0.9238795325112867, 0.3826834323650898},
    {0.9039892931234433, 0.4275550934302821},
    {0.881921264348355, 0.47139673682599764},
    {0.8577286100002721, 0.5141027441932217},
    {0.8314696123025452, 0.5555702330196022},
    {0.8032075314806449, 0.5956993044924334},
    {0.773010453362737, 0.6343932841636455},
    {0.7409511253549591, 0.6715589548470183},
    {0.7071067811865476, 0.7071067811865475},
    {0.6715589548470183, 0.7409511253549591},
    {0.6343932841636455, 0.773010453362737},
    {0.5956993044924335, 0.8032075314806448},
    {0.5555702330196023, 0.8314696123025452},
    {0.5141027441932217, 0.8577286100002721},
    {0.4713967368259978, 0.8819212643483549},
    {0.4275550934302822, 0.9039892931234433},
    {0.38268343236508984, 0.9238795325112867},
    {0.33688985339222005, 0.9415440651830208},
    {0.29028467725446233, 0.9569403357322089},
    {0.24298017990326398, 0.970031253194544},
    {0.19509032201612833, 0.9807852804032304},
    {0.14673047445536175, 0.989176509964781},
    {0.09801714032956077, 0.9951847266721968},
    {0.049067674327418126, 0.9987954562051724},
};

__device__ __forceinline__ int ck(int t, int s) { return 4 * t + s + (t >> 1); }
__device__ __forceinline__ constexpr int br5(int k) {
  return ((k & 1) << 4) | ((k & 2) << 2) | (k & 4) | ((k & 8) >> 2) | ((k & 16) >> 4);
}

// In-register radix-2 DIF DFT of length 32: natural-order input, output
// X[k] in z[br5(k)].  All indices and twiddles are compile-time.
template <int LG>
__device__ __forceinline__ void dif_stage(cplx (&z)[32]) {
  constexpr int len = 1 << LG, half = len >> 1, step = 32 >> LG;
#pragma unroll
  for (int b = 0; b < 32; b += len)
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const cplx a = z[b + i], c = z[b + i + half];
      z[b + i] = {a.re + c.re, a.im + c.im};
      const cplx d = {a.re - c.re, a.im - c.im};
      const int e = i * step;
      if (e == 0) z[b + i + half] = d;
      else if (e == 8) z[b + i + half] = {d.im, -d.re};
      else z[b + i + half] = cmul(d, cplx{c_w32[e][0], c_w32[e][1]});
    }
}

__device__ __forceinline__ void fft32_dif(cplx (&z)[32]) {
  dif_stage<5>(z);
  dif_stage<4>(z);
  dif_stage<3>(z);
  dif_stage<2>(z);
  dif_stage<1>(z);
}

// INV: DCT-III.  z_j = V^a_j + i V^b_j is built from X_j and X_{N-j} of the
// staged tile, and IDFT(z) = conj(DFT(conj z)) / N runs through the same
// four-step DFT; position pos of the result goes to time 2 pos (pos < N/2)
// or 2N - 1 - 2 pos.
// xbf (optional, forward only): also write the tile's input fibres as bf16
// rows [b * rows_pad + fibre][t] -- the K-major operand of the reference-
// operator residual GEMM (residual_bf16.cu), so that kernel need not re-read
// the f64 input.
template <bool INV>
__global__ void __launch_bounds__(32 * D32_WARPS, 2) dct1024_kernel(
    const double* __restrict__ src, double* __restrict__ dst, int64_t rows, int64_t pitch,
    const cplx* __restrict__ gtw, const cplx* __restrict__ gpw, int vec16,
    uint16_t* __restrict__ xbf, int64_t rows_pad) {
  constexpr int N = D32_N, F = 2 * D32_WARPS, NT = 32 * D32_WARPS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* ch = reinterpret_cast<cplx*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t tiles_per_b = (rows + F - 1) / F;
  const int64_t b = blockIdx.x / tiles_per_b;
  const int64_t r0 = (blockIdx.x % tiles_per_b) * F;
  const double* sb = src + b * rows * N + r0;
  double* db = dst + b * rows * N + r0;
  const int nf = int(rows - r0 < F ? rows - r0 : F);  // live fibres of this tile
  // load: chunk q = (t, s) <- fibres r0 + 2s, r0 + 2s + 1 at time t (zero-filled past rows)
  if (vec16) {
#pragma unroll 4
    for (int q = tid; q < 4 * N; q += NT) {
      const int t = q >> 2, s = q & 3;
      cp_async16(&ch[ck(t, s)], sb + 2 * s + int64_t(t) * pitch, 2 * s < nf ? 16 : 0);
    }
  } else {
#pragma unroll 4
    for (int q = tid; q < 4 * N; q += NT) {
      const int t = q >> 2, s = q & 3;
      double* d = reinterpret_cast<double*>(&ch[ck(t, s)]);
      const double* g = sb + 2 * s + int64_t(t) * pitch;
      cp_async8(d, g, 2 * s < nf ? 8 : 0);
      cp_async8(d + 1, g + 1, 2 * s + 1 < nf ? 8 : 0);
    }
  }
  cp_async_commit();
  // twiddles, loaded while the tile is in flight: W_N^{t1 k1} for k1 = 8a + b
  // is wh[a] * wl[b] (two table entries, one product)
  cplx wl[8], wh[4];
#pragma unroll
  for (int b = 1; b < 8; ++b) wl[b] = gtw[lane * b];
#pragma unroll
  for (int a = 1; a < 4; ++a) {
    const int m = lane * 8 * a;
    wh[a] = gtw[m & (N / 2 - 1)];
    if (m & (N / 2)) wh[a] = {-wh[a].re, -wh[a].im};
  }
  cp_async_wait<0>();
  __syncthreads();
  if (!INV && xbf) {
    // warp w packs its own pair (fibres 2w, 2w + 1): lane -> time pair
    // (2 tp, 2 tp + 1), one 4-byte store per fibre (128-byte runs per warp);
    // ck(2 tp, w) = 9 tp + w keeps the 16-byte reads conflict-free
    uint32_t* xo = reinterpret_cast<uint32_t*>(xbf);
    const int64_t rb = b * rows_pad + r0 + 2 * w;
#pragma unroll 4
    for (int tp = lane; tp < N / 2; tp += 32) {
      const cplx u = ch[ck(2 * tp, w)], v = ch[ck(2 * tp + 1, w)];
      auto pk = [](double lo, double hi) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(float(fmin(fmax(lo, -3.0e38), 3.0e38)),
                                                       float(fmin(fmax(hi, -3.0e38), 3.0e38)));
        return *reinterpret_cast<const uint32_t*>(&h);
      };
      if (2 * w < nf) xo[(rb * N) / 2 + tp] = pk(u.re, v.re);
      if (2 * w + 1 < nf) xo[((rb + 1) * N) / 2 + tp] = pk(u.im, v.im);
    }
  }
  const double c0 = sqrt(1.0 / N), c1 = sqrt(2.0 / N);
  const cplx pl = gpw[lane];
  // pass 1: lane t1 holds z[t1 + 32 t2]
  cplx z[32];
  if constexpr (!INV) {
    // Makhoul order: position pos <- time 2 pos (pos < N/2), 2N - 1 - 2 pos otherwise
#pragma unroll
    for (int t2 = 0; t2 < 32; ++t2) {
      const int pos = lane + 32 * t2;
      const int t = t2 < 16 ? 2 * pos : 2 * N - 1 - 2 * pos;
      z[t2] = ch[ck(t, w)];
    }
  } else {
    // V^f_j = e^{i theta_j} (Y_j / c_j - i Y_{N-j} / c_{N-j}), z = conj(V^a + i V^b)
    const double ic0 = 1.0 / c0, ic1 = 1.0 / c1;
#pragma unroll
    for (int t2 = 0; t2 < 32; ++t2) {
      const int j = lane + 32 * t2;
      const cplx y = ch[ck(j, w)], yn = ch[ck((N - j) & (N - 1), w)];
      const double sj = j ? ic1 : ic0, sn = j ? ic1 : 0.0;
      const cplx pw = t2 == 0 ? pl : cmul(pl, cplx{c_pw32[t2][0], c_pw32[t2][1]});
      const cplx va = cmul(pw, cplx{y.re * sj, -yn.re * sn});
      const cplx vb = cmul(pw, cplx{y.im * sj, -yn.im * sn});
      z[t2] = {va.re - vb.im, -(va.im + vb.re)};
    }
  }
  fft32_dif(z);
  // twiddle W_N^{t1 k1}
#pragma unroll
  for (int k1 = 1; k1 < 32; ++k1) {
    const int a = k1 >> 3, b = k1 & 7;
    const cplx tw = a == 0 ? wl[b] : (b == 0 ? wh[a] : cmul(wh[a], wl[b]));
    z[br5(k1)] = cmul(z[br5(k1)], tw);
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) ch[ck(32 * k1 + (lane ^ k1), w)] = z[br5(k1)];
  __syncwarp();
#pragma unroll
  for (int t1 = 0; t1 < 32; ++t1) z[t1] = ch[ck(32 * lane + (t1 ^ lane), w)];
  __syncwarp();
  fft32_dif(z);  // lane k1: Z[k1 + 32 k2] in z[br5(k2)]
  if constexpr (!INV) {
    const int partner = (32 - lane) & 31;
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) {
      const int j = lane + 32 * k2;
      const cplx zj = z[br5(k2)];
      const cplx o = z[br5(31 - k2)], own = z[br5((32 - k2) & 31)];
      cplx zn;
      zn.re = __shfl_sync(0xffffffffu, o.re, partner);
      zn.im = __shfl_sync(0xffffffffu, o.im, partner);
      if (lane == 0) zn = own;  // Z[N - 32 k2] = Z[32 (32 - k2)] (k2 = 0: Z[0])
      const cplx va = {0.5 * (zj.re + zn.re), 0.5 * (zj.im - zn.im)};  // (Z_j + conj Z_{n-j}) / 2
      const cplx vb = {0.5 * (zj.im + zn.im), 0.5 * (zn.re - zj.re)};  // (Z_j - conj Z_{n-j}) / 2i
      const cplx pw = k2 == 0 ? pl : cmul(pl, cplx{c_pw32[k2][0], c_pw32[k2][1]});
      const double cj = j ? c1 : c0;
      ch[ck(j, w)] = {cj * fma(pw.re, va.re, pw.im * va.im), cj * fma(pw.re, vb.re, pw.im * vb.im)};
    }
  } else {
    const double inv = 1.0 / N;
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) {
      const int pos = lane + 32 * k2;
      const int t = k2 < 16 ? 2 * pos : 2 * N - 1 - 2 * pos;
      const cplx r = z[br5(k2)];
      ch[ck(t, w)] = {r.re * inv, -r.im * inv};
    }
  }
  __syncthreads();
  if (vec16 && nf == F) {
#pragma unroll 8
    for (int q = tid; q < 4 * N; q += NT) {
      const int t = q >> 2, s = q & 3;
      const cplx v = ch[ck(t, s)];
      *reinterpret_cast<double2*>(db + 2 * s + int64_t(t) * pitch) = make_double2(v.re, v.im);
    }
  } else {
    for (int q = tid; q < 4 * N; q += NT) {
      const int t = q >> 2, s = q & 3;
      const cplx v = ch[ck(t, s)];
      double* g = db + 2 * s + int64_t(t) * pitch;
      if (2 * s < nf) g[0] = v.re;
      if (2 * s + 1 < nf) g[1] = v.im;
    }
  }
}

struct DctTables {
  cplx* tw[13] = {};
  cplx* pw[13] = {};
};

std::mutex g_dct_mu;
// STARM_DCT_LEGACY=1: the shared-memory radix-4 kernel for every length (A/B runs)
const bool g_dct_legacy = [] {
  const char* e = getenv("STARM_DCT_LEGACY");
  return e && e[0] == '1';
}();
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
int launch_dct(const double* src, double* dst, int64_t rows, int64_t pitch, int64_t batch,
               bool inverse, cudaStream_t st, uint16_t* xbf = nullptr, int64_t rows_pad = 0) {
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
  if (LOGN == 10 && !g_dct_legacy) {
    const size_t sm2 = size_t(D32_CHUNKS) * sizeof(cplx);
    const int64_t t2 = (rows + 2 * D32_WARPS - 1) / (2 * D32_WARPS) * batch;
    const int vec16 = (rows % 2 == 0) && (pitch % 2 == 0) &&
                      (reinterpret_cast<uintptr_t>(src) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(dst) % 16 == 0);
    // hoisted twiddle products at 2 CTAs / SM: 1.33 ms on c2, against 1.44 ms
    // for per-k1 table loads at 3 CTAs / SM and 1.36 ms for the hoisted
    // twiddles squeezed into 168 registers (3 CTAs / SM, spills); loading
    // each lane's 32 values straight from global memory (no staging) 2.4 ms
    auto kern = inverse ? dct1024_kernel<true> : dct1024_kernel<false>;
    STARM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2)));
    kern<<<unsigned(t2), 32 * D32_WARPS, sm2, st>>>(src, dst, rows, pitch, tw, pw, vec16,
                                                    inverse ? nullptr : xbf, rows_pad);
    STARM_LAUNCH_CHECK();
    return STARM_OK;
  }
  auto kern = inverse ? dct_kernel<LOGN, true> : dct_kernel<LOGN, false>;
  STARM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<unsigned(tiles), DCT_THREADS, smem, st>>>(src, dst, rows, pitch, batch, tw, pw);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

}  // namespace
}  // namespace starm

namespace starm {
// Internal launcher (also used by starm_dct_residual_f64): when xbf is set
// and the n = 1024 forward kernel runs, the bf16 operand rows are written
// too; returns whether that happened through *packed.  pitch (0: rows) is
// the distance in doubles between consecutive mode indices of one fibre, so
// a block of `rows` fibres of a wider tensor can be transformed where it
// lies (batch must be 1 when pitch != rows).
int dct_launch(const double* src, double* dst, int64_t rows, int64_t n, int64_t batch, bool inv,
               uint16_t* xbf, int64_t rows_pad, bool* packed, cudaStream_t st, int64_t pitch) {
  if (pitch == 0) pitch = rows;
  if (packed) *packed = xbf && n == 1024 && !inv && !g_dct_legacy;
  switch (n) {
    case 2: return launch_dct<1>(src, dst, rows, pitch, batch, inv, st);
    case 4: return launch_dct<2>(src, dst, rows, pitch, batch, inv, st);
    case 8: return launch_dct<3>(src, dst, rows, pitch, batch, inv, st);
    case 16: return launch_dct<4>(src, dst, rows, pitch, batch, inv, st);
    case 32: return launch_dct<5>(src, dst, rows, pitch, batch, inv, st);
    case 64: return launch_dct<6>(src, dst, rows, pitch, batch, inv, st);
    case 128: return launch_dct<7>(src, dst, rows, pitch, batch, inv, st);
    case 256: return launch_dct<8>(src, dst, rows, pitch, batch, inv, st);
    case 512: return launch_dct<9>(src, dst, rows, pitch, batch, inv, st);
    case 1024: return launch_dct<10>(src, dst, rows, pitch, batch, inv, st, xbf, rows_pad);
    case 2048: return launch_dct<11>(src, dst, rows, pitch, batch, inv, st);
    default: return launch_dct<12>(src, dst, rows, pitch, batch, inv, st);
  }
}
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
  return dct_launch(src, dst, rows, n, batch, inv, nullptr, 0, nullptr, st, 0);
}
