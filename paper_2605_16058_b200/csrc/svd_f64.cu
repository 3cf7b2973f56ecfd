// K3-K6: batched slice SVD -- QR-preconditioned blocked one-sided (Hestenes)
// Jacobi, FP64.
//
// Replaces the per-slice LAPACK dgesvd loop of the reference
// (slicesvd.py:42-62 `_slice_svd`, driven by svd_all_slices :115-136,
// _values_pass :139-168 and svd_truncated_slices :259-292).
//
// Per slice (m x p, column-major) let X be the L x n working matrix
// (L = max(m,p), n = min(m,p)):  X = A if m >= p, X = A^T otherwise.
//
//  1. (tall X, L >= 1.25 n) Householder QR  X = Q R  in a first kernel:
//     16-column panels factored in shared memory, compact-WY trailing
//     updates C -= V (T^T (V^T C)) on FP64 DMMA tiles.  The Jacobi target is
//     then the n x n R (half the work per sweep for c2's 720 x 361 slices).
//     Otherwise the target is X itself.
//  2. Blocked one-sided Jacobi on the target T (columns in blocks of 16,
//     one "pair step" = 32 columns):  Gram G = T_P^T T_P on DMMA (streamed
//     64-row chunks, cp.async double buffering), skip if converged, one
//     inner sweep of round-robin cyclic Jacobi on G in shared memory (16
//     disjoint rotations per round) -> rotation W, T_P <- T_P W (and
//     V_P <- V_P W when vectors are wanted), again on DMMA.
//  3. sigma = column norms of T V (descending bitonic sort).  T V = U_T S so
//     X V = Q U_T S: right singular vectors of X are V, left ones are the
//     normalised columns of X V -- taken directly from T V (no QR) or
//     recomputed as X * V_sel from the untouched input slice (QR path), then
//     re-orthonormalised (CGS2) where sigma_j < 1e-4 sigma_max.
// Because every rotation is applied to the data and every Gram is recomputed
// from it, sigma are column norms of X V with V orthogonal to working
// precision: backward error O(u ||A||) like dgesvd; the Gram only chooses
// rotations.
//
// Scheduling: persistent grids (SMs x resident CTAs) pull slices from atomic
// counters; workspace is per resident CTA (plus one n x n R per slice on the
// QR path).
#include <float.h>
#include <math_constants.h>
#include <limits.h>

#include <mutex>

#include "common.cuh"

namespace starm {
namespace {

constexpr int TPB = 256;
constexpr int GW = 32;        // columns per pair step
constexpr int BW = 16;        // columns per block / QR panel width
constexpr int RCH = 64;       // rows per streamed chunk
constexpr int XS = RCH + 4;   // chunk column stride (doubles)
constexpr int GS = 33;        // Gram row stride
constexpr int WS = 36;        // rotation column stride
constexpr int MAX_NS = 4096;  // largest supported min(m, p) (sort buffer)
constexpr int QR_MAX_LP = 1344;
constexpr int ZS = 20;        // Z (16 x 32) column stride

enum { ST_SLICES = 0, ST_SWEEPS, ST_PAIRS, ST_ROTATED, ST_CYC_GRAM, ST_CYC_EIG, ST_CYC_APPLY,
       ST_CYC_QR, ST_CYC_FINAL, ST_CYC_LOAD, ST_CYC_BAND, ST_CYC_BULGE, ST_CYC_PFACT, ST_CYC_TRAIL,
       ST_CYC_RIGHT, ST_CYC_PMISC, ST_COUNT };

__device__ unsigned long long g_stats[16];

struct SvdParams {
  const double* A;
  int64_t m, p, N;
  const int64_t* ids;
  int64_t count;
  int job;
  double* s;
  double* u;
  double* v;
  const int64_t* ranks;
  const int64_t* u_off;
  const int64_t* g_off;
  double* u_data;
  double* g_data;
  int32_t* status;
  unsigned long long* counter;  // [0] reduce, [1] jacobi / vecout, [2] bulge, [3] orth, [8 + c] bulge chunk c
  int64_t lo, hi;               // bulge / bisect: list positions [lo, hi) of this launch
  int64_t rlo, rhi;             // reduce kernel: list positions [rlo, rhi) of this launch
  int cctr;                     // bulge: counter index of this launch
  double* xslots;               // per-CTA X (LP x NP)
  double* wslots;               // per-CTA V (RP x NP), vector jobs
  double* rbuf;                 // per-slice R (RP x NP), QR path with vectors
  int32_t* flags;               // per-slice load flags (reduce kernel)
  double* bandbuf;              // per-slice 17 diagonals (17 x NP)
  double* debuf;                // per-slice bidiagonal d, e (2 x NP)
  // bidiagonal vector path (vector jobs): logs of the right-side transforms
  double* rvlog;                // per slice, per LQ panel: V (16 x NP) then T (16 x 16)
  double* hhlog;                // per slice: hhcap doubles, right reflectors of the bulge chase
  int64_t hhcap;
  double* hbbuf;                // bulge-chase windows in global memory (large n)
  double* vsel;                 // per slice: right singular vectors (RP x NP)
  double* iiscr;                // inverse-iteration scratch
  int btw;                      // back-transform vectors per pass
  int by_slice;                 // state arrays indexed by slice (state-keeping jobs)
  int qr_stages;                // cp.async ring depth of the reduce kernel
  int64_t L, n, LP, NP, RP;
  int transposed, use_qr, bidiag, stats;
  int wtwo;                     // reduce kernel: two-stage warp rings (else one stage)
  int team_yb;                  // team updates: Y partial buffers (2, or 1 when shared memory is short)
  double tol;
  int max_sweeps, max_inner;
};

struct __align__(16) JacobiSmem {
  double xs[2][GW * XS];
  double g[2][GW * GS];
  double w[2][GW * WS];
  double cd[GW];
  double co[GW];
  double nd[GW];
  int partner[GW];
  int flag[4];
};

// Finalize scratch lives after JacobiSmem (sized by NS = next_pow2(n)), so
// the sort keys survive while the Jacobi staging buffers are reused.
struct FinalView {
  double* key;
  int* idx;
  double* dots;
  double* red;
};

__device__ __forceinline__ FinalView final_view(unsigned char* base, int ns) {
  FinalView f;
  f.key = reinterpret_cast<double*>(base + sizeof(JacobiSmem));
  f.dots = f.key + ns;
  f.red = f.dots + TPB;
  f.idx = reinterpret_cast<int*>(f.red + TPB / 32);
  return f;
}

size_t jacobi_smem_bytes(int ns) {
  return sizeof(JacobiSmem) + size_t(ns) * (sizeof(double) + sizeof(int)) +
         (TPB + TPB / 32) * sizeof(double);
}

constexpr int QR_YZ_DOUBLES = BW * GS + GW * ZS;  // y and z of the streaming updates
struct __align__(16) QrSmemFixed {
  double t[BW * 17];
  double sg[4][BW * 17];  // per row-quarter partial Gram (NT / 128 used)
  // (the streaming updates' y (BW x GS) and z (GW x ZS) live AFTER the panel,
  // just below their per-warp regions: the team updates, which do not use
  // them, put their own buffers over the same space)
  double red[16][BW];     // per-warp partials (NT / 32 used)
  double sums[BW];
  double wv[BW];
  double tau[BW];
  double scal[2 + BW];
  double prow[2][BW];
  double psum[2][BW];
};

// Index of a slice's factorisation state: its list position, or (for the
// state-keeping jobs) the slice number itself so a later call can find it.
__device__ __forceinline__ int64_t state_index(const SvdParams& P, int64_t it) {
  return P.by_slice ? (P.ids ? P.ids[it] : it) : it;
}

__device__ __forceinline__ void stat_add(const SvdParams& P, int k, unsigned long long v) {
  if (P.stats && threadIdx.x == 0) atomicAdd(&g_stats[k], v);
}

__device__ __forceinline__ int64_t gcol(int k, int I, int J) {
  return k < BW ? int64_t(I) * BW + k : int64_t(J) * BW + (k - BW);
}

// Stage rows [r0, r0+RCH) of the 32 pair columns (blocks I, J) of M into buf.
__device__ __forceinline__ void stage_pair(double* buf, const double* M, int64_t ld, int64_t r0,
                                           int I, int J) {
#pragma unroll
  for (int q = 0; q < (GW * RCH / 2) / TPB; ++q) {
    const int c = threadIdx.x + q * TPB;
    const int col = c >> 5;
    const int r2 = (c & 31) * 2;
    cp_async16(buf + col * XS + r2, M + r0 + r2 + gcol(col, I, J) * ld);
  }
  cp_async_commit();
}

// ======================================================================
//                               Jacobi core
// ======================================================================

// G = T_P^T T_P over `rows` rows (multiple of RCH).  Result in g (row-major, GS).
__device__ void gram_pair(JacobiSmem& sm, const double* T, int64_t ld, int64_t rows, int I, int J,
                          double* g) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int ti = warp >> 1, tj0 = (warp & 1) * 2;
  double a00[2] = {0, 0}, a01[2] = {0, 0}, a10[2] = {0, 0}, a11[2] = {0, 0};
  const int64_t nch = rows / RCH;
  stage_pair(sm.xs[0], T, ld, 0, I, J);
  for (int64_t ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      stage_pair(sm.xs[(ch + 1) & 1], T, ld, (ch + 1) * RCH, I, J);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* xs = sm.xs[ch & 1];
    const double* xa = xs + (ti * 8 + gq) * XS + tq;
    const double* xb = xs + (tj0 * 8 + gq) * XS + tq;
#pragma unroll
    for (int k4 = 0; k4 < RCH / 4; ++k4) {
      const double a = xa[k4 * 4];
      dmma884(a00[k4 & 1], a01[k4 & 1], a, xb[k4 * 4]);
      dmma884(a10[k4 & 1], a11[k4 & 1], a, xb[8 * XS + k4 * 4]);
    }
    __syncthreads();
  }
  const int row = ti * 8 + gq;
  g[row * GS + tj0 * 8 + 2 * tq] = a00[0] + a00[1];
  g[row * GS + tj0 * 8 + 2 * tq + 1] = a01[0] + a01[1];
  g[row * GS + (tj0 + 1) * 8 + 2 * tq] = a10[0] + a10[1];
  g[row * GS + (tj0 + 1) * 8 + 2 * tq + 1] = a11[0] + a11[1];
  __syncthreads();
}

// M_P <- M_P * W over `rows` rows (W column-major, stride WS).
__device__ void apply_pair(JacobiSmem& sm, double* M, int64_t ld, int64_t rows, int I, int J,
                           const double* w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t nch = rows / RCH;
  stage_pair(sm.xs[0], M, ld, 0, I, J);
  for (int64_t ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      stage_pair(sm.xs[(ch + 1) & 1], M, ld, (ch + 1) * RCH, I, J);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    double* xs = sm.xs[ch & 1];
    double acc[4][2];
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
    const double* xa = xs + tq * XS + warp * 8 + gq;
    const double* wb = w + gq * WS + tq;
#pragma unroll
    for (int k4 = 0; k4 < GW / 4; ++k4) {
      const double a = xa[k4 * 4 * XS];
#pragma unroll
      for (int c = 0; c < 4; ++c) dmma884(acc[c][0], acc[c][1], a, wb[c * 8 * WS + k4 * 4]);
    }
    // Each warp reads and writes only its own 8 rows: in-place is safe.
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      xs[(c * 8 + 2 * tq) * XS + warp * 8 + gq] = acc[c][0];
      xs[(c * 8 + 2 * tq + 1) * XS + warp * 8 + gq] = acc[c][1];
    }
    __syncthreads();
    const int64_t r0 = ch * RCH;
#pragma unroll
    for (int q = 0; q < (GW * RCH / 2) / TPB; ++q) {
      const int c = threadIdx.x + q * TPB;
      const int col = c >> 5;
      const int r2 = (c & 31) * 2;
      *reinterpret_cast<double2*>(M + r0 + r2 + gcol(col, I, J) * ld) =
          *reinterpret_cast<const double2*>(xs + col * XS + r2);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int rr_pos(int i, int round) {
  return i == 0 ? 0 : ((i - 1 + round) % (GW - 1)) + 1;
}

// Rotation W of the 32x32 Gram in sm.g[0] (cyclic round-robin Jacobi,
// `max_inner` sweeps).  Returns the sm.w buffer index holding W.
__device__ int eig_pair(JacobiSmem& sm, double tol, int max_inner) {
  const int tid = threadIdx.x;
  for (int e = tid; e < GW * GW; e += TPB) {
    const int j = e >> 5, r = e & 31;
    sm.w[0][j * WS + r] = (j == r) ? 1.0 : 0.0;
  }
  int gb = 0, wb = 0;
  for (int sweep = 0; sweep < max_inner; ++sweep) {
    if (tid == 0) sm.flag[1] = 0;
    __syncthreads();
    for (int round = 0; round < GW - 1; ++round) {
      const double* G = sm.g[gb];
      if (tid < GW / 2) {
        const int p = rr_pos(tid, round), q = rr_pos(GW - 1 - tid, round);
        const double a = G[p * GS + p], d = G[q * GS + q], b = G[p * GS + q];
        double c = 1.0, s = 0.0, npp = a, nqq = d;
        if (a > 0.0 && d > 0.0 && fabs(b) > tol * sqrt(a * d)) {
          const double zeta = (d - a) / (2.0 * b);
          double t;
          if (fabs(zeta) > 1e150) {
            t = 0.5 / zeta;
          } else {
            t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          }
          c = rsqrt(1.0 + t * t);
          s = t * c;
          npp = a - t * b;
          nqq = d + t * b;
          sm.flag[1] = 1;
        }
        sm.cd[p] = c;
        sm.cd[q] = c;
        sm.co[p] = -s;
        sm.co[q] = s;
        sm.nd[p] = npp;
        sm.nd[q] = nqq;
        sm.partner[p] = q;
        sm.partner[q] = p;
      }
      __syncthreads();
      double* Gn = sm.g[gb ^ 1];
      const double* W = sm.w[wb];
      double* Wn = sm.w[wb ^ 1];
      const int i = tid >> 3, j0 = tid & 7;
      const double di = sm.cd[i], oi = sm.co[i];
      const int pi = sm.partner[i];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = j0 + 8 * jj;
        const int pj = sm.partner[j];
        const double dj = sm.cd[j], oj = sm.co[j];
        double val;
        if (j == i) {
          val = sm.nd[i];
        } else if (j == pi) {
          val = 0.0;
        } else {
          val = di * (dj * G[i * GS + j] + oj * G[i * GS + pj]) +
                oi * (dj * G[pi * GS + j] + oj * G[pi * GS + pj]);
        }
        Gn[i * GS + j] = val;
        Wn[j * WS + i] = dj * W[j * WS + i] + oj * W[pj * WS + i];
      }
      __syncthreads();
      gb ^= 1;
      wb ^= 1;
    }
    const int any = sm.flag[1];
    __syncthreads();
    if (!any) break;
  }
  return wb;
}

__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < TPB / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

// Orthonormalise column cols[j] of Q (ld, length len) against cols[0..j-1]
// (Gram-Schmidt twice, 8 columns per block pass); a vanished column is
// replaced by the next canonical basis vector orthogonalised likewise.
__device__ void cgs2_fix(FinalView& fs, double* Q, int64_t ld, int64_t len, const int* cols, int j) {
  int64_t basis = 0;
  double* qj = Q + int64_t(cols ? cols[j] : j) * ld;
  // The complement of the j previous columns has dimension len - j, so some
  // canonical vector keeps a residual >= sqrt((len - j) / len): accept the
  // first one above half of that bound.
  const double cthr = 0.5 * sqrt(double(len - j) / double(len));
  for (int64_t attempt = 0; attempt <= len; ++attempt) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int i0 = 0; i0 < j; i0 += TPB / 32) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int i = i0 + warp;
        double d = 0.0;
        if (i < j) {
          const double* qi = Q + int64_t(cols ? cols[i] : i) * ld;
          for (int64_t r = lane; r < len; r += 32) d += qi[r] * qj[r];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0) fs.dots[warp] = d;
        __syncthreads();
        const int cnt = min(TPB / 32, j - i0);
        for (int64_t r = threadIdx.x; r < len; r += TPB) {
          double x = qj[r];
          for (int q = 0; q < cnt; ++q) x -= fs.dots[q] * Q[r + int64_t(cols ? cols[i0 + q] : i0 + q) * ld];
          qj[r] = x;
        }
        __syncthreads();
      }
    }
    double nrm2 = 0.0;
    for (int64_t r = threadIdx.x; r < len; r += TPB) nrm2 += qj[r] * qj[r];
    nrm2 = block_sum(nrm2, fs.red);
    const double nrm = sqrt(nrm2);
    if (nrm > (attempt ? cthr : 0.5) || attempt == len) {
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int64_t r = threadIdx.x; r < len; r += TPB) qj[r] *= inv;
      __syncthreads();
      if (attempt) {  // one more CGS2 pass after a canonical replacement
        for (int i0 = 0; i0 < j; i0 += TPB / 32) {
          const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
          const int i = i0 + warp;
          double d = 0.0;
          if (i < j) {
            const double* qi = Q + int64_t(cols ? cols[i] : i) * ld;
            for (int64_t r = lane; r < len; r += 32) d += qi[r] * qj[r];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (lane == 0) fs.dots[warp] = d;
          __syncthreads();
          const int cnt = min(TPB / 32, j - i0);
          for (int64_t r = threadIdx.x; r < len; r += TPB) {
            double x = qj[r];
            for (int q = 0; q < cnt; ++q) x -= fs.dots[q] * Q[r + int64_t(cols ? cols[i0 + q] : i0 + q) * ld];
            qj[r] = x;
          }
          __syncthreads();
        }
        double n2 = 0.0;
        for (int64_t r = threadIdx.x; r < len; r += TPB) n2 += qj[r] * qj[r];
        n2 = block_sum(n2, fs.red);
        const double iv = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
        for (int64_t r = threadIdx.x; r < len; r += TPB) qj[r] *= iv;
        __syncthreads();
      }
      return;
    }
    for (int64_t r = threadIdx.x; r < len; r += TPB) qj[r] = (r == basis) ? 1.0 : 0.0;
    ++basis;
    __syncthreads();
  }
}

// Copy slice into X (LP x NP, ld LP), transposing when m < p; zero padding.
// Returns flag: 0 ok, 1 all-zero, 2 non-finite.
// Rows [row0, row0 + rows) of X (= A, or A^T when transposed) into the X
// slot (LP x NP, ld LP); rows < 0 means all P.L rows.
template <int NT>
__device__ int load_slice(const SvdParams& P, const double* __restrict__ A, double* __restrict__ X,
                          double* tile, int64_t row0 = 0, int64_t rows = -1, int part = 0, int parts = 1) {
  // part / parts: the CTAs of a cluster each load every parts-th batch / tile
  // of the slice; the return value is then this CTA's share of the flag as
  // bits (1: saw a non-finite entry, 2: saw a nonzero entry) for the caller
  // to combine across the cluster.
  // Batched so that every thread keeps LB loads in flight (the copy is
  // HBM-latency bound otherwise).
  constexpr int LB = 16;
  const int tid = threadIdx.x;
  const int64_t L = rows < 0 ? P.L : rows, n = P.n, LP = P.LP, NP = P.NP;
  int bad = 0, nonzero = 0;
  if (!P.transposed) {
    const int64_t total = LP * NP;
    double v[LB], w[LB];  // batch in hand, next batch in flight
    auto load_batch = [&](double (&d)[LB], int64_t e0) {
#pragma unroll
      for (int u = 0; u < LB; ++u) {
        const int64_t e = e0 + tid + int64_t(u) * NT;
        const int64_t r = e % LP, c = e / LP;
        d[u] = (e < total && r < L && c < n) ? A[(row0 + r) + c * P.m] : 0.0;
      }
    };
    const int64_t bstep = int64_t(NT) * LB * parts;
    load_batch(w, int64_t(NT) * LB * part);
    for (int64_t e0 = int64_t(NT) * LB * part; e0 < total; e0 += bstep) {
#pragma unroll
      for (int u = 0; u < LB; ++u) v[u] = w[u];
      load_batch(w, e0 + bstep);
#pragma unroll
      for (int u = 0; u < LB; ++u) {
        const int64_t e = e0 + tid + int64_t(u) * NT;
        bad |= !isfinite(v[u]);
        nonzero |= (v[u] != 0.0);
        if (e < total) X[e] = v[u];
      }
    }
  } else {
    // 32 (columns of X) x 128 (rows of X) tiles through shared memory; the
    // next tile's loads are issued as soon as this tile is in shared memory,
    // so they fly while this tile is copied out
    constexpr int LT = 4096 / NT;
    const int64_t nrt = (LP + 127) / 128, ntiles = ((NP + 31) / 32) * nrt;
    double v[LT];
    auto load_tile = [&](int64_t t) {
      const int64_t c0 = (t / nrt) * 32, r0 = (t % nrt) * 128;
#pragma unroll
      for (int u = 0; u < LT; ++u) {
        const int e = tid + u * NT;
        const int cc = e & 31, rr = e >> 5;
        const int64_t c = c0 + cc, r = r0 + rr;
        v[u] = (t < ntiles && r < L && c < n) ? A[c + (row0 + r) * P.m] : 0.0;
      }
    };
    load_tile(part);
    for (int64_t t = part; t < ntiles; t += parts) {
      const int64_t c0 = (t / nrt) * 32, r0 = (t % nrt) * 128;
#pragma unroll
      for (int u = 0; u < LT; ++u) {
        const int e = tid + u * NT;
        bad |= !isfinite(v[u]);
        nonzero |= (v[u] != 0.0);
        tile[(e >> 5) * 33 + (e & 31)] = v[u];
      }
      __syncthreads();
      load_tile(t + parts);
#pragma unroll
      for (int u = 0; u < LT; ++u) {
        const int e = tid + u * NT;
        const int rr = e & 127, cc = e >> 7;
        const int64_t c = c0 + cc, r = r0 + rr;
        if (c < NP && r < LP) X[r + c * LP] = tile[rr * 33 + cc];
      }
      __syncthreads();
    }
  }
  bad = __syncthreads_or(bad);
  nonzero = __syncthreads_or(nonzero);
  if (parts > 1) return (bad ? 1 : 0) | (nonzero ? 2 : 0);
  return bad ? 2 : (nonzero ? 0 : 1);
}

// ======================================================================
//                      Householder QR kernel (tall X)
// ======================================================================

__device__ __forceinline__ double& PAN(double* pan, int64_t prs, int c, int64_t r) {
  return pan[c * prs + r];
}

// MUFU rsqrt / rcp refined by Newton steps (FP64 sqrt and division are long
// library sequences on the dependent path of every Householder step).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double rcp_nr(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  return fma(r, e, r);
}

// Sum 16 per-thread partials over the CTA: butterfly inside each warp (16
// shuffles leave lanes 2v, 2v+1 holding warp-sum v), then 8 warp partials.
template <int NT>
__device__ __forceinline__ void reduce16(double (&acc)[BW], double (&red)[16][BW], double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v8[8], v4[4], v2[2], v1;
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4, h2 = lane & 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double keep = h16 ? acc[8 + i] : acc[i];
    const double give = h16 ? acc[i] : acc[8 + i];
    v8[i] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double keep = h8 ? v8[4 + i] : v8[i];
    const double give = h8 ? v8[i] : v8[4 + i];
    v4[i] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double keep = h4 ? v4[2 + i] : v4[i];
    const double give = h4 ? v4[i] : v4[2 + i];
    v2[i] = keep + __shfl_xor_sync(0xffffffffu, give, 4);
  }
  {
    const double keep = h2 ? v2[1] : v2[0];
    const double give = h2 ? v2[0] : v2[1];
    v1 = keep + __shfl_xor_sync(0xffffffffu, give, 2);
  }
  v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
  if (!(lane & 1)) red[warp][(lane >> 1) & 15] = v1;
  __syncthreads();
  if (threadIdx.x < BW) {
    double v[NT / 32];
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) v[w] = red[w][threadIdx.x];
#pragma unroll
    for (int h = 1; h < NT / 32; h <<= 1)
#pragma unroll
      for (int w = 0; w + h < NT / 32; w += 2 * h) v[w] += v[w + h];
    out[threadIdx.x] = v[0];
  }
  __syncthreads();
}

// Unblocked Householder on panel columns [0,16) of pan (rows k0.., ld prs):
// LAPACK dlarfg/dlarf per column.  Leaves R (upper) in rows <= k0+j and v
// below; tau in q.tau.
template <int NT>
__device__ void panel_factor(QrSmemFixed& q, double* pan, int64_t prs, int64_t k0, int64_t LP) {
  const int tid = threadIdx.x;
  for (int j = 0; j < BW; ++j) {
    const int64_t pr = k0 + j;
    double acc[BW];
#pragma unroll
    for (int c = 0; c < BW; ++c) acc[c] = 0.0;
    for (int64_t r = pr + 1 + tid; r < LP; r += NT) {
      const double x = PAN(pan, prs, j, r);
      acc[0] = fma(x, x, acc[0]);
#pragma unroll
      for (int c = 1; c < BW; ++c)
        if (c > j) acc[c] = fma(x, PAN(pan, prs, c, r), acc[c]);
    }
    reduce16<NT>(acc, q.red, q.sums);
    if (tid == 0) {
      const double alpha = PAN(pan, prs, j, pr);
      const double xn2 = q.sums[0];
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      q.tau[j] = tau;
      q.scal[0] = scal;
      q.scal[1] = beta;
      for (int c = j + 1; c < BW; ++c) q.wv[c] = PAN(pan, prs, c, pr) + scal * q.sums[c];
    }
    __syncthreads();
    const double tau = q.tau[j], scal = q.scal[0], beta = q.scal[1];
    if (tau != 0.0) {
      for (int64_t r = pr + tid; r < LP; r += NT) {
        const double x = PAN(pan, prs, j, r);
        const double vr = (r == pr) ? 1.0 : x * scal;
        const double tv = tau * vr;
#pragma unroll
        for (int c = 1; c < BW; ++c)
          if (c > j) PAN(pan, prs, c, r) -= tv * q.wv[c];
        PAN(pan, prs, j, r) = (r == pr) ? beta : vr;
      }
    }
    __syncthreads();
  }
}

// Register-resident variant: thread t owns rows t + i*TPB (i < RPT) of all
// 16 panel columns, so the BLAS2 column steps touch no shared memory; only
// the 16 reductions per column and the pivot row go through it.
// The panel is read straight from global memory: element (r, c) =
// src[r * sr + c * sc] for lo <= r < nrows, 0 otherwise (all loads in flight).
template <int NT, int RPT>
__device__ __noinline__ void panel_factor_reg(QrSmemFixed& q, double* pan, int64_t prs64, int64_t k064,
                                              int64_t nrows64, double* src, int64_t sr,
                                              int64_t sc, int64_t lo64) {
  // Register-resident panel, column loop NOT fully unrolled: b[i][c] holds
  // panel column j + c of this thread's rows; each loop iteration factors
  // two columns (0, then 1) and shifts the window left by two, so every
  // iteration runs the same code (instruction footprint of two columns).
  const int tid = threadIdx.x;
  const int prs = int(prs64), k0 = int(k064), nrows = int(nrows64), lo = int(lo64);
  double b[RPT][BW];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = tid + i * NT;
    const bool in = r >= lo && r < nrows;
#pragma unroll
    for (int c = 0; c < BW; ++c) b[i][c] = in ? src[int64_t(r) * sr + c * sc] : 0.0;
  }
  // One column step on window column C (the pivot), columns C+1.. updated.
#ifdef STARM_PF_PROBE
  long long pt[4] = {0, 0, 0, 0};
#endif
  auto step = [&](const int j, const int C) {
#ifdef STARM_PF_PROBE
    long long p0 = clock64();
#endif
    const int pr = k0 + j;
    const int par = j & 1;  // double-buffered pivot row / sums: 2 barriers per column
    double acc[BW];
#pragma unroll
    for (int c = 0; c < BW; ++c) acc[c] = 0.0;
    // pivot row to SMEM: one thread branches in (the predicated form costs
    // every warp RPT x 8 store slots per column)
    if (tid == (pr & (NT - 1))) {
      const int ip = pr / NT;
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (i == ip) {
#pragma unroll
          for (int c = 0; c < BW; c += 2)
            *reinterpret_cast<double2*>(&q.prow[par][c]) =
                make_double2(c + C < BW ? b[i][c + C] : 0.0, c + 1 + C < BW ? b[i][c + 1 + C] : 0.0);
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = tid + i * NT;
      if (r > pr) {
        const double x = b[i][C];
        acc[0] = fma(x, x, acc[0]);
#pragma unroll
        for (int c = 1; c + C < BW; ++c) acc[c] = fma(x, b[i][c + C], acc[c]);
      }
    }
#ifdef STARM_PF_PROBE
    long long p1 = clock64();
#endif
    reduce16<NT>(acc, q.red, q.psum[par]);
#ifdef STARM_PF_PROBE
    long long p2 = clock64();
#endif
    // every thread derives the reflector (dlarfg) redundantly
    double pw[BW], sw[BW];
#pragma unroll
    for (int c = 0; c < BW; c += 2) {
      const double2 p2 = *reinterpret_cast<const double2*>(&q.prow[par][c]);
      const double2 s2 = *reinterpret_cast<const double2*>(&q.psum[par][c]);
      pw[c] = p2.x;
      pw[c + 1] = p2.y;
      sw[c] = s2.x;
      sw[c + 1] = s2.y;
    }
    const double alpha = pw[0];
    const double xn2 = sw[0];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {  // dlarfg: tau = 1 + |alpha| / nrm, 1 / (alpha - beta) = sign(alpha) / (|alpha| + nrm)
      const double nrm2 = fma(alpha, alpha, xn2);
      double rn, nrm;
      if (nrm2 > 1e-280 && nrm2 < 1e280) {
        rn = rsqrt_nr(nrm2);
        nrm = nrm2 * rn;
      } else {
        nrm = sqrt(nrm2);
        rn = 1.0 / nrm;
      }
      const double aa = fabs(alpha);
      beta = -copysign(nrm, alpha);
      tau = fma(aa, rn, 1.0);
      scal = copysign(rcp_nr(aa + nrm), alpha);
    }
    if (tid == 0) q.tau[j] = tau;
    if (tau != 0.0) {
      double tw[BW];
#pragma unroll
      for (int c = 1; c + C < BW; ++c) tw[c] = tau * fma(scal, sw[c], pw[c]);
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = tid + i * NT;
        if (r >= pr) {
          const double vr = (r == pr) ? 1.0 : b[i][C] * scal;
#pragma unroll
          for (int c = 1; c + C < BW; ++c) b[i][c + C] = fma(-vr, tw[c], b[i][c + C]);
          b[i][C] = (r == pr) ? beta : vr;
        }
      }
    }
    // column j is final: pan gets the explicit V column (0 above the pivot,
    // 1 on it, v below, 0 past nrows) and the R entries (rows k0 .. pr) go
    // straight back to the source matrix
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = tid + i * NT;
      const double bv = b[i][C];
      if (r < prs) pan[j * prs + r] = (r > pr && r < nrows) ? bv : (r == pr ? 1.0 : 0.0);
      if (r >= k0 && r <= pr) src[int64_t(r) * sr + j * sc] = bv;
    }
#ifdef STARM_PF_PROBE
    long long p3 = clock64();
    pt[0] += p1 - p0;
    pt[1] += p2 - p1;
    pt[2] += p3 - p2;
#endif
  };
#pragma unroll 1
  for (int j = 0; j < BW; j += 2) {
    step(j, 0);
    step(j + 1, 1);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
#pragma unroll
      for (int c = 0; c + 2 < BW; ++c) b[i][c] = b[i][c + 2];
      b[i][BW - 2] = b[i][BW - 1] = 0.0;
    }
  }
  __syncthreads();
#ifdef STARM_PF_PROBE
  if (tid == 0) {
    atomicAdd(&g_stats[ST_CYC_GRAM], (unsigned long long)pt[0]);
    atomicAdd(&g_stats[ST_CYC_EIG], (unsigned long long)pt[1]);
    atomicAdd(&g_stats[ST_CYC_APPLY], (unsigned long long)pt[2]);
  }
#endif
}

// Returns true when the register path ran: then pan already holds the
// explicit V and R is written back through src; otherwise the caller copies
// R out of pan and forms V (explicit_v).
template <int NT>
__device__ bool panel_factor_any(QrSmemFixed& q, double* pan, int64_t prs, int64_t k0, int64_t nrows,
                                 double* src, int64_t sr, int64_t sc, int64_t lo) {
  const int64_t rpt = (nrows + NT - 1) / NT;
  switch (rpt) {
    case 1: panel_factor_reg<NT, 1>(q, pan, prs, k0, nrows, src, sr, sc, lo); return true;
    case 2: panel_factor_reg<NT, 2>(q, pan, prs, k0, nrows, src, sr, sc, lo); return true;
    case 3: panel_factor_reg<NT, 3>(q, pan, prs, k0, nrows, src, sr, sc, lo); return true;
    case 4: panel_factor_reg<NT, 4>(q, pan, prs, k0, nrows, src, sr, sc, lo); return true;
    default:
      for (int c = 0; c < BW; ++c)
        for (int64_t r = threadIdx.x; r < prs; r += NT)
          pan[c * prs + r] = (r >= lo && r < nrows) ? src[r * sr + c * sc] : 0.0;
      __syncthreads();
      panel_factor<NT>(q, pan, prs, k0, nrows);
      return false;
  }
}

// S = V^T V (16x16) on DMMA; V = explicit panel (zeros above, 1 on pivots).
// Warp w computes Gram tile (w & 3) over the rows of quarter w >> 2 (NT /
// 128 quarters interleaved in 4-row groups).
template <int NT>
__device__ void panel_gram(QrSmemFixed& q, const double* pan, int64_t prs, int64_t kc, int64_t LP) {
  constexpr int NH = NT / 128, STEP = 4 * NH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int tile = warp & 3, half = warp >> 2;
  const int ti = tile >> 1, tj = tile & 1;
  double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
  const double* pa = pan + (ti * 8 + gq) * prs + tq;
  const double* pb = pan + (tj * 8 + gq) * prs + tq;
  const int lp = int(LP);
  int r0 = int(kc) + half * 4;
  for (; r0 + 3 * STEP < lp; r0 += 4 * STEP) {  // four independent accumulators
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma884(d0[u], d1[u], pa[r0 + STEP * u], pb[r0 + STEP * u]);
  }
  for (; r0 < lp; r0 += STEP) dmma884(d0[0], d1[0], pa[r0], pb[r0]);
  q.sg[half][(ti * 8 + gq) * 17 + tj * 8 + 2 * tq] = (d0[0] + d0[1]) + (d0[2] + d0[3]);
  q.sg[half][(ti * 8 + gq) * 17 + tj * 8 + 2 * tq + 1] = (d1[0] + d1[1]) + (d1[2] + d1[3]);
  __syncthreads();
  // T (forward, columnwise; LAPACK dlarft): T_jj = tau_j,
  // T[i][j] = -tau_j sum_{l=i}^{j-1} T[i][l] S[l][j]   (thread i owns row i)
  const int i = threadIdx.x;
  if (i < BW) {
    for (int j = 0; j < BW; ++j) q.t[i * 17 + j] = 0.0;
    q.t[i * 17 + i] = q.tau[i];
    for (int j = i + 1; j < BW; ++j) {
      double acc = 0.0;
      for (int l = i; l < j; ++l) {
        double sg = q.sg[0][l * 17 + j];
#pragma unroll
        for (int h = 1; h < NH; ++h) sg += q.sg[h][l * 17 + j];
        acc += q.t[i * 17 + l] * sg;
      }
      q.t[i * 17 + j] = -q.tau[j] * acc;
    }
  }
  __syncthreads();
}

struct Ring {
  double* base;
  int nst;
  __device__ __forceinline__ double* buf(int64_t i) const { return base + (i % nst) * (GW * XS); }
};

// ---------------------------------------------------------------------
// Warp-private streaming trailing updates (no CTA barrier per chunk).
// Each warp owns a private region of WREG doubles (a 2-stage cp.async ring
// plus scratch) after the panel in shared memory.
// ---------------------------------------------------------------------
constexpr int WREG = 1280;  // doubles per warp (two-stage ring)
constexpr int WREG1 = 640;  // single-stage variant for panels too tall for WREG
constexpr int CS16 = 20;    // column stride of a staged 16-row chunk

// C <- (I - V T^T V^T) C for all columns [c_start, NP) of X (ld), 32-column
// blocks in turn, rows [kc, nrows) in 16-row chunks dealt round-robin to the
// warps.  Per block: Y = V^T C (pass 1), a cross-warp sum and Z = T^T Y, then
// C -= V Z (pass 2).  Each warp walks one flat sequence of chunk loads
// (block, pass, chunk) through its cp.async ring, so the first chunk of
// pass 2 and of the next block are already in flight during the barriers of
// the reduction.  Index math is 32-bit with per-lane base pointers.
template <int NT, bool TWO>
__device__ void trailing_update_w(QrSmemFixed& q, double* wbase, const double* pan, int64_t prs64,
                                  double* X, int64_t ld64, int64_t nrows64, int64_t NP64,
                                  int64_t kc64, int64_t cs64) {
  constexpr int WR = TWO ? WREG : WREG1;
  constexpr int NW = NT / 32;
  double* const qy = wbase - QR_YZ_DOUBLES;  // y (BW x GS), z (GW x ZS): just below the warp regions
  double* const qz = qy + BW * GS;
  const int prs = int(prs64), ld = int(ld64), nrows = int(nrows64), NP = int(NP64);
  const int kc = int(kc64), c_start = int(cs64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  double* wr = wbase + warp * WR;  // [TWO ? 2 : 1][32 * CS16]
  const int nck = (nrows - kc) / 16;
  const int my = nck > warp ? (nck - warp + NW - 1) / NW : 0;  // chunks of this warp per pass
  const int nb = (NP - c_start + GW - 1) / GW;
  const int total = nb * 2 * my;
  // staging: lane copies rows (sr2, sr2 + 1) of columns scol + 4 i, i < 8
  const int scol = lane >> 3, sr2 = (lane & 7) * 2;
  auto slot_of = [&](int sq) { return TWO ? (sq & 1) : 0; };
  auto issue = [&](int sq) {
    const int b = sq / (2 * my), i = (sq % (2 * my)) % my;
    const int c0 = c_start + b * GW;
    const int nin = (NP - c0 - scol + 3) >> 2;
    double* dst = wr + slot_of(sq) * (GW * CS16) + scol * CS16 + sr2;
    const double* srcp = X + (c0 + scol) * ld + kc + sr2 + (warp + i * NW) * 16;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool in = u < nin;
      cp_async16(dst + 4 * u * CS16, in ? srcp + 4 * u * ld : X, in ? 16 : 0);
    }
    cp_async_commit();
  };
  // before computing step sq: (two-stage) put sq + 1 in flight, wait for sq
  auto begin = [&](int sq) {
    if (TWO && sq + 1 < total) {
      issue(sq + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
  };
  // after computing step sq: (one stage) the slot is free, load sq + 1 --
  // except after the last chunk of pass 1, whose slot takes the partial Y
  auto end = [&](int sq) {
    __syncwarp();
    if (!TWO && sq + 1 < total && (sq % (2 * my)) != my - 1) issue(sq + 1);
  };
  // slot holding warp w's partial Y after pass 1 of block b: the slot of its
  // last pass-1 chunk (free; the two-stage prefetch went to the other one)
  auto part_off = [&](int w, int b) {
    const int myw = nck > w ? (nck - w + NW - 1) / NW : 0;
    return myw ? slot_of(b * 2 * myw + myw - 1) * (GW * CS16) : 0;
  };
  const double* pa0 = pan + gq * prs + kc + tq;  // A fragments of V^T
  const double* pa1 = pa0 + 8 * prs;
  const double* pv = pan + tq * prs + kc + gq;   // A fragments of V
  const double* zb = qz + gq * ZS + tq;
  if (total > 0) issue(0);
  for (int b = 0; b < nb; ++b) {
    const int c0 = c_start + b * GW;
    // ---- pass 1: Y = V^T C (16 x 32), all 8 tiles per warp over its chunks
    double y[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int t = 0; t < 4; ++t) y[a][t][0] = y[a][t][1] = 0.0;
    for (int i = 0; i < my; ++i) {
      const int sq = b * 2 * my + i;
      begin(sq);
      const double* cs = wr + slot_of(sq) * (GW * CS16) + gq * CS16 + tq;
      const int ro = (warp + i * NW) * 16;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        double av[2], bv[4];
        av[0] = pa0[ro + k4 * 4];
        av[1] = pa1[ro + k4 * 4];
#pragma unroll
        for (int t = 0; t < 4; ++t) bv[t] = cs[t * 8 * CS16 + k4 * 4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int t = 0; t < 4; ++t) dmma884(y[a][t][0], y[a][t][1], av[a], bv[t]);
      }
      end(sq);
    }
    // ---- deterministic cross-warp sum (fixed warp order) into q.y
    {
      double* part = wr + part_off(warp, b) + gq * GW + 2 * tq;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          part[a * 8 * GW + t * 8] = y[a][t][0];
          part[a * 8 * GW + t * 8 + 1] = y[a][t][1];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < BW * GW; e += NT) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) sacc += wbase[w * WR + part_off(w, b) + e];
      qy[(e / GW) * GS + (e % GW)] = sacc;
    }
    __syncthreads();
    if (!TWO && my > 0) issue(b * 2 * my + my);  // first chunk of pass 2
    // ---- Z = T^T Y (16 x 32), column-major (stride ZS) for B fragments
    for (int e = threadIdx.x; e < BW * GW; e += NT) {
      const int ii = e & 15, c = e >> 4;
      double sacc = 0.0;
      for (int l = 0; l <= ii; ++l) sacc += q.t[l * 17 + ii] * qy[l * GS + c];
      qz[c * ZS + ii] = sacc;
    }
    __syncthreads();
    double zf[4][4];  // B fragments of Z
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4)
#pragma unroll
      for (int t = 0; t < 4; ++t) zf[k4][t] = zb[t * 8 * ZS + k4 * 4];
    // ---- pass 2: C -= V Z per chunk
    const int nin = (NP - c0 - scol + 3) >> 2;
    double* xl = X + (c0 + scol) * ld + kc + sr2;
    for (int i = 0; i < my; ++i) {
      const int sq = b * 2 * my + my + i;
      begin(sq);
      double* csb = wr + slot_of(sq) * (GW * CS16);
      const int ro = (warp + i * NW) * 16;
      double acc[2][4][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[a][t][0] = acc[a][t][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < BW / 4; ++k4) {
        double av[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) av[a] = pv[k4 * 4 * prs + ro + a * 8];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int t = 0; t < 4; ++t) dmma884(acc[a][t][0], acc[a][t][1], av[a], zf[k4][t]);
      }
      double* cw = csb + 2 * tq * CS16 + gq;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          cw[t * 8 * CS16 + a * 8] -= acc[a][t][0];
          cw[t * 8 * CS16 + CS16 + a * 8] -= acc[a][t][1];
        }
      __syncwarp();
      const double* cr = csb + scol * CS16 + sr2;
      double* xw = xl + ro;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < nin)
          *reinterpret_cast<double2*>(xw + 4 * u * ld) = *reinterpret_cast<const double2*>(cr + 4 * u * CS16);
      end(sq);
    }
    __syncthreads();  // q.z is rewritten by the next block
  }
  cp_async_wait<0>();
  __syncthreads();
}

// LQ half-step update, warp-private:  C <- C (I - V T V^T) for columns
// [j0, NP) and rows [rmin, nrows) of A (ld).  Each warp owns 8-row tiles
// (rows rc + 8*t, t = warp, warp+8, ...) end to end: Y = C V, Z = Y T (on
// DMMA) and C -= Z V^T never leave the warp.  V[j][c] = pan2[c * prs + j].
constexpr int CS8 = 12;  // column stride of a staged 8-row tile

template <int NT, bool TWO>
__device__ void right_update_w(QrSmemFixed& q, double* wbase, const double* pan2, int64_t prs64,
                               double* A, int64_t ld64, int64_t nrows64, int64_t NP64, int64_t rc64,
                               int64_t rmin64, int64_t j064) {
  constexpr int WR = TWO ? WREG : WREG1;
  constexpr int NW = NT / 32;
  const int prs = int(prs64), ld = int(ld64), nrows = int(nrows64), NP = int(NP64);
  const int rc = int(rc64), rmin = int(rmin64), j0 = int(j064);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  double* wr = wbase + warp * WR;              // ring [TWO ? 2 : 1][32 * CS8]
  double* zs = wr + (TWO ? 2 : 1) * GW * CS8;  // Y / Z scratch [16 * CS8]
  const int nblk = (NP - j0 + GW - 1) / GW;
  const int ntile = (nrows - rc) / 8;
  // staging: lane copies rows (sr2, sr2 + 1) of columns scol + 8 i, i < 4
  const int scol = lane >> 2, sr2 = (lane & 3) * 2;
  double* al = A + (j0 + scol) * ld + sr2;  // + r0 + (32 b + 8 i) ld
  auto stage = [&](int r0, int b, int slot) {
    double* dst = wr + slot * (GW * CS8) + scol * CS8 + sr2;
    const double* srcp = al + r0 + b * GW * ld;
    const int lim = NP - j0 - b * GW - scol;  // column scol + 8 i in range  <=>  8 i < lim
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool in = 8 * i < lim;
      cp_async16(dst + 8 * i * CS8, in ? srcp + 8 * i * ld : A, in ? 16 : 0);
    }
    cp_async_commit();
  };
  const double* pvy = pan2 + gq * prs + j0 + tq;  // Y pass B: V[jb+k4*4+tq][ct*8+gq]
  const double* pvz = pan2 + tq * prs + j0 + gq;  // Z pass B: V[jb+c*8+gq][k4*4+tq]
  // T as B fragments (T[k][n], n = ct*8+gq, k = k4*4+tq), loop-invariant
  double tf[4][2];
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4)
#pragma unroll
    for (int ct = 0; ct < 2; ++ct) tf[k4][ct] = q.t[(k4 * 4 + tq) * 17 + ct * 8 + gq];
  for (int tile = warp; tile < ntile; tile += NW) {
    const int r0 = rc + tile * 8;
    if (r0 + 8 <= rmin) continue;  // rows above the panel are final
    // ---- Y = C V (8 x 16)
    double y[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};  // [ct][k4&1][e]
    stage(r0, 0, 0);
    for (int b = 0; b < nblk; ++b) {
      if (!TWO && b > 0) stage(r0, b, 0);
      if (TWO && b + 1 < nblk) {
        stage(r0, b + 1, (b + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const double* cs = wr + (TWO ? (b & 1) : 0) * (GW * CS8) + tq * CS8 + gq;
      const double* pb = pvy + b * GW;
#pragma unroll
      for (int k4 = 0; k4 < GW / 4; ++k4) {
        const double a = cs[k4 * 4 * CS8];
#pragma unroll
        for (int ct = 0; ct < 2; ++ct)
          dmma884(y[ct][k4 & 1][0], y[ct][k4 & 1][1], a, pb[ct * 8 * prs + k4 * 4]);
      }
      __syncwarp();
    }
    // ---- Z = Y T (8 x 16) on DMMA: Y -> zs row-major, Z -> zs column-major (A fragments)
#pragma unroll
    for (int ct = 0; ct < 2; ++ct) {
      zs[gq * 16 + ct * 8 + 2 * tq] = y[ct][0][0] + y[ct][1][0];
      zs[gq * 16 + ct * 8 + 2 * tq + 1] = y[ct][0][1] + y[ct][1][1];
    }
    __syncwarp();
    double z[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const double a = zs[gq * 16 + k4 * 4 + tq];
#pragma unroll
      for (int ct = 0; ct < 2; ++ct) dmma884(z[ct][0], z[ct][1], a, tf[k4][ct]);
    }
    __syncwarp();
#pragma unroll
    for (int ct = 0; ct < 2; ++ct) {
      zs[(ct * 8 + 2 * tq) * CS8 + gq] = z[ct][0];
      zs[(ct * 8 + 2 * tq + 1) * CS8 + gq] = z[ct][1];
    }
    __syncwarp();
    double zf[4];
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) zf[k4] = zs[(k4 * 4 + tq) * CS8 + gq];
    // ---- C -= Z V^T, block by block
    stage(r0, 0, 0);
    for (int b = 0; b < nblk; ++b) {
      if (!TWO && b > 0) stage(r0, b, 0);
      if (TWO && b + 1 < nblk) {
        stage(r0, b + 1, (b + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      double* csb = wr + (TWO ? (b & 1) : 0) * (GW * CS8);
      const double* pb = pvz + b * GW;
      double acc[4][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < BW / 4; ++k4)
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma884(acc[c][0], acc[c][1], zf[k4], pb[k4 * 4 * prs + c * 8]);
      double* cw = csb + 2 * tq * CS8 + gq;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        cw[c * 8 * CS8] -= acc[c][0];
        cw[c * 8 * CS8 + CS8] -= acc[c][1];
      }
      __syncwarp();
      const double* cr = csb + scol * CS8 + sr2;
      double* aw = al + r0 + b * GW * ld;
      const int lim = NP - j0 - b * GW - scol;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (8 * i < lim)
          *reinterpret_cast<double2*>(aw + 8 * i * ld) = *reinterpret_cast<const double2*>(cr + 8 * i * CS8);
      __syncwarp();
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// ---------------------------------------------------------------------
// Register-resident team updates (one HBM/L2 read + one write of every
// trailing block per panel).
//
// The warps form teams of TW in {1, 2, 4, 8}; a team owns one 8-column group
// (left update) or one 8-row tile (right update) at a time and holds it in
// registers across both passes: each warp keeps up to TT 8x8 blocks, two
// doubles per lane, in a layout that is at once the B (A) fragment of
// pass 1 and the accumulator of pass 2 (pass 1 sums over the rows (columns)
// in the order the lane holds them; pass 2's k index is permuted to
// pi(h, e, t) = 8h + t + 4e, which the T fragments of Z absorb).  While a
// group is processed, the warp's blocks of its next group stream into a
// per-warp SMEM stage by cp.async, so the global latency hides behind the
// DMMA work.  The team sums its partial Y through SMEM in a fixed warp
// order (deterministic), every warp forms Z on DMMA, and pass 2 accumulates
// -Z V^T straight into the held blocks.  TW is the smallest team whose
// registers cover the rows (columns); beyond 8 * TT blocks the caller falls
// back to the ring path.
//
// SMEM (after the panel): ybuf 2 x NW x 128 doubles, then the stage
// NW x TT x 64 doubles.
// ---------------------------------------------------------------------
constexpr int TT = 16;  // 8x8 blocks per warp held in registers
constexpr int YB = 144;  // doubles per warp partial of Y (padded: conflict-free 16-byte reads)
constexpr int TEAM_SMEM_DOUBLES = 2 * 8 * YB + 8 * TT * 64;   // for 8 warps, two Y buffers
constexpr int TEAM_SMEM_DOUBLES1 = 1 * 8 * YB + 8 * TT * 64;  // one Y buffer (an extra team barrier per group)

// Team sum of the warps' partial Y (fixed warp order): lane gets the four
// values Y[4kk + tq][gq] (left) / Y[gq][4kk + tq] (right), stored at
// gq * 18 + tq * 4 + kk of every warp's block.
template <int tw>
__device__ __forceinline__ void team_ysum(const double* tb, int gq, int tq, double (&a)[4]) {
  const double* src = tb + gq * 18 + tq * 4;
  double2 s0 = *reinterpret_cast<const double2*>(src), s1 = *reinterpret_cast<const double2*>(src + 2);
#pragma unroll
  for (int w = 1; w < tw; ++w) {
    const double2 u0 = *reinterpret_cast<const double2*>(src + w * YB);
    const double2 u1 = *reinterpret_cast<const double2*>(src + w * YB + 2);
    s0.x += u0.x;
    s0.y += u0.y;
    s1.x += u1.x;
    s1.y += u1.y;
  }
  a[0] = s0.x;
  a[1] = s0.y;
  a[2] = s1.x;
  a[3] = s1.y;
}

__device__ __forceinline__ int64_t round_up16(int64_t v) { return (v + 15) & ~int64_t(15); }

__device__ __forceinline__ void team_sync(int team, int tw) {
  if (tw == 1) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(tw * 32) : "memory");
}

template <int NT>
__device__ __forceinline__ int team_width(int blocks) {
  int tw = 1;
  while (tw < NT / 32 && tw * TT < blocks) tw <<= 1;
  return tw * TT >= blocks ? tw : 0;
}

// T as B fragments of Z^T = Y^T T' / Z = Y T' with T'[l][8h + 2t + e] =
// T[l][8h + t + 4e]: tf[kk][h] = T[4kk + tq][8h + phi(gq)], phi(j) = (j >> 1) + 4 (j & 1).
__device__ __forceinline__ void load_tf(const QrSmemFixed& q, double (&tf)[4][2], int gq, int tq) {
  const int ph = (gq >> 1) + 4 * (gq & 1);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int h = 0; h < 2; ++h) tf[kk][h] = q.t[(4 * kk + tq) * 17 + 8 * h + ph];
}

// A slice may be factored by a CLUSTER of CTAs (few slices, many SMs): every
// CTA factors each panel redundantly (same arithmetic, same bits, the panel
// and T in its own shared memory) and takes every csize-th column group /
// row tile of the trailing updates; the matrix lives in global memory (L2),
// so a cluster barrier (release / acquire) after every update orders them.
struct ClusterPos {
  int rank, size;
};
__device__ __forceinline__ ClusterPos cluster_pos() {
  unsigned r, n;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return ClusterPos{int(r), int(n)};
}
__device__ __forceinline__ void cluster_sync(const ClusterPos& cp) {
  if (cp.size > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// C <- (I - V T^T V^T) C on rows [r0, r0 + 8 ntiles) x columns [c_start, NP)
// of X (ld); V = pan (explicit: zero above the pivots), T = q.t.
// Lane (gq, tq) holds C[2tq + ks][gq] of each block (ks = 0, 1).
template <int NT, int tw, bool CL, int nyb>
__device__ __noinline__ void team_left_update_t(QrSmemFixed& q, double* ybuf, const double* pan, int prs,
                                                double* X, int ld, int ntiles, int NP, int r0, int c_start,
                                                ClusterPos cpin) {
  const ClusterPos cp = CL ? cpin : ClusterPos{0, 1};  // (compile-time 1 CTA: the unsplit code)
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  const int nteams = (NW / tw) * cp.size, team = (warp / tw) * cp.size + cp.rank, wit = warp % tw;
  const int lteam = warp / tw;  // team inside this CTA (barrier id, Y partials)
  const int my = wit < ntiles ? (ntiles - wit + tw - 1) / tw : 0;
  const int ngroups = (NP - c_start) >> 3;
  double tf[4][2];
  load_tf(q, tf, gq, tq);
  const int rw = r0 + wit * 8;
  constexpr int ts = tw * 8;                        // row stride between a warp's blocks
  const double* pA = pan + gq * prs + rw + 2 * tq;  // V[row 2tq (+ks)][col gq (+8h)]
  const double* pB = pan + tq * prs + rw + gq;      // V[row gq][col tq (+8h+4e)]
  double* st = ybuf + nyb * NW * YB + warp * (TT * 64) + 2 * lane;  // stage slot i: st + 64 i
  auto issue = [&](int g) {
    const double* src = X + (c_start + 8 * g + gq) * ld + rw + 2 * tq;
#pragma unroll
    for (int i = 0; i < TT; ++i)
      if (i < my) cp_async16(st + 64 * i, src + i * ts);
    cp_async_commit();
  };
  if (team < ngroups) issue(team);
  int it = 0;
  for (int g = team; g < ngroups; g += nteams, ++it) {
    cp_async_wait<0>();
    double c[TT][2];
#pragma unroll
    for (int i = 0; i < TT; ++i)
      if (i < my) {
        const double2 v = *reinterpret_cast<const double2*>(st + 64 * i);
        c[i][0] = v.x;
        c[i][1] = v.y;
      } else {
        c[i][0] = c[i][1] = 0.0;  // (ends the block's liveness across groups)
      }
    if (g + nteams < ngroups) issue(g + nteams);  // own slots were just read
    // pass 1: Y = V^T C (16 x 8); lane accumulates Y[8h + gq][2tq + e] in
    // four chains per half
    double y[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < 4; ++u) y[h][u][0] = y[h][u][1] = 0.0;
#pragma unroll
    for (int i = 0; i < TT; ++i) {
      if (i >= my) break;  // (a branch, not predication: predicated-off DMMAs still occupy the pipe)
      {
        const double* pa = pA + i * ts;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 va = *reinterpret_cast<const double2*>(pa + 8 * h * prs);
          dmma884n(y[h][(2 * i) & 3][0], y[h][(2 * i) & 3][1], va.x, c[i][0]);
          dmma884n(y[h][(2 * i + 1) & 3][0], y[h][(2 * i + 1) & 3][1], va.y, c[i][1]);
        }
      }
    }
    double* yb = ybuf + (nyb == 2 ? (it & 1) : 0) * NW * YB;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {  // Y[r = 8h + gq][c = 2tq + e] -> c * 18 + (r & 3) * 4 + (r >> 2)
        const int r = 8 * h + gq;
        yb[warp * YB + (2 * tq + e) * 18 + (r & 3) * 4 + (r >> 2)] =
            (y[h][0][e] + y[h][1][e]) + (y[h][2][e] + y[h][3][e]);
      }
    team_sync(lteam, tw);
    // Z^T = Y^T T': A[gq][tq] of k-step kk = Y[4kk + tq][gq]; lane ends with
    // zt[h][e] = Z[8h + tq + 4e][gq]
    double zt[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    double ya[4];
    team_ysum<tw>(yb + lteam * tw * YB, gq, tq, ya);
    if (nyb == 1) team_sync(lteam, tw);  // one Y buffer: all reads before the next group's writes
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int h = 0; h < 2; ++h) dmma884n(zt[h][0], zt[h][1], ya[kk], tf[kk][h]);
    // pass 2: C^T += (-Z^T) V^T, k-step (h, e) <-> k = 8h + tq + 4e,
    // k-step-major so consecutive DMMAs update different blocks
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const double nz = -zt[kk >> 1][kk & 1];
      const double* pb = pB + (8 * (kk >> 1) + 4 * (kk & 1)) * prs;
#pragma unroll
      for (int i = 0; i < TT; ++i) {
        if (i >= my) break;
        dmma884n(c[i][0], c[i][1], nz, pb[i * ts]);
      }
    }
    double* xc = X + (c_start + 8 * g + gq) * ld + rw + 2 * tq;
#pragma unroll
    for (int i = 0; i < TT; ++i)
      if (i < my) *reinterpret_cast<double2*>(xc + i * ts) = make_double2(c[i][0], c[i][1]);
  }
}

template <int NT, bool CL>
__device__ bool team_left_update(QrSmemFixed& q, double* ybuf, const double* pan, int prs, double* X,
                                 int ld, int nrows, int NP, int r0, int c_start, ClusterPos cp, int nyb) {
  const int ntiles = (nrows - r0) >> 3;
  switch (team_width<NT>(ntiles)) {
    case 1:
      if (nyb == 2) team_left_update_t<NT, 1, CL, 2>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      else team_left_update_t<NT, 1, CL, 1>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      break;
    case 2:
      if (nyb == 2) team_left_update_t<NT, 2, CL, 2>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      else team_left_update_t<NT, 2, CL, 1>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      break;
    case 4:
      if (nyb == 2) team_left_update_t<NT, 4, CL, 2>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      else team_left_update_t<NT, 4, CL, 1>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      break;
    case 8:
      if (nyb == 2) team_left_update_t<NT, 8, CL, 2>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      else team_left_update_t<NT, 8, CL, 1>(q, ybuf, pan, prs, X, ld, ntiles, NP, r0, c_start, cp);
      break;
    default: return false;
  }
  __syncthreads();
  return true;
}

// C <- C (I - V T V^T) on rows [rmin, nrows) x columns [j0, NP) of A (ld);
// V[j][c] = pan2[c * prs + j] (explicit, zero left of the pivots).
// Lane (gq, tq) holds C[gq][2tq + e] of each block.
template <int NT, int tw, bool CL, int nyb>
__device__ __noinline__ void team_right_update_t(QrSmemFixed& q, double* ybuf, const double* pan2, int prs,
                                                 double* A, int ld, int nrows, int nch, int rmin, int j0,
                                                 ClusterPos cpin) {
  const ClusterPos cp = CL ? cpin : ClusterPos{0, 1};
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  const int nteams = (NW / tw) * cp.size, team = (warp / tw) * cp.size + cp.rank, wit = warp % tw;
  const int lteam = warp / tw;
  const int my = wit < nch ? (nch - wit + tw - 1) / tw : 0;
  const int ntile = (nrows - rmin) >> 3;
  double tf[4][2];
  load_tf(q, tf, gq, tq);
  const int cw = j0 + wit * 8;
  constexpr int cs = tw * 8;                          // column stride between a warp's blocks
  const double* pB1 = pan2 + gq * prs + cw + 2 * tq;  // V[col 2tq (+e)][8h + gq]
  const double* pB2 = pan2 + tq * prs + cw + gq;      // V[col gq][8h + tq + 4e]
  double* st = ybuf + nyb * NW * YB + warp * (TT * 64) + 2 * lane;
  int ldc = cs * ld;
  auto issue = [&](int t) {
    const double* src = A + (cw + 2 * tq) * ld + rmin + 8 * t + gq;
#pragma unroll
    for (int i = 0; i < TT; ++i)
      if (i < my) {
        cp_async8(st + 64 * i, src + i * ldc);
        cp_async8(st + 64 * i + 1, src + i * ldc + ld);
      }
    cp_async_commit();
  };
  if (team < ntile) issue(team);
  int it = 0;
  for (int t = team; t < ntile; t += nteams, ++it) {
    cp_async_wait<0>();
    double c[TT][2];
#pragma unroll
    for (int i = 0; i < TT; ++i)
      if (i < my) {
        const double2 v = *reinterpret_cast<const double2*>(st + 64 * i);
        c[i][0] = v.x;
        c[i][1] = v.y;
      } else {
        c[i][0] = c[i][1] = 0.0;
      }
    if (t + nteams < ntile) issue(t + nteams);
    // pass 1: Y = C V (8 x 16); lane accumulates Y[gq][8h + 2tq + e]
    double y[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < 4; ++u) y[h][u][0] = y[h][u][1] = 0.0;
#pragma unroll
    for (int i = 0; i < TT; ++i) {
      if (i >= my) break;
      {
        const double* pb = pB1 + i * cs;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 vb = *reinterpret_cast<const double2*>(pb + 8 * h * prs);
          dmma884n(y[h][(2 * i) & 3][0], y[h][(2 * i) & 3][1], c[i][0], vb.x);
          dmma884n(y[h][(2 * i + 1) & 3][0], y[h][(2 * i + 1) & 3][1], c[i][1], vb.y);
        }
      }
    }
    double* yb = ybuf + (nyb == 2 ? (it & 1) : 0) * NW * YB;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {  // Y[r = gq][c = 8h + 2tq + e] -> r * 18 + (c & 3) * 4 + (c >> 2)
        const int c = 8 * h + 2 * tq + e;
        yb[warp * YB + gq * 18 + (c & 3) * 4 + (c >> 2)] = (y[h][0][e] + y[h][1][e]) + (y[h][2][e] + y[h][3][e]);
      }
    team_sync(lteam, tw);
    // Z = Y T': A[gq][tq] of k-step kk = Y[gq][4kk + tq]; lane ends with
    // z[h][e] = Z[gq][8h + tq + 4e]
    double z[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    double ya[4];
    team_ysum<tw>(yb + lteam * tw * YB, gq, tq, ya);
    if (nyb == 1) team_sync(lteam, tw);  // one Y buffer: all reads before the next group's writes
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int h = 0; h < 2; ++h) dmma884n(z[h][0], z[h][1], ya[kk], tf[kk][h]);
    // pass 2: C += (-Z) V^T, k-step (h, e) <-> k = 8h + tq + 4e
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const double nz = -z[kk >> 1][kk & 1];
      const double* pb = pB2 + (8 * (kk >> 1) + 4 * (kk & 1)) * prs;
#pragma unroll
      for (int i = 0; i < TT; ++i) {
        if (i >= my) break;
        dmma884n(c[i][0], c[i][1], nz, pb[i * cs]);
      }
    }
    double* xr = A + (cw + 2 * tq) * ld + rmin + 8 * t + gq;
    asm volatile("" : "+r"(ldc));
#pragma unroll
    for (int i = 0; i < TT; ++i)
      if (i < my) {
        xr[i * ldc] = c[i][0];
        xr[i * ldc + ld] = c[i][1];
      }
  }
}

template <int NT, bool CL>
__device__ bool team_right_update(QrSmemFixed& q, double* ybuf, const double* pan2, int prs, double* A,
                                  int ld, int nrows, int NP, int rmin, int j0, ClusterPos cp, int nyb) {
  const int nch = (NP - j0) >> 3;
  switch (team_width<NT>(nch)) {
    case 1:
      if (nyb == 2) team_right_update_t<NT, 1, CL, 2>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      else team_right_update_t<NT, 1, CL, 1>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      break;
    case 2:
      if (nyb == 2) team_right_update_t<NT, 2, CL, 2>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      else team_right_update_t<NT, 2, CL, 1>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      break;
    case 4:
      if (nyb == 2) team_right_update_t<NT, 4, CL, 2>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      else team_right_update_t<NT, 4, CL, 1>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      break;
    case 8:
      if (nyb == 2) team_right_update_t<NT, 8, CL, 2>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      else team_right_update_t<NT, 8, CL, 1>(q, ybuf, pan2, prs, A, ld, nrows, nch, rmin, j0, cp);
      break;
    default: return false;
  }
  __syncthreads();
  return true;
}

// Panel -> explicit V (zeros above the pivot, 1 on it) for rows [0, prs).
template <int NT>
__device__ __forceinline__ void explicit_v(double* pan, int64_t prs, int64_t k0, int64_t nrows) {
  for (int c = 0; c < BW; ++c) {
    double* col = pan + c * prs;
    for (int64_t r = threadIdx.x; r < prs; r += NT) {
      if (r < k0 + c || r >= nrows) col[r] = 0.0;
      else if (r == k0 + c) col[r] = 1.0;
    }
  }
  __syncthreads();
}

// Householder QR of the tall X (LP rows, NP columns, ld LP) in 16-column
// panels with compact-WY trailing updates; leaves R in the leading NP x NP
// block and zeros below it.
template <int NT, bool CL = false>
__device__ __noinline__ void qr_phase(const SvdParams& P, QrSmemFixed& q, double* pan, int64_t prs,
                         double* wbase, double* X, int64_t live, long long& pf, long long& tr,
                         ClusterPos cpin = ClusterPos{0, 1}) {
  const ClusterPos cp = CL ? cpin : ClusterPos{0, 1};
  const int64_t LP = P.LP, NP = P.NP;
  const int tid = threadIdx.x;
  for (int64_t k0 = 0; k0 < NP; k0 += BW) {
    const int64_t kc = (k0 / RCH) * RCH;
    bool reg;
    { long long _a = clock64(); reg = panel_factor_any<NT>(q, pan, prs, k0, LP, X + k0 * LP, 1, LP, 0); pf += clock64() - _a; }
    if (!reg) {
      if (tid < BW * BW) {
        const int c = tid / BW, r = tid % BW;
        if (r <= c) X[(k0 + r) + (k0 + c) * LP] = pan[c * prs + k0 + r];
      }
      __syncthreads();
    }
    if (k0 + BW < NP) {
      if (!reg) explicit_v<NT>(pan, prs, k0, LP);
      panel_gram<NT>(q, pan, prs, kc, LP);
      long long _a = clock64();
      if (!(NT == 256 && P.team_yb &&
            team_left_update<NT, CL>(q, wbase, pan, int(prs), X, int(LP), int(live), int(NP), int(k0),
                                 int(k0 + BW), cp, P.team_yb))) {
        if (cp.rank == 0)  // (the streaming fallback is not split: one CTA of the cluster runs it)
          P.wtwo ? trailing_update_w<NT, true>(q, wbase + QR_YZ_DOUBLES, pan, prs, X, LP, LP, NP, kc, k0 + BW)
                 : trailing_update_w<NT, false>(q, wbase + QR_YZ_DOUBLES, pan, prs, X, LP, LP, NP, kc, k0 + BW);
      }
      tr += clock64() - _a;
    }
    __syncthreads();
    cluster_sync(cp);  // the next panel reads columns every CTA of the cluster updated
  }
  // keep only R (upper triangle of the leading NP x NP block): zero below the
  // diagonal in the rows the band phase reads (< RP; TSQR masks r <= c itself)
  const int zr = int(P.RP < LP ? P.RP : LP), lp = int(LP);
  for (int c = 0; c < int(NP); ++c)
    for (int r = c + 1 + tid; r < zr; r += NT) X[r + int64_t(c) * lp] = 0.0;
  __syncthreads();
  cluster_sync(cp);  // (every CTA writes the same zeros; none may run ahead into the band phase)
}

// Load / factorisation kernel (one CTA per slice, persistent):
//   X (L x n) -> [Householder QR if L > n] -> n x n matrix A (upper
//   triangular R or X itself) -> band reduction  A = Q1 B P1^T  with B
//   upper band (bandwidth 16) by alternating 16-column QR and 16-row LQ
//   panels (compact-WY updates on DMMA, nst-stage cp.async ring) -> the 17
//   diagonals of B to bandbuf.  Vector jobs also log P1's panels (V, T).
template <int NT, bool CL>
__global__ void __launch_bounds__(NT, 1) svd_reduce_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrSmemFixed& q = *reinterpret_cast<QrSmemFixed*>(smem_raw);
  const int64_t LP = P.LP, NP = P.NP, RP = P.RP, n = P.n;
  const int64_t prs = LP + 36;
  double* pan = reinterpret_cast<double*>(smem_raw + sizeof(QrSmemFixed));
  const Ring ring{pan + BW * prs, P.qr_stages};
  double* wbase = pan + BW * prs;  // team buffers / y, z + per-warp regions (aliases the ring)
  __shared__ int64_t cur;
  const int tid = threadIdx.x;
  const ClusterPos cp = CL ? cluster_pos() : ClusterPos{0, 1};
  const int64_t cid = int64_t(blockIdx.x) / cp.size, ncl = int64_t(gridDim.x) / cp.size;
  double* X = P.xslots + cid * LP * NP;  // one working matrix per cluster
  int64_t next_static = P.rlo + cid;

  for (;;) {
    // one CTA per slice: dynamic work counter; a cluster per slice: clusters
    // stride over the list (equal work per slice, no cross-CTA broadcast)
    if (cp.size == 1) {
      if (tid == 0) cur = P.rlo + int64_t(atomicAdd(&P.counter[0], 1ull));
    } else if (tid == 0) {
      cur = next_static;
    }
    next_static += ncl;
    __syncthreads();
    const int64_t it = cur;
    __syncthreads();
    if (it >= P.rhi) break;
    const int64_t si = state_index(P, it);
    const int64_t slice = P.ids ? P.ids[it] : it;
    long long t0 = clock64();
    int flag;
    if (cp.size == 1) {
      flag = load_slice<NT>(P, P.A + slice * P.m * P.p, X, ring.buf(0));
    } else {
      // the cluster's CTAs load interleaved shares of the slice and exchange
      // their flag bits through distributed shared memory
      __shared__ int fbits[8];
      const int mine = load_slice<NT>(P, P.A + slice * P.m * P.p, X, ring.buf(0), 0, -1, cp.rank, cp.size);
      if (tid < cp.size) {  // thread r writes this CTA's bits into CTA r's fbits[rank]
        unsigned long long remote;
        asm volatile("mapa.u64 %0, %1, %2;"
                     : "=l"(remote)
                     : "l"(reinterpret_cast<unsigned long long>(&fbits[cp.rank])), "r"(unsigned(tid)));
        *reinterpret_cast<volatile int*>(remote) = mine;
      }
      cluster_sync(cp);
      int bits = 0;
      for (int r = 0; r < cp.size; ++r) bits |= fbits[r];
      flag = (bits & 1) ? 2 : ((bits & 2) ? 0 : 1);
    }
    if (tid == 0 && cp.rank == 0) {
      P.flags[si] = flag;
      if (flag == 2) atomicMin(&P.status[0], int32_t(slice));
    }
    // (no CTA of a cluster may update X before all have finished writing it;
    // the second barrier also keeps the next slice's flag exchange off fbits)
    cluster_sync(cp);
    if (flag) continue;
    long long t1 = clock64();
    long long pf = 0, tr = 0, ru = 0;
    // ---------------- QR of the tall X (rows LP)
    if (P.L > P.n) qr_phase<NT, CL>(P, q, pan, prs, wbase, X, round_up16(P.L), pf, tr, cp);
    long long t2 = clock64();
    // ---------------- band reduction of the leading NP x NP block (rows RP)
    for (int64_t k = 0; k < NP; k += BW) {
      const int64_t kc = (k / RCH) * RCH;
      bool reg;
      { long long _a = clock64(); reg = panel_factor_any<NT>(q, pan, prs, k, RP, X + k * LP, 1, LP, 0); pf += clock64() - _a; }
      if (!reg) {
        if (tid < BW * BW) {
          const int c = tid / BW, r = tid % BW;
          if (r <= c) X[(k + r) + (k + c) * LP] = pan[c * prs + k + r];
        }
        __syncthreads();
      }
      if (k + BW >= NP) break;
      if (!reg) explicit_v<NT>(pan, prs, k, RP);
      panel_gram<NT>(q, pan, prs, kc, RP);
      {
        long long _a = clock64();
        if (!(NT == 256 && P.team_yb &&
              team_left_update<NT, CL>(q, wbase, pan, int(prs), X, int(LP), int(NP), int(NP), int(k),
                                   int(k + BW), cp, P.team_yb))) {
          if (cp.rank == 0)
            P.wtwo ? trailing_update_w<NT, true>(q, wbase + QR_YZ_DOUBLES, pan, prs, X, LP, RP, NP, kc, k + BW)
                   : trailing_update_w<NT, false>(q, wbase + QR_YZ_DOUBLES, pan, prs, X, LP, RP, NP, kc, k + BW);
        }
        tr += clock64() - _a;
      }
      __syncthreads();
      cluster_sync(cp);  // the LQ panel reads rows every CTA of the cluster updated
      // LQ half-step on rows [k, k+16), columns [k+16, NP)
      const int64_t j0 = k + BW;
      { long long _a = clock64(); reg = panel_factor_any<NT>(q, pan, prs, j0, NP, X + k, LP, 1, j0); pf += clock64() - _a; }
      if (!reg) {
        if (tid < BW * BW) {
          const int c = tid / BW, r = tid % BW;  // R2[r][c] -> A[k+c][j0+r]
          if (r <= c) X[(k + c) + (j0 + r) * LP] = pan[c * prs + j0 + r];
        }
        __syncthreads();
        explicit_v<NT>(pan, prs, j0, NP);
      }
      panel_gram<NT>(q, pan, prs, (j0 / 8) * 8, NP);
      if (P.rvlog && cp.rank == 0) {  // vector jobs: keep P1's panel (V, T) for the back-transformation
        double* dst = P.rvlog + (si * (NP / BW) + k / BW) * (BW * NP + BW * BW);
        for (int c = 0; c < BW; ++c)
          for (int64_t jj = tid; jj < NP; jj += NT) dst[c * NP + jj] = pan[c * prs + jj];
        if (tid < BW * BW) dst[BW * NP + tid] = q.t[(tid / BW) * 17 + (tid % BW)];
      }
      {
        long long _a = clock64();
        if (NT == 256 && P.team_yb &&
            team_right_update<NT, CL>(q, wbase, pan, int(prs), X, int(LP), int(NP), int(NP), int(j0), int(j0),
                                  cp, P.team_yb)) {
        } else if (cp.rank != 0) {
        } else if (P.wtwo) {
          right_update_w<NT, true>(q, wbase + QR_YZ_DOUBLES, pan, prs, X, LP, RP, NP, (j0 / RCH) * RCH, j0, j0);
        } else {
          right_update_w<NT, false>(q, wbase + QR_YZ_DOUBLES, pan, prs, X, LP, RP, NP, (j0 / RCH) * RCH, j0, j0);
        }
        ru += clock64() - _a;
      }
      __syncthreads();
      cluster_sync(cp);  // the next QR panel reads columns every CTA of the cluster updated
    }
    // ---------------- the 17 diagonals of the band (every CTA of a cluster
    // writes the same values; the barrier keeps the next load off X meanwhile)
    double* band = P.bandbuf + si * (BW + 1) * NP;
    for (int d = 0; d <= BW; ++d)
      for (int64_t i = tid; i < NP; i += NT) band[d * NP + i] = (i + d < n) ? X[i + (i + d) * LP] : 0.0;
    __syncthreads();
    cluster_sync(cp);
    long long t3 = clock64();
    stat_add(P, ST_CYC_LOAD, (unsigned long long)(t1 - t0));
    stat_add(P, ST_CYC_QR, (unsigned long long)(t2 - t1));
    stat_add(P, ST_CYC_BAND, (unsigned long long)(t3 - t2));
    stat_add(P, ST_CYC_PFACT, (unsigned long long)pf);
    stat_add(P, ST_CYC_TRAIL, (unsigned long long)tr);
    stat_add(P, ST_CYC_RIGHT, (unsigned long long)ru);
  }
}

// TSQR first level for tall-skinny slices whose 16-column panel does not
// fit in shared memory (e.g. 8192 x 64): block b of a slice is rows
// [b BR, (b + 1) BR) of X; its Householder QR (qr_phase) leaves R_b, which
// goes to rows [b NP, b NP + NP) of the slice's stacked matrix S (SP x n,
// column-major).  S^T S = X^T X, so the bidiagonal path on S gives X's sigma
// and right vectors; the left vectors are formed from X itself (vecout).
template <int NT>
__global__ void __launch_bounds__(NT) svd_tsqr_kernel(SvdParams P, double* S, int64_t BR,
                                                       int64_t nbk, int64_t SP) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrSmemFixed& q = *reinterpret_cast<QrSmemFixed*>(smem_raw);
  const int64_t LP = P.LP, NP = P.NP, n = P.n;
  const int64_t prs = LP + 36;
  double* pan = reinterpret_cast<double*>(smem_raw + sizeof(QrSmemFixed));
  const Ring ring{pan + BW * prs, P.qr_stages};
  double* wbase = pan + BW * prs;
  __shared__ int64_t cur;
  const int tid = threadIdx.x;
  double* X = P.xslots + int64_t(blockIdx.x) * LP * NP;
  long long pf = 0, tr = 0;
  for (;;) {
    if (tid == 0) cur = int64_t(atomicAdd(&P.counter[5], 1ull));
    __syncthreads();
    const int64_t item = cur;
    __syncthreads();
    if (item >= P.count * nbk) break;
    const int64_t it = item / nbk, b = item % nbk;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int64_t row0 = b * BR, rows = P.L - row0 < BR ? P.L - row0 : BR;
    const int flag = load_slice<NT>(P, P.A + slice * P.m * P.p, X, ring.buf(0), row0, rows);
    double* Sd = S + slice * SP * n + b * NP;  // rows b NP .., ld SP
    if (flag == 2) {  // non-finite: poison the block so the stacked pass names the slice
      for (int64_t e = tid; e < NP * n; e += NT) Sd[(e % NP) + (e / NP) * SP] = CUDART_NAN;
      __syncthreads();
      continue;
    }
    if (flag == 0) qr_phase<NT>(P, q, pan, prs, wbase, X, LP, pf, tr);
    for (int64_t e = tid; e < NP * n; e += NT) {
      const int64_t r = e % NP, c = e / NP;
      Sd[r + c * SP] = (flag == 0 && r <= c) ? X[r + c * LP] : 0.0;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------
// Band (upper bandwidth BW) -> upper bidiagonal by Householder bulge
// chasing.  Sweep i (for row i) runs tasks k = 0, 1, ...; task (i, k) has
//   c0 = i + k*BW + 1,  c1 = min(c0 + BW - 1, n - 1),  L = c1 - c0 + 1:
//   right: reflector H on columns [c0, c1] that annihilates row rho's
//          entries (c0, c1] (rho = i for k = 0, else c0 - BW), applied to
//          rows [rho, c1]  (creates fill below the diagonal);
//   left:  reflector G on rows [c0, c1] that annihilates column c0 below
//          the diagonal, applied to columns [c0, min(c0 + 2 BW - 1, n - 1)]
//          (creates the bulge above the band that task k + 1 removes).
// Every task stays inside rows [c0 - BW, c0 + BW - 1] x columns
// [c0, c0 + 2 BW - 1], so tasks whose c0 differ by >= 2 BW are independent.
// Sweep i starts at time step 3 i: tasks of one step have c0 differing by
// >= 3 BW - 1, and every conflicting pair runs in the sequential
// (sweep-major) order, so the result equals the sequential algorithm's bit
// for bit.  One warp per task, a CTA barrier per time step, ~3n steps.
// The working matrix is kept as a diagonal window per row (offsets
// -(BW-1) .. 2 BW - 1, stride HB): in shared memory when it fits, else in a
// per-CTA global (L2-resident) buffer.  Vector jobs log each right
// reflector as 16 doubles (tau, v_1 .. v_{BW-1}).
// ----------------------------------------------------------------------
constexpr int HB = 3 * BW;    // window row stride (odd HB - 1: conflict-free columns)
constexpr int HOFF = BW - 1;  // window index of the diagonal
constexpr int HLOG = BW;      // doubles per logged reflector

__host__ __device__ __forceinline__ int64_t hb_tasks(int64_t n, int64_t i) {  // tasks of sweep i
  return (i >= 0 && i <= n - 3) ? (n - 3 - i) / BW + 1 : 0;
}
__host__ __device__ __forceinline__ int64_t hb_kmax(int64_t n) { return n >= 3 ? hb_tasks(n, 0) : 1; }
__host__ __device__ __forceinline__ int64_t hb_steps(int64_t n) {
  return n >= 3 ? 3 * (n - 3) + hb_tasks(n, n - 3) : 0;
}
__host__ __device__ __forceinline__ int hb_warps(int64_t n, int cap) {  // ceil(kmax / 3) sweeps overlap
  const int64_t w = (hb_kmax(n) + 2) / 3;
  return int(w < 1 ? 1 : (w > cap ? cap : w));
}
__device__ __forceinline__ double& HEL(double* W, int r, int c) { return W[r * (HB - 1) + c + HOFF]; }

// Window accessors of the chase: one flat window (shared or global memory),
// or the rows split over the two CTAs of a cluster (rows < H in rank 0's
// shared memory, the rest in rank 1's; both pointers are generic addresses
// from cluster.map_shared_rank, so either CTA reaches either half).
struct WinFlat {
  double* W;
  __device__ __forceinline__ double* at(int r, int c) const { return W + r * (HB - 1) + c + HOFF; }
};
struct WinSplit {
  double* W0;
  double* W1;
  int H;
  __device__ __forceinline__ double* at(int r, int c) const {
    // (element (r, c) sits at row * HB + (c - r) + HOFF of its half)
    return r < H ? W0 + r * (HB - 1) + c + HOFF : W1 + (r - H) * (HB - 1) + (c - H) + HOFF;
  }
};


// Warp-wide dlarfg: lanes 0..L-1 hold x (0 beyond); on return x holds v
// (lane 0: 1, 0 beyond L), beta the new leading entry; returns tau (0: H = I).
// sqrt and the two divisions go through MUFU rsqrt/rcp + Newton steps:
// tau = 1 + |alpha| / norm, 1 / (alpha - beta) = sign(alpha) / (|alpha| + norm).
// Lanes 16..31 carry a mirror of lanes 0..15 (x of lane l & 15), so the sum
// needs four butterfly levels and both half-warps end with it.
__device__ __forceinline__ double warp_house(double& x, int lane, double& beta) {
  double s2 = (lane & 15) ? x * x : 0.0;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  const double alpha = __shfl_sync(0xffffffffu, x, 0);
  beta = alpha;
  if (s2 == 0.0) return 0.0;
  const double nrm2 = fma(alpha, alpha, s2);
  double rn, nrm;
  if (nrm2 > 1e-280 && nrm2 < 1e280) {
    rn = rsqrt_nr(nrm2);
    nrm = nrm2 * rn;
  } else {
    nrm = sqrt(nrm2);
    rn = 1.0 / nrm;
  }
  const double aa = fabs(alpha);
  beta = -copysign(nrm, alpha);
  const double tau = fma(aa, rn, 1.0);
  const double scal = copysign(rcp_nr(aa + nrm), alpha);
  x = lane ? x * scal : 1.0;
  return tau;
}

// One task of the chase (see above).  The window has BW zero rows of
// padding below row n - 1, so the reflector loops run over all BW entries
// with v_l = 0 beyond L and constant offsets from one base pointer.
// Inactive warps (act false) run the shuffles on zeros and touch nothing, so
// every warp reaches each shuffle converged.
template <class Win>
__device__ __forceinline__ void hb_task(const Win& W, int n, int i, int k, bool act, int lane,
                                        double* vs, double* lg) {
  const int c0 = i + k * BW + 1;
  const int c1 = min(c0 + BW - 1, n - 1);
  const int L = act ? c1 - c0 + 1 : 0;
  const int rho = k ? c0 - BW : i;
  double beta;
  // ---- right reflector from row rho, applied to rows (rho, c1]
  double x = (lane & 15) < L ? *W.at(rho, c0 + (lane & 15)) : 0.0;  // mirrored halves
  const double tau = warp_house(x, lane, beta);
  if (act && lg && lane < BW) lg[lane] = lane ? x : tau;
  double col0 = 0.0;  // this lane's updated A(rho + 1 + lane, c0)
  if (tau != 0.0) {
    if (lane < L) *W.at(rho, c0 + lane) = lane ? 0.0 : beta;
    vs[lane] = x;
    __syncwarp();
    const int r = rho + 1 + lane;
    if (r <= c1) {
      double* row = W.at(r, c0);  // row[l] = A(r, c0 + l)
      double a[BW];
#pragma unroll
      for (int l = 0; l < BW; ++l) a[l] = row[l];
      double w4[4] = {0.0, 0.0, 0.0, 0.0};  // four chains: half the dependent depth
#pragma unroll
      for (int l = 0; l < BW; ++l) w4[l & 3] = fma(a[l], vs[l], w4[l & 3]);
      const double w = ((w4[0] + w4[1]) + (w4[2] + w4[3])) * tau;
      col0 = fma(-w, vs[0], a[0]);
      row[0] = col0;
#pragma unroll
      for (int l = 1; l < BW; ++l) row[l] = fma(-w, vs[l], a[l]);
    }
    __syncwarp();
  }
  // ---- left reflector from column c0, applied to columns (c0, c0 + 2 BW - 1].
  // Its column c0 entries were just produced in registers by lanes
  // c0 + l - rho - 1 (when the right reflector was applied): shuffle them.
  const double ysh = __shfl_sync(0xffffffffu, col0, (c0 + (lane & 15) - rho - 1) & 31);
  double y = (lane & 15) < L ? (tau != 0.0 ? ysh : *W.at(c0 + (lane & 15), c0)) : 0.0;
  const double tl = warp_house(y, lane, beta);
  if (tl != 0.0) {
    if (lane < L) *W.at(c0 + lane, c0) = lane ? 0.0 : beta;
    vs[lane] = y;
    __syncwarp();
    const int c = c0 + 1 + lane;
    if (c < n) {
      double a[BW];
#pragma unroll
      for (int l = 0; l < BW; ++l) a[l] = *W.at(c0 + l, c);  // A(c0 + l, c)
      double w4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < BW; ++l) w4[l & 3] = fma(vs[l], a[l], w4[l & 3]);
      const double w = ((w4[0] + w4[1]) + (w4[2] + w4[3])) * tl;
#pragma unroll
      for (int l = 0; l < BW; ++l) *W.at(c0 + l, c) = fma(-w, vs[l], a[l]);
    }
    __syncwarp();
  }
}

template <bool GMEM>
__global__ void __launch_bounds__(GMEM ? 1024 : 512) svd_bulge_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double vsh[32][32];
  __shared__ int64_t cur;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = int(P.n);
  const int64_t NP = P.NP;
  double* W = GMEM ? P.hbbuf + int64_t(blockIdx.x) * (n + BW) * HB : reinterpret_cast<double*>(smem_raw);
  const WinFlat Wf{W};
  const int64_t kmax = hb_kmax(n), T = hb_steps(n);
  for (;;) {
    if (threadIdx.x == 0) cur = P.lo + int64_t(atomicAdd(&P.counter[P.cctr], 1ull));
    __syncthreads();
    const int64_t it = cur;
    __syncthreads();
    if (it >= P.hi) break;
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    long long t0 = clock64();
    const double* band = P.bandbuf + si * (BW + 1) * NP;
    for (int64_t e = threadIdx.x; e < int64_t(n + BW) * HB; e += blockDim.x) {
      const int r = int(e / HB), d = int(e % HB) - HOFF;
      W[e] = (d >= 0 && d <= BW && r + d < n) ? band[d * NP + r] : 0.0;
    }
    __syncthreads();
    double* lg = P.hhlog ? P.hhlog + si * P.hhcap : nullptr;
    // this warp runs sweeps i == warp (mod nw); sweep i is active at steps
    // [3 i, 3 i + K_i).  With 3 nw >= kmax a warp has at most one active
    // sweep; otherwise (n > 96 BW) older sweeps are finished in extra passes.
    int cur = -1, next = warp;
    for (int64_t t = 0; t < T; ++t) {
      if (3 * int64_t(next) == t) {
        cur = next;
        next += nw;
      }
      if (!GMEM || 3 * nw >= kmax) {
        const int k = int(t - 3 * int64_t(cur));
        const bool act = cur >= 0 && k < hb_tasks(n, cur);
        if (act)  // (warp-uniform: idle warps go straight to the step barrier)
          hb_task(Wf, n, cur, k, true, lane, vsh[warp], lg ? lg + (int64_t(cur) * kmax + k) * HLOG : nullptr);
      } else {
        for (int i = cur; i >= 0 && t - 3 * int64_t(i) < kmax; i -= nw) {
          const int k = int(t - 3 * int64_t(i));
          const bool act = k < hb_tasks(n, i);
          hb_task(Wf, n, act ? i : 0, act ? k : 0, act, lane, vsh[warp],
                  lg ? lg + (int64_t(i) * kmax + k) * HLOG : nullptr);
        }
      }
      __syncthreads();
    }
    double* de = P.debuf + si * 2 * NP;
    for (int64_t q = threadIdx.x; q < NP; q += blockDim.x) {
      de[q] = q < n ? HEL(W, int(q), int(q)) : 0.0;
      de[NP + q] = q + 1 < n ? HEL(W, int(q), int(q) + 1) : 0.0;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && P.stats) atomicAdd(&g_stats[ST_CYC_BULGE], (unsigned long long)(t1 - t0));
  }
}

// The same chase for windows beyond one SM's shared memory (616 < n <= 1160,
// e.g. c3's 1024 x 1024 slices: 385 KB): a cluster of two CTAs holds the
// window in distributed shared memory (rows < H on rank 0, the rest on rank
// 1).  Both CTAs walk the same step loop; the task of sweep i at step t is
// run by the CTA that owns its pivot column c0 (warp = sweep mod nw, as in
// the one-CTA kernel), reaching across the boundary through DSMEM where its
// rows straddle it, and one cluster barrier per step orders the steps.
// Every task does the arithmetic of hb_task in the same order, so d, e and
// the reflector log are bitwise those of the other variants.  Clusters take
// slices lo + c, lo + c + (clusters), ... (equal work per slice).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(768, 1) svd_bulge_cluster_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double vsh[32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = int(P.n);
  const int64_t NP = P.NP;
  unsigned rank, nclusters, cid;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(nclusters));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  const int R = n + BW, H = (R + 1) / 2;
  double* mine = reinterpret_cast<double*>(smem_raw);
  // generic addresses of both halves (mapa: this CTA's shared address in the
  // peer's window)
  WinSplit Ws;
  {
    unsigned long long g0, g1;
    const unsigned long long self = reinterpret_cast<unsigned long long>(mine);
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(g0) : "l"(self), "r"(0u));
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(g1) : "l"(self), "r"(1u));
    Ws.W0 = reinterpret_cast<double*>(g0);
    Ws.W1 = reinterpret_cast<double*>(g1);
    Ws.H = H;
  }
  auto cluster_sync = [] {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  };
  const int r_lo = rank ? H : 0, r_hi = rank ? R : H;  // window rows held here
  const int64_t kmax = hb_kmax(n), T = hb_steps(n);
  for (int64_t it = P.lo + cid; it < P.hi; it += nclusters) {
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;  // (cluster-uniform)
    long long t0 = clock64();
    const double* band = P.bandbuf + si * (BW + 1) * NP;
    for (int e = threadIdx.x; e < (r_hi - r_lo) * HB; e += blockDim.x) {
      const int r = r_lo + e / HB, d = e % HB - HOFF;
      mine[e] = (d >= 0 && d <= BW && r + d < n) ? band[d * NP + r] : 0.0;
    }
    cluster_sync();
    double* lg = P.hhlog ? P.hhlog + si * P.hhcap : nullptr;
    int cur = -1, next = warp;
    for (int64_t t = 0; t < T; ++t) {
      if (3 * int64_t(next) == t) {
        cur = next;
        next += nw;
      }
      const int k = int(t - 3 * int64_t(cur));
      const bool act = cur >= 0 && k < hb_tasks(n, cur);
      if (act) {
        const int c0 = cur + k * BW + 1;
        if ((c0 < H ? 0u : 1u) == rank)
          hb_task(Ws, n, cur, k, true, lane, vsh[warp], lg ? lg + (int64_t(cur) * kmax + k) * HLOG : nullptr);
      }
      cluster_sync();
    }
    double* de = P.debuf + si * 2 * NP;
    for (int64_t q = r_lo + threadIdx.x; q < r_hi && q < NP; q += blockDim.x) {
      de[q] = q < n ? *Ws.at(int(q), int(q)) : 0.0;
      de[NP + q] = q + 1 < n ? *Ws.at(int(q), int(q) + 1) : 0.0;
    }
    for (int64_t q = R + threadIdx.x; rank == 1 && q < NP; q += blockDim.x) de[q] = de[NP + q] = 0.0;
    cluster_sync();  // the next slice's fill must not overtake these reads
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0 && P.stats)
      atomicAdd(&g_stats[ST_CYC_BULGE], (unsigned long long)(t1 - t0));
  }
}

// ----------------------------------------------------------------------
// Singular values of the upper bidiagonal (d, e) by bisection on the
// Golub-Kahan tridiagonal T_GK (zero diagonal, off-diagonals d0,e0,d1,...),
// whose eigenvalues are +-sigma: #sigma < x = (#negative Sturm pivots of
// T_GK - x I) - n.  One thread per (slice, sigma_j), sigma_j the j-th
// largest; interval shrunk to 2u * max(sigma_j, 1e-3 * bound).
// ----------------------------------------------------------------------
// Pivots use rcp_nr (relative error ~1e-15): a Sturm pivot computed this
// way is the exact pivot of T_GK with off-diagonals perturbed by a few ulps,
// which is all the count needs.

__device__ __forceinline__ int count_below(const double* d, const double* e, int n, double x,
                                           double pivmin) {
  int neg = 0;
  double q = -x;
  neg += (q < 0.0);
  for (int k = 0; k < n; ++k) {
    const double dk = d[k];
    if (fabs(q) < pivmin) q = -pivmin;
    q = fma(-dk * dk, rcp_nr(q), -x);
    neg += (q < 0.0);
    if (k + 1 < n) {
      const double ek = e[k];
      if (fabs(q) < pivmin) q = -pivmin;
      q = fma(-ek * ek, rcp_nr(q), -x);
      neg += (q < 0.0);
    }
  }
  return neg - n;
}

// Sturm count of T_GK - x I plus the log-derivatives of f(x) = det(T_GK - x I):
// with pivots q_i (q_0 = -x, q_i = -x - b_{i-1}^2 / q_{i-1}),
//   G = f'/f = sum q_i'/q_i,  H = -(f'/f)' = sum (q_i'/q_i)^2 - q_i''/q_i.
__device__ __forceinline__ int count_lag(const double* d, const double* e, int n, double x,
                                         double pivmin, double& G, double& H) {
  int neg = 0;
  double q = -x, dq = -1.0, d2 = 0.0;
  G = 0.0;
  H = 0.0;
  neg += (q < 0.0);
  for (int k = 0; k < 2 * n - 1; ++k) {
    const double b = (k & 1) ? e[k >> 1] : d[k >> 1];
    if (fabs(q) < pivmin) q = -pivmin;
    const double r = rcp_nr(q);
    const double g = dq * r;
    G += g;
    H = fma(g, g, fma(-d2, r, H));
    const double t = b * b * r;
    const double tr = t * r;
    d2 = tr * fma(-2.0 * dq, g, d2);  // b^2 r^2 (q'' - 2 q'^2 r)
    dq = fma(tr, dq, -1.0);
    q = -x - t;
    neg += (q < 0.0);
  }
  if (fabs(q) < pivmin) q = -pivmin;
  const double r = rcp_nr(q);
  const double g = dq * r;
  G += g;
  H = fma(g, g, fma(-d2, r, H));
  return neg - n;
}

// sigma_j: bisection on Sturm counts until [lo, hi) isolates it (count(lo) =
// target, count(hi) = target + 1), then Laguerre's method on det(T_GK - x I)
// (cubically convergent; T_GK is real-rooted, and the branch is chosen by
// the count so the iterate moves toward the bracketed root), safeguarded by
// the bracket, which every evaluation tightens.  Clusters that never
// isolate, and Laguerre runs that do not converge, finish by bisection to
// 2u * max(sigma, 1e-3 * bound).  The phases are warp-uniform (a lane waits
// for the warp before the next phase) so bisection and Laguerre steps never
// diverge inside a warp.
__global__ void svd_bisect_kernel(SvdParams P) {
  const int64_t n = P.n, NP = P.NP;
  // one warp per (slice, block of 32 consecutive j): the multisection below
  // shares probes inside a warp, so the composition of a warp must depend
  // on the slice alone (sigma bitwise identical whichever job or chunk
  // computes it)
  const int64_t jblocks = (n + 31) >> 5;
  const int64_t wtotal = (P.hi - P.lo) * jblocks;
  const double N2 = 2.0 * double(n);
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; w < wtotal; w += warps) {
    const int64_t jv = (w % jblocks) * 32 + lane;
    const bool valid = jv < n;
    const int64_t it = P.lo + w / jblocks, j = valid ? jv : 0;
    const int64_t si = state_index(P, it);
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int flag = valid ? P.flags[si] : 1;
    const double* d = P.debuf + si * 2 * NP;
    const double* e = d + NP;
    double bound = 0.0, amax = 0.0;
    if (flag == 0) {
      for (int64_t k = 0; k < n; ++k) {
        const double dk = fabs(d[k]), ek = (k + 1 < n) ? fabs(e[k]) : 0.0;
        const double ekm = k > 0 ? fabs(e[k - 1]) : 0.0;
        bound = fmax(bound, fmax(dk + ek, dk + ekm));
        amax = fmax(amax, fmax(dk, ek));
      }
    }
    const double pivmin = fmax(DBL_MIN, amax * amax * 1e-300);
    const int64_t target = n - 1 - j;  // want count_below(x) <= target
    double lo = 0.0, hi = bound * (1.0 + 4.0 * DBL_EPSILON) + DBL_MIN;
    int64_t clo = 0, chi = n;
    double sigma = 0.0, x = 0.0;
    int state = (flag == 0 && bound > 0.0) ? 0 : 3;  // 0 isolate, 1 Laguerre, 2 bisect, 3 done
    auto converged = [&]() {
      const double mid = 0.5 * (lo + hi);
      return !(mid > lo && mid < hi) || hi - lo <= 2.0 * DBL_EPSILON * fmax(lo, 1e-3 * bound);
    };
    // ---- phase A: cooperative multisection until isolated.  A Sturm count
    // at x tells every sigma of the slice which side of x it lies on, so
    // the lanes of a warp (consecutive j of one slice) share their probes:
    // lanes whose brackets coincide split that bracket into k + 1 parts
    // with k distinct probes, and every lane tightens its bracket with all
    // probes of its slice (32 probes per Sturm sweep instead of 1).
    int nA = 0, nB = 0, nC = 0;  // sweeps of this warp per phase (diagnostic counters)
    while (__any_sync(0xffffffffu, state == 0)) {
      ++nA;
      bool probe = false;
      if (state == 0) {
        if (converged()) {
          sigma = 0.5 * (lo + hi);
          state = 3;
        } else if (clo == target && chi == target + 1) {
          x = 0.5 * (lo + hi);
          state = 1;
        } else {
          probe = true;
        }
      }
      // runs of lanes with the same (slice, bracket) among the probing lanes
      const double plo = __shfl_up_sync(0xffffffffu, lo, 1), phi = __shfl_up_sync(0xffffffffu, hi, 1);
      const int64_t pit = __shfl_up_sync(0xffffffffu, it, 1);
      const bool pprobe = __shfl_up_sync(0xffffffffu, probe, 1);
      const bool cont = lane > 0 && probe && pprobe && pit == it && plo == lo && phi == hi;
      const unsigned starts = __ballot_sync(0xffffffffu, !cont);  // run heads (and non-probing lanes)
      const int head = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
      const unsigned after = starts & ~(0xffffffffu >> (31 - lane));  // heads beyond this lane
      const int next = after ? __ffs(after) - 1 : 32;
      const int rank = lane - head, k = next - head;
      double xp = 0.0;
      int64_t cp = 0;
      if (probe) {
        xp = lo + (hi - lo) * (double(rank + 1) / double(k + 1));
        if (!(xp > lo && xp < hi)) xp = 0.5 * (lo + hi);
        cp = count_below(d, e, int(n), xp, pivmin);
      }
#pragma unroll 4
      for (int m = 0; m < 32; ++m) {
        const double xm = __shfl_sync(0xffffffffu, xp, m);
        const int64_t cm = __shfl_sync(0xffffffffu, cp, m);
        const int64_t im = __shfl_sync(0xffffffffu, it, m);
        const bool pm = __shfl_sync(0xffffffffu, probe, m);
        if (state == 0 && pm && im == it) {
          if (cm <= target) {
            if (xm > lo) {
              lo = xm;
              clo = cm;
            }
          } else if (xm < hi) {
            hi = xm;
            chi = cm;
          }
        }
      }
    }
    // ---- phase B: Laguerre inside the bracket
    for (int lt = 0; lt < 16 && __any_sync(0xffffffffu, state == 1); ++lt) {
      ++nB;
      if (state == 1) {
        double G, H;
        const int64_t c = count_lag(d, e, int(n), x, pivmin, G, H);
        const bool below = c <= target;  // x below sigma_j: step up
        if (below) {
          lo = x;
          clo = c;
        } else {
          hi = x;
          chi = c;
        }
        const double disc = sqrt(fmax((N2 - 1.0) * fma(N2, H, -G * G), 0.0));
        const double den = below ? G - disc : G + disc;
        double xn = den != 0.0 ? x - N2 / den : 0.5 * (lo + hi);
        const double tol = 2.0 * DBL_EPSILON * fmax(fabs(xn), 1e-3 * bound);
        if (fabs(xn - x) <= tol || hi - lo <= tol) {
          sigma = (xn >= lo && xn <= hi) ? xn : x;
          state = 3;
        } else {
          if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
          x = xn;
        }
      }
    }
    if (state == 1) state = 2;
    // ---- phase C: bisection to the end for the rest
    while (__any_sync(0xffffffffu, state == 2)) {
      ++nC;
      if (state == 2) {
        if (converged()) {
          sigma = 0.5 * (lo + hi);
          state = 3;
        } else {
          const double mid = 0.5 * (lo + hi);
          if (count_below(d, e, int(n), mid, pivmin) <= target) lo = mid;
          else hi = mid;
        }
      }
    }
    if (valid && flag != 2) P.s[j + slice * n] = sigma;
    if (P.stats && lane == 0) {
      atomicAdd(&g_stats[ST_SWEEPS], (unsigned long long)nA);
      atomicAdd(&g_stats[ST_PAIRS], (unsigned long long)nB);
      atomicAdd(&g_stats[ST_ROTATED], (unsigned long long)nC);
      atomicMax(&g_stats[ST_CYC_FINAL], (unsigned long long)(nA * 1000000 + nB * 1000 + nC));
    }
  }
}

// ======================================================================
//                     Jacobi + finalize kernel
// ======================================================================

// Qside (L x k, ld LP, columns 0..k-1) = X * V[:, idx[0..k)] from the
// untouched slice (X = A or A^T), on DMMA.  Uses sm.xs / sm.w as staging.
__device__ void gemm_xv(const SvdParams& P, JacobiSmem& sm, const double* A, const double* V,
                        const int* idx, int64_t k, double* Q) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t L = P.L, n = P.n, LP = P.LP, NP = P.NP, RP = P.RP;
  for (int64_t kb = 0; kb < k; kb += GW) {
    for (int64_t r0 = 0; r0 < LP; r0 += RCH) {
      double acc[4][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
      for (int64_t kk = 0; kk < NP; kk += GW) {
        double* xs = sm.xs[0];
        double* wt = sm.w[0];
        // X tile: rows r0..r0+63, cols kk..kk+31 -> xs[col*XS + row]
        // (all loads of a tile are issued before any store: one latency per tile)
        constexpr int XN = GW * RCH / TPB, WN = GW * GW / TPB;
        double xv[XN], wv[WN];
#pragma unroll
        for (int u = 0; u < XN; ++u) {
          const int e = tid + u * TPB;
          int col, row;
          if (P.transposed) { col = e & 31; row = e >> 5; }   // consecutive col -> contiguous A
          else { row = e & 63; col = e >> 6; }                // consecutive row -> contiguous A
          const int64_t r = r0 + row, c = kk + col;
          xv[u] = (r < L && c < n) ? (P.transposed ? A[c + r * P.m] : A[r + c * P.m]) : 0.0;
        }
        // W tile: W[kk+i][idx[kb+j]] -> wt[j*WS + i]
#pragma unroll
        for (int u = 0; u < WN; ++u) {
          const int e = tid + u * TPB;
          const int i = e & 31, j = e >> 5;
          const int64_t jj = kb + j;
          wv[u] = (jj < k) ? V[(kk + i) + int64_t(idx[jj]) * RP] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < XN; ++u) {
          const int e = tid + u * TPB;
          int col, row;
          if (P.transposed) { col = e & 31; row = e >> 5; }
          else { row = e & 63; col = e >> 6; }
          xs[col * XS + row] = xv[u];
        }
#pragma unroll
        for (int u = 0; u < WN; ++u) {
          const int e = tid + u * TPB;
          wt[(e >> 5) * WS + (e & 31)] = wv[u];
        }
        __syncthreads();
        const double* xa = xs + tq * XS + warp * 8 + gq;
        const double* wb = wt + gq * WS + tq;
#pragma unroll
        for (int k4 = 0; k4 < GW / 4; ++k4) {
          const double a = xa[k4 * 4 * XS];
#pragma unroll
          for (int c = 0; c < 4; ++c) dmma884(acc[c][0], acc[c][1], a, wb[c * 8 * WS + k4 * 4]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = kb + c * 8 + 2 * tq + e;
          const int64_t row = r0 + warp * 8 + gq;
          if (col < k && row < L) Q[row + col * LP] = acc[c][e];
        }
    }
  }
  __syncthreads();
}


// slicesvd.py:51-54: an all-zero slice has zero values and identity bases.
__device__ void emit_zero_slice(const SvdParams& P, int64_t slice) {
  const int tid = threadIdx.x;
  const int64_t r = P.n;
  if (P.s)
    for (int64_t j = tid; j < r; j += blockDim.x) P.s[j + slice * r] = 0.0;
  if (P.job == STARM_SVD_FULL) {
    double* U = P.u + slice * P.m * r;
    double* Vo = P.v + slice * P.p * r;
    for (int64_t e = tid; e < P.m * r; e += blockDim.x) U[e] = ((e % P.m) == (e / P.m)) ? 1.0 : 0.0;
    for (int64_t e = tid; e < P.p * r; e += blockDim.x) Vo[e] = ((e % P.p) == (e / P.p)) ? 1.0 : 0.0;
  } else if (P.job == STARM_SVD_TRUNCATED) {
    const int64_t k = P.ranks[slice];
    double* U = P.u_data + P.u_off[slice];
    double* G = P.g_data + P.g_off[slice];
    for (int64_t e = tid; e < P.m * k; e += blockDim.x) U[e] = ((e % P.m) == (e / P.m)) ? 1.0 : 0.0;
    for (int64_t e = tid; e < k * P.p; e += blockDim.x) G[e] = 0.0;
  }
  __syncthreads();
}

// Write the requested factors of one slice given the right singular vectors
// of the working matrix X (columns vidx[j] of V, ld RP, j in descending sigma
// order) and sigma in P.s.  The other side is X V normalised: recomputed
// from the input slice (qgemm) or taken from the Jacobi target T (= X V).
// Columns whose sigma is below 1e-4 sigma_max are re-orthonormalised (CGS2).
__device__ void emit_vectors(const SvdParams& P, JacobiSmem& sm, FinalView& fs, int64_t slice,
                             const double* A, const double* V, const int* vidx, double* Xslot,
                             bool qgemm, double* T, int64_t ldt) {
  const int tid = threadIdx.x;
  const int64_t L = P.L, n = P.n, LP = P.LP, RP = P.RP, r = n;
  const double* sg = P.s + slice * r;
  const double smax = sg[0];
  const int64_t kout = (P.job == STARM_SVD_FULL) ? r : P.ranks[slice];
  double* Qb;
  int64_t ldq;
  const int* qc;
  if (qgemm) {
    gemm_xv(P, sm, A, V, vidx, kout, Xslot);
    Qb = Xslot;
    ldq = LP;
    qc = nullptr;
  } else {
    Qb = T;
    ldq = ldt;
    qc = vidx;
  }
  // normalise by the actual column norms (deterministic warp-per-column sums)
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int64_t j = warp; j < kout; j += TPB / 32) {
      double* col = Qb + int64_t(qc ? qc[j] : j) * ldq;
      double acc = 0.0;
      for (int64_t rr = lane; rr < L; rr += 32) acc += col[rr] * col[rr];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const double nrm = sqrt(acc);
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int64_t rr = lane; rr < L; rr += 32) col[rr] *= inv;
    }
  }
  __syncthreads();
  for (int64_t j = 0; j < kout; ++j)
    if (!(sg[j] > 1e-4 * smax)) cgs2_fix(fs, Qb, ldq, L, qc, int(j));
  __syncthreads();
  if (P.job == STARM_SVD_FULL) {
    double* Uo = P.u + slice * P.m * r;
    double* Vo = P.v + slice * P.p * r;
    double* Qd = P.transposed ? Vo : Uo;  // ld L
    double* Wd = P.transposed ? Uo : Vo;  // ld n
    for (int64_t j = 0; j < kout; ++j) {
      const double* qcol = Qb + int64_t(qc ? qc[j] : j) * ldq;
      for (int64_t rr = tid; rr < L; rr += TPB) Qd[rr + j * L] = qcol[rr];
      const double* vcol = V + int64_t(vidx[j]) * RP;
      for (int64_t rr = tid; rr < n; rr += TPB) Wd[rr + j * n] = vcol[rr];
    }
  } else {
    double* Uk = P.u_data + P.u_off[slice];
    double* G = P.g_data + P.g_off[slice];
    if (!P.transposed) {
      for (int64_t j = 0; j < kout; ++j) {
        const double* qcol = Qb + int64_t(qc ? qc[j] : j) * ldq;
        for (int64_t rr = tid; rr < L; rr += TPB) Uk[rr + j * L] = qcol[rr];
      }
      for (int64_t e = tid; e < kout * n; e += TPB) {
        const int64_t j = e % kout, col = e / kout;
        G[e] = sg[j] * V[col + int64_t(vidx[j]) * RP];
      }
    } else {
      for (int64_t j = 0; j < kout; ++j) {
        const double* vcol = V + int64_t(vidx[j]) * RP;
        for (int64_t rr = tid; rr < n; rr += TPB) Uk[rr + j * n] = vcol[rr];
      }
      for (int64_t e = tid; e < kout * L; e += TPB) {
        const int64_t j = e % kout, col = e / kout;
        G[e] = sg[j] * Qb[col + int64_t(qc ? qc[j] : j) * ldq];
      }
    }
  }
  __syncthreads();
}

// ======================================================================
//        Vectors on the bidiagonal path (no Jacobi): inverse iteration
//        on T_GK + back-transformation through the logged right-side
//        transformations (bulge column rotations, band LQ reflectors).
// ======================================================================

__device__ __forceinline__ int64_t kout_of(const SvdParams& P, int64_t slice) {
  return (P.job == STARM_SVD_FULL) ? P.n : P.ranks[slice];
}

// Right singular vectors of the bidiagonal (d, e) for sigma_j, j < k, by
// inverse iteration on T_GK - sigma_j I (tridiagonal LU with partial
// pivoting, LAPACK dgttrf/dgttrs), 3 solves from a fixed start vector.  The
// even entries of the T_GK eigenvector are v (B v = sigma u).
// Close singular values (gap <= 1e-6 ||T||) form clusters that one thread
// processes in order, as LAPACK dstein does: equal shifts are separated by
// 10 eps ||T|| and every iterate is orthogonalised (MGS) against the cluster's
// earlier eigenvectors z = [v; B v / sigma] (rebuilt from the stored v), so a
// degenerate pair yields two orthogonal vectors of its eigenspace instead of
// the same one twice.  Clusters are cut into chunks of II_CMAX vectors.
// One thread per (slice, cluster head); per-thread scratch of 6 x 2n doubles.
constexpr int II_CMAX = 32;

// Per-thread scratch vectors are interleaved within a warp (element i of a
// lane's vector at i * 32 + lane), so a warp's accesses to the same index
// are one coalesced line and each warp walks its own region sequentially;
// the recurrences carry their state in registers and prefetch the next
// step's operands.
struct Strided {
  double* p;
  int64_t s;
  __device__ __forceinline__ double& operator[](int64_t i) const { return p[i * s]; }
};

// LU with partial pivoting of T_GK - lam I (zero diagonal, off-diagonals
// b_k = d0, e0, d1, ...; LAPACK dgttrf): outputs the reciprocal pivots rdd,
// super-diagonals du, du2, multipliers dl and the interchange flags z.  The
// sequential recurrence runs from registers in blocks of IB steps whose
// operands are loaded (and results stored) together.
constexpr int IB = 8;

__device__ void ii_factor(const double* bd, const double* be, int64_t N2, double lam, double pert,
                          Strided rdd, Strided du, Strided du2, Strided dl, Strided z) {
  auto b_at = [&](int64_t i) { return i < N2 - 1 ? ((i & 1) ? be[i >> 1] : bd[i >> 1]) : 0.0; };
  double cdd = -lam;                    // dd[i] as modified so far
  double cdu = b_at(0);                 // du[i] as modified so far
  // original b_i .. b_{i+IB} of the current block; the next block's are
  // loaded one block ahead (software pipelining of the read-only inputs)
  double nb[IB + 1];
#pragma unroll
  for (int u = 0; u <= IB; ++u) nb[u] = b_at(u);
  for (int64_t i0 = 0; i0 + 1 < N2; i0 += IB) {
    double bb[IB + 1];
#pragma unroll
    for (int u = 0; u <= IB; ++u) bb[u] = nb[u];
#pragma unroll
    for (int u = 0; u <= IB; ++u) nb[u] = b_at(i0 + IB + u);
    double o_rdd[IB], o_du[IB], o_du2[IB], o_dl[IB], o_z[IB];
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      const int64_t i = i0 + u;
      o_rdd[u] = o_du[u] = o_du2[u] = o_dl[u] = o_z[u] = 0.0;
      if (i + 1 < N2) {
        const double bi = bb[u], bnext = bb[u + 1];  // b_{N2-1} = 0 by b_at
        double ddi, ndd, ndu;
        if (fabs(cdd) >= fabs(bi)) {
          ddi = cdd == 0.0 ? pert : cdd;
          const double fact = bi / ddi;
          o_dl[u] = fact;
          o_du[u] = cdu;
          ndd = -lam - fact * cdu;
          ndu = bnext;
        } else {
          const double fact = cdd / bi;
          ddi = bi;
          o_dl[u] = fact;
          o_du[u] = -lam;  // the old dd[i + 1]
          ndd = cdu + fact * lam;
          o_du2[u] = bnext;
          ndu = -fact * bnext;
          o_z[u] = 1.0;
        }
        o_rdd[u] = 1.0 / ddi;
        cdd = ndd;
        cdu = ndu;
      }
    }
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      const int64_t i = i0 + u;
      if (i + 1 < N2) {
        rdd[i] = o_rdd[u];
        du[i] = o_du[u];
        du2[i] = o_du2[u];
        dl[i] = o_dl[u];
        z[i] = o_z[u];
      }
    }
  }
  rdd[N2 - 1] = 1.0 / (cdd == 0.0 ? pert : cdd);
}

__device__ void ii_solve(int64_t N2, Strided rdd, Strided du, Strided du2, Strided dl, Strided z,
                         Strided x) {
  // forward: apply L and the row interchanges; x[i] carried in a register
  double xi = x[0];
  // block operands loaded one block ahead (the next block never reads an x
  // this block stores: it reads x[i0 + IB + 1 ..], this one stores x[i0 .. i0 + IB - 1])
  double ndl[IB], nz[IB], nx[IB];
  auto fwd_load = [&](int64_t b0) {
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      const int64_t i = b0 + u;
      const bool in = i + 1 < N2;
      ndl[u] = in ? dl[i] : 0.0;
      nz[u] = in ? z[i] : 0.0;
      nx[u] = in ? x[i + 1] : 0.0;
    }
  };
  fwd_load(0);
  for (int64_t i0 = 0; i0 + 1 < N2; i0 += IB) {
    double dlv[IB], zv[IB], xv[IB];
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      dlv[u] = ndl[u];
      zv[u] = nz[u];
      xv[u] = nx[u];
    }
    fwd_load(i0 + IB);
    double xo[IB];
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      if (i0 + u + 1 >= N2) break;  // the chain must stop at the last row
      if (zv[u] != 0.0) {
        xo[u] = xv[u];
        xi = xi - dlv[u] * xv[u];
      } else {
        xo[u] = xi;
        xi = xv[u] - dlv[u] * xi;
      }
    }
#pragma unroll
    for (int u = 0; u < IB; ++u)
      if (i0 + u + 1 < N2) x[i0 + u] = xo[u];
  }
  // backward: U has diagonal 1/rdd, super du, second super du2
  double x1 = xi * rdd[N2 - 1];  // x[N2 - 1]
  x[N2 - 1] = x1;
  if (N2 < 2) return;
  double x0 = (x[N2 - 2] - du[N2 - 2] * x1) * rdd[N2 - 2];
  x[N2 - 2] = x0;
  double nxv[IB], nduv[IB], ndu2v[IB], nrv[IB];  // next block, loaded one block ahead
  auto bwd_load = [&](int64_t b1) {
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      const int64_t i = b1 - u;
      const bool in = i >= 0;
      nxv[u] = in ? x[i] : 0.0;
      nduv[u] = in ? du[i] : 0.0;
      ndu2v[u] = in ? du2[i] : 0.0;
      nrv[u] = in ? rdd[i] : 0.0;
    }
  };
  bwd_load(N2 - 3);
  for (int64_t i1 = N2 - 3; i1 >= 0; i1 -= IB) {  // block i1, i1 - 1, ..., i1 - IB + 1
    double xv[IB], duv[IB], du2v[IB], rv[IB];
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      xv[u] = nxv[u];
      duv[u] = nduv[u];
      du2v[u] = ndu2v[u];
      rv[u] = nrv[u];
    }
    bwd_load(i1 - IB);
    double xo[IB];
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      const double v = (xv[u] - duv[u] * x0 - du2v[u] * x1) * rv[u];
      xo[u] = v;
      x1 = x0;
      x0 = v;
    }
#pragma unroll
    for (int u = 0; u < IB; ++u)
      if (i1 - u >= 0) x[i1 - u] = xo[u];
  }
}

// x -= (x.z / z.z) z for the T_GK eigenvector z of a previous cluster member
// (v = stored right vector, sig its shift; u = B v / sig, 0 when sig == 0).
__device__ void ii_orth(const double* bd, const double* be, int64_t n, const double* v, double sig,
                        Strided x) {
  const double rs = sig > 0.0 ? 1.0 / sig : 0.0;
  double dot = 0.0, nz = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double zv = v[i];
    const double zu = (bd[i] * v[i] + (i + 1 < n ? be[i] * v[i + 1] : 0.0)) * rs;
    dot += x[2 * i] * zv + x[2 * i + 1] * zu;
    nz += zv * zv + zu * zu;
  }
  if (nz <= 0.0) return;
  const double c = dot / nz;
  for (int64_t i = 0; i < n; ++i) {
    const double zv = v[i];
    const double zu = (bd[i] * v[i] + (i + 1 < n ? be[i] * v[i + 1] : 0.0)) * rs;
    x[2 * i] -= c * zv;
    x[2 * i + 1] -= c * zu;
  }
}

// The items of one thread: g = gtid, gtid + nthreads, ... over (vector j,
// list position it) pairs, vector index major (the few real items, j < k, of
// every slice come first and spread over all threads / warps); scratch
// vectors through the Strided views (global, warp-interleaved, or one
// compact region per thread in shared memory).
// Vector j of list position `it` (a no-op unless j heads a cluster chunk).
__device__ __forceinline__ void bdvec_one(const SvdParams& P, int64_t j, int64_t it, Strided rdd,
                                          Strided du, Strided du2, Strided dl, Strided z, Strided x) {
  const int64_t n = P.n, NP = P.NP, RP = P.RP, N2 = 2 * P.n;
  {
    const int64_t si = state_index(P, it);
    if (P.flags[si]) return;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int64_t kout = kout_of(P, slice);
    if (j >= kout) return;
    const double* bd = P.debuf + si * 2 * NP;
    const double* be = bd + NP;
    const double* sv = P.s + slice * n;
    double tnorm = 0.0;
    for (int64_t k = 0; k < n; ++k) tnorm = fmax(tnorm, fabs(bd[k]) + (k + 1 < n ? fabs(be[k]) : 0.0));
    const double pert = fmax(tnorm * DBL_EPSILON, DBL_MIN);
    const double ctol = 1e-6 * tnorm;
    // cluster run containing j: [r0, ...); j heads a chunk iff (j - r0) % II_CMAX == 0
    int64_t r0 = j;
    while (r0 > 0 && sv[r0 - 1] - sv[r0] <= ctol) --r0;
    if ((j - r0) % II_CMAX) return;
    int64_t jend = j + 1;
    while (jend < kout && jend - j < II_CMAX && sv[jend - 1] - sv[jend] <= ctol) ++jend;
    double lprev = 0.0;
    for (int64_t jj = j; jj < jend; ++jj) {
      double lam = sv[jj];
      if (jj > j && lam > lprev - 10.0 * pert) lam = lprev - 10.0 * pert;  // separate equal shifts
      lprev = lam;
      ii_factor(bd, be, N2, lam, pert, rdd, du, du2, dl, z);
      for (int64_t i = 0; i < N2; ++i)
        x[i] = 1.0 + 0.25 * double(((i + 1) * 7919 + (jj + 1) * 104729) % 97) / 97.0;
      for (int iter = 0; iter < 3; ++iter) {
        for (int64_t q = j; q < jj; ++q) ii_orth(bd, be, n, P.vsel + si * RP * NP + q * RP, sv[q], x);
        ii_solve(N2, rdd, du, du2, dl, z, x);
        double nrm = 0.0;
        for (int64_t i = 0; i < N2; ++i) nrm = fmax(nrm, fabs(x[i]));
        const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
        for (int64_t i = 0; i < N2; ++i) x[i] *= inv;
      }
      for (int64_t q = j; q < jj; ++q) ii_orth(bd, be, n, P.vsel + si * RP * NP + q * RP, sv[q], x);
      // v = even entries, unit 2-norm
      double nv = 0.0;
      for (int64_t i = 0; i < n; ++i) nv += x[2 * i] * x[2 * i];
      const double inv = nv > 0.0 ? 1.0 / sqrt(nv) : 0.0;
      double* vout = P.vsel + si * RP * NP + jj * RP;
      for (int64_t i = 0; i < RP; ++i) vout[i] = (i < n) ? x[2 * i] * inv : 0.0;
    }
  }
}

__device__ __forceinline__ void bdvec_items(const SvdParams& P, int64_t total_work, int64_t gtid,
                                            int64_t nthreads, Strided rdd, Strided du, Strided du2,
                                            Strided dl, Strided z, Strided x) {
  // vector index major: the few real items (j < k) of every slice come first
  // and spread over all threads / warps
  for (int64_t g = gtid; g < total_work; g += nthreads)
    bdvec_one(P, g / P.count, g % P.count, rdd, du, du2, dl, z, x);
}

// Number of vectors the job computes (sum of k over the listed slices) into
// counter[5]: the two launches below pick the scratch placement from it.
__global__ void __launch_bounds__(256) svd_bdvec_count_kernel(SvdParams P) {
  // also the exclusive prefix sums of k over the list (count + 1 entries at
  // the start of the global scratch, which only the other launch uses) so
  // the shared-memory launch can enumerate exactly the real vectors
  __shared__ long long sc[256];
  __shared__ long long base;
  long long* prefix = reinterpret_cast<long long*>(P.iiscr);
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < P.count; c0 += 256) {
    const int64_t it = c0 + threadIdx.x;
    long long k = 0;
    if (it < P.count && !P.flags[state_index(P, it)]) k = kout_of(P, P.ids ? P.ids[it] : it);
    sc[threadIdx.x] = k;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {  // inclusive scan
      const long long v = threadIdx.x >= o ? sc[threadIdx.x - o] : 0;
      __syncthreads();
      sc[threadIdx.x] += v;
      __syncthreads();
    }
    if (it < P.count) prefix[it] = base + sc[threadIdx.x] - k;
    __syncthreads();
    if (threadIdx.x == 255) base += sc[255];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    prefix[P.count] = base;
    P.counter[5] = (unsigned long long)base;
  }
}

// Few vectors (at most II_SMEM_OVERSUB per shared-memory slot, e.g. the
// pruned c2 step's 336 or c1's 640): every thread keeps its six scratch
// vectors in a compact region of shared memory, so the recurrences run at
// shared-memory latency instead of walking 2 MB of interleaved scratch per
// warp through L2.  Same arithmetic, same results.
constexpr int II_SMEM_OVERSUB = 2;

__global__ void svd_bdvec_kernel(SvdParams P, int64_t total_work, int64_t smem_slots) {
  if (int64_t(P.counter[5]) <= II_SMEM_OVERSUB * smem_slots) return;  // the shared-memory launch ran
  const int64_t NP = P.NP;
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  // scratch interleaved within each warp (element i of lane l at i * 32 + l):
  // coalesced per index, sequential per warp (TLB-friendly)
  const int64_t vl = 2 * NP;
  double* wscr = P.iiscr + (gtid >> 5) * (6 * vl * 32) + (gtid & 31);
  bdvec_items(P, total_work, gtid, nthreads, Strided{wscr, 32}, Strided{wscr + 1 * vl * 32, 32},
              Strided{wscr + 2 * vl * 32, 32}, Strided{wscr + 3 * vl * 32, 32},
              Strided{wscr + 4 * vl * 32, 32}, Strided{wscr + 5 * vl * 32, 32});
}

__global__ void svd_bdvec_smem_kernel(SvdParams P, int64_t total_work, int64_t smem_slots) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (int64_t(P.counter[5]) > II_SMEM_OVERSUB * smem_slots) return;
  // one vector per WARP (lane 0 works): the pivoting branches of different
  // vectors would serialise inside a warp, and with this few vectors the
  // chain's instruction latency is all that matters (6 threads of one warp:
  // 0.84 ms on c2; one lane per warp: see DESIGN)
  if (threadIdx.x & 31) return;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t vl = 2 * P.NP;
  const int64_t nthreads = int64_t(gridDim.x) * nwarps;
  // slot-major over CTAs so consecutive items land on different SMs
  const int64_t gtid = int64_t(warp) * gridDim.x + blockIdx.x;
  double* w = reinterpret_cast<double*>(smem_raw) + int64_t(warp) * (6 * vl + 2);
  const long long* prefix = reinterpret_cast<const long long*>(P.iiscr);
  const int64_t total = int64_t(P.counter[5]);
  for (int64_t q = gtid; q < total; q += nthreads) {
    int64_t lo = 0, hi = P.count;  // prefix[lo] <= q < prefix[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (prefix[mid] <= q) lo = mid;
      else hi = mid;
    }
    bdvec_one(P, q - prefix[lo], lo, Strided{w, 1}, Strided{w + vl, 1}, Strided{w + 2 * vl, 1},
              Strided{w + 3 * vl, 1}, Strided{w + 4 * vl, 1}, Strided{w + 5 * vl, 1});
  }
}

// One warp per slice: Gram-Schmidt twice of the k bidiagonal vectors in
// order (a vanished vector is replaced by a canonical basis vector).
__global__ void __launch_bounds__(32) svd_orth_kernel(SvdParams P) {
  const int lane = threadIdx.x;
  const int64_t n = P.n, NP = P.NP, RP = P.RP;
  for (;;) {
    int64_t it = 0;
    if (lane == 0) it = int64_t(atomicAdd(&P.counter[3], 1ull));
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= P.count) break;
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int64_t k = kout_of(P, slice);
    double* Vb = P.vsel + si * RP * NP;
    for (int64_t j = 0; j < k; ++j) {
      double* vj = Vb + j * RP;
      int64_t basis = 0;
      const double cthr = 0.5 * sqrt(double(n - j) / double(n));  // see cgs2_fix
      for (int64_t attempt = 0; attempt <= n; ++attempt) {
        for (int pass = 0; pass < (attempt ? 3 : 2); ++pass) {
          for (int64_t i = 0; i < j; ++i) {
            const double* vi = Vb + i * RP;
            double d = 0.0;
            for (int64_t q = lane; q < n; q += 32) d += vi[q] * vj[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            for (int64_t q = lane; q < n; q += 32) vj[q] -= d * vi[q];
            __syncwarp();
          }
        }
        double nr = 0.0;
        for (int64_t q = lane; q < n; q += 32) nr += vj[q] * vj[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nr += __shfl_xor_sync(0xffffffffu, nr, o);
        nr = sqrt(nr);
        if (nr > (attempt ? cthr : 0.5) || attempt == n) {
          const double inv = nr > 0.0 ? 1.0 / nr : 0.0;
          for (int64_t q = lane; q < n; q += 32) vj[q] *= inv;
          __syncwarp();
          break;
        }
        for (int64_t q = lane; q < n; q += 32) vj[q] = (q == basis) ? 1.0 : 0.0;
        ++basis;
        __syncwarp();
      }
    }
  }
}

// Blocked variant (RP <= 1024): one CTA (8 warps) per slice.  Vectors are
// taken 16 at a time into shared memory (W); the block is projected against
// all earlier, finished vectors Q = V[:, 0:j0] by block-MGS over 64-column
// chunks of Q, twice (C = Q_c^T W, W -= Q_c C, both on DMMA), then
// orthonormalised internally (CGS2, one warp per dot product) and written
// back.  A vector that vanishes (norm <= 1/2 of its unit input) falls back
// to canonical basis vectors projected against every earlier vector, as the
// one-warp kernel above.  Vector j depends only on vectors < j (block
// boundaries at multiples of 16), so the leading k vectors are the same bits
// whatever the slice's rank.  Work per slice: 4 n k^2 flops on DMMA instead
// of k^2 dependent warp dot products.
constexpr int OB = 16;   // vectors per block
constexpr int OQ = 64;   // earlier vectors per chunk
constexpr int OCS = 24;  // C row stride (conflict-free B fragments)
__host__ __device__ __forceinline__ size_t orth_smem(int64_t RP) {
  return (size_t(OB) * size_t(RP + 4) + size_t(OQ) * OCS + 32) * sizeof(double);
}

__device__ __forceinline__ double cta_sum256(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const double s = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(256) svd_orth_block_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n = int(P.n), rp = int(P.RP), ws = rp + 4;
  const int64_t NP = P.NP, RP = P.RP;
  double* W = reinterpret_cast<double*>(smem_raw);  // [OB][ws]: column c at W + c * ws
  double* Cs = W + OB * ws;                         // [OQ][OCS]
  double* red = Cs + OQ * OCS;                      // [8] CTA partials
  double* dots = red + 8;                           // [16]
  __shared__ int64_t cur;
  for (;;) {
    if (tid == 0) cur = int64_t(atomicAdd(&P.counter[3], 1ull));
    __syncthreads();
    const int64_t it = cur;
    __syncthreads();
    if (it >= P.count) break;
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int k = int(kout_of(P, slice));
    double* Vb = P.vsel + si * RP * NP;
    int64_t basis = 0;
    for (int j0 = 0; j0 < k; j0 += OB) {
      const int kb = min(OB, k - j0);
      for (int e = tid; e < OB * rp; e += 256) {
        const int c = e / rp, q = e - c * rp;
        W[c * ws + q] = (c < kb && q < n) ? Vb[int64_t(j0 + c) * RP + q] : 0.0;
      }
      __syncthreads();
      for (int pass = 0; pass < 2 && j0 > 0; ++pass) {
        for (int i0 = 0; i0 < j0; i0 += OQ) {
          {  // Cs[i][c] = sum_q V[q][i0 + i] W[c][q]; warp w: i in [8w, 8w + 8)
            const int col = i0 + 8 * warp + g;
            const bool live = col < j0;
            const double* qa = Vb + int64_t(live ? col : 0) * RP + t;
            const double* wb = W + g * ws + t;
            double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll 8
            for (int r = 0; r < n; r += 4) {
              const double a = live ? qa[r] : 0.0;
              dmma884n(d0, d1, a, wb[r]);
              dmma884n(e0, e1, a, wb[r + 8 * ws]);
            }
            double* cr = Cs + (8 * warp + g) * OCS + 2 * t;
            cr[0] = d0;
            cr[1] = d1;
            cr[8] = e0;
            cr[9] = e1;
          }
          __syncthreads();
          {  // W[c][q] -= sum_i V[q][i0 + i] Cs[i][c]; warp w: row tiles w, w + 8, ...
            const int nic = min(OQ, j0 - i0);  // a multiple of OB
            for (int r0 = 8 * warp; r0 < n; r0 += 64) {
              const double* qa = Vb + int64_t(i0 + t) * RP + r0 + g;
              const double* cb = Cs + t * OCS + g;
              double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll 4
              for (int kk = 0; kk < nic; kk += 4) {
                const double a = qa[int64_t(kk) * RP];
                dmma884n(d0, d1, a, cb[kk * OCS]);
                dmma884n(e0, e1, a, cb[kk * OCS + 8]);
              }
              double* wr = W + 2 * t * ws + r0 + g;
              wr[0] -= d0;
              wr[ws] -= d1;
              wr[8 * ws] -= e0;
              wr[9 * ws] -= e1;
            }
          }
          __syncthreads();
        }
      }
      for (int c = 0; c < kb; ++c) {
        double* wc = W + c * ws;
        for (int pass = 0; pass < 2 && c > 0; ++pass) {
          for (int i = warp; i < c; i += 8) {
            const double* wi = W + i * ws;
            double sd = 0.0;
            for (int q = lane; q < n; q += 32) sd = fma(wi[q], wc[q], sd);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
            if (lane == 0) dots[i] = sd;
          }
          __syncthreads();
          for (int q = tid; q < n; q += 256) {
            double v = wc[q];
            for (int i = 0; i < c; ++i) v = fma(-dots[i], W[i * ws + q], v);
            wc[q] = v;
          }
          __syncthreads();
        }
        double sq = 0.0;
        for (int q = tid; q < n; q += 256) sq = fma(wc[q], wc[q], sq);
        double nr = sqrt(cta_sum256(sq, red));
        if (!(nr > 0.5)) {
          // vanished: canonical basis vectors, each projected (3 passes, MGS)
          // against every earlier vector, until one keeps norm > cthr
          const int j = j0 + c;
          const double cthr = 0.5 * sqrt(double(n - j) / double(n));
          for (int attempt = 1; attempt <= n; ++attempt) {
            for (int q = tid; q < n; q += 256) wc[q] = (q == basis) ? 1.0 : 0.0;
            ++basis;
            __syncthreads();
            for (int pass = 0; pass < 3; ++pass) {
              for (int i = 0; i < j; ++i) {
                const double* vi = i < j0 ? Vb + int64_t(i) * RP : W + (i - j0) * ws;
                double sd = 0.0;
                for (int q = tid; q < n; q += 256) sd = fma(vi[q], wc[q], sd);
                const double dd = cta_sum256(sd, red);
                for (int q = tid; q < n; q += 256) wc[q] = fma(-dd, vi[q], wc[q]);
                __syncthreads();
              }
            }
            sq = 0.0;
            for (int q = tid; q < n; q += 256) sq = fma(wc[q], wc[q], sq);
            nr = sqrt(cta_sum256(sq, red));
            if (nr > cthr) break;
          }
        }
        const double inv = nr > 0.0 ? 1.0 / nr : 0.0;
        for (int q = tid; q < n; q += 256) wc[q] *= inv;
        __syncthreads();
      }
      for (int e = tid; e < kb * rp; e += 256) {
        const int c = e / rp, q = e - c * rp;
        if (q < n) Vb[int64_t(j0 + c) * RP + q] = W[c * ws + q];
      }
      __syncthreads();
    }
  }
}

// Back-transformation v <- P1 P2 v of the right vectors: the bulge chase's
// right reflectors in reverse order, then the band reduction's LQ panels
// (I - V T V^T) from the last to the first.  One CTA per (slice, group of G
// vectors), one warp per vector.  Every log record is staged into shared
// memory once per CTA (cp.async, one sweep ahead) and applied by all G
// warps, so the logs are read once per group rather than once per vector.
// The tasks of one sweep act on disjoint 16-column ranges: lane k applies
// task k (chunks of 32 tasks), a CTA barrier between sweeps.  The LQ panels
// are streamed in 128-row chunks, each warp forming V^T x (butterfly
// reduced), T (V^T x), then x -= V z.  Vectors live in shared memory with a
// skewed index (q + q / 16) so the lanes' 16-element ranges fall in
// distinct banks; records are padded to 17 doubles for the same reason.
constexpr int BT_REC = 17;   // padded record stride
constexpr int BT_ROWS = 64;  // LQ panel rows per staged chunk (double-buffered)
// Sweep-record buffers (records staged BT_NRB - 1 sweeps ahead) and the L2
// prefetch distance in sweeps.  Measured (ncu, cold caches): c2 (85 MB of
// log) 0.65 ms without prefetch, 0.52 with; c1 (33 MB) 0.42 without, 0.35
// with; deeper staging (4, 8 buffers) changes neither.
constexpr int BT_NRB = 2;
constexpr int BT_PF = 16;
__host__ __device__ __forceinline__ int64_t bt_stride(int64_t n) { return n + n / 16 + 48; }
__host__ __device__ __forceinline__ size_t bt_smem(int64_t n, int g) {
  return (size_t(g) * bt_stride(n) + BT_NRB * size_t(hb_kmax(n)) * BT_REC + 2 * BW * BT_ROWS + BW * BW) *
         sizeof(double);
}
__device__ __forceinline__ int sx(int q) { return q + (q >> 4); }

template <bool PF>
__global__ void __launch_bounds__(256) svd_backtransform_kernel(SvdParams P, int G, int lq) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nthr = blockDim.x;
  const int n = int(P.n);
  const int64_t NP = P.NP, RP = P.RP;
  const int npan = int(NP / BW);
  const int64_t stride = bt_stride(n);
  const int kmax = int(hb_kmax(n));
  double* xs = reinterpret_cast<double*>(smem_raw);    // [G][stride]
  double* rb = xs + G * stride;                        // [BT_NRB][kmax * BT_REC] sweep records
  double* vc = rb + BT_NRB * kmax * BT_REC;            // [2][BW][BT_ROWS] LQ chunks
  double* ts = vc + 2 * BW * BT_ROWS;                  // [BW * BW] LQ T
  double* x = xs + warp * stride;
  const int ngroups = (n + G - 1) / G;
  for (int64_t cta = blockIdx.x; cta < P.count * ngroups; cta += gridDim.x) {
    const int64_t it = cta / ngroups;
    const int grp = int(cta % ngroups);
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int kv = int(kout_of(P, slice));
    const int j0 = grp * G;
    if (j0 >= kv) continue;
    const int j = j0 + warp;
    const bool act = j < kv;
    double* vg = P.vsel + si * RP * NP + int64_t(j) * RP;
    for (int q = lane; q < stride; q += 32) x[q] = 0.0;
    __syncwarp();
    if (act)
      for (int q = lane; q < n; q += 32) x[sx(q)] = vg[q];
    // ---- bulge-chase reflectors, last sweep first
    const double* lg = P.hhlog + si * P.hhcap;
    // The records of a sweep are read once, from the log the bulge chase
    // wrote (L2 or HBM): one sweep of lookahead (~400 cycles of work) cannot
    // cover that latency, so they are prefetched to L2 BT_PF sweeps ahead and
    // staged into shared memory BT_NRB - 1 sweeps ahead.
    auto stage = [&](int i) {  // records of sweep i -> rb[i % BT_NRB] (empty group for i < 0)
      if (i >= 0) {
        const int K = int(hb_tasks(n, i));
        double* dst = rb + (i % BT_NRB) * kmax * BT_REC;
        const double* src = lg + int64_t(i) * kmax * HLOG;
        for (int e = threadIdx.x; e < K * HLOG; e += nthr) {  // padded rows: 8-byte copies
          const int k = e / HLOG, h = e % HLOG;
          cp_async8(dst + k * BT_REC + h, src + k * HLOG + h);
        }
      }
      cp_async_commit();
    };
    auto prefetch = [&](int i) {  // one 128-byte line per thread
      if (PF && i >= 0) {
        const int lines = (int(hb_tasks(n, i)) * HLOG * 8 + 127) / 128;
        if (int(threadIdx.x) < lines)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(lg + int64_t(i) * kmax * HLOG + threadIdx.x * 16));
      }
    };
    if (PF)
      for (int d = 0; d < BT_PF; ++d) prefetch(n - 3 - d);
    for (int d = 0; d < BT_NRB - 1; ++d) stage(n - 3 - d);
    for (int i = n - 3; i >= 0; --i) {
      stage(i - (BT_NRB - 1));
      if (PF) prefetch(i - BT_PF);
      cp_async_wait<BT_NRB - 1>();
      __syncthreads();
      const int K = int(hb_tasks(n, i));
      const double* rbuf = rb + (i % BT_NRB) * kmax * BT_REC;
      if (act) {
        for (int kb = 0; kb < K; kb += 32) {  // tasks of one sweep are disjoint
          const int k = kb + lane;
          if (k < K) {
            const double* r = rbuf + k * BT_REC;
            const double tau = r[0];
            if (tau != 0.0) {
              const int c0 = i + k * BW + 1;
              const int base = sx(c0), b16 = BW - (c0 & 15);  // skew steps by one at l = b16
              double xv[BW];
#pragma unroll
              for (int l = 0; l < BW; ++l) xv[l] = x[base + l + (l >= b16)];
              double w0 = xv[0], w1 = 0.0;
#pragma unroll
              for (int l = 1; l < BW; l += 2) {
                w1 = fma(r[l], xv[l], w1);
                if (l + 1 < BW) w0 = fma(r[l + 1], xv[l + 1], w0);
              }
              const double w = (w0 + w1) * tau;
              x[base] = xv[0] - w;
#pragma unroll
              for (int l = 1; l < BW; ++l) x[base + l + (l >= b16)] = fma(-w, r[l], xv[l]);
            }
          }
        }
      }
      __syncthreads();  // rb[i % BT_NRB] is restaged BT_NRB sweeps later
    }
    // ---- LQ panels of the band reduction, last first.  Per panel one flat
    // sequence of 2 nq chunk loads (pass 1: V^T x, pass 2: x -= V z) through
    // a two-buffer cp.async ring.
    const double* rv = P.rvlog + si * int64_t(npan) * (BW * NP + BW * BW);
    for (int pk = lq ? npan - 2 : -1; pk >= 0; --pk) {
      const double* Vp = rv + int64_t(pk) * (BW * NP + BW * BW);  // V[c][q], q < NP
      const int jlo = pk * BW + BW;
      const int nq = (n - jlo + BT_ROWS - 1) / BT_ROWS;
      if (nq <= 0) continue;
      auto issue = [&](int t) {
        const int q0 = jlo + (t % nq) * BT_ROWS;
        double* dst = vc + (t & 1) * BW * BT_ROWS;
        for (int e = threadIdx.x; e < BW * (BT_ROWS / 2); e += nthr) {
          const int c = e / (BT_ROWS / 2), r2 = (e % (BT_ROWS / 2)) * 2;
          const int left = n - (q0 + r2);
          const int bytes = left >= 2 ? 16 : (left == 1 ? 8 : 0);
          cp_async16(dst + c * BT_ROWS + r2, bytes ? Vp + int64_t(c) * NP + q0 + r2 : Vp, bytes);
        }
        cp_async_commit();
      };
      for (int e = threadIdx.x; e < BW * BW; e += nthr) ts[e] = Vp[BW * NP + e];
      issue(0);
      double y[BW], zz[BW];
#pragma unroll
      for (int c = 0; c < BW; ++c) y[c] = 0.0;
      for (int t = 0; t < 2 * nq; ++t) {
        if (t + 1 < 2 * nq) {
          issue(t + 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* cb = vc + (t & 1) * BW * BT_ROWS;
        const int q0 = jlo + (t % nq) * BT_ROWS;
        if (t == nq) {  // pass 1 done: y = V^T x (warp sum), z = T y
#pragma unroll
          for (int c = 0; c < BW; ++c) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) y[c] += __shfl_xor_sync(0xffffffffu, y[c], o);
          }
#pragma unroll
          for (int a = 0; a < BW; ++a) {
            double acc = 0.0;
#pragma unroll
            for (int b2 = 0; b2 < BW; ++b2) acc = fma(ts[a * BW + b2], y[b2], acc);
            zz[a] = acc;
          }
        }
        if (act) {
          for (int r = lane; r < BT_ROWS && q0 + r < n; r += 32) {
            if (t < nq) {
              const double xq = x[sx(q0 + r)];
#pragma unroll
              for (int c = 0; c < BW; ++c) y[c] = fma(cb[c * BT_ROWS + r], xq, y[c]);
            } else {
              double acc = x[sx(q0 + r)];
#pragma unroll
              for (int c = 0; c < BW; ++c) acc = fma(-cb[c * BT_ROWS + r], zz[c], acc);
              x[sx(q0 + r)] = acc;
            }
          }
        }
        __syncthreads();  // the buffer is refilled two steps later
      }
    }
    __syncwarp();
    if (act)
      for (int q = lane; q < RP; q += 32) vg[q] = q < n ? x[sx(q)] : 0.0;
    __syncthreads();
  }
}

// LQ panels of the band reduction applied to KB right vectors at once on
// DMMA (after svd_backtransform_kernel has applied the bulge reflectors):
// X <- (I - V_p T_p V_p^T) X for p = last .. first, X (n x KB) resident in
// shared memory, V_p streamed from the panel log.  Per panel: Y = V_p^T X
// (16 x KB tiles, one per warp, K split in two when KB = 16), Z = T_p Y,
// X -= V_p Z.  Column v of X depends only on itself, so vector j is the
// same bits whatever the slice's rank.  4 n^2 flops per vector on DMMA.
constexpr int LQ_ZS = 40;  // Z row stride (= 8 mod 32: conflict-free B fragments)
__host__ __device__ __forceinline__ int lq_xs(int64_t n) { return int(((n + 31) / 32) * 32 + 4); }
__host__ __device__ __forceinline__ size_t lq_smem(int64_t n, int kb) {
  return (size_t(kb) * lq_xs(n) + 2 * BW * 40 + BW * LQ_ZS + BW * BW) * sizeof(double);
}

template <int KB>
__global__ void __launch_bounds__(256) svd_lqapply_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NT8 = KB / 8, TILES = 2 * NT8, KS = 8 / TILES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n = int(P.n), npan = int(P.NP / BW), xs = lq_xs(P.n);
  const int64_t NP = P.NP, RP = P.RP;
  double* X = reinterpret_cast<double*>(smem_raw);  // [KB][xs]: vector v at X + v * xs
  double* Ys = X + KB * xs;                         // [KS][16][40]
  double* Zs = Ys + 2 * BW * 40;                    // [16][LQ_ZS]
  double* Ts = Zs + BW * LQ_ZS;                     // [16][16]
  const int ngroups = (n + KB - 1) / KB;
  const int tile = warp % TILES, ks = warp / TILES, mt = tile / NT8, nt = tile % NT8;
  for (int64_t cta = blockIdx.x; cta < P.count * ngroups; cta += gridDim.x) {
    const int64_t it = cta / ngroups;
    const int j0 = int(cta % ngroups) * KB;
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int kv = int(kout_of(P, slice));
    if (j0 >= kv) continue;
    double* vb = P.vsel + si * RP * NP;
    for (int e = tid; e < KB * xs; e += 256) {
      const int v = e / xs, q = e - v * xs;
      X[e] = (j0 + v < kv && q < n) ? vb[int64_t(j0 + v) * RP + q] : 0.0;
    }
    const double* rv = P.rvlog + si * int64_t(npan) * (BW * NP + BW * BW);
    for (int pk = npan - 2; pk >= 0; --pk) {
      const double* Vp = rv + int64_t(pk) * (BW * NP + BW * BW);  // V[c][q] at Vp[c * NP + q]
      const int jlo = pk * BW + BW;                               // V rows < jlo are zero
      if (jlo >= n) continue;
      Ts[tid] = Vp[BW * NP + tid];  // T[a][b] at a * 16 + b (256 threads, 256 entries)
      if (pk > 0 && tid < BW) {     // next panel's live rows -> L2 while this one runs
        const double* nv = Vp - (BW * NP + BW * BW) + int64_t(tid) * NP;
        const int lo = (jlo - BW) & ~1, bytes = (n - lo) * 8 & ~15;
        if (bytes > 0) bulk_prefetch_l2(nv + lo, bytes);
      }
      __syncthreads();
      {  // Y = V^T X: warp -> (mt, nt) tile, rows split KS ways (4-aligned)
        const int r0 = jlo & ~3, span = ((n - r0 + 4 * KS - 1) / (4 * KS)) * 4;
        const int rb = r0 + ks * span, re = min(n, rb + span);
        const double* va = Vp + int64_t(8 * mt + g) * NP + t;
        const double* xb = X + (8 * nt + g) * xs + t;
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
        int r = rb;
#pragma unroll 4
        for (; r + 4 < re; r += 8) {
          dmma884n(d0, d1, va[r], xb[r]);
          dmma884n(e0, e1, va[r + 4], xb[r + 4]);
        }
        if (r < re) dmma884n(d0, d1, va[r], xb[r]);
        double* yr = Ys + (ks * BW + 8 * mt + g) * 40 + 8 * nt + 2 * t;
        yr[0] = d0 + e0;
        yr[1] = d1 + e1;
      }
      __syncthreads();
      for (int e = tid; e < BW * KB; e += 256) {  // Z = T Y
        const int a = e / KB, v = e - a * KB;
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < BW; ++b) {
          double y = Ys[b * 40 + v];
          if (KS == 2) y += Ys[(BW + b) * 40 + v];
          acc = fma(Ts[a * BW + b], y, acc);
        }
        Zs[a * LQ_ZS + v] = acc;
      }
      __syncthreads();
#pragma unroll 2
      for (int r0 = (jlo & ~7) + 8 * warp; r0 < n; r0 += 64) {  // X -= V Z, 8-row tiles
        double acc[NT8][2];
#pragma unroll
        for (int c = 0; c < NT8; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < BW; kk += 4) {
          const double a = Vp[int64_t(kk + t) * NP + r0 + g];
#pragma unroll
          for (int c = 0; c < NT8; ++c) dmma884n(acc[c][0], acc[c][1], a, Zs[(kk + t) * LQ_ZS + 8 * c + g]);
        }
#pragma unroll
        for (int c = 0; c < NT8; ++c) {
          X[(8 * c + 2 * t) * xs + r0 + g] -= acc[c][0];
          X[(8 * c + 2 * t + 1) * xs + r0 + g] -= acc[c][1];
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < KB * int(RP); e += 256) {
      const int v = e / int(RP), q = e - v * int(RP);
      if (j0 + v < kv) vb[int64_t(j0 + v) * RP + q] = q < n ? X[v * xs + q] : 0.0;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------
// Blocked back-transformation of the bulge-chase reflectors on DMMA
// (n > 400: c3, c4).  The right reflectors H_{i,k} (sweep i, task k) act on
// coordinates c0 = i + 16k + 1 .. c0 + 15 and must be applied to every
// vector x in the reverse of the chase order.  Grouping 16 consecutive
// sweeps with the same task index, B(g, k) = H_{16g,k} ... H_{16g+15,k},
// gives a compact-WY block I - V T V^T on the 32-row window
// [16 (g + k), 16 (g + k) + 32) (V lower trapezoidal: column j holds
// v_{16g+j,k} at window rows j + 1 .. j + 16).  Reflectors of different
// blocks overlap only as follows: B(g, k) meets B(g, k - 1) and
// B(g + 1, k - 2 .. k), and in every overlapping pair the reverse chase
// order applies the larger sweep first -- i.e. B(g + 1, .) before B(g, .),
// and within a group B(g, k - 1) before B(g, k) (H_{i',k-1} with i' > i
// overlaps H_{i,k}; H_{i,k-1} with i' < i does not).  So the schedule
// g = G - 1 .. 0, k = 0 .. K_g - 1 is the sequential product exactly.
// T (16 x 16, dlarft forward) of every block is built once per slice by
// svd_bt_tlog_kernel; svd_bt_blocked_kernel keeps KB vectors resident in
// shared memory and applies each block with three DMMA phases per warp
// (warp = 8 vectors): Y^T = X_R^T V, Z^T = Y^T T^T, X_R^T -= Z^T V^T, the
// K index of the last two permuted to (2t, 2t+1, 8+2t, 9+2t) so the
// accumulators of one phase are the A fragments of the next (no shuffle, no
// shared-memory round trip).  Every vector depends only on itself: the
// truncated factors stay the leading full factors bit for bit.
// ----------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t bt_groups(int64_t n) { return n >= 3 ? (n - 3) / BW + 1 : 0; }
__host__ __device__ __forceinline__ int64_t bt_gtasks(int64_t n, int64_t g) { return hb_tasks(n, g * BW); }
__host__ __device__ __forceinline__ int64_t bt_nblocks(int64_t n) {
  int64_t t = 0;
  for (int64_t g = 0; g < bt_groups(n); ++g) t += bt_gtasks(n, g);
  return t;
}
constexpr int BTV_S = 20;  // V window row stride (doubles, = 4 mod 16: conflict-free B fragments)
constexpr int BTT_S = 20;  // T row stride
constexpr int BT_NST = 8;  // blocks in flight (records + T): covers the L2/HBM latency of a block
constexpr int BTR_S = 18;  // staged record stride (16 would put the 16 records of a block in one bank pair:
                           // the V-window build read them 16-way conflicted, 47% of the kernel's wavefronts)

// T of every block of every slice: one warp per (list position, block).
__global__ void __launch_bounds__(128) svd_bt_tlog_kernel(SvdParams P, double* tlog, int64_t nblk) {
  __shared__ double vbuf[4][32 * 17];
  __shared__ double gbuf[4][16 * 17];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = int(P.n);
  const int64_t kmax = hb_kmax(n), G = bt_groups(n);
  double* V = vbuf[warp];
  double* Gm = gbuf[warp];
  const int64_t total = P.count * nblk;
  for (int64_t w = int64_t(blockIdx.x) * 4 + warp; w < total; w += int64_t(gridDim.x) * 4) {
    const int64_t it = w / nblk, b = w % nblk;
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    // block index b -> (g, k): groups from the last one down
    int64_t g = G - 1, rem = b;
    while (rem >= bt_gtasks(n, g)) rem -= bt_gtasks(n, g--);
    const int64_t k = rem;
    const double* lg = P.hhlog + si * P.hhcap;
    for (int e = lane; e < 32 * 17; e += 32) V[e] = 0.0;
    __syncwarp();
    double tau = 0.0;
    if (lane < BW) {  // lane j: reflector of sweep 16 g + j (identity if the task does not exist)
      const int64_t i = g * BW + lane;
      if (i <= n - 3 && k < hb_tasks(n, i)) {
        const double* rec = lg + (i * kmax + k) * HLOG;
        tau = rec[0];
        if (tau != 0.0) {
          V[(lane + 1) * 17 + lane] = 1.0;
          for (int l = 1; l < BW; ++l) V[(lane + 1 + l) * 17 + lane] = rec[l];
        }
      }
    }
    __syncwarp();
    // Gram G[a][c] = sum_l V[l][a] V[l][c] (8 entries per lane)
    for (int e = lane; e < BW * BW; e += 32) {
      const int a = e >> 4, c = e & 15;
      double acc = 0.0;
      for (int l = 0; l < 32; ++l) acc = fma(V[l * 17 + a], V[l * 17 + c], acc);
      Gm[a * 17 + c] = acc;
    }
    __syncwarp();
    // dlarft (forward, columnwise): lane i owns row i of T
    double* T = tlog + (si * nblk + b) * (BW * BW);
    const double taui = __shfl_sync(0xffffffffu, tau, lane & 15);
    if (lane < BW) {
      double row[BW];
#pragma unroll
      for (int j = 0; j < BW; ++j) row[j] = 0.0;
#pragma unroll
      for (int j = 0; j < BW; ++j) {
        const double tj = __shfl_sync(0x0000ffffu, tau, j);
        if (j == lane) row[j] = taui;
        if (j > lane) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < BW; ++l)
            if (l >= lane && l < j) acc = fma(row[l], Gm[l * 17 + j], acc);
          row[j] = -tj * acc;
        }
      }
#pragma unroll
      for (int j = 0; j < BW; ++j) T[lane * BW + j] = row[j];
    }
    __syncwarp();
  }
}

template <int KB>
__global__ void __launch_bounds__(KB * 4) svd_bt_blocked_kernel(SvdParams P, const double* tlog,
                                                               int64_t nblk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int n = int(P.n), xs = lq_xs(P.n);
  const int64_t NP = P.NP, RP = P.RP, kmax = hb_kmax(n), G = bt_groups(n);
  double* X = reinterpret_cast<double*>(smem_raw);   // [KB][xs]
  double* Vb = X + KB * xs;                          // [2][32 * BTV_S]
  double* Tb = Vb + 2 * 32 * BTV_S;                  // [BT_NST][16 * BTT_S]
  double* Rb = Tb + BT_NST * BW * BTT_S;             // [BT_NST][16 records * BTR_S] raw log records
  const int ngroups = (n + KB - 1) / KB;
  for (int64_t cta = blockIdx.x; cta < P.count * ngroups; cta += gridDim.x) {
    const int64_t it = cta / ngroups;
    const int j0 = int(cta % ngroups) * KB;
    const int64_t si = state_index(P, it);
    if (P.flags[si]) continue;
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int kv = int(kout_of(P, slice));
    if (j0 >= kv) continue;
    double* vb = P.vsel + si * RP * NP;
    for (int e = tid; e < KB * xs; e += KB * 4) {
      const int v = e / xs, q = e - v * xs;
      X[e] = (j0 + v < kv && q < n) ? vb[int64_t(j0 + v) * RP + q] : 0.0;
    }
    const double* lg = P.hhlog + si * P.hhcap;
    const double* tl = tlog + si * nblk * (BW * BW);
    // stage block b (records + T) into buffer slot: records of sweeps 16 g + j, task k
    auto stage = [&](int64_t b, int64_t g, int64_t k, int slot) {
      double* rb = Rb + slot * (BW * BTR_S);
      double* tb = Tb + slot * (BW * BTT_S);
      for (int e = tid; e < BW * (BW / 2); e += KB * 4) {
        const int j = e / (BW / 2), h = (e % (BW / 2)) * 2;
        const int64_t i = g * BW + j;
        const bool live = i <= n - 3 && k < hb_tasks(n, i);
        cp_async16(rb + j * BTR_S + h, live ? lg + (i * kmax + k) * HLOG + h : lg, live ? 16 : 0);
        const int a = e / (BW / 2), c = (e % (BW / 2)) * 2;
        cp_async16(tb + a * BTT_S + c, tl + b * (BW * BW) + a * BW + c, 16);
      }
      cp_async_commit();
    };
    int64_t gcur = G - 1, kcur = 0;
    auto advance = [&](int64_t& g, int64_t& k) {
      if (++k >= bt_gtasks(n, g)) {
        --g;
        k = 0;
      }
    };
    // ring of BT_NST blocks: blocks b .. b + BT_NST - 2 in flight
    int64_t gs = gcur, ks = kcur;
    for (int q = 0; q < BT_NST - 1; ++q) {
      if (q < nblk) {
        stage(q, gs, ks, q);
        advance(gs, ks);
      } else {
        cp_async_commit();
      }
    }
    const double* xw = X + (8 * warp + g8) * xs;   // this lane's vector (row = vector g8 of the warp)
    double* xwm = X + (8 * warp + g8) * xs;
    for (int64_t b = 0; b < nblk; ++b) {
      const int slot = int(b % BT_NST), vslot = int(b & 1);
      cp_async_wait<BT_NST - 2>();
      __syncthreads();
      {  // V window of block b from its staged records
        double* Vw = Vb + vslot * (32 * BTV_S);
        const double* rb = Rb + slot * (BW * BTR_S);
        for (int e = tid; e < 32 * BW; e += KB * 4) {
          const int l = e / BW, j = e % BW;
          const int d = l - 1 - j;
          double v = 0.0;
          if (d >= 0 && d < BW && rb[j * BTR_S] != 0.0) v = d == 0 ? 1.0 : rb[j * BTR_S + d];
          Vw[l * BTV_S + j] = v;
        }
      }
      if (b + BT_NST - 1 < nblk) {  // refill the slot block b - 1 used
        stage(b + BT_NST - 1, gs, ks, int((b + BT_NST - 1) % BT_NST));
        advance(gs, ks);
      } else {
        cp_async_commit();
      }
      __syncthreads();
      const int rb0 = int(BW * (gcur + kcur));          // window rows rb0 .. rb0 + 31
      const double* V = Vb + vslot * (32 * BTV_S);
      const double* T = Tb + slot * (BW * BTT_S);
      // Y^T (8 vectors x 16) = X_R^T V: K = 32 window rows
      double y[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int s4 = 0; s4 < 8; ++s4) {
        const int rr = 4 * s4 + t4;
        const double a = rb0 + rr < xs ? xw[rb0 + rr] : 0.0;
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma884n(y[ni][0], y[ni][1], a, V[rr * BTV_S + 8 * ni + g8]);
      }
      // Z^T = Y^T T^T: K order (2t, 2t+1, 8+2t, 9+2t) = (y[0][0], y[0][1], y[1][0], y[1][1])
      double z[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const int cs[4] = {2 * t4, 2 * t4 + 1, 8 + 2 * t4, 9 + 2 * t4};
      const double ya[4] = {y[0][0], y[0][1], y[1][0], y[1][1]};
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
          dmma884n(z[ni][0], z[ni][1], ya[s4], T[(8 * ni + g8) * BTT_S + cs[s4]]);
      // X_R^T -= Z^T V^T: 4 row tiles of 8, same K order
      const double za[4] = {-z[0][0], -z[0][1], -z[1][0], -z[1][1]};
      __syncwarp();
#pragma unroll
      for (int ri = 0; ri < 4; ++ri) {
        const int r = rb0 + 8 * ri + 2 * t4;
        double d0 = r < xs ? xwm[r] : 0.0, d1 = r + 1 < xs ? xwm[r + 1] : 0.0;
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) dmma884n(d0, d1, za[s4], V[(8 * ri + g8) * BTV_S + cs[s4]]);
        __syncwarp();
        if (r < xs) xwm[r] = d0;
        if (r + 1 < xs) xwm[r + 1] = d1;
      }
      advance(gcur, kcur);
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int e = tid; e < KB * int(RP); e += KB * 4) {
      const int v = e / int(RP), q = e - v * int(RP);
      if (j0 + v < kv) vb[int64_t(j0 + v) * RP + q] = q < n ? X[v * xs + q] : 0.0;
    }
    __syncthreads();
  }
}

// Output kernel of the bidiagonal vector path: sigma are in P.s (bisection),
// right singular vectors of X in vsel (sorted order); emit U / V / packed
// factors through the shared emit_vectors (other side = X V / ||X V||).
__global__ void __launch_bounds__(TPB) svd_vecout_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacobiSmem& sm = *reinterpret_cast<JacobiSmem*>(smem_raw);
  int NS = 1;
  while (NS < P.n) NS <<= 1;
  FinalView fs = final_view(smem_raw, NS);
  __shared__ int64_t cur;
  const int tid = threadIdx.x;
  const int64_t LP = P.LP, NP = P.NP, RP = P.RP;
  double* Xslot = P.xslots + int64_t(blockIdx.x) * LP * NP;
  for (;;) {
    if (tid == 0) cur = int64_t(atomicAdd(&P.counter[1], 1ull));
    __syncthreads();
    const int64_t it = cur;
    __syncthreads();
    if (it >= P.count) break;
    const int64_t si = state_index(P, it);
    const int64_t slice = P.ids ? P.ids[it] : it;
    const int flag = P.flags[si];
    if (flag == 2) continue;
    if (flag == 1) {
      emit_zero_slice(P, slice);
      continue;
    }
    for (int j = tid; j < NS; j += TPB) fs.idx[j] = j;
    __syncthreads();
    emit_vectors(P, sm, fs, slice, P.A + slice * P.m * P.p, P.vsel + si * RP * NP, fs.idx, Xslot,
                 true, nullptr, 0);
  }
}

template <bool WANTV>
__global__ void __launch_bounds__(TPB, 3) svd_jacobi_kernel(SvdParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacobiSmem& sm = *reinterpret_cast<JacobiSmem*>(smem_raw);
  int NS = 1;
  while (NS < P.n) NS <<= 1;
  FinalView fs = final_view(smem_raw, NS);
  __shared__ int64_t cur;
  const int tid = threadIdx.x;
  const int64_t n = P.n, LP = P.LP, NP = P.NP, RP = P.RP;
  double* Xslot = P.xslots + int64_t(blockIdx.x) * LP * NP;
  double* V = WANTV ? P.wslots + int64_t(blockIdx.x) * RP * NP : nullptr;
  const int nb = int(NP / BW);

  for (;;) {
    if (tid == 0) cur = int64_t(atomicAdd(&P.counter[1], 1ull));
    __syncthreads();
    const int64_t it = cur;
    __syncthreads();
    if (it >= P.count) break;
    const int64_t si = state_index(P, it);
    const int64_t slice = P.ids ? P.ids[it] : it;
    const double* A = P.A + slice * P.m * P.p;
    long long t0 = clock64();

    double* T;
    int64_t ldt, rows;
    int flag;
    if (P.use_qr) {
      flag = P.flags[si];
      T = P.rbuf + it * RP * NP;
      ldt = RP;
      rows = RP;
    } else {
      flag = load_slice<TPB>(P, A, Xslot, sm.xs[0]);
      T = Xslot;
      ldt = LP;
      rows = LP;
    }
    if (flag == 2) {
      if (tid == 0) atomicMin(&P.status[0], int32_t(slice));
      __syncthreads();
      continue;
    }
    const int64_t r = n;
    if (flag == 1) {
      emit_zero_slice(P, slice);
      continue;
    }
    if (WANTV) {
      for (int64_t c = 0; c < NP; ++c)
        for (int64_t rr = tid; rr < RP; rr += TPB) V[rr + c * RP] = (rr == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned long long cg = 0, ce = 0, ca = 0, npairs = 0, nrot = 0;

    // ---- Jacobi sweeps over block pairs
    int converged = 0, sweeps = 0;
    for (int sweep = 0; sweep < P.max_sweeps && !converged; ++sweep) {
      int rotated = 0;
      ++sweeps;
      for (int I = 0; I < nb - 1; ++I) {
        for (int J = I + 1; J < nb; ++J) {
          long long a0 = clock64();
          gram_pair(sm, T, ldt, rows, I, J, sm.g[0]);
          int need = 0;
          const double* G = sm.g[0];
          for (int e = tid; e < GW * GW; e += TPB) {
            const int i = e >> 5, j = e & 31;
            if (i < j) {
              const double a = G[i * GS + i], d = G[j * GS + j];
              if (a > 0.0 && d > 0.0 && fabs(G[i * GS + j]) > P.tol * sqrt(a * d)) need = 1;
            }
          }
          need = __syncthreads_or(need);
          long long a1 = clock64();
          cg += a1 - a0;
          ++npairs;
          if (!need) continue;
          rotated = 1;
          ++nrot;
          const int wb = eig_pair(sm, P.tol, P.max_inner);
          long long a2 = clock64();
          apply_pair(sm, T, ldt, rows, I, J, sm.w[wb]);
          if (WANTV) apply_pair(sm, V, RP, RP, I, J, sm.w[wb]);
          long long a3 = clock64();
          ce += a2 - a1;
          ca += a3 - a2;
        }
      }
      converged = !rotated;
    }
    if (!converged && tid == 0) atomicMin(&P.status[1], int32_t(slice));
    __syncthreads();
    long long t2 = clock64();

    // ---- finalize: column norms of T (= sigma), descending sort
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int64_t c = warp; c < NS; c += TPB / 32) {
        double acc = 0.0;
        if (c < n)
          for (int64_t rr = lane; rr < rows; rr += 32) {
            const double x = T[rr + c * ldt];
            acc += x * x;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          fs.key[c] = (c < n) ? sqrt(acc) : -1.0;
          fs.idx[c] = (c < n) ? int(c) : INT_MAX;
        }
      }
    }
    __syncthreads();
    for (int k = 2; k <= NS; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < NS; i += TPB) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const double ka = fs.key[i], kb = fs.key[ixj];
            const int ia = fs.idx[i], ib = fs.idx[ixj];
            const bool up = (i & k) == 0;
            const bool sw = up ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
            if (sw) {
              fs.key[i] = kb;
              fs.key[ixj] = ka;
              fs.idx[i] = ib;
              fs.idx[ixj] = ia;
            }
          }
        }
        __syncthreads();
      }
    }
    // Reported sigma: the bidiagonal/bisection values when that path ran
    // (so values-only, full and truncated jobs agree bitwise), else the
    // Jacobi column norms.
    if (P.s && !P.bidiag)
      for (int64_t j = tid; j < r; j += TPB) P.s[j + slice * r] = fs.key[j];
    __syncthreads();

    if (WANTV && P.job != STARM_SVD_VALUES) {
      __syncthreads();
      emit_vectors(P, sm, fs, slice, A, V, fs.idx, Xslot, P.use_qr, T, ldt);
    }
    __syncthreads();
    long long t3 = clock64();
    stat_add(P, ST_SLICES, 1);
    stat_add(P, ST_SWEEPS, sweeps);
    stat_add(P, ST_PAIRS, npairs);
    stat_add(P, ST_ROTATED, nrot);
    stat_add(P, ST_CYC_GRAM, cg);
    stat_add(P, ST_CYC_EIG, ce);
    stat_add(P, ST_CYC_APPLY, ca);
    stat_add(P, ST_CYC_LOAD, (unsigned long long)(t1 - t0));
    stat_add(P, ST_CYC_FINAL, (unsigned long long)(t3 - t2));
  }
}

__global__ void reset_status_kernel(int32_t* status, unsigned long long* counters) {
  if (threadIdx.x < 2) status[threadIdx.x] = INT32_MAX;
  counters[threadIdx.x] = 0ull;  // 32 counters
}

// ---------------------------------------------------------------- host side

struct Plan {
  int64_t L, n, LP, NP, RP;
  int job;                  // effective job after the fallback mapping
  bool transposed, use_qr, wantv, bidiag, run_jacobi, internal_s, wtwo;
  int team_yb;
  int reduce_nt;
  bool logs;                // right-side transformation logs (vector machinery buffers)
  bool run_front;           // reduce / bulge / bisect
  bool run_vec;             // inverse iteration / back-transform / output
  bool by_slice;            // state kept per slice across calls
  int ns;
  size_t jsmem, rsmem, bsmem;
  int slots_j, slots_r, slots_b, bisect_blocks, slots_v, slots_t, ii_threads, btw, qr_stages, bt_g;
  int64_t hhcap, count;
  bool hb_gmem;
  bool hb_cluster;  // window split over a 2-CTA cluster (DSMEM); slots_b counts clusters
  int hb_threads;
  size_t vsmem, tsmem;
  size_t off_x, off_w, off_r, off_f, off_band, off_de, off_s, off_rv, off_rcs, off_rcol, off_rcnt,
      off_vsel, off_ii, off_tlog, total;
  int bt_kb;                // blocked back-transformation: vectors per CTA (0 = per-warp kernel)
  int64_t bt_nblk;
};

int g_tune_inner = 1;
// inverse-iteration threads per SM (env STARM_II_PER_SM; each owns 12 n doubles of scratch)
const int g_ii_per_sm = [] {
  // measured on c4 (895 K vectors): 128 -> 173 ms, 512 -> 111 ms, 1024 -> 110 ms
  const char* e = getenv("STARM_II_PER_SM");
  const int v = e ? atoi(e) : 512;
  return (v >= 32 && v <= 2048) ? (v / 32) * 32 : 512;
}();
// STARM_BT_BLOCKED=0: the per-warp back-transformation for n > 400 too (A/B runs)
const bool g_bt_blocked = [] {
  const char* e = getenv("STARM_BT_BLOCKED");
  return !(e && e[0] == '0');
}();
size_t bt_blocked_smem(int64_t n, int kb) {
  return (size_t(kb) * lq_xs(n) + 2 * 32 * BTV_S + size_t(BT_NST) * (BW * BTT_S + BW * BTR_S)) *
         sizeof(double);
}
// reduce-kernel CTA size: 0 = automatic, else 256 or 512 (env STARM_REDUCE_THREADS)
int g_reduce_threads = [] {
  const char* e = getenv("STARM_REDUCE_THREADS");
  const int v = e ? atoi(e) : 256;
  return (v == 0 || v == 256 || v == 512) ? v : 256;
}();
int g_tune_sweeps = 60;
// STARM_LQ_WARP=1: LQ panels applied per warp inside the back-transformation (A/B runs)
const bool g_lq_warp = [] {
  const char* e = getenv("STARM_LQ_WARP");
  return e && e[0] == '1';
}();
// STARM_ORTH_WARP=1: the one-warp-per-slice orthonormalisation everywhere (A/B runs)
const bool g_orth_warp = [] {
  const char* e = getenv("STARM_ORTH_WARP");
  return e && e[0] == '1';
}();
// bisection blocks per launch on the side stream (env STARM_BISECT_SIDE_PER_SM, per SM)
int g_bisect_side_blocks = [] {
  const char* e = getenv("STARM_BISECT_SIDE_PER_SM");
  const int per = e ? atoi(e) : 4;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (per >= 1 && per <= 64 ? per : 4) * sms;
}();
// 1 = bidiagonal values path when the panel fits, 0 = Jacobi only, 2 = bidiagonal
// with the bulge-chase window in global memory, 3 = diagnostic: the values
// pass stops after the reduce kernel (outputs undefined; for timing it alone)
int g_tune_mode = 1;
const bool g_team_off = [] {  // STARM_TEAM_UPDATES=0: streaming trailing updates only (A/B runs)
  const char* e = getenv("STARM_TEAM_UPDATES");
  return e && e[0] == '0';
}();
const bool g_reduce_cluster = [] {
  const char* e = getenv("STARM_REDUCE_CLUSTER");
  return !(e && e[0] == '0');
}();
const int g_reduce_cluster_max = [] {  // largest cluster tried (2, 4 or 8)
  const char* e = getenv("STARM_REDUCE_CLUSTER_MAX");
  const int v = e ? atoi(e) : 8;
  return v >= 2 && v <= 8 ? v : 8;
}();
const bool g_bulge_cluster = [] {
  const char* e = getenv("STARM_BULGE_CLUSTER");
  return !(e && e[0] == '0');
}();
int g_stats_on = 0;

int occupancy(const void* fn, int threads, size_t smem, int* per_sm) {
  STARM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  STARM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fn, threads, smem));
  if (*per_sm < 1) *per_sm = 1;
  return STARM_OK;
}

int make_plan(int64_t m, int64_t p, int64_t count, int64_t nslices, int job, bool have_s, Plan* pl) {
  Plan g{};
  g.L = m > p ? m : p;
  g.n = m < p ? m : p;
  g.transposed = m < p;
  g.LP = round_up(g.L, RCH);
  g.NP = round_up(g.n, BW);
  if (g.NP < GW) g.NP = GW;
  g.RP = round_up(g.NP, RCH);
  g.ns = 1;
  while (g.ns < g.n) g.ns <<= 1;
  g.jsmem = jacobi_smem_bytes(g.ns);
  g.bidiag = g_tune_mode >= 1 && g.LP <= QR_MAX_LP;
  {
    const size_t fixed = sizeof(QrSmemFixed) + size_t(BW) * size_t(g.LP + 36) * sizeof(double);
    const size_t ring = size_t(GW) * XS * sizeof(double);
    g.qr_stages = 2;
    // after the panel: the streaming updates' y, z and per-warp rings, or
    // (aliased) the team updates' Y partials + stages, or the load ring
    auto smem_for = [&](int nt, bool two, int team_yb = 0) {
      const size_t extra = size_t(g.qr_stages) * ring;
      size_t w = (size_t(QR_YZ_DOUBLES) + size_t(nt / 32) * (two ? WREG : WREG1)) * sizeof(double);
      const size_t team = team_yb == 2   ? size_t(TEAM_SMEM_DOUBLES) * sizeof(double)
                          : team_yb == 1 ? size_t(TEAM_SMEM_DOUBLES1) * sizeof(double)
                                         : 0;
      if (team > w) w = team;
      return fixed + (w > extra ? w : extra);
    };
    const size_t cap = size_t(227 * 1024);
    // 16 warps (single-stage rings) when they fit next to the panel, else 8
    // warps with two-stage rings when those fit, else one stage
    int nt = g_reduce_threads;
    if (nt == 0) nt = smem_for(512, false) <= cap ? 512 : 256;
    if (nt == 512 && smem_for(512, false) > cap) nt = 256;
    g.reduce_nt = nt;
    g.wtwo = smem_for(nt, true) <= cap;
    // team updates (256 threads): two Y-partial buffers when they fit, one
    // (an extra team barrier per group) for tall panels (c3: LP = 1024)
    g.team_yb = 0;
    if (nt == 256) g.team_yb = smem_for(nt, g.wtwo, 2) <= cap ? 2 : (smem_for(nt, g.wtwo, 1) <= cap ? 1 : 0);
    if (g_team_off) g.team_yb = 0;
    g.rsmem = smem_for(nt, g.wtwo, g.team_yb);
    if (g.rsmem > cap) g.bidiag = false;  // panel does not fit: Jacobi path
  }
  // Without the bidiagonal path the state-keeping jobs degrade to the plain
  // ones (the Jacobi kernel recomputes).
  if (!g.bidiag && job == STARM_SVD_VALUES_STATE) job = STARM_SVD_VALUES;
  if (!g.bidiag && job == STARM_SVD_TRUNCATED_STATE) job = STARM_SVD_TRUNCATED;
  g.job = job;
  g.by_slice = job == STARM_SVD_VALUES_STATE || job == STARM_SVD_TRUNCATED_STATE;
  if (g.by_slice) count = nslices;  // state for every slice, indexed by slice
  g.count = count;
  g.wantv = job == STARM_SVD_FULL || job == STARM_SVD_TRUNCATED || job == STARM_SVD_TRUNCATED_STATE;
  g.use_qr = false;  // the Jacobi fallback works on X directly
  g.run_jacobi = !g.bidiag;
  g.logs = g.bidiag && job != STARM_SVD_VALUES;
  g.run_front = g.bidiag && job != STARM_SVD_TRUNCATED_STATE;
  g.run_vec = g.bidiag && g.wantv;
  // (the state-keeping truncated job always receives the values pass's s,
  //  so its workspace has exactly the values-state layout)
  g.internal_s = g.wantv && !have_s && !g.by_slice;
  g.bsmem = size_t(g.n + BW) * HB * sizeof(double);
  g.hb_gmem = g_tune_mode == 2 || g.bsmem > size_t(216 * 1024);
  // too large for one SM but each half fits: the 2-CTA cluster kernel
  // (STARM_BULGE_CLUSTER=0 keeps the global-memory window for A/B runs)
  const size_t half = size_t((g.n + BW + 1) / 2) * HB * sizeof(double);
  g.hb_cluster = g.hb_gmem && g_tune_mode != 2 && half <= size_t(216 * 1024) && g_bulge_cluster &&
                 3 * hb_warps(g.n, 24) >= hb_kmax(g.n);  // (one active sweep per warp)
  g.hb_threads = 32 * hb_warps(g.n, g.hb_cluster ? 24 : (g.hb_gmem ? 32 : 16));
  if (g.hb_gmem) g.bsmem = 0;
  if (g.hb_cluster) {
    g.hb_gmem = false;
    g.bsmem = half;
  }
  int dev = 0, sms = 0, per = 0;
  STARM_CUDA_TRY(cudaGetDevice(&dev));
  STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  auto clampc = [&](int64_t v) { return int(v < 1 ? 1 : (v > count ? count : v)); };
  int rc;
  if (g.run_jacobi) {
    rc = g.wantv ? occupancy((const void*)svd_jacobi_kernel<true>, TPB, g.jsmem, &per)
                 : occupancy((const void*)svd_jacobi_kernel<false>, TPB, g.jsmem, &per);
    if (rc) return rc;
    g.slots_j = clampc(int64_t(sms) * per);
  }
  if (g.logs) {
    rc = occupancy((const void*)svd_vecout_kernel, TPB, g.jsmem, &per);
    if (rc) return rc;
    g.slots_v = clampc(int64_t(sms) * per);
    g.slots_j = g.slots_v;  // vecout uses the X slots
    g.slots_t = clampc(int64_t(sms) * 8);  // CGS2 warps (one per slice)
    g.bt_g = 8;  // vectors (warps) per back-transform CTA
    while (g.bt_g > 1 && bt_smem(g.n, g.bt_g) > size_t(200 * 1024)) --g.bt_g;
    g.tsmem = bt_smem(g.n, g.bt_g);
    rc = occupancy((const void*)svd_backtransform_kernel<true>, 32 * g.bt_g, g.tsmem, &per);
    if (!rc) rc = occupancy((const void*)svd_backtransform_kernel<false>, 32 * g.bt_g, g.tsmem, &per);
    if (rc) return rc;
    g.btw = per;  // back-transform CTAs per SM
    const int64_t work = count * g.n;
    const int64_t iicap = int64_t(sms) * g_ii_per_sm;
    g.ii_threads = int(work < iicap ? work : iicap);
    g.ii_threads = int(round_up(g.ii_threads < 1 ? 1 : g.ii_threads, 128));  // whole blocks
    g.hhcap = (g.n >= 3 ? (g.n - 2) : 1) * hb_kmax(g.n) * HLOG;
  }
  if (g.bidiag) {
    rc = g.reduce_nt == 512 ? occupancy((const void*)svd_reduce_kernel<512, false>, 512, g.rsmem, &per)
                            : occupancy((const void*)svd_reduce_kernel<256, false>, 256, g.rsmem, &per);
    if (rc) return rc;
    g.slots_r = clampc(int64_t(sms) * per);
    if (const char* e = getenv("STARM_REDUCE_SLOTS")) {  // experiment: fewer slices in flight
      const int v = atoi(e);
      if (v >= 1 && v < g.slots_r) g.slots_r = v;
    }
    if (g.hb_cluster) {
      STARM_CUDA_TRY(cudaFuncSetAttribute((const void*)svd_bulge_cluster_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(g.bsmem)));
      g.slots_b = clampc(int64_t(sms) / 2);  // clusters (one CTA per SM, two per cluster)
    } else {
      rc = occupancy(g.hb_gmem ? (const void*)svd_bulge_kernel<true> : (const void*)svd_bulge_kernel<false>,
                     g.hb_threads, g.bsmem, &per);
      if (rc) return rc;
      g.slots_b = clampc(int64_t(sms) * per);
    }
    int64_t bb = (count * g.n + 127) / 128;
    g.bisect_blocks = int(bb < int64_t(sms) * 16 ? bb : int64_t(sms) * 16);
    if (g.bisect_blocks < 1) g.bisect_blocks = 1;
  }
  const int64_t xslots = g.slots_j > g.slots_r ? g.slots_j : g.slots_r;
  size_t off = 256;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  g.off_x = take(size_t(xslots) * g.LP * g.NP * sizeof(double));
  g.off_w = take(g.wantv && g.run_jacobi ? size_t(g.slots_j) * g.RP * g.NP * sizeof(double) : 0);
  g.off_r = take(0);
  g.off_f = take(size_t(count) * 4);
  g.off_band = take(g.bidiag ? size_t(count) * (BW + 1) * g.NP * sizeof(double) : 0);
  g.off_de = take(g.bidiag ? size_t(count) * 2 * g.NP * sizeof(double) : 0);
  g.off_s = take(g.internal_s ? size_t(nslices) * g.n * sizeof(double) : 0);
  const size_t npan = size_t(g.NP / BW);
  g.off_rv = take(g.logs ? size_t(count) * npan * (BW * g.NP + BW * BW) * sizeof(double) : 0);
  g.off_rcs = take(g.logs ? size_t(count) * g.hhcap * sizeof(double) : 0);
  g.off_rcol = take(g.hb_gmem ? size_t(g.slots_b) * (g.n + BW) * HB * sizeof(double) : 0);
  g.off_rcnt = take(0);
  g.off_vsel = take(g.logs ? size_t(count) * g.RP * g.NP * sizeof(double) : 0);
  g.off_ii = take(g.logs ? size_t(g.ii_threads) * 6 * 2 * g.NP * sizeof(double) : 0);
  // blocked back-transformation (n > 400, the DMMA LQ-panel range): T of
  // every 16-sweep block per slice, 32 or 16 resident vectors per CTA
  g.bt_kb = 0;
  g.bt_nblk = 0;
  if (g.logs && g.n > 400 && g_bt_blocked) {
    auto btsm = [&](int kb) { return bt_blocked_smem(g.n, kb); };
    // measured: c4 (n = 512, 32 vectors / 4 warps per CTA) 238 -> 172 ms against the
    // per-warp kernel; c3 (n = 1024: only 16 vectors / 2 warps fit) 26 -> 55 ms,
    // so the 16-vector form is not used
    g.bt_kb = btsm(32) <= size_t(200 * 1024) ? 32 : 0;
    if (g.bt_kb) g.bt_nblk = bt_nblocks(g.n);
  }
  g.off_tlog = take(g.bt_kb ? size_t(count) * g.bt_nblk * BW * BW * sizeof(double) : 0);
  g.total = off;
  *pl = g;
  return STARM_OK;
}

// TSQR route for tall-skinny slices whose panel does not fit in shared memory
// (L padded > QR_MAX_LP, n <= 256): row blocks of BR = 1024 rows are reduced
// to their R factors (svd_tsqr_kernel) into a stacked SP x n matrix per slice
// (SP = ceil(L / BR) * NP <= QR_MAX_LP), the bidiagonal path runs on that, and
// vecout forms the left vectors from the original slices.  Workspace: the
// inner plan's layout first (so a state-keeping pair sees the same offsets),
// then S, the block-QR X slots and the vecout X slots.
struct TsqrPlan {
  bool on = false;
  int64_t BR = 0, nbk = 0, SP = 0, LPo = 0, blk_L = 0;
  int slots_q = 0;
  Plan inner{}, blk{};
  size_t off_S = 0, off_q = 0, off_vx = 0, total = 0;
};

int make_tsqr_plan(int64_t m, int64_t p, int64_t count, int64_t nslices, int job, bool have_s,
                   TsqrPlan* tp) {
  TsqrPlan t{};
  const int64_t L = m > p ? m : p, n = m < p ? m : p;
  const int64_t LP0 = round_up(L, RCH);
  if (g_tune_mode >= 1 && g_tune_mode != 3 && LP0 > QR_MAX_LP && n <= 256) {
    t.BR = 1024;
    t.nbk = (L + t.BR - 1) / t.BR;
    int64_t NP = round_up(n, BW);
    if (NP < GW) NP = GW;
    t.SP = t.nbk * NP;
    if (t.SP <= QR_MAX_LP && t.SP > n) {
      int rc = make_plan(t.SP, n, count, nslices, job, have_s, &t.inner);
      if (rc != STARM_OK) return rc;
      rc = make_plan(t.BR, n, count, nslices, STARM_SVD_VALUES, false, &t.blk);
      if (rc != STARM_OK) return rc;
      if (t.inner.bidiag && t.blk.bidiag && t.blk.reduce_nt == 256) {
        int dev = 0, sms = 0, per = 0;
        STARM_CUDA_TRY(cudaGetDevice(&dev));
        STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        rc = occupancy((const void*)svd_tsqr_kernel<256>, 256, t.blk.rsmem, &per);
        if (rc != STARM_OK) return rc;
        const int64_t items = t.inner.count * t.nbk;
        t.slots_q = int(int64_t(sms) * per < items ? int64_t(sms) * per : items);
        if (t.slots_q < 1) t.slots_q = 1;
        t.on = true;
        t.blk_L = L;
        t.LPo = LP0;
        size_t off = (t.inner.total + 255) & ~size_t(255);
        auto take = [&](size_t bytes) {
          const size_t o = off;
          off += (bytes + 255) & ~size_t(255);
          return o;
        };
        t.off_S = take(size_t(nslices) * t.SP * n * sizeof(double));
        t.off_q = take(size_t(t.slots_q) * t.blk.LP * t.blk.NP * sizeof(double));
        const bool vec = t.inner.run_vec || t.inner.by_slice;
        t.off_vx = take(vec ? size_t(t.inner.slots_v) * LP0 * t.inner.NP * sizeof(double) : 0);
        t.total = off;
      }
    }
  }
  *tp = t;
  return STARM_OK;
}

}  // namespace
}  // namespace starm

using namespace starm;

extern "C" size_t starm_svd_workspace_bytes(int64_t m, int64_t p, int64_t nslices, int64_t count,
                                            int job) {
  if (m < 1 || p < 1 || nslices < 1) return 0;
  if (count < 1 || count > nslices) count = nslices;
  TsqrPlan tp;
  if (make_tsqr_plan(m, p, count, nslices, job, false, &tp) != STARM_OK) return 0;
  if (tp.on) return tp.total;
  Plan pl;
  if (make_plan(m, p, count, nslices, job, false, &pl) != STARM_OK) return 0;
  return pl.total;
}

extern "C" int starm_svd_tune(int max_inner, int max_sweeps, int mode, int stats) {
  if (max_inner > 0) g_tune_inner = max_inner;
  if (max_sweeps > 0) g_tune_sweeps = max_sweeps;
  if (mode >= 0) g_tune_mode = mode;
  if (stats >= 0) g_stats_on = stats;
  return STARM_OK;
}

extern "C" int starm_svd_stats(unsigned long long* host16, int reset) {
  STARM_CUDA_TRY(cudaDeviceSynchronize());
  STARM_CUDA_TRY(cudaMemcpyFromSymbol(host16, g_stats, sizeof(unsigned long long) * 16));
  if (reset) {
    unsigned long long z[16] = {0};
    STARM_CUDA_TRY(cudaMemcpyToSymbol(g_stats, z, sizeof(z)));
  }
  return STARM_OK;
}

namespace starm {
namespace {
// Library-owned side stream + events per device for the chunked bulge /
// sigma overlap (created on first use, never destroyed).
// The fork ... join enqueue sequence of one call holds `mu`, so host threads
// running SVDs on different streams of one device cannot interleave their
// event records / waits on the shared side stream.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, ev[16] = {};
  std::mutex mu;
};
std::mutex g_side_mu;
SideStream g_side[64];

SideStream* side_stream() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_side_mu);
  SideStream& x = g_side[dev];
  if (!x.s) {
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
    for (auto& e : x.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return &x;
}
}  // namespace
}  // namespace starm

namespace starm {
namespace {
// Left-vector source for the TSQR route: vecout forms U from the original
// slices (X V / sigma) while everything else ran on the stacked R factors.
struct VecOverride {
  const double* A;
  int64_t m, p, L, LP;
  int transposed;
  double* xslots;
};

int svd_core(const double* ahat, int64_t m, int64_t p, int64_t nslices, const int64_t* slice_ids,
             int64_t count, int job, double* s, double* u, double* v, const int64_t* ranks,
             const int64_t* u_off, const int64_t* g_off, double* u_data, double* g_data,
             int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st,
             unsigned long long* counters, const VecOverride* vo) {
  Plan pl;
  int rc = make_plan(m, p, count, nslices, job, s != nullptr, &pl);
  if (rc != STARM_OK) return rc;
  STARM_CHECK_ARG(ws_bytes >= pl.total, "svd: workspace too small (%zu < %zu)", ws_bytes, pl.total);
  char* base = reinterpret_cast<char*>(ws);

  SvdParams P{};
  P.A = ahat;
  P.m = m;
  P.p = p;
  P.N = nslices;
  P.ids = slice_ids;
  P.count = count;
  P.job = pl.job == STARM_SVD_TRUNCATED_STATE ? STARM_SVD_TRUNCATED
          : pl.job == STARM_SVD_VALUES_STATE  ? STARM_SVD_VALUES
                                              : pl.job;
  P.s = pl.internal_s ? reinterpret_cast<double*>(base + pl.off_s) : s;
  P.u = u;
  P.v = v;
  P.ranks = ranks;
  P.u_off = u_off;
  P.g_off = g_off;
  P.u_data = u_data;
  P.g_data = g_data;
  P.status = status;
  P.counter = counters;
  P.xslots = reinterpret_cast<double*>(base + pl.off_x);
  P.wslots = reinterpret_cast<double*>(base + pl.off_w);
  P.rbuf = nullptr;
  P.flags = reinterpret_cast<int32_t*>(base + pl.off_f);
  P.bandbuf = reinterpret_cast<double*>(base + pl.off_band);
  P.qr_stages = pl.qr_stages;
  P.debuf = reinterpret_cast<double*>(base + pl.off_de);
  P.L = pl.L;
  P.n = pl.n;
  P.LP = pl.LP;
  P.NP = pl.NP;
  P.RP = pl.RP;
  P.transposed = pl.transposed;
  P.use_qr = pl.use_qr;
  P.bidiag = pl.bidiag;
  P.wtwo = pl.wtwo;
  P.team_yb = pl.team_yb;
  P.lo = 0;
  P.hi = count;
  P.cctr = 2;
  P.by_slice = pl.by_slice;
  P.hbbuf = reinterpret_cast<double*>(base + pl.off_rcol);
  P.stats = g_stats_on;
  // Jacobi convergence: every |cos(x_i, x_j)| <= L * eps (LAPACK dgesvj uses M*EPS).
  P.tol = double(pl.L > 32 ? pl.L : 32) * DBL_EPSILON;
  P.max_sweeps = g_tune_sweeps;
  P.max_inner = g_tune_inner;
  if (pl.logs) {
    P.rvlog = reinterpret_cast<double*>(base + pl.off_rv);
    P.hhlog = reinterpret_cast<double*>(base + pl.off_rcs);
    P.hhcap = pl.hhcap;
    P.vsel = reinterpret_cast<double*>(base + pl.off_vsel);
    P.iiscr = reinterpret_cast<double*>(base + pl.off_ii);
    P.btw = pl.btw;
  }
  if (pl.run_front) {
    // Few slices (at most half the SMs): a cluster of 2 / 4 / 8 CTAs per slice
    // splits the trailing updates (team path only).  STARM_REDUCE_CLUSTER=0
    // keeps one CTA per slice (A/B runs).  A launch of several waves whose
    // last wave fills at most half the SMs (c3: 512 slices = 3 waves of 148
    // + 68) runs that remainder as a second launch on clusters.
    int dev = 0, sms = 0;
    STARM_CUDA_TRY(cudaGetDevice(&dev));
    STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool can_cluster = pl.reduce_nt == 256 && pl.team_yb > 0 && g_reduce_cluster;
    auto launch_reduce = [&](int64_t lo, int64_t hi) -> int {
      if (lo >= hi) return STARM_OK;
      SvdParams Pr = P;
      Pr.rlo = lo;
      Pr.rhi = hi;
      const int64_t cnt = hi - lo;
      int csz = 1;
      if (can_cluster)
        while (csz < g_reduce_cluster_max && cnt * int64_t(2 * csz) <= int64_t(sms)) csz *= 2;
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute at[1];
      if (csz > 1) {
        STARM_CUDA_TRY(cudaFuncSetAttribute((const void*)svd_reduce_kernel<256, true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.rsmem)));
        // halve the cluster until the device can co-schedule at least one
        // (a partitioned or smaller GPU may not place 8 CTAs of this size)
        for (; csz > 1; csz /= 2) {
          cfg.gridDim = dim3(unsigned(cnt * csz), 1, 1);
          cfg.blockDim = dim3(256, 1, 1);
          cfg.dynamicSmemBytes = pl.rsmem;
          cfg.stream = st;
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = unsigned(csz);
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          int nclusters = 0;
          if (cudaOccupancyMaxActiveClusters(&nclusters, svd_reduce_kernel<256, true>, &cfg) == cudaSuccess &&
              nclusters >= 1)
            break;
          (void)cudaGetLastError();
        }
      }
      if (csz > 1) {
        STARM_CUDA_TRY(cudaLaunchKernelEx(&cfg, svd_reduce_kernel<256, true>, Pr));
      } else if (pl.reduce_nt == 512) {
        svd_reduce_kernel<512, false><<<pl.slots_r, 512, pl.rsmem, st>>>(Pr);
      } else {
        svd_reduce_kernel<256, false><<<pl.slots_r, 256, pl.rsmem, st>>>(Pr);
      }
      STARM_LAUNCH_CHECK();
      return STARM_OK;
    };
    {
      const int64_t rem = count % pl.slots_r;
      const bool split = can_cluster && count > pl.slots_r && pl.slots_r == sms && rem > 0 &&
                         2 * rem <= int64_t(sms);
      int rcl = launch_reduce(0, split ? count - rem : count);
      if (rcl) return rcl;
      if (split) {
        rcl = launch_reduce(count - rem, count);
        if (rcl) return rcl;
      }
    }
    if (g_tune_mode == 3) return STARM_OK;
    // Bulge chase and sigma in NCH slice chunks: sigma of chunk c (FP64-pipe
    // bound, no shared memory) runs on a side stream next to the bulge chase
    // of chunk c + 1 (latency bound, one CTA per SM); fork / join by events,
    // so stream capture sees an ordinary fork-join.
    const int nch = count >= 4 * int64_t(pl.slots_b) ? 4 : 1;
    SideStream* ss = nch > 1 ? side_stream() : nullptr;
    if (nch > 1 && !ss) return STARM_CUDA;
    std::unique_lock<std::mutex> side_lock;
    if (ss) side_lock = std::unique_lock<std::mutex>(ss->mu);
    if (ss) {
      STARM_CUDA_TRY(cudaEventRecord(ss->fork, st));
      STARM_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    }
    // chunk sizes in whole waves of the one-CTA-per-SM bulge chase (c2:
    // 296, 296, 296, 136 = 7 waves, where four equal chunks of 256 take 8),
    // which also leaves the smallest chunk's sigma as the exposed tail
    const int64_t per = round_up(ceil_div(count, nch), int64_t(pl.slots_b));
    for (int c = 0; c < nch; ++c) {
      SvdParams Pc = P;
      Pc.lo = per * c < count ? per * c : count;
      Pc.hi = per * (c + 1) < count ? per * (c + 1) : count;
      Pc.cctr = nch > 1 ? 8 + c : 2;
      if (Pc.lo >= Pc.hi) continue;
      if (pl.hb_cluster) svd_bulge_cluster_kernel<<<2 * pl.slots_b, pl.hb_threads, pl.bsmem, st>>>(Pc);
      else if (pl.hb_gmem) svd_bulge_kernel<true><<<pl.slots_b, pl.hb_threads, 0, st>>>(Pc);
      else svd_bulge_kernel<false><<<pl.slots_b, pl.hb_threads, pl.bsmem, st>>>(Pc);
      STARM_LAUNCH_CHECK();
      if (ss) {
        STARM_CUDA_TRY(cudaEventRecord(ss->ev[c], st));
        STARM_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->ev[c], 0));
        // beside the bulge chase: at most BISECT_SIDE_PER_SM blocks per SM, so
        // the next chunk's bulge CTA (27 K registers) always finds room
        // instead of queueing behind a register file full of bisection warps
        const int side = pl.bisect_blocks < g_bisect_side_blocks ? pl.bisect_blocks : g_bisect_side_blocks;
        svd_bisect_kernel<<<side, 128, 0, ss->s>>>(Pc);
      } else {
        svd_bisect_kernel<<<pl.bisect_blocks, 128, 0, st>>>(Pc);
      }
      STARM_LAUNCH_CHECK();
    }
    if (ss) {
      STARM_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
      STARM_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
    }
  }
  if (pl.run_vec) {
    {
      // scratch placement by the number of vectors (device-side count): the
      // shared-memory launch for few vectors, the global-scratch one otherwise
      int dev = 0, sms = 0;
      STARM_CUDA_TRY(cudaGetDevice(&dev));
      STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const size_t per = size_t(6 * 2 * pl.NP + 2) * sizeof(double);
      int tpc = int((216 * 1024) / per);
      tpc = tpc > 8 ? 8 : tpc;  // (215 registers per thread: at most 9 warps)
      const int64_t slots = int64_t(tpc) * sms;
      svd_bdvec_count_kernel<<<1, 256, 0, st>>>(P);
      STARM_LAUNCH_CHECK();
      if (tpc >= 1) {
        STARM_CUDA_TRY(cudaFuncSetAttribute(svd_bdvec_smem_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(per * tpc)));
        svd_bdvec_smem_kernel<<<sms, 32 * tpc, per * tpc, st>>>(P, count * pl.n, slots);
        STARM_LAUNCH_CHECK();
      }
      svd_bdvec_kernel<<<pl.ii_threads / 128, 128, 0, st>>>(P, count * pl.n, tpc >= 1 ? slots : 0);
      STARM_LAUNCH_CHECK();
    }
    STARM_LAUNCH_CHECK();
    if (pl.RP <= 1024 && !g_orth_warp) {
      const size_t osm = orth_smem(pl.RP);
      int dev = 0, sms = 0;
      STARM_CUDA_TRY(cudaGetDevice(&dev));
      STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      STARM_CUDA_TRY(cudaFuncSetAttribute(svd_orth_block_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(osm)));
      int per = int((227 * 1024) / (osm + 1024));
      per = per < 1 ? 1 : (per > 4 ? 4 : per);
      int64_t grid = int64_t(sms) * per;
      if (grid > count) grid = count;
      svd_orth_block_kernel<<<unsigned(grid), 256, osm, st>>>(P);
    } else {
      svd_orth_kernel<<<pl.slots_t, 32, 0, st>>>(P);
    }
    STARM_LAUNCH_CHECK();
    {
      // one CTA per (slice, group of bt_g vectors); groups beyond a slice's
      // rank exit at once
      int64_t blocks = count * ((pl.n + pl.bt_g - 1) / pl.bt_g);
      int dev = 0, sms = 0;
      STARM_CUDA_TRY(cudaGetDevice(&dev));
      STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const int64_t cap = int64_t(sms) * pl.btw * 8;
      if (blocks > cap) blocks = cap;
      // LQ panels on DMMA over blocks of 32 (n <= 636) or 16 (n <= 1276) vectors
      // for n > 400 (measured: c4 n = 512 truncated pass 762 -> 733 ms, c3 n =
      // 1024 420 -> 409 ms); below that the separate launch costs more than
      // the per-warp panels inside the back-transformation (c2 n = 361: +0.34 ms)
      const int lkb = (g_lq_warp || pl.n <= 400) ? 0
                      : (lq_smem(pl.n, 32) <= size_t(200 * 1024) ? 32
                         : (lq_smem(pl.n, 16) <= size_t(200 * 1024) ? 16 : 0));
      if (lkb && pl.bt_kb) {
        double* tlog = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + pl.off_tlog);
        const int64_t warps = count * pl.bt_nblk;
        int64_t tb = (warps + 3) / 4;
        if (tb > int64_t(sms) * 16) tb = int64_t(sms) * 16;
        svd_bt_tlog_kernel<<<unsigned(tb), 128, 0, st>>>(P, tlog, pl.bt_nblk);
        STARM_LAUNCH_CHECK();
        const size_t bsm = bt_blocked_smem(pl.n, pl.bt_kb);
        auto bk = pl.bt_kb == 32 ? svd_bt_blocked_kernel<32> : svd_bt_blocked_kernel<16>;
        STARM_CUDA_TRY(cudaFuncSetAttribute(bk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bsm)));
        int per = int((227 * 1024) / (bsm + 1024));
        per = per < 1 ? 1 : (per > 4 ? 4 : per);
        int64_t bb = count * ((pl.n + pl.bt_kb - 1) / pl.bt_kb);
        if (bb > int64_t(sms) * per) bb = int64_t(sms) * per;
        bk<<<unsigned(bb), pl.bt_kb * 4, bsm, st>>>(P, tlog, pl.bt_nblk);
      } else {
        // L2 prefetch of the sweep records 16 sweeps ahead (STARM_BT_PREFETCH=0:
        // the plain instantiation, for A/B runs)
        int pf = 1;
        if (const char* e = getenv("STARM_BT_PREFETCH")) pf = e[0] == '1';
        // (measured, ncu, with both instantiations in the library: c2 0.65 -> 0.52 ms,
        // c1 0.42 -> 0.35 ms; the timing of this kernel is sensitive to code layout)
        if (pf) svd_backtransform_kernel<true><<<unsigned(blocks), 32 * pl.bt_g, pl.tsmem, st>>>(P, pl.bt_g, lkb == 0);
        else svd_backtransform_kernel<false><<<unsigned(blocks), 32 * pl.bt_g, pl.tsmem, st>>>(P, pl.bt_g, lkb == 0);
      }
      STARM_LAUNCH_CHECK();
      if (lkb) {
        const size_t lsm = lq_smem(pl.n, lkb);
        auto lk = lkb == 32 ? svd_lqapply_kernel<32> : svd_lqapply_kernel<16>;
        STARM_CUDA_TRY(cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(lsm)));
        int per = int((227 * 1024) / (lsm + 1024));
        per = per < 1 ? 1 : (per > 4 ? 4 : per);
        int64_t lb = count * ((pl.n + lkb - 1) / lkb);
        if (lb > int64_t(sms) * per) lb = int64_t(sms) * per;
        lk<<<unsigned(lb), 256, lsm, st>>>(P);
      }
    }
    STARM_LAUNCH_CHECK();
    SvdParams Pv = P;
    if (vo) {
      Pv.A = vo->A;
      Pv.m = vo->m;
      Pv.p = vo->p;
      Pv.L = vo->L;
      Pv.LP = vo->LP;
      Pv.transposed = vo->transposed;
      Pv.xslots = vo->xslots;
    }
    svd_vecout_kernel<<<pl.slots_v, TPB, pl.jsmem, st>>>(Pv);
    STARM_LAUNCH_CHECK();
  }
  if (pl.run_jacobi) {
    if (pl.wantv)
      svd_jacobi_kernel<true><<<pl.slots_j, TPB, pl.jsmem, st>>>(P);
    else
      svd_jacobi_kernel<false><<<pl.slots_j, TPB, pl.jsmem, st>>>(P);
    STARM_LAUNCH_CHECK();
  }
  return STARM_OK;
}
}  // namespace
}  // namespace starm

extern "C" int starm_svd_f64(const double* ahat, int64_t m, int64_t p, int64_t nslices,
                             const int64_t* slice_ids, int64_t count, int job, double* s,
                             double* u, double* v, const int64_t* ranks, const int64_t* u_off,
                             const int64_t* g_off, double* u_data, double* g_data,
                             int32_t* status, void* ws, size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(m >= 1 && p >= 1 && nslices >= 1, "svd: extents must be positive");
  STARM_CHECK_ARG(job >= STARM_SVD_VALUES && job <= STARM_SVD_TRUNCATED_STATE,
                  "svd: unknown job %d", job);
  const int64_t r = m < p ? m : p;
  if (r > MAX_NS) {
    set_error("svd: min(m, p) = %lld exceeds the supported %d", (long long)r, MAX_NS);
    return STARM_UNSUPPORTED;
  }
  STARM_CHECK_ARG(ahat && status && ws, "svd: null pointer");
  STARM_CHECK_ARG((job != STARM_SVD_VALUES && job != STARM_SVD_VALUES_STATE) || s,
                  "svd: values jobs need s");
  STARM_CHECK_ARG(job != STARM_SVD_FULL || (s && u && v), "svd: full job needs s, u, v");
  STARM_CHECK_ARG((job != STARM_SVD_TRUNCATED && job != STARM_SVD_TRUNCATED_STATE) ||
                      (ranks && u_off && g_off && u_data && g_data),
                  "svd: truncated jobs need ranks, offsets and packed buffers");
  STARM_CHECK_ARG(job != STARM_SVD_TRUNCATED_STATE || s,
                  "svd: the state-keeping truncated job needs the values pass's s");
  STARM_CHECK_ARG(job != STARM_SVD_VALUES_STATE || !slice_ids,
                  "svd: the state-keeping values job factors every slice (slice_ids must be NULL)");
  if (!slice_ids) count = nslices;
  cudaStream_t st = as_stream(stream);
  unsigned long long* counters = reinterpret_cast<unsigned long long*>(ws);
  reset_status_kernel<<<1, 32, 0, st>>>(status, counters);
  STARM_LAUNCH_CHECK();
  if (count <= 0) return STARM_OK;
  TsqrPlan tp;
  int rc = make_tsqr_plan(m, p, count, nslices, job, s != nullptr, &tp);
  if (rc != STARM_OK) return rc;
  if (!tp.on)
    return svd_core(ahat, m, p, nslices, slice_ids, count, job, s, u, v, ranks, u_off, g_off, u_data,
                    g_data, status, ws, ws_bytes, st, counters, nullptr);
  STARM_CHECK_ARG(ws_bytes >= tp.total, "svd: workspace too small (%zu < %zu)", ws_bytes, tp.total);
  char* base = reinterpret_cast<char*>(ws);
  double* S = reinterpret_cast<double*>(base + tp.off_S);
  {  // first level: R of every row block into S
    SvdParams Q{};
    Q.A = ahat;
    Q.m = m;
    Q.p = p;
    Q.N = nslices;
    Q.ids = slice_ids;
    Q.count = count;
    Q.status = status;
    Q.counter = counters;
    Q.xslots = reinterpret_cast<double*>(base + tp.off_q);
    Q.qr_stages = tp.blk.qr_stages;
    Q.L = tp.blk_L;
    Q.n = tp.blk.n;
    Q.LP = tp.blk.LP;
    Q.NP = tp.blk.NP;
    Q.RP = tp.blk.RP;
    Q.transposed = m < p;
    Q.wtwo = tp.blk.wtwo;
    Q.team_yb = tp.blk.team_yb;
    Q.stats = g_stats_on;
    svd_tsqr_kernel<256><<<tp.slots_q, 256, tp.blk.rsmem, st>>>(Q, S, tp.BR, tp.nbk, tp.SP);
    STARM_LAUNCH_CHECK();
  }
  const int64_t n = m < p ? m : p;
  VecOverride vo{ahat, m, p, tp.blk_L, tp.LPo, m < p ? 1 : 0,
                 reinterpret_cast<double*>(base + tp.off_vx)};
  return svd_core(S, tp.SP, n, nslices, slice_ids, count, job, s, u, v, ranks, u_off, g_off, u_data,
                  g_data, status, ws, tp.inner.total, st, counters, &vo);
}
