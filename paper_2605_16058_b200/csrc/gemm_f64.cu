// K1 / K11: batched column-major FP64 GEMM on the DMMA tensor pipe.
//
//   C_b (M x N) = A_b (M x K) * B_b (K x N),  b in [0, batch)
//
// Used for the mode-k TTM (ttm.py:113-135: the row-major view
// dst[b] = mat @ src[b] is, column-major, dst_b = src_b * mat^T with
// M = rows, K = inner, N = out_cols) and for the facewise product of
// starm_product (tsvdm.py:205-216).
//
// Tiling: CTA tile 128 x 64 x 16, 8 warps (4 along M x 2 along N), warp
// tile 32 x 32 = 4 x 4 DMMA.8x8x4 accumulators (64 FP64 registers).  A 4-stage
// cp.async ring stages A[k][m] (m contiguous, +4 pad) and B[n][k] (k
// contiguous, +4 pad) tiles; the pads make every fragment load
// bank-conflict free (half-warp lanes (g,t) hit banks 8t+2g / 8g+2t).
// Grid: x = (M-tile, N-tile) with the N-tile fastest so all CTAs that read
// one A panel run back to back and A streams from HBM once; z = batch.
#include "common.cuh"

namespace starm {
namespace {

// c3-shaped transform (scripts/run_gemm.py): BK 16 x 4 stages 32.3 TFLOP/s
// (2 CTAs / SM), 16 x 3 30.0, 32 x 2 32.0, 32 x 3 25.5 (1 CTA / SM)
#ifndef GEMM_BK
#define GEMM_BK 16
#endif
#ifndef GEMM_STAGES
#define GEMM_STAGES 4
#endif
constexpr int BM = 128, BN = 64, BK = GEMM_BK, STAGES = GEMM_STAGES, THREADS = 256;
constexpr int APAD = BM + 4;  // doubles per k-row of the A tile
constexpr int BPAD = BK + 4;  // doubles per n-column of the B tile
constexpr int A_TILE = BK * APAD;
constexpr int B_TILE = BN * BPAD;
constexpr size_t SMEM_BYTES = size_t(STAGES) * (A_TILE + B_TILE) * sizeof(double);

struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  int64_t M, N, K, lda, ldb, ldc, sA, sB, sC;
  int64_t tiles_n;
  int64_t tiles;           // tiles per batch block
  // ERR epilogue (K10 fused into the writer of C): reference tensor E with
  // ld ldc; per CTA {sum (E - C)^2, sum E^2} over the tile -> epart[2 tile]
  const double* E;
  double* epart;
};

template <int VA, int VB>
__device__ __forceinline__ void load_stage(const GemmArgs& g, const double* A, const double* B,
                                           double* As, double* Bs, int64_t m0, int64_t n0,
                                           int64_t k0) {
  const int tid = threadIdx.x;
  // A tile: BK columns x BM contiguous rows.
  constexpr int A_CHUNKS = BK * BM / VA;
#pragma unroll
  for (int c = tid; c < A_CHUNKS; c += THREADS) {
    const int kk = c / (BM / VA);
    const int mm = (c % (BM / VA)) * VA;
    const int64_t gm = m0 + mm, gk = k0 + kk;
    double* dst = As + kk * APAD + mm;
    const bool in = (gk < g.K) && (gm < g.M);
    const double* src = in ? A + gm + gk * g.lda : A;
    if (VA == 2) {
      // M is even on this path, so a chunk is either fully in or fully out.
      cp_async16(dst, src, in ? 16 : 0);
    } else {
      cp_async8(dst, src, in ? 8 : 0);
    }
  }
  // B tile: BN columns x BK contiguous k.
  constexpr int B_CHUNKS = BN * BK / VB;
#pragma unroll
  for (int c = tid; c < B_CHUNKS; c += THREADS) {
    const int nn = c / (BK / VB);
    const int kk = (c % (BK / VB)) * VB;
    const int64_t gn = n0 + nn, gk = k0 + kk;
    double* dst = Bs + nn * BPAD + kk;
    const bool in = (gn < g.N) && (gk < g.K);
    const double* src = in ? B + gk + gn * g.ldb : B;
    if (VB == 2) {
      cp_async16(dst, src, in ? 16 : 0);
    } else {
      cp_async8(dst, src, in ? 8 : 0);
    }
  }
}

template <int VA, int VB, bool ERR>
__global__ void __launch_bounds__(THREADS, 2) gemm_f64_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_TILE;

  const int64_t tile = blockIdx.x;
  const int64_t tn = tile % g.tiles_n;
  const int64_t tm = tile / g.tiles_n;
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const int64_t b = blockIdx.z;
  const double* A = g.A + b * g.sA;
  const double* B = g.B + b * g.sB;
  double* C = g.C + b * g.sC;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t KT = (g.K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage<VA, VB>(g, A, B, As + s * A_TILE, Bs + s * B_TILE, m0, n0, s * BK);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      const int slot = int(nk % STAGES);
      if (nk < KT) load_stage<VA, VB>(g, A, B, As + slot * A_TILE, Bs + slot * B_TILE, m0, n0, nk * BK);
      cp_async_commit();
    }
    const int slot = int(kt % STAGES);
    const double* as = As + slot * A_TILE + wm * 32 + gq;
    const double* bs = Bs + slot * B_TILE + (wn * 32 + gq) * BPAD + tq;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(k4 * 4 + tq) * APAD + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * BPAD + k4 * 4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: D[g][2t], D[g][2t+1] -> C(m, n), C(m, n+1); with ERR also the
  // tile's error partials against E (fixed reduction order: deterministic).
  double sd = 0.0, sa = 0.0;
  // ERR: the E values of a half are loaded before its first store to C (C
  // and E may alias as far as the compiler knows, so loads interleaved
  // with the stores would each wait out a full memory latency); two halves
  // of 16 values: 32 at once would spill at 128 registers.
#pragma unroll
  for (int ih = 0; ih < 4; ih += 2) {
    double ev[ERR ? 2 : 1][4][2];
    if (ERR) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t m = m0 + wm * 32 + (ih + i) * 8 + gq;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t n = n0 + wn * 32 + j * 8 + 2 * tq;
          ev[i][j][0] = (m < g.M && n < g.N) ? __ldg(g.E + m + n * g.ldc) : 0.0;
          ev[i][j][1] = (m < g.M && n + 1 < g.N) ? __ldg(g.E + m + (n + 1) * g.ldc) : 0.0;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t m = m0 + wm * 32 + (ih + i) * 8 + gq;
      if (m >= g.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t n = n0 + wn * 32 + j * 8 + 2 * tq;
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          if (n + e2 < g.N) {
            const double v = acc[ih + i][j][e2];
            C[m + (n + e2) * g.ldc] = v;
            if (ERR) {
              const double e = ev[i][j][e2];
              const double d = e - v;
              sd = fma(d, d, sd);
              sa = fma(e, e, sa);
            }
          }
        }
      }
    }
  }
  if (ERR) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sd += __shfl_xor_sync(0xffffffffu, sd, o);
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
    }
    __syncthreads();  // the stage buffers are free: reuse them for the warp partials
    if (lane == 0) {
      smem[2 * warp] = sd;
      smem[2 * warp + 1] = sa;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < THREADS / 32; ++w) {
        s0 += smem[2 * w];
        s1 += smem[2 * w + 1];
      }
      g.epart[2 * tile] = s0;
      g.epart[2 * tile + 1] = s1;
    }
  }
}

// Persistent over the tiles of one batch block: CTA c runs tiles c, c + grid,
// ... and the cp.async ring runs straight across tile boundaries (k-tile
// stream s = (tile index, kt)), so the loads of the next tile are in flight
// while the epilogue of the current one stores C (and, with ERR, reads E).
// With a short K (the fused reconstruction has K = nnz = 64: four k-tiles)
// a per-tile prologue would otherwise expose a full memory latency per tile.
template <int VA, int VB, bool ERR>
__global__ void __launch_bounds__(THREADS, 2) gemm_f64_pers_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double wred[2 * THREADS / 32];
  double* As = smem;
  double* Bs = smem + STAGES * A_TILE;

  const int64_t b = blockIdx.z;
  const double* A = g.A + b * g.sA;
  const double* B = g.B + b * g.sB;
  double* C = g.C + b * g.sC;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;

  const int64_t KT = (g.K + BK - 1) / BK;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t mine = first < g.tiles ? (g.tiles - first + stride - 1) / stride : 0;
  const int64_t total = mine * KT;  // k-tile steps of this CTA

  // prefetch cursor (k-tile step ps of the stream): tile origin and kt kept
  // incrementally (no divisions in the loop)
  int64_t ps = 0, pkt = 0, ptile = first;
  int64_t pm0 = (ptile / g.tiles_n) * BM, pn0 = (ptile % g.tiles_n) * BN;
  auto issue = [&]() {
    if (ps < total) {
      const int slot = int(ps % STAGES);
      load_stage<VA, VB>(g, A, B, As + slot * A_TILE, Bs + slot * B_TILE, pm0, pn0, pkt * BK);
      ++ps;
      if (++pkt == KT) {
        pkt = 0;
        ptile += stride;
        pm0 = (ptile / g.tiles_n) * BM;
        pn0 = (ptile % g.tiles_n) * BN;
      }
    }
    cp_async_commit();
  };
  // L2 prefetch of the E values of a tile (read by its epilogue).
  auto prefetch_e = [&](int64_t tile) {
    const int64_t m0 = (tile / g.tiles_n) * BM, n0 = (tile % g.tiles_n) * BN;
#pragma unroll
    for (int q = 0; q < BM * BN / 16 / THREADS; ++q) {  // one prefetch per 128-byte line
      const int e = threadIdx.x + q * THREADS;
      const int64_t m = m0 + (e % (BM / 16)) * 16, n = n0 + e / (BM / 16);
      if (m < g.M && n < g.N) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.E + m + n * g.ldc));
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue();

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int64_t kt = 0, ti = 0;
  if (ERR && mine > 0) prefetch_e(first);
  for (int64_t s = 0; s < total; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue();
    const int slot = int(s % STAGES);
    const double* as = As + slot * A_TILE + wm * 32 + gq;
    const double* bs = Bs + slot * B_TILE + (wn * 32 + gq) * BPAD + tq;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(k4 * 4 + tq) * APAD + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * BPAD + k4 * 4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (++kt < KT) continue;
    kt = 0;

    // Epilogue of tile ti: D[g][2t], D[g][2t+1] -> C(m, n), C(m, n+1); with
    // ERR also the tile's error partials against E (fixed reduction order:
    // deterministic).
    const int64_t tile = first + ti * stride;
    ++ti;
    const int64_t m0 = (tile / g.tiles_n) * BM, n0 = (tile % g.tiles_n) * BN;
    if (ERR && ti < mine) prefetch_e(first + ti * stride);
    double sd = 0.0, sa = 0.0;
    // ERR: the E values of a half are loaded before its first store to C (C
    // and E may alias as far as the compiler knows, so loads interleaved
    // with the stores would each wait out a full memory latency); two halves
    // of 16 values: 32 at once would spill at 128 registers.
#pragma unroll
    for (int ih = 0; ih < 4; ih += 2) {
      double ev[ERR ? 2 : 1][4][2];
      if (ERR) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int64_t m = m0 + wm * 32 + (ih + i) * 8 + gq;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t n = n0 + wn * 32 + j * 8 + 2 * tq;
            ev[i][j][0] = (m < g.M && n < g.N) ? __ldg(g.E + m + n * g.ldc) : 0.0;
            ev[i][j][1] = (m < g.M && n + 1 < g.N) ? __ldg(g.E + m + (n + 1) * g.ldc) : 0.0;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t m = m0 + wm * 32 + (ih + i) * 8 + gq;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t n = n0 + wn * 32 + j * 8 + 2 * tq;
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            if (n + e2 < g.N) {
              const double v = acc[ih + i][j][e2];
              C[m + (n + e2) * g.ldc] = v;
              if (ERR) {
                const double e = ev[i][j][e2];
                const double d = e - v;
                sd = fma(d, d, sd);
                sa = fma(e, e, sa);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (ERR) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sd += __shfl_xor_sync(0xffffffffu, sd, o);
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
      }
      if (lane == 0) {
        wred[2 * warp] = sd;
        wred[2 * warp + 1] = sa;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < THREADS / 32; ++w) {
          s0 += wred[2 * w];
          s1 += wred[2 * w + 1];
        }
        g.epart[2 * tile] = s0;
        g.epart[2 * tile + 1] = s1;
      }
      // (the next write of wred is behind the next step's CTA barrier)
    }
  }
  cp_async_wait<0>();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int VA, int VB, bool ERR = false>
int launch_t(const GemmArgs& g, int64_t batch, cudaStream_t st) {
  // the attribute is per device: set it on every launch (a cheap host call)
  STARM_CUDA_TRY(cudaFuncSetAttribute(gemm_f64_kernel<VA, VB, ERR>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(SMEM_BYTES)));
  STARM_CUDA_TRY(cudaFuncSetAttribute(gemm_f64_pers_kernel<VA, VB, ERR>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(SMEM_BYTES)));
  const int64_t tiles = g.tiles_n * ceil_div(g.M, BM);
  // persistent: at most 2 CTAs per SM per batch block when there is a single
  // block (batched launches keep one tile per CTA: the blocks fill the GPU)
  int dev = 0, sms = 148;
  STARM_CUDA_TRY(cudaGetDevice(&dev));
  STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // ... and only for a short K, where the per-tile prologue is what costs: a
  // long K loop hides it, and one tile per CTA lets the hardware stagger the
  // CTAs (c3's K = 512 transform: 17.0 ms against 19.4 ms persistent)
  const bool persistent = batch == 1 && g.K <= 8 * BK && tiles > 2 * int64_t(sms);
  const int64_t gx = persistent ? 2 * int64_t(sms) : tiles;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    GemmArgs gb = g;
    gb.tiles = tiles;
    gb.A += b0 * g.sA;
    gb.B += b0 * g.sB;
    gb.C += b0 * g.sC;
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    dim3 grid(unsigned(gx), 1, unsigned(nb));
    if (persistent) gemm_f64_pers_kernel<VA, VB, ERR><<<grid, THREADS, SMEM_BYTES, st>>>(gb);
    else gemm_f64_kernel<VA, VB, ERR><<<grid, THREADS, SMEM_BYTES, st>>>(gb);
    STARM_LAUNCH_CHECK();
  }
  return STARM_OK;
}

}  // namespace

// Internal entry point shared by the C ABI functions below and other .cu files.
int gemm_f64(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K,
             int64_t lda, int64_t ldb, int64_t ldc, int64_t sA, int64_t sB, int64_t sC,
             int64_t batch, cudaStream_t st) {
  if (M <= 0 || N <= 0 || batch <= 0) return STARM_OK;
  if (K <= 0) {
    // Empty contraction: C = 0.
    for (int64_t b = 0; b < batch; ++b)
      STARM_CUDA_TRY(cudaMemset2DAsync(C + b * sC, size_t(ldc) * 8, 0, size_t(M) * 8, size_t(N), st));
    return STARM_OK;
  }
  GemmArgs g{A, B, C, M, N, K, lda, ldb, ldc, sA, sB, sC, ceil_div(N, BN), 0, nullptr, nullptr};
  const bool va = (M % 2 == 0) && (lda % 2 == 0) && (sA % 2 == 0) && aligned16(A);
  const bool vb = (K % 2 == 0) && (ldb % 2 == 0) && (sB % 2 == 0) && aligned16(B);
  if (va && vb) return launch_t<2, 2>(g, batch, st);
  if (va) return launch_t<2, 1>(g, batch, st);
  if (vb) return launch_t<1, 2>(g, batch, st);
  return launch_t<1, 1>(g, batch, st);
}

// C = A * B (batch 1) with the K10 error partials of E against C fused into
// the epilogue: epart[2 t], epart[2 t + 1] for tile t < gemm_f64_tiles(M, N).
int64_t gemm_f64_tiles(int64_t M, int64_t N) { return ceil_div(M, BM) * ceil_div(N, BN); }

int gemm_f64_err(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K,
                 int64_t lda, int64_t ldb, int64_t ldc, const double* E, double* epart,
                 cudaStream_t st) {
  if (M <= 0 || N <= 0) return STARM_OK;
  STARM_CHECK_ARG(K > 0, "gemm_f64_err: empty contraction");
  GemmArgs g{A, B, C, M, N, K, lda, ldb, ldc, 0, 0, 0, ceil_div(N, BN), 0, E, epart};
  const bool va = (M % 2 == 0) && (lda % 2 == 0) && aligned16(A);
  const bool vb = (K % 2 == 0) && (ldb % 2 == 0) && aligned16(B);
  if (va && vb) return launch_t<2, 2, true>(g, 1, st);
  if (va) return launch_t<2, 1, true>(g, 1, st);
  if (vb) return launch_t<1, 2, true>(g, 1, st);
  return launch_t<1, 1, true>(g, 1, st);
}

}  // namespace starm

extern "C" int starm_ttm_f64(const double* src, const double* mat, double* dst, int64_t rows,
                             int64_t inner, int64_t batch, int64_t out_cols, void* stream) {
  STARM_CHECK_ARG(rows >= 1 && inner >= 1 && batch >= 1 && out_cols >= 1,
                  "ttm: extents must be positive (rows=%lld inner=%lld batch=%lld out_cols=%lld)",
                  (long long)rows, (long long)inner, (long long)batch, (long long)out_cols);
  STARM_CHECK_ARG(src && mat && dst, "ttm: null pointer");
  // dst_b (rows x out_cols) = src_b (rows x inner) * B, B(l, j) = mat[j*inner + l].
  return starm::gemm_f64(src, mat, dst, rows, out_cols, inner, rows, inner, rows, rows * inner, 0,
                         rows * out_cols, batch, starm::as_stream(stream));
}

// The same product restricted to the fibre block [f0, f0 + nf) of a 3-way
// tensor (batch 1): src and dst are the FULL tensors' buffers (leading
// dimension `rows`), so the transform can run block by block, e.g. behind the
// host-to-device copy of each block (the reference's np.matmul in
// ttm.py:113-135 needs the whole unfolding in memory).
extern "C" int starm_ttm_block_f64(const double* src, const double* mat, double* dst, int64_t rows,
                                   int64_t inner, int64_t out_cols, int64_t f0, int64_t nf,
                                   void* stream) {
  STARM_CHECK_ARG(rows >= 1 && inner >= 1 && out_cols >= 1 && f0 >= 0 && nf >= 0 && f0 + nf <= rows,
                  "ttm block: bad extents (rows=%lld inner=%lld out_cols=%lld f0=%lld nf=%lld)",
                  (long long)rows, (long long)inner, (long long)out_cols, (long long)f0, (long long)nf);
  if (nf == 0) return STARM_OK;
  STARM_CHECK_ARG(src && mat && dst, "ttm block: null pointer");
  return starm::gemm_f64(src + f0, mat, dst + f0, nf, out_cols, inner, rows, inner, rows, 0, 0, 0, 1,
                         starm::as_stream(stream));
}

extern "C" int starm_facewise_gemm_f64(const double* a, const double* b, double* c, int64_t m,
                                       int64_t p, int64_t l, int64_t nslices, void* stream) {
  STARM_CHECK_ARG(m >= 1 && p >= 1 && l >= 1 && nslices >= 1,
                  "facewise gemm: extents must be positive");
  STARM_CHECK_ARG(a && b && c, "facewise gemm: null pointer");
  return starm::gemm_f64(a, b, c, m, l, p, m, p, m, m * p, p * l, m * l, nslices,
                         starm::as_stream(stream));
}
