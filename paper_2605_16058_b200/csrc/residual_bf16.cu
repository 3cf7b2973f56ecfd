// K1c: the reference operator's residual on the 5th-generation tensor cores.
//
// The reference applies its DCT as a dense product with the matrix that
// dct_matrix() builds in float64 (transforms.py:75-91, ttm.py:113-135).
// Those entries carry rounding of the cos ARGUMENT, up to ~2.4e-14 for
// n = 1024 -- structured, not random, so on c2 it leaks the strong seasonal
// slices into the noise slices and moves their sigma by up to 4e-10
// (VERDICT r1 weak #1).  The fast path computes the exact DCT-II by FFT
// (dct.cu) and then adds the residual operator Delta = M_ref - M_exact:
//
//     dst_b  +=  2^-e * (Delta_bf16 @ bf16(src_b))          (b < batch)
//
// Delta is tiny, so its product needs only ~3 significant digits: bf16
// operands with fp32 accumulation bring the result within a few u of the
// reference's own fl(M_ref @ x) (numpy emulation on c2-shaped fibres:
// noise-slice sigma from 1.5e-10 to 2e-13 of the reference).  The product is
// a (fibres x n) x (n x n) GEMM: 545 GFLOP on c2, which the DMMA pipe would
// need 17 ms for; tcgen05 kind::f16 does it at HBM speed of the epilogue.
//
// Kernels
//  * residual_pack_kernel: src (column-major: element (f, k) of batch b at
//    b*rows*n + k*rows + f) -> ws bf16 [b][f][k] (k contiguous, fibre rows
//    padded to a multiple of 128 and zero-filled): the K-major operand layout.
//  * residual_gemm_kernel: persistent, warp-specialised, 1 CTA / SM.
//      warp 0      TMA producer: 128 x 64 fibre tile and 256 x 64 Delta tile
//                  per stage (SWIZZLE_128B), 4-stage mbarrier ring;
//      warp 1      TMEM allocation (512 columns = two 128 x 256 fp32
//                  accumulators) and the single-thread tcgen05.mma issuer
//                  (M = 128 fibres, N = 256 outputs, K = 16 per instruction);
//      warps 2..9  epilogue: tcgen05.ld of 32 columns per chunk, then
//                  dst += 2^-e * acc with 32 coalesced f64 loads in flight per
//                  thread (warp w reads TMEM lanes 32*(w%4).., columns half
//                  (w-2)/4).  The two accumulators let the epilogue of tile
//                  i overlap the MMAs of tile i+1.
#include "common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <mutex>

namespace starm {
namespace {

constexpr int RB_M = 128;          // fibres per tile (TMEM lanes)
constexpr int RB_N = 256;          // transform outputs per tile
constexpr int RB_K = 64;           // k per stage: one 128-byte swizzle row of bf16
constexpr int RB_STAGES = 4;
constexpr int RB_EPI_WARPS = 8;
constexpr int RB_THREADS = 32 * (2 + RB_EPI_WARPS);
constexpr int RB_A_BYTES = RB_M * RB_K * 2;     // 16 KB
constexpr int RB_B_BYTES = RB_N * RB_K * 2;     // 32 KB
constexpr int RB_STAGE_BYTES = RB_A_BYTES + RB_B_BYTES;
constexpr size_t RB_SMEM = size_t(RB_STAGES) * RB_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t RB_TMEM_COLS = 512;

// ---------------------------------------------------------------- PTX

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 in, fp32 accumulate.
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// UMMA shared-memory descriptor: K-major operand, SWIZZLE_128B, rows of
// 128 bytes, 8-row groups 1024 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;              // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;      // SBO
  d |= uint64_t(1) << 46;              // descriptor version
  d |= uint64_t(2) << 61;              // SWIZZLE_128B
  return d;
}
// Instruction descriptor: c = f32, a = b = bf16, both K-major, M = 128, N = 256.
constexpr uint32_t RB_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(RB_N >> 3) << 17) |
                              (uint32_t(RB_M >> 4) << 24);

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- kernels

__global__ void __launch_bounds__(256) residual_pack_kernel(const double* __restrict__ src,
                                                            uint16_t* __restrict__ ws,
                                                            int64_t rows, int64_t n,
                                                            int64_t rows_pad, int64_t pitch) {
  __shared__ float tile[64][65];
  const int tid = threadIdx.x;
  const int64_t f0 = int64_t(blockIdx.x) * 64;
  const int64_t k0 = int64_t(blockIdx.y) * 64;
  const int64_t b = blockIdx.z;
  const double* s = src + b * rows * n;
#pragma unroll 4
  for (int i = tid; i < 64 * 64; i += 256) {
    const int kk = i >> 6, ff = i & 63;
    const int64_t f = f0 + ff;
    double x = f < rows ? __ldg(s + (k0 + kk) * pitch + f) : 0.0;
    // bf16 saturates instead of overflowing: a fibre beyond 3.4e38 keeps the
    // FFT result's accuracy (its residual term is then inexact, not inf)
    x = fmin(fmax(x, -3.0e38), 3.0e38);
    tile[kk][ff] = float(x);
  }
  __syncthreads();
  uint16_t* o = ws + (b * rows_pad + f0) * n + k0;
  for (int i = tid; i < 64 * 8; i += 256) {
    const int ff = i >> 3, kc = (i & 7) * 8;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(tile[kc + 2 * j][ff], tile[kc + 2 * j + 1][ff]);
      w[j] = *reinterpret_cast<const uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(o + int64_t(ff) * n + kc) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

struct ResidualArgs {
  double* dst;
  int64_t rows, n, rows_pad, batch;
  int64_t nout;            // output columns (n, or the selected rows of Delta)
  int64_t tiles, nblk;     // total tiles, output blocks per fibre block (nout padded / RB_N)
  double scale;            // 2^-e
};

__global__ void __launch_bounds__(RB_THREADS, 1)
    residual_gemm_kernel(const __grid_constant__ CUtensorMap map_x,
                         const __grid_constant__ CUtensorMap map_d, const ResidualArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RB_STAGES * RB_STAGE_BYTES);
  uint64_t* empty = full + RB_STAGES;
  uint64_t* tfull = empty + RB_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = int(g.n / RB_K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < RB_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], RB_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_d)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(RB_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
        const int fb = int(tile / g.nblk);
        const int nb = int(tile % g.nblk);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * RB_STAGE_BYTES;
          mbar_expect_tx(&full[s], RB_STAGE_BYTES);
          tma_load_2d(sa, &map_x, &full[s], kb * RB_K, fb * RB_M);
          tma_load_2d(sa + RB_A_BYTES, &map_d, &full[s], kb * RB_K, nb * RB_N);
          if (++s == RB_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * RB_N);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * RB_STAGE_BYTES);
          const uint32_t sb = sa + RB_A_BYTES;
#pragma unroll
          for (int k = 0; k < RB_K / 16; ++k)
            tc_mma_bf16(d_tmem, sw128_desc(sa + 32 * k), sw128_desc(sb + 32 * k), RB_IDESC,
                        uint32_t(kb | k));
          tc_commit(&empty[s]);
          if (++s == RB_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else {
    // epilogue warps
    const int q = warp & 3;                // TMEM lane quadrant this warp may read
    const int half = (warp - 2) >> 2;      // column half
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
      const int64_t fb = tile / g.nblk;
      const int64_t nb = tile % g.nblk;
      const int64_t grow = fb * RB_M;                  // padded global fibre row
      const int64_t b = grow / g.rows_pad;
      const int64_t f = grow - b * g.rows_pad + 32 * q + lane;
      const bool live = f < g.rows;
      double* out = g.dst + b * g.rows * g.nout + f;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < RB_N / 2; c += 32) {
        const int col = half * (RB_N / 2) + c;
        float v[32];
        tmem_ld32(tmem_base + (uint32_t(32 * q) << 16) + uint32_t(acc * RB_N + col), v);
        const int64_t col0 = nb * RB_N + col;
        if (live && col0 + 32 <= g.nout) {
          double* p = out + col0 * g.rows;
          double x[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] = p[int64_t(j) * g.rows];
#pragma unroll
          for (int j = 0; j < 32; ++j) p[int64_t(j) * g.rows] = fma(double(v[j]), g.scale, x[j]);
        } else if (live && col0 < g.nout) {   // last, partial block of selected columns
          double* p = out + col0 * g.rows;
          const int lim = int(g.nout - col0);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < lim) p[int64_t(j) * g.rows] = fma(double(v[j]), g.scale, p[int64_t(j) * g.rows]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(RB_TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- host

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_encode_mu;

int get_encoder() {
  std::lock_guard<std::mutex> lk(g_encode_mu);
  if (g_encode) return STARM_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  STARM_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return STARM_CUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return STARM_OK;
}

int make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
             uint32_t box_outer) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
    return STARM_CUDA;
  }
  return STARM_OK;
}

int64_t rows_padded(int64_t rows) { return round_up(rows, RB_M); }

}  // namespace
}  // namespace starm

using namespace starm;

extern "C" size_t starm_ttm_residual_workspace_bytes(int64_t rows, int64_t n, int64_t batch) {
  if (rows <= 0 || n <= 0 || batch <= 0) return 0;
  return size_t(rows_padded(rows)) * size_t(n) * size_t(batch) * 2;
}

namespace starm {
namespace {
// Pack (unless the DCT kernel already wrote the bf16 rows) + tcgen05 GEMM.
int residual_run(const double* pack_src, const uint16_t* delta_bf16, int log2_scale, double* dst,
                 int64_t rows, int64_t n, int64_t batch, const void* ws, cudaStream_t st,
                 int64_t nout = -1) {
  if (nout < 0) nout = n;
  const int64_t nout_pad = round_up(nout, RB_N);
  const int64_t rows_pad = rows_padded(rows);
  const int64_t total_rows = rows_pad * batch;
  STARM_CHECK_ARG(total_rows < (int64_t(1) << 31) && n <= 65536 && batch <= 65535,
                  "ttm residual: tensor too large for one launch");
  int rc = get_encoder();
  if (rc) return rc;
  if (pack_src) {
    dim3 grid(unsigned(rows_pad / 64), unsigned(n / 64), unsigned(batch));
    residual_pack_kernel<<<grid, 256, 0, st>>>(pack_src, static_cast<uint16_t*>(const_cast<void*>(ws)),
                                               rows, n, rows_pad, rows);
    STARM_LAUNCH_CHECK();
  }
  CUtensorMap map_x, map_d;
  rc = make_map(&map_x, ws, uint64_t(n), uint64_t(total_rows), RB_K, RB_M);
  if (rc) return rc;
  rc = make_map(&map_d, delta_bf16, uint64_t(n), uint64_t(nout_pad), RB_K, RB_N);
  if (rc) return rc;
  int dev = 0, sms = 148;
  STARM_CUDA_TRY(cudaGetDevice(&dev));
  STARM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // the attribute is per device: set it on every launch (cheap)
  STARM_CUDA_TRY(cudaFuncSetAttribute(residual_gemm_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(RB_SMEM)));
  ResidualArgs g;
  g.dst = dst;
  g.rows = rows;
  g.n = n;
  g.rows_pad = rows_pad;
  g.batch = batch;
  g.nout = nout;
  g.nblk = nout_pad / RB_N;
  g.tiles = (total_rows / RB_M) * g.nblk;
  g.scale = ldexp(1.0, -log2_scale);
  const int64_t grid = g.tiles < sms ? g.tiles : sms;
  residual_gemm_kernel<<<unsigned(grid), RB_THREADS, RB_SMEM, st>>>(map_x, map_d, g);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

int residual_args(const double* src, const uint16_t* delta_bf16, double* dst, int64_t n, void* ws,
                  size_t ws_bytes, int64_t rows, int64_t batch) {
  STARM_CHECK_ARG(src && delta_bf16 && dst && ws, "ttm residual: null pointer");
  STARM_CHECK_ARG(src != dst, "ttm residual: src and dst alias");
  if (n % RB_N != 0) {
    set_error("ttm residual: n = %lld must be a multiple of %d", (long long)n, RB_N);
    return STARM_UNSUPPORTED;
  }
  STARM_CHECK_ARG(ws_bytes >= size_t(rows_padded(rows)) * size_t(n) * size_t(batch) * 2,
                  "ttm residual: workspace too small");
  STARM_CHECK_ARG((reinterpret_cast<uintptr_t>(ws) & 127) == 0 &&
                      (reinterpret_cast<uintptr_t>(delta_bf16) & 127) == 0,
                  "ttm residual: workspace and Delta must be 128-byte aligned");
  return STARM_OK;
}
}  // namespace
}  // namespace starm

extern "C" int starm_ttm_residual_bf16(const double* src, const uint16_t* delta_bf16, int log2_scale,
                                       double* dst, int64_t rows, int64_t n, int64_t batch,
                                       void* ws, size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(rows >= 0 && n >= 0 && batch >= 0, "ttm residual: negative extent");
  if (rows == 0 || batch == 0 || n == 0) return STARM_OK;
  const int rc = residual_args(src, delta_bf16, dst, n, ws, ws_bytes, rows, batch);
  if (rc) return rc;
  return residual_run(src, delta_bf16, log2_scale, dst, rows, n, batch, ws, as_stream(stream));
}

extern "C" int starm_dct_residual_f64(const double* src, double* dst, int64_t rows, int64_t n,
                                      int64_t batch, int inverse, const uint16_t* delta_bf16,
                                      int log2_scale, void* ws, size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(rows >= 0 && n >= 0 && batch >= 0, "dct residual: negative extent");
  if (rows == 0 || batch == 0 || n == 0) return STARM_OK;
  int rc = residual_args(src, delta_bf16, dst, n, ws, ws_bytes, rows, batch);
  if (rc) return rc;
  if ((n & (n - 1)) != 0 || n > 4096) {
    set_error("dct residual: the fast path needs a power-of-two length in [256, 4096]");
    return STARM_UNSUPPORTED;
  }
  const cudaStream_t st = as_stream(stream);
  bool packed = false;
  rc = dct_launch(src, dst, rows, n, batch, inverse != 0, static_cast<uint16_t*>(ws),
                  rows_padded(rows), &packed, st);
  if (rc) return rc;
  return residual_run(packed ? nullptr : src, delta_bf16, log2_scale, dst, rows, n, batch, ws, st);
}

extern "C" int starm_dct_pack_f64(const double* src, double* dst, int64_t rows, int64_t n,
                                  int64_t batch, int inverse, void* ws, size_t ws_bytes,
                                  void* stream) {
  STARM_CHECK_ARG(rows >= 0 && n >= 0 && batch >= 0, "dct pack: negative extent");
  if (rows == 0 || batch == 0 || n == 0) return STARM_OK;
  STARM_CHECK_ARG(src && dst && ws && src != dst, "dct pack: null or aliased pointer");
  if ((n & (n - 1)) != 0 || n < RB_N || n > 4096) {
    set_error("dct pack: the fast path needs a power-of-two length in [256, 4096]");
    return STARM_UNSUPPORTED;
  }
  STARM_CHECK_ARG(ws_bytes >= starm_ttm_residual_workspace_bytes(rows, n, batch) &&
                      (reinterpret_cast<uintptr_t>(ws) & 127) == 0,
                  "dct pack: workspace too small or not 128-byte aligned");
  const cudaStream_t st = as_stream(stream);
  bool packed = false;
  int rc = dct_launch(src, dst, rows, n, batch, inverse != 0, static_cast<uint16_t*>(ws),
                      rows_padded(rows), &packed, st);
  if (rc || packed) return rc;
  const int64_t rows_pad = rows_padded(rows);
  dim3 grid(unsigned(rows_pad / 64), unsigned(n / 64), unsigned(batch));
  residual_pack_kernel<<<grid, 256, 0, st>>>(src, static_cast<uint16_t*>(ws), rows, n, rows_pad, rows);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

// Fibre block [f0, f0 + nf) of a (rows x n) tensor, transformed where it
// lies: src/dst/ws are the FULL tensor's buffers, so a caller can run the
// forward DCT block by block (e.g. behind the host-to-device copy of each
// block) and end with exactly the buffers starm_dct_pack_f64 leaves.
extern "C" int starm_dct_pack_block_f64(const double* src, double* dst, int64_t rows, int64_t n,
                                        int64_t f0, int64_t nf, void* ws, size_t ws_bytes,
                                        void* stream) {
  STARM_CHECK_ARG(rows >= 0 && n >= 0 && f0 >= 0 && nf >= 0 && f0 + nf <= rows,
                  "dct pack block: bad extents");
  if (nf == 0 || n == 0) return STARM_OK;
  STARM_CHECK_ARG(src && dst && ws && src != dst, "dct pack block: null or aliased pointer");
  if ((n & (n - 1)) != 0 || n < RB_N || n > 4096) {
    set_error("dct pack block: the fast path needs a power-of-two length in [256, 4096]");
    return STARM_UNSUPPORTED;
  }
  STARM_CHECK_ARG(f0 % RB_M == 0 && (f0 + nf == rows || nf % RB_M == 0),
                  "dct pack block: blocks must start and end on multiples of 128 fibres");
  STARM_CHECK_ARG(ws_bytes >= starm_ttm_residual_workspace_bytes(rows, n, 1) &&
                      (reinterpret_cast<uintptr_t>(ws) & 127) == 0,
                  "dct pack block: workspace too small or not 128-byte aligned");
  const cudaStream_t st = as_stream(stream);
  uint16_t* wsb = static_cast<uint16_t*>(ws) + f0 * n;
  bool packed = false;
  int rc = dct_launch(src + f0, dst + f0, nf, n, 1, false, wsb, rows_padded(nf), &packed, st, rows);
  if (rc || packed) return rc;
  const int64_t rows_pad = rows_padded(nf);
  dim3 grid(unsigned(rows_pad / 64), unsigned(n / 64), 1);
  residual_pack_kernel<<<grid, 256, 0, st>>>(src + f0, wsb, nf, n, rows_pad, rows);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

extern "C" int starm_residual_apply_f64(const void* ws, const uint16_t* delta_bf16, int log2_scale,
                                        double* dst, int64_t rows, int64_t n, int64_t nout,
                                        int64_t batch, void* stream) {
  STARM_CHECK_ARG(rows >= 0 && n >= 0 && nout >= 0 && batch >= 0, "residual apply: negative extent");
  if (rows == 0 || batch == 0 || n == 0 || nout == 0) return STARM_OK;
  STARM_CHECK_ARG(ws && delta_bf16 && dst, "residual apply: null pointer");
  if (n % RB_N != 0) {
    set_error("residual apply: n = %lld must be a multiple of %d", (long long)n, RB_N);
    return STARM_UNSUPPORTED;
  }
  STARM_CHECK_ARG((reinterpret_cast<uintptr_t>(ws) & 127) == 0 &&
                      (reinterpret_cast<uintptr_t>(delta_bf16) & 127) == 0,
                  "residual apply: operands must be 128-byte aligned");
  return residual_run(nullptr, delta_bf16, log2_scale, dst, rows, n, batch, ws, as_stream(stream),
                      nout);
}
