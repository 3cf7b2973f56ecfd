// K8 packed offsets, K9 facewise reconstruction, K10 error sums, and the
// C-ABI error plumbing.
#include <string.h>

#include <atomic>
#include <string>

#include "common.cuh"

namespace starm {

namespace {
thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

namespace {

// ---------------------------------------------------------------- offsets
// slicesvd.py:208-211 -- exclusive scans of ranks*m and ranks*p, one CTA.
__global__ void __launch_bounds__(1024) offsets_kernel(const int64_t* ranks, int64_t N, int64_t m,
                                                       int64_t p, int64_t* u_off, int64_t* g_off) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t chunk = (N + 1023) / 1024;
  const int64_t lo = t * chunk;
  const int64_t hi = lo + chunk < N ? lo + chunk : N;
  int64_t local = 0;
  for (int64_t i = lo; i < hi; ++i) local += ranks[i];
  part[t] = local;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < 1024; ++i) {
      const int64_t x = part[i];
      part[i] = acc;
      acc += x;
    }
  }
  __syncthreads();
  int64_t acc = part[t];
  if (t == 0) {
    u_off[0] = 0;
    g_off[0] = 0;
  }
  for (int64_t i = lo; i < hi; ++i) {
    acc += ranks[i];
    u_off[i + 1] = acc * m;
    g_off[i + 1] = acc * p;
  }
}

// ------------------------------------------------- facewise U_i G_i tiles
// chat_i (m x p) = U_i (m x k) * G_i (k x p), k = ranks[i] (0 -> zeros), on
// DMMA: 64 x 64 output tile per CTA, 8 warps of 32 x 16 (4 x 2 m8n8k4
// accumulators), K in chunks of 16 staged in shared memory with row stride
// 72 (= 8 mod 32: the (g, t) fragment lanes hit distinct banks).
constexpr int RT = 64, KC = 16, US = RT + 8;

// ids (optional): slot j of chat holds slice ids[j] (the compacted nonzero
// slices of the fused reconstruction); NULL: slot j = slice j.
__global__ void __launch_bounds__(256) unpack_kernel(const double* u_data, const double* g_data,
                                                     const int64_t* ranks, const int64_t* u_off,
                                                     const int64_t* g_off, int64_t m, int64_t p,
                                                     int64_t tiles_m, int64_t tiles_p,
                                                     double* chat, const int64_t* ids) {
  __shared__ double us[KC][US];  // us[k][row]
  __shared__ double gs[KC][US];  // gs[k][col]
  const int64_t per_slice = tiles_m * tiles_p;
  const int64_t slot = blockIdx.x / per_slice;
  const int64_t slice = ids ? ids[slot] : slot;
  const int64_t tile = blockIdx.x % per_slice;
  const int64_t m0 = (tile % tiles_m) * RT, p0 = (tile / tiles_m) * RT;
  const int64_t k = ranks[slice];
  const double* U = u_data + u_off[slice];
  const double* G = g_data + g_off[slice];
  double* C = chat + slot * m * p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;  // rows 32 wm .., cols 16 wn ..
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t k0 = 0; k0 < k; k0 += KC) {
    for (int e = threadIdx.x; e < KC * RT; e += 256) {
      const int kk = e / RT, rr = e % RT;  // U: consecutive threads, consecutive rows
      const int64_t row = m0 + rr, kx = k0 + kk;
      us[kk][rr] = (row < m && kx < k) ? U[row + kx * m] : 0.0;
      const int cc = e / KC, k2 = e % KC;  // G: consecutive threads, consecutive k
      const int64_t col = p0 + cc, ky = k0 + k2;
      gs[k2][cc] = (col < p && ky < k) ? G[ky + col * k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < KC; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = us[k4 + tq][32 * wm + 8 * i + gq];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = gs[k4 + tq][16 * wn + 8 * j + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884n(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + 32 * wm + 8 * i + gq;
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t col = p0 + 16 * wn + 8 * j + 2 * tq;
      if (col < p) C[row + col * m] = acc[i][j][0];
      if (col + 1 < p) C[row + (col + 1) * m] = acc[i][j][1];
    }
  }
}

// ------------------------------------------------------------- error sums
constexpr int ES_THREADS = 256, ES_BLOCKS = 148 * 4;

__global__ void __launch_bounds__(ES_THREADS) err_partial_kernel(const double* a, const double* b,
                                                                 int64_t count, double* part) {
  __shared__ double red[2][ES_THREADS / 32];
  double d2 = 0.0, a2 = 0.0;
  for (int64_t i = blockIdx.x * int64_t(ES_THREADS) + threadIdx.x; i < count;
       i += int64_t(ES_BLOCKS) * ES_THREADS) {
    const double x = a[i], y = b[i];
    const double d = x - y;
    d2 = fma(d, d, d2);
    a2 = fma(x, x, a2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][warp] = d2;
    red[1][warp] = a2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < ES_THREADS / 32; ++w) {
      s0 += red[0][w];
      s1 += red[1][w];
    }
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

// Fixed-order sum of nparts (d2, a2) partial pairs: each of 256 threads sums a
// contiguous run, then a fixed tree (deterministic for a given nparts).
__global__ void __launch_bounds__(256) err_final_kernel(const double* part, int64_t nparts,
                                                        double* out2) {
  __shared__ double red[2][256];
  const int64_t per = (nparts + 255) / 256;
  const int64_t lo = threadIdx.x * per, hi = lo + per < nparts ? lo + per : nparts;
  double s0 = 0.0, s1 = 0.0;
  for (int64_t b = lo; b < hi; ++b) {
    s0 += part[2 * b];
    s1 += part[2 * b + 1];
  }
  red[0][threadIdx.x] = s0;
  red[1][threadIdx.x] = s1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] += red[0][threadIdx.x + o];
      red[1][threadIdx.x] += red[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out2[0] = red[0][0];
    out2[1] = red[1][0];
  }
}

// B (K x n, column-major) of the fused reconstruction: B[i][t] = minv[t][ids[i]]
// (minv row-major n x n), i.e. the columns of M^-1 that meet a nonzero slice.
__global__ void gather_inverse_kernel(const double* minv, const int64_t* ids, int64_t K, int64_t n,
                                      double* B) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= K * n) return;
  const int64_t i = e % K, t = e / K;
  B[e] = minv[t * n + (ids ? ids[i] : i)];
}


// ------------------------------------------------------- pack from full
__global__ void pack_full_kernel(const double* s, const double* u, const double* v, int64_t m,
                                 int64_t p, int64_t r, const int64_t* ranks, const int64_t* u_off,
                                 const int64_t* g_off, double* u_data, double* g_data) {
  const int64_t i = blockIdx.x;
  const int64_t k = ranks[i];
  if (k == 0) return;
  const double* ui = u + i * m * r;
  const double* vi = v + i * p * r;
  const double* si = s + i * r;
  double* ud = u_data + u_off[i];
  double* gd = g_data + g_off[i];
  for (int64_t e = threadIdx.x; e < m * k; e += blockDim.x) ud[e] = ui[e];
  for (int64_t e = threadIdx.x; e < k * p; e += blockDim.x) {
    const int64_t j = e % k, c = e / k;
    gd[e] = si[j] * vi[c + j * p];
  }
}

__global__ void __launch_bounds__(256) tail_energy_kernel(const double* s, int64_t r, int64_t N,
                                                          int64_t rank, double* out2) {
  __shared__ double red[2][256];
  double tail = 0.0, tot = 0.0;
  for (int64_t e = threadIdx.x; e < r * N; e += 256) {
    const double x = s[e];
    const double sq = x * x;
    tot += sq;
    if (e % r >= rank) tail += sq;
  }
  red[0][threadIdx.x] = tail;
  red[1][threadIdx.x] = tot;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] += red[0][threadIdx.x + o];
      red[1][threadIdx.x] += red[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out2[0] = red[0][0];
    out2[1] = red[1][0];
  }
}

}  // namespace
}  // namespace starm

using namespace starm;

extern "C" int starm_pack_from_full_f64(const double* s, const double* u, const double* v,
                                        int64_t m, int64_t p, int64_t nslices,
                                        const int64_t* ranks, const int64_t* u_off,
                                        const int64_t* g_off, double* u_data, double* g_data,
                                        void* stream) {
  STARM_CHECK_ARG(m >= 1 && p >= 1 && nslices >= 1, "pack_from_full: bad extents");
  STARM_CHECK_ARG(s && u && v && ranks && u_off && g_off && u_data && g_data,
                  "pack_from_full: null pointer");
  STARM_CHECK_ARG(nslices < (int64_t(1) << 31), "pack_from_full: too many slices");
  const int64_t r = m < p ? m : p;
  pack_full_kernel<<<unsigned(nslices), 256, 0, as_stream(stream)>>>(s, u, v, m, p, r, ranks, u_off,
                                                                     g_off, u_data, g_data);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

extern "C" int starm_tail_energy_f64(const double* s, int64_t r, int64_t nslices, int64_t rank,
                                     double* out2, void* stream) {
  STARM_CHECK_ARG(r >= 1 && nslices >= 1 && rank >= 0, "tail_energy: bad extents");
  STARM_CHECK_ARG(s && out2, "tail_energy: null pointer");
  tail_energy_kernel<<<1, 256, 0, as_stream(stream)>>>(s, r, nslices, rank, out2);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

extern "C" int starm_abi_version(void) { return STARM_ABI_VERSION; }

extern "C" long long starm_launch_count_reset(void) { return g_launches.exchange(0); }

extern "C" size_t starm_last_error(char* buf, size_t len) {
  const std::string& e = g_last_error;
  if (buf && len) {
    const size_t n = e.size() < len - 1 ? e.size() : len - 1;
    memcpy(buf, e.data(), n);
    buf[n] = 0;
  }
  return e.size();
}

extern "C" int starm_pack_offsets(const int64_t* ranks, int64_t nslices, int64_t m, int64_t p,
                                  int64_t* u_off, int64_t* g_off, void* stream) {
  STARM_CHECK_ARG(nslices >= 0 && m >= 1 && p >= 1, "pack_offsets: bad extents");
  STARM_CHECK_ARG(u_off && g_off && (ranks || nslices == 0), "pack_offsets: null pointer");
  offsets_kernel<<<1, 1024, 0, as_stream(stream)>>>(ranks, nslices, m, p, u_off, g_off);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

extern "C" int starm_unpack_facewise_f64(const double* u_data, const double* g_data,
                                         const int64_t* ranks, const int64_t* u_off,
                                         const int64_t* g_off, int64_t m, int64_t p,
                                         int64_t nslices, double* chat, void* stream) {
  STARM_CHECK_ARG(m >= 1 && p >= 1 && nslices >= 1, "unpack: bad extents");
  STARM_CHECK_ARG(ranks && u_off && g_off && chat, "unpack: null pointer");
  const int64_t tm = ceil_div(m, RT), tp = ceil_div(p, RT);
  const int64_t blocks = tm * tp * nslices;
  STARM_CHECK_ARG(blocks < (int64_t(1) << 31), "unpack: grid too large");
  unpack_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(u_data, g_data, ranks, u_off,
                                                                 g_off, m, p, tm, tp, chat, nullptr);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

extern "C" size_t starm_error_sums_workspace_bytes(int64_t count) {
  (void)count;
  return size_t(2) * ES_BLOCKS * sizeof(double);
}

extern "C" int starm_error_sums_f64(const double* a, const double* b, int64_t count, double* out2,
                                    void* ws, size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(count >= 0, "error sums: bad count");
  STARM_CHECK_ARG(a && b && out2 && ws, "error sums: null pointer");
  STARM_CHECK_ARG(ws_bytes >= starm_error_sums_workspace_bytes(count), "error sums: workspace too small");
  double* part = reinterpret_cast<double*>(ws);
  cudaStream_t st = as_stream(stream);
  err_partial_kernel<<<ES_BLOCKS, ES_THREADS, 0, st>>>(a, b, count, part);
  STARM_LAUNCH_CHECK();
  err_final_kernel<<<1, 256, 0, st>>>(part, ES_BLOCKS, out2);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

// ------------------------------------------- K9 + inverse transform + K10
// Workspace: compacted slices (F x nnz), the gathered inverse columns
// (nnz x n), error partials (2 per GEMM tile, or per error block).
extern "C" size_t starm_reconstruct_workspace_bytes(int64_t m, int64_t p, int64_t n, int64_t nnz) {
  if (m < 1 || p < 1 || n < 1 || nnz < 0) return 0;
  const int64_t F = m * p;
  const int64_t tiles = gemm_f64_tiles(F, n);
  const int64_t parts = tiles > ES_BLOCKS ? tiles : ES_BLOCKS;
  return size_t(F * nnz + nnz * n + 2 * parts) * sizeof(double) + 256;
}

extern "C" int starm_reconstruct_f64(const double* u_data, const double* g_data,
                                     const int64_t* ranks, const int64_t* u_off,
                                     const int64_t* g_off, int64_t m, int64_t p, int64_t n,
                                     const int64_t* nz_ids, int64_t nnz, const double* minv,
                                     const double* a, double* out, double* err2, void* ws,
                                     size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(m >= 1 && p >= 1 && n >= 1 && nnz >= 0 && nnz <= n,
                  "reconstruct: bad extents (m=%lld p=%lld n=%lld nnz=%lld)", (long long)m,
                  (long long)p, (long long)n, (long long)nnz);
  STARM_CHECK_ARG(ranks && u_off && g_off && minv && out && ws, "reconstruct: null pointer");
  STARM_CHECK_ARG(!a || err2, "reconstruct: err2 is required with a");
  STARM_CHECK_ARG(ws_bytes >= starm_reconstruct_workspace_bytes(m, p, n, nnz),
                  "reconstruct: workspace too small");
  const cudaStream_t st = as_stream(stream);
  const int64_t F = m * p;
  double* chat = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  double* B = chat + F * nnz;
  double* part = B + nnz * n;
  if (nnz == 0) {  // every rank is zero: the reconstruction is 0
    STARM_CUDA_TRY(cudaMemsetAsync(out, 0, size_t(F * n) * sizeof(double), st));
    if (a) {
      err_partial_kernel<<<ES_BLOCKS, ES_THREADS, 0, st>>>(a, out, F * n, part);
      STARM_LAUNCH_CHECK();
      err_final_kernel<<<1, 256, 0, st>>>(part, ES_BLOCKS, err2);
      STARM_LAUNCH_CHECK();
    }
    return STARM_OK;
  }
  const int64_t tm = ceil_div(m, RT), tp = ceil_div(p, RT);
  const int64_t blocks = tm * tp * nnz;
  STARM_CHECK_ARG(blocks < (int64_t(1) << 31), "reconstruct: grid too large");
  unpack_kernel<<<unsigned(blocks), 256, 0, st>>>(u_data, g_data, ranks, u_off, g_off, m, p, tm, tp,
                                                 chat, nz_ids);
  STARM_LAUNCH_CHECK();
  gather_inverse_kernel<<<unsigned(ceil_div(nnz * n, 256)), 256, 0, st>>>(minv, nz_ids, nnz, n, B);
  STARM_LAUNCH_CHECK();
  // out (F x n, column-major = the (m, p, n) tensor) = chat_nz (F x nnz) * B
  if (a) {
    const int rc = gemm_f64_err(chat, B, out, F, n, nnz, F, nnz, F, a, part, st);
    if (rc) return rc;
    err_final_kernel<<<1, 256, 0, st>>>(part, gemm_f64_tiles(F, n), err2);
    STARM_LAUNCH_CHECK();
  } else {
    const int rc = starm_ttm_f64(chat, B, out, F, nnz, 1, n, stream);  // out = chat_nz * B
    if (rc) return rc;
  }
  return STARM_OK;
}

// ---------------------------------------------------------- float32 twins
// The reference upcasts float32 input to float64 on construction
// (tensor.py:87); on the device the upcast runs after an f32 H2D (half the
// PCIe bytes of the f64 tensor).
namespace starm {
namespace {
__global__ void upcast_kernel(const float* __restrict__ src, double* __restrict__ dst, int64_t count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    dst[i] = double(src[i]);
}
__global__ void downcast_kernel(const double* __restrict__ src, float* __restrict__ dst, int64_t count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    dst[i] = float(src[i]);
}
unsigned stream_grid(int64_t count) {
  const int64_t b = ceil_div(count, 256);
  return unsigned(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}
}  // namespace
}  // namespace starm

extern "C" int starm_upcast_f32_f64(const float* src, double* dst, int64_t count, void* stream) {
  STARM_CHECK_ARG(count >= 0, "upcast: negative count");
  if (count == 0) return STARM_OK;
  STARM_CHECK_ARG(src && dst, "upcast: null pointer");
  upcast_kernel<<<stream_grid(count), 256, 0, as_stream(stream)>>>(src, dst, count);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

extern "C" size_t starm_ttm_f32_workspace_bytes(int64_t rows, int64_t inner, int64_t batch,
                                                int64_t out_cols) {
  if (rows < 1 || inner < 1 || batch < 1 || out_cols < 1) return 0;
  return size_t(rows * batch * (inner + out_cols) + inner * out_cols) * sizeof(double) + 256;
}

extern "C" int starm_ttm_f32(const float* src, const float* mat, float* dst, int64_t rows,
                             int64_t inner, int64_t batch, int64_t out_cols, void* ws,
                             size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(rows >= 1 && inner >= 1 && batch >= 1 && out_cols >= 1,
                  "ttm: extents must be positive (rows=%lld inner=%lld batch=%lld out_cols=%lld)",
                  (long long)rows, (long long)inner, (long long)batch, (long long)out_cols);
  STARM_CHECK_ARG(src && mat && dst && ws, "ttm: null pointer");
  STARM_CHECK_ARG(ws_bytes >= starm_ttm_f32_workspace_bytes(rows, inner, batch, out_cols),
                  "ttm f32: workspace too small");
  const cudaStream_t st = as_stream(stream);
  double* s64 = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  double* d64 = s64 + rows * batch * inner;
  double* m64 = d64 + rows * batch * out_cols;
  upcast_kernel<<<stream_grid(rows * batch * inner), 256, 0, st>>>(src, s64, rows * batch * inner);
  STARM_LAUNCH_CHECK();
  upcast_kernel<<<stream_grid(inner * out_cols), 256, 0, st>>>(mat, m64, inner * out_cols);
  STARM_LAUNCH_CHECK();
  const int rc = starm_ttm_f64(s64, m64, d64, rows, inner, batch, out_cols, stream);
  if (rc) return rc;
  downcast_kernel<<<stream_grid(rows * batch * out_cols), 256, 0, st>>>(d64, dst, rows * batch * out_cols);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

// ------------------------------------------------------ per-slice energy
// f[i] = sum of squares of slice i (slice_elems contiguous doubles), one CTA
// per slice, fixed reduction order (deterministic).  sigma_max(slice)^2 <=
// f[i]: the bound the pruned tolerance path uses.
namespace starm {
namespace {
__global__ void __launch_bounds__(256) slice_energy_kernel(const double* __restrict__ a,
                                                           int64_t elems, int64_t pitch,
                                                           double* __restrict__ f) {
  __shared__ double red[256];
  const double* x = a + int64_t(blockIdx.x) * pitch;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t i = threadIdx.x;
  for (; i + 768 < elems; i += 1024) {
    const double x0 = x[i], x1 = x[i + 256], x2 = x[i + 512], x3 = x[i + 768];
    acc[0] = fma(x0, x0, acc[0]);
    acc[1] = fma(x1, x1, acc[1]);
    acc[2] = fma(x2, x2, acc[2]);
    acc[3] = fma(x3, x3, acc[3]);
  }
  for (; i < elems; i += 256) acc[0] = fma(x[i], x[i], acc[0]);
  red[threadIdx.x] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) f[blockIdx.x] = red[0];
}
}  // namespace
}  // namespace starm

extern "C" int starm_slice_energy_f64(const double* a, int64_t slice_elems, int64_t nslices,
                                      double* f_out, void* stream) {
  STARM_CHECK_ARG(slice_elems >= 1 && nslices >= 0, "slice energy: bad extents");
  if (nslices == 0) return STARM_OK;
  STARM_CHECK_ARG(a && f_out, "slice energy: null pointer");
  STARM_CHECK_ARG(nslices < (int64_t(1) << 31), "slice energy: too many slices");
  slice_energy_kernel<<<unsigned(nslices), 256, 0, as_stream(stream)>>>(a, slice_elems, slice_elems,
                                                                        f_out);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

// The same sums over the fibre block [f0, f0 + nf) of every slice
// (f_out[i] = sum of squares of a[i * slice_elems + f0 .. + nf)): partial
// energies of a tensor whose fibre blocks become available one at a time.
extern "C" int starm_slice_energy_block_f64(const double* a, int64_t slice_elems, int64_t nslices,
                                            int64_t f0, int64_t nf, double* f_out, void* stream) {
  STARM_CHECK_ARG(slice_elems >= 1 && nslices >= 0 && f0 >= 0 && nf >= 1 && f0 + nf <= slice_elems,
                  "slice energy block: bad extents");
  if (nslices == 0) return STARM_OK;
  STARM_CHECK_ARG(a && f_out, "slice energy block: null pointer");
  STARM_CHECK_ARG(nslices < (int64_t(1) << 31), "slice energy block: too many slices");
  slice_energy_kernel<<<unsigned(nslices), 256, 0, as_stream(stream)>>>(a + f0, nf, slice_elems, f_out);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}

// Strided host-to-device copy (cudaMemcpy2DAsync): `height` runs of `width`
// bytes, pitches in bytes -- one fibre block of a host tensor into the same
// place of its device copy.  Asynchronous for page-locked host memory.
extern "C" int starm_copy2d_h2d(void* dst, size_t dpitch, const void* src, size_t spitch,
                                size_t width, size_t height, void* stream) {
  if (width == 0 || height == 0) return STARM_OK;
  STARM_CHECK_ARG(dst && src && dpitch >= width && spitch >= width, "copy2d: bad arguments");
  STARM_CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice,
                                   as_stream(stream)));
  return STARM_OK;
}

// ------------------------------------------------------------- mode Gram
// G = sum_b A_b^T A_b for the `batch` column-major (rows x inner) blocks of
// the mode-k view (TTMPlan): G = unfold(k) unfold(k)^T, the Gram matrix of
// the data-driven transform (transforms.py:94-110).  64 x 64 output tiles on
// DMMA (8 warps of 32 x 16), K = rows x batch split over `ks` CTA slices
// whose partial tiles are summed in a fixed order (deterministic), then
// symmetrised.
namespace starm {
namespace {
constexpr int GR_T = 64, GR_KC = 16, GR_S = GR_T + 8;

__global__ void __launch_bounds__(256) gram_partial_kernel(const double* __restrict__ a, int64_t rows,
                                                           int64_t inner, int64_t batch, int64_t kchunk,
                                                           int64_t tiles1, double* __restrict__ part) {
  __shared__ double us[GR_KC][GR_S];
  __shared__ double gs[GR_KC][GR_S];
  const int64_t tile = blockIdx.x, ks = blockIdx.y;
  const int64_t i0 = (tile % tiles1) * GR_T, j0 = (tile / tiles1) * GR_T;
  const int64_t K = rows * batch;
  const int64_t k_lo = ks * kchunk, k_hi = k_lo + kchunk < K ? k_lo + kchunk : K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[4][2][2] = {};
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += GR_KC) {
    for (int e = threadIdx.x; e < GR_KC * GR_T; e += 256) {
      const int kk = e % GR_KC, c = e / GR_KC;
      const int64_t k = k0 + kk;
      const bool in = k < k_hi;
      const int64_t b = in ? k / rows : 0, r = in ? k - b * rows : 0;
      const double* blk = a + b * rows * inner + r;
      us[kk][c] = (in && i0 + c < inner) ? blk[(i0 + c) * rows] : 0.0;
      gs[kk][c] = (in && j0 + c < inner) ? blk[(j0 + c) * rows] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < GR_KC; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = us[k4 + tq][32 * wm + 8 * i + gq];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = gs[k4 + tq][16 * wn + 8 * j + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884n(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* out = part + (ks * gridDim.x + tile) * (GR_T * GR_T);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = 32 * wm + 8 * i + gq, c = 16 * wn + 8 * j + 2 * tq;
      out[r + c * GR_T] = acc[i][j][0];
      out[r + (c + 1) * GR_T] = acc[i][j][1];
    }
}

__global__ void gram_final_kernel(const double* __restrict__ part, int64_t inner, int64_t tiles1,
                                  int64_t ntiles, int64_t nks, double* __restrict__ g) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= inner * inner) return;
  const int64_t i = e % inner, j = e / inner;
  auto at = [&](int64_t r, int64_t c) {
    const int64_t tile = (r / GR_T) + (c / GR_T) * tiles1;
    const int64_t off = (r % GR_T) + (c % GR_T) * GR_T;
    double s = 0.0;
    for (int64_t ks = 0; ks < nks; ++ks) s += part[(ks * ntiles + tile) * (GR_T * GR_T) + off];
    return s;
  };
  g[e] = 0.5 * (at(i, j) + at(j, i));   // exact symmetry
}

int64_t gram_ksplit(int64_t rows, int64_t inner, int64_t batch) {
  const int64_t tiles1 = (inner + GR_T - 1) / GR_T;
  const int64_t K = rows * batch;
  int64_t ks = (4 * 148 + tiles1 * tiles1 - 1) / (tiles1 * tiles1);   // ~4 CTAs per SM
  const int64_t maxks = (K + 4 * GR_KC - 1) / (4 * GR_KC);
  if (ks > maxks) ks = maxks;
  return ks < 1 ? 1 : ks;
}
}  // namespace
}  // namespace starm

extern "C" size_t starm_gram_workspace_bytes(int64_t rows, int64_t inner, int64_t batch) {
  if (rows < 1 || inner < 1 || batch < 1) return 0;
  const int64_t tiles1 = (inner + GR_T - 1) / GR_T;
  return size_t(gram_ksplit(rows, inner, batch) * tiles1 * tiles1 * GR_T * GR_T) * sizeof(double);
}

extern "C" int starm_gram_f64(const double* a, int64_t rows, int64_t inner, int64_t batch, double* g,
                              void* ws, size_t ws_bytes, void* stream) {
  STARM_CHECK_ARG(rows >= 1 && inner >= 1 && batch >= 1, "gram: extents must be positive");
  STARM_CHECK_ARG(a && g && ws, "gram: null pointer");
  STARM_CHECK_ARG(ws_bytes >= starm_gram_workspace_bytes(rows, inner, batch), "gram: workspace too small");
  const cudaStream_t st = as_stream(stream);
  const int64_t tiles1 = (inner + GR_T - 1) / GR_T, ntiles = tiles1 * tiles1;
  const int64_t ks = gram_ksplit(rows, inner, batch);
  const int64_t K = rows * batch;
  const int64_t kchunk = round_up(ceil_div(K, ks), GR_KC);
  STARM_CHECK_ARG(ntiles < (int64_t(1) << 31) && ks < 65536, "gram: too large");
  const dim3 grid{unsigned(ntiles), unsigned(ks), 1u};
  gram_partial_kernel<<<grid, 256, 0, st>>>(a, rows, inner, batch, kchunk, tiles1,
                                           static_cast<double*>(ws));
  STARM_LAUNCH_CHECK();
  gram_final_kernel<<<unsigned(ceil_div(inner * inner, 256)), 256, 0, st>>>(
      static_cast<const double*>(ws), inner, tiles1, ntiles, ks, g);
  STARM_LAUNCH_CHECK();
  return STARM_OK;
}
