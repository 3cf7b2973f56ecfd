// K7: tolerance-driven rank selection on the device, bit-for-bit the
// semantics of compute_threshold (tsvdm.py:85-115):
//
//   sq = s*s; v = sort(sq) ascending; w = cumsum(v) (sequential fp64);
//   total = w[-1]; budget = eps*eps*total; j = searchsorted(w, budget, 'left');
//   tau = v[j-1] (0 if j == 0); keep = sq > tau;
//   discarded = sum(sq[~keep])   <- numpy pairwise add-reduce over the C-order
//                                   (row-major) masked copy of the (r, N) matrix
//   if discarded >= budget and tau > 0: keep = sq >= tau; discarded = sum(sq[~keep])
//   ranks = keep.sum(axis=0)
//
// Pipeline (one stream, no host round trip):
//   square_keys -> radix sort (64-bit keys: non-negative doubles order like
//   their bit patterns) -> sequential running sums + lower_bound -> masks for
//   both candidate rules in C order -> exclusive scans -> order-preserving
//   compaction -> numpy-pairwise sums of both candidates (the pairwise tree
//   cut at depth 10 into 1024 subtrees per candidate, summed by 64 CTAs of
//   32 threads, then recombined level by level in the same shape by one CTA)
//   -> tie rule -> per-slice ranks.
// All products use __dmul_rn so no FMA contraction changes a rounding.
#include <cub/cub.cuh>

#include "common.cuh"

namespace starm {
namespace {

#ifndef PW_LOG
#define PW_LOG 10
#endif
constexpr int PW_DEPTH = PW_LOG;  // 2^PW_DEPTH == PW_THREADS
constexpr int PW_THREADS = 1 << PW_DEPTH;

struct ThState {
  double budget;
  double tau;
  double total;
  double disc[2];  // candidate discarded sums: [0] strict rule, [1] tie-retain rule
  int64_t j;
  int64_t cnt[2];
  int mode;        // -1: all-zero total, 0: keep sq > tau, 1: keep sq >= tau
  // pruned form (starm_threshold_pruned_f64): e0 = energy of the slices left
  // out (every one of their sigma^2 <= tbound); cert = the crossing value
  // v[j] exceeds tbound, i.e. all values <= tbound are discarded whatever
  // they are.  e0 = 0, tbound = -1 for the plain call (bitwise unchanged).
  double e0;
  double tbound;
  int cert;
};

__global__ void square_keys_kernel(const double* s, int64_t count, unsigned long long* keys) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double x = s[i];
    keys[i] = __double_as_longlong(__dmul_rn(x, x));
  }
}

// Sequential running sums (np.cumsum) and the lower_bound search.
// Two warps: warp 1 streams tiles of 1024 sorted values into shared memory
// (and the running sums of the previous tile back out) while lane 0 of warp 0
// runs the strictly sequential fp64 chain on the current tile; loads of the
// next 8 values are issued ahead of the 8 dependent adds so the chain runs
// at DADD latency.  The chain is the only serial part of the threshold.
constexpr int CS_TILE = 1024;

__global__ void __launch_bounds__(64) cumsum_search_kernel(const unsigned long long* vbits,
                                                           int64_t count, double eps, double* w,
                                                           double* v_out, ThState* st, double e0,
                                                           double tbound) {
  __shared__ __align__(16) double tile[2][CS_TILE];
  __shared__ __align__(16) double wt[2][CS_TILE];
  __shared__ double acc_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* v = reinterpret_cast<const double*>(vbits);
  const int64_t ntiles = (count + CS_TILE - 1) / CS_TILE;
  auto tlen = [&](int64_t t) { return int(count - t * CS_TILE < CS_TILE ? count - t * CS_TILE : CS_TILE); };
  if (warp == 1 && ntiles > 0) {
    const int len = tlen(0);
    for (int k = lane; k < len; k += 32) {
      const double x = v[k];
      tile[0][k] = x;
      if (v_out) v_out[k] = x;
    }
  }
  __syncthreads();
  double acc = 0.0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int b = int(t & 1);
    if (warp == 0) {
      if (lane == 0) {
        const double* tl = tile[b];
        double* wl = wt[b];
        const int len = tlen(t);
        int k = 0;
        if (t == 0) {
          acc = e0 == 0.0 ? tl[0] : __dadd_rn(e0, tl[0]);  // pruned form: the left-out energy first
          wl[0] = acc;
          for (k = 1; k < 8 && k < len; ++k) {
            acc = __dadd_rn(acc, tl[k]);
            wl[k] = acc;
          }
        }
        // running sums leave as 16-byte pairs
        auto chain8 = [&](const double (&c)[8], int k0) {
          double w8[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            acc = __dadd_rn(acc, c[q]);
            w8[q] = acc;
          }
#pragma unroll
          for (int q = 0; q < 8; q += 2)
            *reinterpret_cast<double2*>(wl + k0 + q) = make_double2(w8[q], w8[q + 1]);
        };
        // three banks: each bank's loads are issued two banks (16 dependent
        // adds, ~128 cycles) before its adds, covering the ~60-cycle
        // shared-memory latency that a one-bank lead only just covered
        auto load8 = [&](double (&c)[8], int k0) {
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const double2 v2 = *reinterpret_cast<const double2*>(tl + k0 + q);
            c[q] = v2.x;
            c[q + 1] = v2.y;
          }
        };
        double ra[8], rb[8], rc[8];
        if (k + 8 <= len) load8(ra, k);
        if (k + 16 <= len) load8(rb, k + 8);
        for (; k + 24 <= len; k += 24) {
          load8(rc, k + 16);
          chain8(ra, k);
          if (k + 32 <= len) load8(ra, k + 24);
          chain8(rb, k + 8);
          if (k + 40 <= len) load8(rb, k + 32);
          chain8(rc, k + 16);
        }
        if (k + 8 <= len) {
          chain8(ra, k);
          k += 8;
        }
        if (k + 8 <= len) {
          chain8(rb, k);
          k += 8;
        }
        for (; k < len; ++k) {
          acc = __dadd_rn(acc, tl[k]);
          wl[k] = acc;
        }
      }
    } else {
      if (t + 1 < ntiles) {  // prefetch the next tile: all loads in flight at once
        const int len = tlen(t + 1);
        const int64_t base = (t + 1) * CS_TILE;
        constexpr int PER = CS_TILE / 32;
        double x[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = lane + 32 * u;
          x[u] = k < len ? v[base + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = lane + 32 * u;
          if (k < len) {
            tile[b ^ 1][k] = x[u];
            if (v_out) v_out[base + k] = x[u];
          }
        }
      }
      if (t > 0) {  // running sums of the previous tile out
        const int len = tlen(t - 1);
        const int64_t base = (t - 1) * CS_TILE;
        for (int k = lane; k < len; k += 32) w[base + k] = wt[b ^ 1][k];
      }
    }
    __syncthreads();
  }
  if (warp == 1 && ntiles > 0) {
    const int64_t t = ntiles - 1;
    const int len = tlen(t);
    for (int k = lane; k < len; k += 32) w[t * CS_TILE + k] = wt[t & 1][k];
  }
  if (threadIdx.x == 0) acc_sh = acc;
  __syncthreads();
  acc = acc_sh;
  if (threadIdx.x != 0) return;
  const double total = count ? acc : e0;
  st->total = total;
  st->e0 = e0;
  st->tbound = tbound;
  st->cert = 0;
  if (total == 0.0) {
    st->mode = -1;
    st->j = 0;
    st->tau = 0.0;
    st->budget = 0.0;
    st->cert = 1;
    return;
  }
  const double budget = __dmul_rn(__dmul_rn(eps, eps), total);
  // searchsorted(w, budget, side='left'): first k with w[k] >= budget.
  int64_t lo = 0, hi = count;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (w[mid] < budget)
      lo = mid + 1;
    else
      hi = mid;
  }
  st->budget = budget;
  st->j = lo;
  st->tau = lo > 0 ? v[lo - 1] : 0.0;
  st->mode = 0;
  st->cert = lo < count && v[lo] > tbound;
}

// Masks in C (row-major) order of the (r, N) matrix: c = row*N + slice.
__global__ void mask_kernel(const double* s, int64_t r, int64_t N, const ThState* st, int* fa,
                            int* fb) {
  const int64_t count = r * N;
  const double tau = st->tau;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < count;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = c / N, slice = c % N;
    const double x = s[row + slice * r];
    const double sq = __dmul_rn(x, x);
    fa[c] = !(sq > tau);   // dropped under keep = sq > tau
    fb[c] = !(sq >= tau);  // dropped under keep = sq >= tau
  }
}

__global__ void scatter_kernel(const double* s, int64_t r, int64_t N, const int* fa, const int* fb,
                               const int* pa, const int* pb, double* da, double* db) {
  const int64_t count = r * N;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < count;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = c / N, slice = c % N;
    const double x = s[row + slice * r];
    const double sq = __dmul_rn(x, x);
    if (fa[c]) da[pa[c]] = sq;
    if (fb[c]) db[pb[c]] = sq;
  }
}

// numpy DOUBLE_pairwise_sum (loops_utils.h.src), recursive.
__device__ double pw_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int64_t i = 8;
    const int64_t stop = n - (n % 8);
    for (; i < stop; i += 8) {
      r0 = __dadd_rn(r0, a[i + 0]);
      r1 = __dadd_rn(r1, a[i + 1]);
      r2 = __dadd_rn(r2, a[i + 2]);
      r3 = __dadd_rn(r3, a[i + 3]);
      r4 = __dadd_rn(r4, a[i + 4]);
      r5 = __dadd_rn(r5, a[i + 5]);
      r6 = __dadd_rn(r6, a[i + 6]);
      r7 = __dadd_rn(r7, a[i + 7]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_sum(a, n2), pw_sum(a + n2, n - n2));
}

__device__ __forceinline__ int64_t pw_split(int64_t n) {
  int64_t n2 = n / 2;
  return n2 - n2 % 8;
}

// Subtree t of the pairwise tree cut at depth PW_DEPTH (0 when t is not the
// owner of a leaf that ends above the cut).
__device__ double pw_leaf(const double* a, int64_t n, int t) {
  int64_t lo = 0, len = n;
  for (int depth = 0; depth < PW_DEPTH; ++depth) {
    if (len <= 128) {
      // Leaf above the cut: only the all-zero-suffix descendant computes it.
      return (t & ((1 << (PW_DEPTH - depth)) - 1)) == 0 ? pw_sum(a + lo, len) : 0.0;
    }
    const int64_t n2 = pw_split(len);
    if ((t >> (PW_DEPTH - 1 - depth)) & 1) {
      lo += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  return pw_sum(a + lo, len);
}

// Recombine the PW_THREADS subtree sums in part[] bottom-up, one tree level
// per step, in the tree's own order: node (d, p) lives at part[p << (D - d)]
// (its left child's slot), so every internal node adds its two children in
// place.  Nodes that were leaves above the cut (n <= 128) already hold their
// sum; nodes below such a leaf do not exist.  One CTA of PW_THREADS threads.
__device__ double pw_combine_levels(int64_t n, double* part) {
  const int t = threadIdx.x;
  for (int d = PW_DEPTH - 1; d >= 0; --d) {
    if (t < (1 << d)) {
      int64_t l = n;
      bool exists = true;
      for (int q = 0; q < d; ++q) {  // replay the splits from the root
        if (l <= 128) {
          exists = false;
          break;
        }
        const int64_t n2 = pw_split(l);
        l = ((t >> (d - 1 - q)) & 1) ? l - n2 : n2;
      }
      if (exists && l > 128) {
        const int i = t << (PW_DEPTH - d);
        part[i] = __dadd_rn(part[i], part[i + (1 << (PW_DEPTH - d - 1))]);
      }
    }
    __syncthreads();
  }
  const double res = (n == 0) ? 0.0 : __dadd_rn(0.0, part[0]);
  __syncthreads();
  return res;
}

// The 2 x PW_THREADS subtree sums (both candidate masks), 32 per CTA so the
// strided per-thread reads spread over many SMs' L1s.
constexpr int PW_LEAF_CTA = 32;
__global__ void __launch_bounds__(PW_LEAF_CTA) pairwise_leaves_kernel(const int* fa, const int* fb,
                                                                      const int* pa, const int* pb,
                                                                      const double* da,
                                                                      const double* db, int64_t count,
                                                                      const ThState* st, double* parts) {
  if (st->mode < 0) return;
  const int g = blockIdx.x * PW_LEAF_CTA + threadIdx.x;  // [0, 2 PW_THREADS)
  const int which = g / PW_THREADS, t = g % PW_THREADS;
  const int64_t na = count ? int64_t(pa[count - 1]) + fa[count - 1] : 0;
  const int64_t nb = count ? int64_t(pb[count - 1]) + fb[count - 1] : 0;
  parts[g] = which ? pw_leaf(db, nb, t) : pw_leaf(da, na, t);
}

__global__ void __launch_bounds__(PW_THREADS) pairwise_kernel(const int* fa, const int* fb,
                                                               const int* pa, const int* pb,
                                                               int64_t count, const double* parts,
                                                               ThState* st) {
  __shared__ double part[PW_THREADS];
  if (st->mode < 0) return;
  const int64_t na = count ? int64_t(pa[count - 1]) + fa[count - 1] : 0;
  const int64_t nb = count ? int64_t(pb[count - 1]) + fb[count - 1] : 0;
  part[threadIdx.x] = parts[threadIdx.x];
  __syncthreads();
  const double sa = pw_combine_levels(na, part);
  part[threadIdx.x] = parts[PW_THREADS + threadIdx.x];
  __syncthreads();
  const double sb = pw_combine_levels(nb, part);
  if (threadIdx.x == 0) {
    // pruned form: the left-out slices' energy is discarded too (e0 = 0 otherwise)
    const double da = st->e0 == 0.0 ? sa : __dadd_rn(st->e0, sa);
    const double dbb = st->e0 == 0.0 ? sb : __dadd_rn(st->e0, sb);
    st->disc[0] = da;
    st->disc[1] = dbb;
    st->cnt[0] = na;
    st->cnt[1] = nb;
    st->mode = (da >= st->budget && st->tau > 0.0) ? 1 : 0;
  }
}

__global__ void ranks_kernel(const double* s, int64_t r, int64_t N, const ThState* st,
                             int64_t* ranks, double* scal, int64_t* j_out) {
  const int mode = st->mode;
  const double tau = st->tau;
  // one warp per slice: lanes stride the r values (coalesced), integer counts
  // summed by shuffles (one thread per slice walked its column serially:
  // 0.09 ms for c2's 70 x 361 values)
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; i < N; i += warps) {
    int k = 0;
    if (mode >= 0) {
      for (int64_t row = lane; row < r; row += 32) {
        const double x = s[row + i * r];
        const double sq = __dmul_rn(x, x);
        k += (mode == 0) ? (sq > tau) : (sq >= tau);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if (lane == 0) ranks[i] = k;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (mode < 0) {
      scal[0] = 0.0;
      scal[1] = 0.0;
      scal[2] = 0.0;
      *j_out = 0;
    } else {
      scal[0] = tau;
      scal[1] = st->disc[mode];
      scal[2] = st->total;
      *j_out = st->j;
    }
  }
}

struct ThLayout {
  size_t keys, sorted, w, fa, fb, pa, pb, da, db, state, parts, cub, total;
  size_t cub_bytes;
};

ThLayout layout(int64_t count) {
  ThLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  L.keys = take(count * 8);
  L.sorted = take(count * 8);
  L.w = take(count * 8);
  L.fa = take(count * 4);
  L.fb = take(count * 4);
  L.pa = take(count * 4);
  L.pb = take(count * 4);
  L.da = take(count * 8);
  L.db = take(count * 8);
  L.state = take(sizeof(ThState));
  L.parts = take(2 * PW_THREADS * sizeof(double));  // pairwise subtree sums of both candidates
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, int(count));
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int*)nullptr, (int*)nullptr,
                                int(count));
  L.cub_bytes = sort_bytes > scan_bytes ? sort_bytes : scan_bytes;
  L.cub = take(L.cub_bytes);
  L.total = off;
  return L;
}

int grid_for(int64_t count) {
  int64_t g = (count + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return int(g);
}

}  // namespace
}  // namespace starm

using namespace starm;

extern "C" size_t starm_threshold_workspace_bytes(int64_t r, int64_t nslices) {
  if (r < 1 || nslices < 1) return 0;
  return layout(r * nslices).total;
}

namespace starm {
namespace {
int threshold_run(const double* s, int64_t r, int64_t nslices, double epsilon, double* v_out,
                  double* w_out, int64_t* ranks_out, double* scal_out, int64_t* j_out, void* ws,
                  size_t ws_bytes, void* stream, double e0, double tbound, int32_t* cert_out);
}  // namespace
}  // namespace starm

extern "C" int starm_threshold_f64(const double* s, int64_t r, int64_t nslices, double epsilon,
                                   double* v_out, double* w_out, int64_t* ranks_out,
                                   double* scal_out, int64_t* j_out, void* ws, size_t ws_bytes,
                                   void* stream) {
  return threshold_run(s, r, nslices, epsilon, v_out, w_out, ranks_out, scal_out, j_out, ws,
                       ws_bytes, stream, 0.0, -1.0, nullptr);
}

extern "C" int starm_threshold_pruned_f64(const double* s, int64_t r, int64_t nslices,
                                          double epsilon, double e0, double tbound,
                                          int64_t* ranks_out, double* scal_out, int64_t* j_out,
                                          int32_t* cert_out, void* ws, size_t ws_bytes,
                                          void* stream) {
  STARM_CHECK_ARG(e0 >= 0.0 && tbound >= 0.0 && cert_out, "threshold pruned: bad e0 / tbound");
  return threshold_run(s, r, nslices, epsilon, nullptr, nullptr, ranks_out, scal_out, j_out, ws,
                       ws_bytes, stream, e0, tbound, cert_out);
}

__global__ void cert_kernel(const starm::ThState* st, int32_t* cert) { *cert = st->cert; }

namespace starm {
namespace {
int threshold_run(const double* s, int64_t r, int64_t nslices, double epsilon, double* v_out,
                  double* w_out, int64_t* ranks_out, double* scal_out, int64_t* j_out, void* ws,
                  size_t ws_bytes, void* stream, double e0, double tbound, int32_t* cert_out) {
  STARM_CHECK_ARG(r >= 1 && nslices >= 1, "threshold: extents must be positive");
  STARM_CHECK_ARG(epsilon > 0.0 && epsilon < 1.0, "tolerance must lie in (0, 1), got %g", epsilon);
  const int64_t count = r * nslices;
  STARM_CHECK_ARG(count < (int64_t(1) << 31), "threshold: too many values (%lld)", (long long)count);
  STARM_CHECK_ARG(s && ranks_out && scal_out && j_out && ws, "threshold: null pointer");
  const ThLayout L = layout(count);
  STARM_CHECK_ARG(ws_bytes >= L.total, "threshold: workspace too small (%zu < %zu)", ws_bytes, L.total);
  char* base = reinterpret_cast<char*>(ws);
  auto* keys = reinterpret_cast<unsigned long long*>(base + L.keys);
  auto* sorted = reinterpret_cast<unsigned long long*>(base + L.sorted);
  double* w = w_out ? w_out : reinterpret_cast<double*>(base + L.w);
  int* fa = reinterpret_cast<int*>(base + L.fa);
  int* fb = reinterpret_cast<int*>(base + L.fb);
  int* pa = reinterpret_cast<int*>(base + L.pa);
  int* pb = reinterpret_cast<int*>(base + L.pb);
  double* da = reinterpret_cast<double*>(base + L.da);
  double* db = reinterpret_cast<double*>(base + L.db);
  ThState* stt = reinterpret_cast<ThState*>(base + L.state);
  void* cubtmp = base + L.cub;
  size_t cub_bytes = L.cub_bytes;
  cudaStream_t st = as_stream(stream);
  const int grid = grid_for(count);

  square_keys_kernel<<<grid, 256, 0, st>>>(s, count, keys);
  STARM_LAUNCH_CHECK();
  STARM_CUDA_TRY(cub::DeviceRadixSort::SortKeys(cubtmp, cub_bytes, keys, sorted, int(count), 0, 64, st));
  count_launch(3);  // the three CUB device-wide calls of this function
  cumsum_search_kernel<<<1, 64, 0, st>>>(sorted, count, epsilon, w, v_out, stt, e0, tbound);
  STARM_LAUNCH_CHECK();
  mask_kernel<<<grid, 256, 0, st>>>(s, r, nslices, stt, fa, fb);
  STARM_LAUNCH_CHECK();
  cub_bytes = L.cub_bytes;
  STARM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cubtmp, cub_bytes, fa, pa, int(count), st));
  cub_bytes = L.cub_bytes;
  STARM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cubtmp, cub_bytes, fb, pb, int(count), st));
  scatter_kernel<<<grid, 256, 0, st>>>(s, r, nslices, fa, fb, pa, pb, da, db);
  STARM_LAUNCH_CHECK();
  double* parts = reinterpret_cast<double*>(base + L.parts);
  pairwise_leaves_kernel<<<2 * PW_THREADS / PW_LEAF_CTA, PW_LEAF_CTA, 0, st>>>(fa, fb, pa, pb, da, db,
                                                                              count, stt, parts);
  STARM_LAUNCH_CHECK();
  pairwise_kernel<<<1, PW_THREADS, 0, st>>>(fa, fb, pa, pb, count, parts, stt);
  STARM_LAUNCH_CHECK();
  ranks_kernel<<<grid_for(nslices * 32), 256, 0, st>>>(s, r, nslices, stt, ranks_out, scal_out, j_out);
  STARM_LAUNCH_CHECK();
  if (cert_out) {
    cert_kernel<<<1, 1, 0, st>>>(stt, cert_out);
    STARM_LAUNCH_CHECK();
  }
  return STARM_OK;
}
}  // namespace
}  // namespace starm
