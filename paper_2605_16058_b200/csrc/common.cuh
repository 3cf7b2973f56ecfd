// Shared helpers for libstarm: error state, launch checks and sm_100a PTX
// wrappers (cp.async staging, FP64 DMMA tiles).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <stdio.h>
#include <stdarg.h>

#include "starm.h"

namespace starm {

// Thread-local last error message, read back by starm_last_error().
void set_error(const char* fmt, ...);

// Process-wide count of kernel launches issued by this library (bench claim
// `gpu_launches`); CUB device-wide calls count as one launch each.
void count_launch(int n = 1);

#define STARM_CHECK_ARG(cond, ...)                                   \
  do {                                                               \
    if (!(cond)) {                                                   \
      ::starm::set_error(__VA_ARGS__);                               \
      return STARM_INVALID_ARG;                                      \
    }                                                                \
  } while (0)

#define STARM_CUDA_TRY(expr)                                         \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) {                                         \
      ::starm::set_error("%s: %s (%s:%d)", #expr,                    \
                         cudaGetErrorString(_e), __FILE__, __LINE__);\
      return STARM_CUDA;                                             \
    }                                                                \
  } while (0)

#define STARM_LAUNCH_CHECK()                                         \
  do {                                                               \
    ::starm::count_launch(1);                                        \
    STARM_CUDA_TRY(cudaGetLastError());                              \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// dct.cu: the fast DCT-II / DCT-III; with xbf the n = 1024 forward kernel
// also writes the bf16 operand rows of the residual GEMM (*packed = true).
// pitch: doubles between consecutive mode indices of a fibre (0 = rows).
int dct_launch(const double* src, double* dst, int64_t rows, int64_t n, int64_t batch, bool inv,
               uint16_t* xbf, int64_t rows_pad, bool* packed, cudaStream_t st, int64_t pitch = 0);

// gemm_f64.cu: C = A * B (batch 1, column-major) with the K10 error partials
// of E against C fused into the epilogue (epart: 2 doubles per tile).
int64_t gemm_f64_tiles(int64_t M, int64_t N);
int gemm_f64_err(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K,
                 int64_t lda, int64_t ldb, int64_t ldc, const double* E, double* epart,
                 cudaStream_t st);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------- PTX

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy; src_bytes < 16 zero-fills the rest.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes = 16) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
// 8-byte async copy (cache-all path; .cg only supports 16 bytes).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes = 8) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor pipe (SASS DMMA.8x8x4).
// Fragment ownership (lane = 4*g + t, g = lane>>2, t = lane&3):
//   a = A[g][t], b = B[t][g], d0/d1 = D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Bulk (TMA-engine) prefetch of [ptr, ptr + bytes) into L2; ptr 16-byte
// aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* ptr, int bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// Same, without `volatile`: lets the compiler schedule the DMMA among loads.
__device__ __forceinline__ void dmma884n(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

}  // namespace starm
