// common.cuh — shared host/device helpers for the ozb200 C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/ozb200.h"

namespace oz {

// ---------------------------------------------------------------------------
// Host-side error plumbing: thread-local message + status code.
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
const char* last_error();

#define OZ_CHECK_CUDA(expr)                                                       \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::oz::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,               \
                      cudaGetErrorString(_e));                                    \
      return OZ_CUDA_ERROR;                                                       \
    }                                                                             \
  } while (0)

// One-time, per-process setup (kernel attributes): C++11 thread-safe static
// initialisation, so concurrent callers (harness worker threads on their own
// streams) never race on it; the error of the first attempt is sticky.
#define OZ_ONCE(expr)                                          \
  do {                                                         \
    static const cudaError_t oz_once_err_ = [&] { return (expr); }(); \
    OZ_CHECK_CUDA(oz_once_err_);                               \
  } while (0)


// Every kernel launched by this library is counted (bench.py reports it as
// gpu_launches); cuBLAS launches are not ours and are not counted.
void count_launch();
#define OZ_CHECK_LAUNCH()                                                         \
  do {                                                                            \
    ::oz::count_launch();                                                         \
    OZ_CHECK_CUDA(cudaGetLastError());                                            \
  } while (0)

// Optional per-phase timing (CUDA events on the launching stream), enabled by
// oz_prof_enable(); used by bench.py for the roofline of the dominant kernel.
enum ProfKind { PROF_EMU_GEMM = 0, PROF_PANEL = 1, PROF_DGEMM = 2, PROF_SPLIT = 3,
                PROF_LASWP = 4, PROF_TRSM = 5, PROF_SOLVE = 6, PROF_OTHER = 7,
                PROF_COMPOSE = 8, PROF_DGEMM_PANEL = 9, PROF_DGEMM_TRSM = 10,
                PROF_GEMM_SMS = 11,  // emulated GEMM time x (SMs it may use / all SMs)
                PROF_KINDS = 12 };
int prof_start(cudaStream_t st);
void prof_stop(int tag, cudaStream_t st, int kind, double work, int sms = 0);

#define OZ_REQUIRE(cond, code, ...)                                               \
  do {                                                                            \
    if (!(cond)) {                                                                \
      ::oz::set_error(__VA_ARGS__);                                               \
      return (code);                                                              \
    }                                                                             \
  } while (0)

#define OZ_TRY(expr)                                                              \
  do {                                                                            \
    int _s = (expr);                                                              \
    if (_s != OZ_OK) return _s;                                                   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();  // cached per device

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------------------
// Device helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 2^e as a double for e in [-1022, 1023] (exact construction of the bits).
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}

// ldexp that is exact (correctly rounded) for every input: multiply by an
// exactly representable power of two when possible, fall back to ldexp().
static __device__ __noinline__ double ldexp_slow(double x, int e) { return ldexp(x, e); }
__device__ __forceinline__ double ldexp_exact(double x, int e) {
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, pow2(e));
  return ldexp_slow(x, e);  // out-of-line: keeps unrolled epilogues small
}

// frexp exponent of |x| (x finite, x != 0): x = m * 2^e with 0.5 <= m < 1.
__device__ __forceinline__ int frexp_exp(double x) { return ilogb(x) + 1; }

// Atomic max on the IEEE bits of a non-negative double (monotone as uint64).
__device__ __forceinline__ void atomic_max_abs(unsigned long long* dst, double v) {
  atomicMax(dst, static_cast<unsigned long long>(__double_as_longlong(fabs(v))));
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = v > w ? v : w;
  }
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace oz
