// Shared helpers for the colbandit_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <type_traits>
#include <algorithm>

#include "../../include/colbandit_b200.h"

#if defined(__CUDA_ARCH__) && !defined(__CUDA_ARCH_FEAT_SM100_ALL)
#error "colbandit_b200 kernels are written for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace cbx {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define CBX_CUDA_CHECK(expr)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::cbx::cuda_fail(_e, #expr); \
  } while (0)

#define CBX_LAUNCH_CHECK(what)                                       \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::cbx::cuda_fail(_e, what);        \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
__host__ __device__ __forceinline__ size_t align_up_dev(size_t x, size_t a) { return (x + a - 1) / a * a; }

int sm_count();

// ----------------------------------------------------------------- element loads
template <typename T> struct Elem;
template <> struct Elem<float> {
  static __device__ __forceinline__ float to_f(float x) { return x; }
  static __device__ __forceinline__ double to_d(float x) { return (double)x; }
};
template <> struct Elem<double> {
  static __device__ __forceinline__ float to_f(double x) { return (float)x; }
  static __device__ __forceinline__ double to_d(double x) { return x; }
};
template <> struct Elem<__half> {
  static __device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
  static __device__ __forceinline__ double to_d(__half x) { return (double)__half2float(x); }
};
template <> struct Elem<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ double to_d(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
};

inline size_t dtype_size(int dtype) {
  switch (dtype) {
    case CBX_F32: return 4;
    case CBX_F16: return 2;
    case CBX_BF16: return 2;
    case CBX_F64: return 8;
  }
  return 0;
}

// ----------------------------------------------------------------- ordered keys
// Ascending key order == (descending score, ascending index); -0.0 folds to +0.0
// so the two zeros tie like they do under np.lexsort.
__device__ __forceinline__ uint64_t desc_key_f32(float s) {
  s = s + 0.0f;
  uint32_t u = __float_as_uint(s);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // ascending with s
  return (uint64_t)(~u);                             // descending with s
}
__device__ __forceinline__ uint64_t desc_key_f64(double s) {
  s = s + 0.0;
  uint64_t u = (uint64_t)__double_as_longlong(s);
  u = (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
  return ~u;
}

// ----------------------------------------------------------------- exact summation
// CPython math.fsum (Modules/mathmodule.c: Shewchuk partials + half-even
// correction) on a small expansion held in registers. Values are finite.
// Partials are non-overlapping, increasing in magnitude, never zero; the
// exact sum is order independent, so growing one expansion incrementally and
// rounding it gives bit-for-bit the fsum of the same multiset of values.
template <int CAP>
struct Expansion {
  double p[CAP];
  int n;
  __device__ __forceinline__ void clear() { n = 0; }
  // add x exactly; returns false on capacity overflow
  __device__ __forceinline__ bool add(double x) {
    int i = 0;
#pragma unroll
    for (int j = 0; j < CAP; ++j) {
      if (j < n) {
        double y = p[j];
        if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
        double hi = __dadd_rn(x, y);
        double lo = __dsub_rn(y, __dsub_rn(hi, x));
        if (lo != 0.0) {
#pragma unroll
          for (int s = 0; s <= j; ++s)
            if (s == i) p[s] = lo;
          ++i;
        }
        x = hi;
      }
    }
    if (x != 0.0) {
      if (i >= CAP) { n = i; return false; }
#pragma unroll
      for (int s = 0; s < CAP; ++s)
        if (s == i) p[s] = x;
      ++i;
    }
    n = i;
    return true;
  }
  // correctly rounded value of the expansion (0.0 when empty)
  __device__ __forceinline__ double round() const {
    double hi = 0.0, lo = 0.0;
    int m = n;
    double pm = 0.0;  // p[m - 1] after the loop
    if (m > 0) {
#pragma unroll
      for (int s = 0; s < CAP; ++s)
        if (s == m - 1) hi = p[s];
      --m;
      bool stop = false;
#pragma unroll
      for (int s = CAP - 2; s >= 0; --s) {
        if (!stop && s == m - 1) {
          double x = hi;
          double y = p[s];
          hi = __dadd_rn(x, y);
          double yr = __dsub_rn(hi, x);
          lo = __dsub_rn(y, yr);
          --m;
          if (lo != 0.0) stop = true;
        }
      }
#pragma unroll
      for (int s = 0; s < CAP; ++s)
        if (s == m - 1) pm = p[s];
      if (m > 0 && ((lo < 0.0 && pm < 0.0) || (lo > 0.0 && pm > 0.0))) {
        double y = __dmul_rn(lo, 2.0);
        double x = __dadd_rn(hi, y);
        double yr = __dsub_rn(x, hi);
        if (y == yr) hi = x;
      }
    }
    return hi;
  }
};

}  // namespace cbx
