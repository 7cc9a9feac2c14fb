// common.cuh — shared device helpers of libprony (sm_100a).
// Complex FP64 is carried as double2 {x = re, y = im}, bit-identical to prony_c128.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/prony.h"

namespace prony {

constexpr int kWarp = 32;

// Debug builds (-DPRONY_DEBUG, tools/ab_variants.py "debug"): index checks on the gather paths count
// violations in a device counter (read with prony_debug_violations()) and clamp the access instead of
// faulting. Release builds compile the checks away.
#ifdef PRONY_DEBUG
#define PRONY_CHECK_INDEX(idx, lo, hi)                          \
  do {                                                          \
    if ((idx) < (lo) || (idx) >= (hi)) {                        \
      atomicAdd(&::prony::g_prony_violations, 1ull);            \
      (idx) = (lo);                                             \
    }                                                           \
  } while (0)
#else
#define PRONY_CHECK_INDEX(idx, lo, hi) \
  do {                                 \
  } while (0)
#endif

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// First device-side error wins.
__device__ __forceinline__ void set_status(int32_t* st, int32_t code) {
  if (st) atomicCAS(st, 0, code);
}

inline int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size): the call costs microseconds
// of host time, which small launch-bound pencils paid on every launch (api.cu)
cudaError_t ensure_smem_attr(const void* fn, int bytes);
template <typename K>
cudaError_t ensure_smem_attr(K* fn, size_t bytes) {
  return ensure_smem_attr(reinterpret_cast<const void*>(fn), (int)bytes);
}

}  // namespace prony
