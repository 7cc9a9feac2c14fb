// common.cuh — shared device helpers of libprony (sm_100a).
// Complex FP64 is carried as double2 {x = re, y = im}, bit-identical to prony_c128.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/prony.h"

namespace prony {

constexpr int kWarp = 32;

// ----------------------------------------------------------------------------------------
// FP64 tensor-pipe MMA: D(16x8) += A(16x4) * B(4x8), all f64 (PTX mma.sync m16n8k4 .f64,
// SASS DMMA.8x8x4 on sm_100a). Fragment ownership per lane (g = lane>>2, q = lane&3):
//   a0 = A[g][q], a1 = A[g+8][q];  b = B[q][g];
//   c0 = C[g][2q], c1 = C[g][2q+1], c2 = C[g+8][2q], c3 = C[g+8][2q+1].
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// Complex 16x8x4 tile update, 4M form (4 real products):
//   Re += Ar Br - Ai Bi ;  Im += Ar Bi + Ai Br
__device__ __forceinline__ void cmma16x8x4_4m(double (&re)[4], double (&im)[4], double2 a0, double2 a1,
                                              double2 b) {
  dmma16x8x4(re, a0.x, a1.x, b.x);
  dmma16x8x4(re, -a0.y, -a1.y, b.y);
  dmma16x8x4(im, a0.x, a1.x, b.y);
  dmma16x8x4(im, a0.y, a1.y, b.x);
}

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

}  // namespace prony
