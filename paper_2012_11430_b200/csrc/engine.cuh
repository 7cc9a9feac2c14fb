// engine.cuh — the complex-FP64 DMMA warp engine and async-copy / mbarrier primitives shared by
// k_project, k_reduce (project.cu) and k_vls (vandermonde_ls.cu). sm_100a.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

namespace prony {

// compile-time loop: f(std::integral_constant<int, 0>{}) ... f(std::integral_constant<int, N - 1>{})
template <typename F, int... J>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, J...>) {
  (f(std::integral_constant<int, J>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// ---------------------------------------------------------------------------- warp engine
// non-volatile so ptxas may interleave independent MMAs
__device__ __forceinline__ void mma16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// Complex warp tile C(16 x 8*NA) += A(16 x 4) B(4 x 8*NA) for one k-step of 4, operands in shared
// memory in k-major planes: Ac[k*lda + row] (re, im), As[k*ldas + row] (re+im), Bc[k*ldb + col],
// Bs[k*ldbs + col]. Lane (g = lane>>2, q = lane&3) reads A rows g, g+8 at k = q and B column g at
// k = q (conflict-free LDS: strides are = 2 (double2) / 4 (double) mod 16 x 8 bytes).
// MODE 3 (3M): acc0 += Ar Br, acc1 += Ai Bi, acc2 += (Ar+Ai)(Br+Bi)
// MODE 4 (4M): acc0 += Ar Br - Ai Bi, acc1 += Ar Bi + Ai Br
// NA <= NT n-tiles are active (compile-time, so no predicated MMAs).
// PK (packed last n-tile, MODE 3): n-tile NA-1 holds w = m % 8 <= 4 valid columns; it is
// computed as Ar [Br | Bi] (acc0) and Ai [Br | Bi] (acc1) on ONE 8-wide B fragment — lane column g reads
// column (g & 3) of the tile, the real part for g < 4 and the imaginary part for g >= 4 — so 2 real DMMA
// products instead of the 3 of a half-empty 3M tile; acc_packed_to_complex recombines (4M form).
// SREG (MODE 3): the sum operands Re+Im of A and Re+Im (Re-Im for CONJB) of B are formed in registers from
// the complex fragments (As, Bs unused): no sum planes in shared memory, one DADD per n-tile per k-step.
template <int NT, int NA, int MODE, bool CONJB = false, bool PK = false, bool SREG = false>
__device__ __forceinline__ void warp_cmma_k4(double (&acc)[3][NT][4], const double2* __restrict__ Ac,
                                             const double* __restrict__ As, int lda, int ldas,
                                             const double2* __restrict__ Bc, const double* __restrict__ Bs,
                                             int ldb, int ldbs, int g, int q) {
  // CONJB: the B operand is conj(Bc) (its sum plane Bs must then hold Re - Im)
  const double2 a0 = Ac[q * lda + g];
  const double2 a1 = Ac[q * lda + g + 8];
  double s0 = 0.0, s1 = 0.0;
  if constexpr (MODE == 3) {
    if constexpr (SREG) {
      s0 = a0.x + a0.y;
      s1 = a1.x + a1.y;
    } else {
      s0 = As[q * ldas + g];
      s1 = As[q * ldas + g + 8];
    }
  }
  const double2* brow = Bc + q * ldb + g;
  const double* bsrow = SREG ? nullptr : Bs + q * ldbs + g;
  constexpr double sb = CONJB ? -1.0 : 1.0;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    if constexpr (PK && MODE == 3) {
      if (j == NA - 1) {
        const double2 bb = brow[8 * j - (g & 4)];  // column 8j + (g & 3) of the tile
        const double bp = (g & 4) ? bb.y : bb.x;
        mma16x8x4(acc[0][j], a0.x, a1.x, bp);
        mma16x8x4(acc[1][j], a0.y, a1.y, bp);
        continue;
      }
    }
    {
      const double2 b = brow[8 * j];
      if constexpr (MODE == 3) {
        double bs;
        if constexpr (SREG) bs = CONJB ? b.x - b.y : b.x + b.y;
        else bs = bsrow[8 * j];
        mma16x8x4(acc[0][j], a0.x, a1.x, b.x);
        mma16x8x4(acc[1][j], sb * a0.y, sb * a1.y, b.y);  // Ai (sb Bi): sign folded into the A operand
        mma16x8x4(acc[2][j], s0, s1, bs);
      } else {
        mma16x8x4(acc[0][j], a0.x, a1.x, b.x);
        mma16x8x4(acc[1][j], sb * a0.x, sb * a1.x, b.y);
        mma16x8x4(acc[0][j], -sb * a0.y, -sb * a1.y, b.y);
        mma16x8x4(acc[1][j], a0.y, a1.y, b.x);
      }
    }
  }
}

// dispatch on the warp's active n-tile count (warp-uniform) so each variant is fully unrolled
template <int NT, int MODE, bool CONJB = false>
__device__ __forceinline__ void warp_cmma_k4_n(int nt_active, double (&acc)[3][NT][4], const double2* Ac,
                                               const double* As, int lda, int ldas, const double2* Bc,
                                               const double* Bs, int ldb, int ldbs, int g, int q) {
  if (nt_active == NT) {
    warp_cmma_k4<NT, NT, MODE, CONJB>(acc, Ac, As, lda, ldas, Bc, Bs, ldb, ldbs, g, q);
  } else if constexpr (NT > 1) {
    if (nt_active == NT - 1) {
      warp_cmma_k4<NT, NT - 1, MODE, CONJB>(acc, Ac, As, lda, ldas, Bc, Bs, ldb, ldbs, g, q);
    } else if constexpr (NT > 2) {
      if (nt_active == NT - 2) {
        warp_cmma_k4<NT, NT - 2, MODE, CONJB>(acc, Ac, As, lda, ldas, Bc, Bs, ldb, ldbs, g, q);
      } else if constexpr (NT > 3) {
        if (nt_active == NT - 3)
          warp_cmma_k4<NT, NT - 3, MODE, CONJB>(acc, Ac, As, lda, ldas, Bc, Bs, ldb, ldbs, g, q);
      }
    }
  }
}

// packed last n-tile (PK): lane q < 2 holds columns 2q, 2q+1 of Ar Br (acc0) and Ai Br (acc1); its partner
// q + 2 (lane ^ 2) holds the same columns of Ar Bi and Ai Bi. A B: Re = Ar Br - Ai Bi, Im = Ar Bi + Ai Br;
// A conj(B) (CONJB): Re = Ar Br + Ai Bi, Im = Ai Br - Ar Bi. Valid on lanes q < 2 (the tile's columns 0..3);
// lanes q >= 2 get 0 (padding columns). All 32 lanes must call it.
template <int NT, bool CONJB = false>
__device__ __forceinline__ void acc_packed_to_complex(const double (&acc)[3][NT][4], int j, int q, double (&re)[4],
                                                      double (&im)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const double p0 = __shfl_xor_sync(0xffffffffu, acc[0][j][e], 2);
    const double p1 = __shfl_xor_sync(0xffffffffu, acc[1][j][e], 2);
    if constexpr (CONJB) {
      re[e] = q < 2 ? acc[0][j][e] + p1 : 0.0;
      im[e] = q < 2 ? acc[1][j][e] - p0 : 0.0;
    } else {
      re[e] = q < 2 ? acc[0][j][e] - p1 : 0.0;
      im[e] = q < 2 ? p0 + acc[1][j][e] : 0.0;
    }
  }
}

template <int NT, int MODE>
__device__ __forceinline__ void acc_to_complex(const double (&acc)[3][NT][4], int j, double (&re)[4],
                                               double (&im)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if constexpr (MODE == 3) {
      re[e] = acc[0][j][e] - acc[1][j][e];
      im[e] = acc[2][j][e] - acc[0][j][e] - acc[1][j][e];
    } else {
      re[e] = acc[0][j][e];
      im[e] = acc[1][j][e];
    }
  }
}

__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(uint32_t sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(src_bytes));
}
// the same with a compile-time byte offset folded into the shared address (an immediate of the LDGSTS)
template <int OFF>
__device__ __forceinline__ void cp_async16_at(uint32_t sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0+%3], [%1], 16, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(src_bytes), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void cp_async8_at(uint32_t sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0+%3], [%1], 8, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(src_bytes), "n"(OFF));
}
__device__ __forceinline__ void cp_async16_cg(uint32_t sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------- mbarrier helpers
__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(addr) : "memory");
}
// arrive on the mbarrier once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void mbar_arrive_cp_async(uint32_t addr) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// expect `bytes` of bulk-copy transactions on the mbarrier (counts as one arrival)
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t addr, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(addr), "r"(bytes)
               : "memory");
}
// bulk global -> shared copy (size multiple of 16, 16-byte aligned), completes on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t sdst, const void* gsrc, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sdst),
               "l"(gsrc), "r"(bytes), "r"(mbar)
               : "memory");
}
template <int R>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R));
}
template <int R>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(R));
}


}  // namespace prony
