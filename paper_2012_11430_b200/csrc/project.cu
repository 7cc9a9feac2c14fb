// project.cu — S_l = U* T_l V Sigma^-1 (eq_generateSl) on sm_100a.
//
// Launches per call:
//   k_prep      P(k) = sum_i k_i L^(d-1-i) for k in I_n (linear box offset of k, so that
//               T_l[k,h] = grid[P(k) - P(h) + L^(d-l) + C0], C0 = n sum_i L^i; F5),
//               gsum = Re+Im of the grid and Vsum = Re+Im of V (3M operand planes)
//   k_project   Y_c = T_l[rows, chunk c] V[chunk c, :] — implicit-Toeplitz gather of T_l straight
//               from the L2-resident sample grid into shared memory (T_l is never written
//               anywhere), complex FP64 on the DMMA pipe, split-K over column chunks c
//   k_reduce    S_part[p] = U[rows_p]^* (sum_c Y_c[rows_p])   (same DMMA warp engine)
//   k_finalize  S_l = (sum_p S_part[p]) diag(1/sigma)          (fixed order -> deterministic)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "engine.cuh"
#include "project.cuh"

namespace prony {

#ifdef PRONY_DEBUG
__device__ unsigned long long g_prony_violations = 0;  // gather-index violations (debug builds only)
#endif

// complex product formulation: 3 (Gauss/3M, default) or 4 (4M); env PRONY_CMUL=4m selects 4M
static int cmul_mode() {
  const char* e = getenv("PRONY_CMUL");
  return (e && (e[0] == '4')) ? 4 : 3;
}

// ---------------------------------------------------------------------------- prep
// Vsum[h][c] = Re+Im of V[h][c] (0 for the padding columns c >= m), rows [r0, r1), with 4 independent loads in
// flight per thread (the loop is HBM-latency bound otherwise); 32-bit index arithmetic when (r1 - r0) NP fits
template <typename I>
__device__ __forceinline__ void vsum_rows_t(int r0, int r1, int m, int ldv, int NP, const double2* __restrict__ V,
                                            double* __restrict__ vsum) {
  const I nv = (I)(r1 - r0) * NP;
  const I stride = (I)gridDim.x * blockDim.x;
  I e = (I)blockIdx.x * blockDim.x + threadIdx.x;
  double* out = vsum + (size_t)r0 * NP;
  for (; e + 3 * stride < nv; e += 4 * stride) {
    double sv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const I eu = e + u * stride;
      const I h = r0 + eu / NP;
      const int c = (int)(eu % NP);
      sv[u] = 0.0;
      if (c < m) {
        const double2 v = __ldg(V + (size_t)h * ldv + c);
        sv[u] = v.x + v.y;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) out[e + u * stride] = sv[u];
  }
  for (; e < nv; e += stride) {
    const I h = r0 + e / NP;
    const int c = (int)(e % NP);
    double sv = 0.0;
    if (c < m) {
      const double2 v = __ldg(V + (size_t)h * ldv + c);
      sv = v.x + v.y;
    }
    out[e] = sv;
  }
}
__device__ __forceinline__ void vsum_rows(int r0, int r1, int m, int ldv, int NP, const double2* __restrict__ V,
                                          double* __restrict__ vsum) {
  if ((int64_t)(r1 - r0) * NP + 4LL * gridDim.x * blockDim.x < 2147483647LL)
    vsum_rows_t<int>(r0, r1, m, ldv, NP, V, vsum);
  else
    vsum_rows_t<int64_t>(r0, r1, m, ldv, NP, V, vsum);
}

__device__ __forceinline__ void prep_ext_rows(int d, int n, int64_t E, int32_t* __restrict__ etab,
                                              int32_t* __restrict__ umap);

// The staging kernel of a projection: P table, gsum plane, the Vsum rows [0, vrows), and in the same launch
// (one launch instead of three host API calls for small, launch-bound pencils) the shared-row tables when etab
// is given, the split-K arrival counters zeroed, and optionally the caller's status word zeroed (prony_pencil).
__global__ void k_prep(int d, int n, int N, int m, int ldv, int NP, int64_t box, const double2* __restrict__ grid,
                       const double2* __restrict__ V, int32_t* __restrict__ ptab, double* __restrict__ gsum,
                       double* __restrict__ vsum, int vrows, int64_t E, int32_t* __restrict__ etab,
                       int32_t* __restrict__ umap, int* __restrict__ counters, int ncounters,
                       int32_t* __restrict__ zero_status) {
  if (etab) prep_ext_rows(d, n, E, etab, umap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncounters; i += gridDim.x * blockDim.x) counters[i] = 0;
  if (zero_status && blockIdx.x == 0 && threadIdx.x == 0) *zero_status = 0;
  const int L = 2 * n + 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t k = t0; k < N + kPtabPad; k += stride) {
    if (k >= N) {
      ptab[k] = 0;
      continue;
    }
    int r = (int)k, P = 0, s = 1;
    for (int i = d - 1; i >= 0; --i) {  // last coordinate fastest, stride 1
      P += (r % (n + 1)) * s;
      r /= (n + 1);
      s *= L;
    }
    ptab[k] = P;
  }
  for (int64_t e = t0; e < box; e += stride) {
    const double2 v = grid[e];
    gsum[e] = v.x + v.y;
  }
  vsum_rows(0, vrows, m, ldv, NP, V, vsum);
}

// Vsum rows [r0, r1) (the part of V that arrives after k_prep ran, prony_pencil_host)
__global__ void k_vsum(int r0, int r1, int m, int ldv, int NP, const double2* __restrict__ V, double* __restrict__ vsum) {
  vsum_rows(r0, r1, m, ldv, NP, V, vsum);
}

// Shared-row tables (F8): for e in E = {0..n+1}^d with coordinates c (base n+2, last
// fastest): etab[e] = sum_i c_i L^(d-1-i), so T_E[e,h] = grid[etab[e] - P(h) + C0]; and for each l,
// umap[l][e] = index in I_n of k = c - e_l when that k lies in I_n (then T_l[k,:] = T_E[e,:]), else -1.
__device__ __forceinline__ void prep_ext_rows(int d, int n, int64_t E, int32_t* __restrict__ etab,
                                              int32_t* __restrict__ umap) {
  const int L = 2 * n + 2, Le = n + 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E + kPtabPad;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e >= E) {
      etab[e] = 0;
      continue;
    }
    int c[PRONY_MAX_D];
    int64_t r = e;
    for (int i = d - 1; i >= 0; --i) {
      c[i] = (int)(r % Le);
      r /= Le;
    }
    int P = 0, s = 1;
    for (int i = d - 1; i >= 0; --i) {
      P += c[i] * s;
      s *= L;
    }
    etab[e] = P;
    for (int l = 0; l < d; ++l) {  // S_{l+1}: shift e_{l+1} is coordinate l
      int idx = 0;
      bool ok = c[l] >= 1;
      for (int i = 0; i < d; ++i) {
        const int k = c[i] - (i == l ? 1 : 0);
        ok = ok && k <= n;
        idx = idx * (n + 1) + k;
      }
      umap[(int64_t)l * E + e] = ok ? idx : -1;
    }
  }
}

// ---------------------------------------------------------------------------- projection
// Warp-specialized CTA of kThreads = 512 threads: warpgroups 0-2 are consumers (12 warps =
// WM x WN, warp tile 16 rows x 8*nt_active columns, 3M/4M DMMA; setmaxnreg 152 registers),
// warpgroup 3 is the producer (setmaxnreg 40): it fills a kStages-deep ring of kBK-column stages
// with cp.async and signals each stage on a "full" mbarrier (cp.async.mbarrier.arrive); consumers
// release a stage on its "empty" mbarrier. No CTA-wide barrier in the main loop.
//   A planes  Ac[kc][r] = T_l[k_r][h0+kc] = grid[P(k_r) + s_l + C0 - P(h0+kc)],  As = gsum[same]
//             (implicit Toeplitz gather straight from the L2/L1-resident grid, zero-filled outside)
//   B planes  Bc[kc][c] = V[h0+kc][c], Bs[kc][c] = Vsum[h0+kc][c] (zero-filled for c >= m, h >= h_end)
// CTA tile: BM = 16*WM rows of T_l x NP = 8*ceil(m/8) columns of V (n-tiles split near-evenly
// over the WN column warps, <= NT <= 4 each).
#ifndef PRONY_CONSUMER_WARPS
#define PRONY_CONSUMER_WARPS 12
#endif
constexpr int kConsumerWarps = PRONY_CONSUMER_WARPS;    // 12 (3 warpgroups) or 8 (2 warpgroups)
constexpr int kThreads = 32 * (kConsumerWarps + 4);     // + the producer warpgroup
constexpr int kReduceThreads = 512;
constexpr int kGatherThreads = 96;  // producer threads doing the A gather (warp 3 issues the B bulk copies)
#ifndef PRONY_CONSUMER_REGS
#define PRONY_CONSUMER_REGS (PRONY_CONSUMER_WARPS == 12 ? 160 : 232)
#endif
#ifndef PRONY_PRODUCER_REGS
#define PRONY_PRODUCER_REGS (PRONY_CONSUMER_WARPS == 12 ? 32 : 40)
#endif
#ifndef PRONY_KK_UNROLL
#define PRONY_KK_UNROLL 4
#endif
#ifndef PRONY_PROJ_SREG
#define PRONY_PROJ_SREG 0
#endif
// SREG: the 3M sum operands formed in the consumers' registers (no gsum / Vsum planes gathered or copied)
constexpr bool kProjSreg = PRONY_PROJ_SREG != 0;
constexpr int kKkUnroll = PRONY_KK_UNROLL;
constexpr int kConsumerRegs = PRONY_CONSUMER_REGS;  // 384 x 160 + 128 x 32 = 65536 (12 warps); 256 x 240 + 4096 (8)
constexpr int kProducerRegs = PRONY_PRODUCER_REGS;
// setmaxnreg only redistributes the CTA's launch-time register pool (kThreads x the per-thread count
// ptxas assigns under __launch_bounds__(kThreads, 1), a multiple of 8): the split must fit in it or
// the consumers' allocation never succeeds
constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8 > 255 ? 255 : (65536 / kThreads) / 8 * 8;
static_assert(kConsumerRegs * 32 * kConsumerWarps + kProducerRegs * 128 <= kLaunchRegs * kThreads,
              "setmaxnreg split exceeds the CTA register pool");

template <int NT, int WN>
struct ProjTile {
  static constexpr int WM = kConsumerWarps / WN;
  static constexpr int BM = 16 * WM;
  static constexpr int NPMAX = 8 * NT * WN;          // smem capacity (NP <= NPMAX)
  static constexpr int LDA = BM + 2, LDAS = BM + 4;  // double2 / double strides (conflict-free)
  static constexpr int LDB = NPMAX + 2, LDBS = NPMAX + 4;
  static constexpr int A_C = 0;                      // offsets in doubles within a stage
  static constexpr int A_S = A_C + kBK * LDA * 2;
  static constexpr int B_C = A_S + kBK * LDAS;
  static constexpr int B_S = B_C + kBK * LDB * 2;
  static constexpr int STAGE = B_S + kBK * LDBS;
  static constexpr int BAR = kStages * STAGE;        // mbarriers after the stages (2 per stage)
  static constexpr int PAT = BAR + 2 * kStages;      // row table P(k_r) + s_l + C0 (BM ints)
  static constexpr size_t SMEM = (size_t)PAT * sizeof(double) + (size_t)(BM + 4) * sizeof(int);
  static_assert(STAGE % 2 == 0, "stage must keep 16-byte alignment");
  // A-gather threads of the producer warpgroup: warps 0-2 (warp 3 issues the B bulk copies). ROWOWNER: BM divides
  // them (BM = 96, 48: the m <= 80 shapes), so every gather thread owns whole rows of the tile. For BM = 64 (m > 80)
  // the element-strided gather is kept: the row-owner forms measured slower there (64 owners: 29.0 ms, all 128
  // producer threads with warp 3 also gathering: 29.4 ms, vs 28.5 ms at cfg4) — that producer already runs ahead
  // of the DMMA-bound consumers, and the variants changed the consumers' register allocation (spills in the loop)
  static constexpr bool ROWOWNER = 96 % BM == 0 && kBK % (96 / BM) == 0;
  static constexpr int GT = 96;
  static_assert(!ROWOWNER || (GT % BM == 0 && kBK % (GT / BM) == 0), "gather threads must own whole tile rows");
};

template <int NT, int WN, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_project(ProjParams p) {
  using T = ProjTile<NT, WN>;
  constexpr int WM = T::WM, BM = T::BM;
  extern __shared__ __align__(16) double smem[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t full0 = sbase + (uint32_t)T::BAR * 8u;       // full[s]  at full0 + 8 s
  const uint32_t empty0 = full0 + (uint32_t)kStages * 8u;     // empty[s] at empty0 + 8 s

  const int tid = threadIdx.x;
  const int l = blockIdx.z;
  const int rows = p.rows[l];
  const int rb0 = blockIdx.x * BM;
  if (rb0 >= rows) return;  // whole CTA exits together
  const int chunk = blockIdx.y + p.chunk_base;
  const int h_begin = chunk == 0 ? 0 : p.chunk0_w + (chunk - 1) * p.chunk_w;
  const int h_end = min(h_begin + (chunk == 0 ? p.chunk0_w : p.chunk_w), p.N);
  const int KT = (h_end - h_begin + kBK - 1) / kBK;
  const int m = p.m, N = p.N, NP = p.NP;

  // zero the B planes of every slot once: padding columns [m, NP) are never written by the bulk
  // copies, and rows past h_end of a partial last stage must not hold garbage (A is 0 there)
  for (int s = 0; s < kStages; ++s)
    for (int e = tid; e < kBK * (T::LDB * 2 + T::LDBS); e += kThreads) smem[s * T::STAGE + T::B_C + e] = 0.0;
  int* sPA = reinterpret_cast<int*>(smem + T::PAT);
  for (int r = tid; r < BM; r += kThreads)
    sPA[r] = (rb0 + r < rows) ? p.rtab[p.kb[l] + rb0 + r] + p.shift[l] : -1;  // -1: row outside
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8u * s, T::GT + 1);  // A-gather cp.async arrivals + B expect_tx
      mbar_init(empty0 + 8u * s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= kConsumerWarps * 32) {
    // ================================================================== producer warpgroup
    setmaxnreg_dec<kProducerRegs>();
    const int pt = tid - kConsumerWarps * 32;  // 0..127
    const int plane = pt & 31;
    const int32_t* __restrict__ ptab = p.ptab;
    if constexpr (T::ROWOWNER) {
      // A gather, row-owner form (BM = 96, 48): gather thread pt < GT owns row ra = pt % BM of the tile for the
      // whole CTA (its P(k_ra) + shift read once from the row table) and columns kc0, kc0 + TPR, ... of every stage;
      // P(h0 + kc) comes from lane kc (shfl). Per element: one shfl, one subtraction, the two cp.async (immediate
      // smem offsets). (The round-1/2 form decomposed e = pt + 96 j into (kc, ra) and re-read the row table per
      // element, ~30 instructions per element: at m = 30 its consumers waited on the full barrier 7.8% of their
      // samples.) Warp 3 first issues the stage's B rows: one bulk copy per V row (lanes 0..15) and per Vsum row
      // (lanes 16..31), completing on the same full barrier (expect_tx).
      const double2* __restrict__ grid = p.grid;
      const double* __restrict__ gsum = p.gsum;
      const double2* __restrict__ V = p.V;
      const double* __restrict__ vsum = p.vsum;
      constexpr int TPR = T::GT / BM, KPT = kBK / TPR;
      const bool gather = pt < T::GT, bwarp = pt >= 96;
      const int ra = pt % BM, kc0 = (pt / BM) % TPR;
      const int pa = sPA[ra];
      const uint32_t dA = (uint32_t)(T::A_C + 2 * (kc0 * T::LDA + ra)) * 8u;
      const uint32_t dS = (uint32_t)(T::A_S + kc0 * T::LDAS + ra) * 8u;
      const int kr = plane & (kBK - 1);
      const bool sum_plane = plane >= kBK;
      const uint32_t bytes_row = (uint32_t)m * 16u + (MODE == 3 && !kProjSreg ? (uint32_t)NP * 8u : 0u);
      // lane i < kBK holds P(h0 + i) of the stage being issued (prefetched one stage ahead)
      int ph_next = (plane < kBK && h_begin + plane < N) ? __ldg(ptab + h_begin + plane) : 0;
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % kStages;
        const int h0 = h_begin + kt * kBK;
        const int ph = ph_next;
        const int hn = h0 + kBK + plane;
        ph_next = (plane < kBK && hn < N) ? __ldg(ptab + hn) : 0;
        if (kt >= kStages) mbar_wait(empty0 + 8u * s, (uint32_t)((kt / kStages) - 1) & 1u);
        const uint32_t st = sbase + (uint32_t)(s * T::STAGE) * 8u;
        if (bwarp) {
          const int nrows = min(kBK, h_end - h0);
          if (plane == 0) mbar_arrive_expect_tx(full0 + 8u * s, bytes_row * (uint32_t)nrows);
          __syncwarp();
          if (plane < 2 * kBK && kr < nrows) {
            const int h = h0 + kr;
            if (!sum_plane) {
              bulk_g2s(st + (uint32_t)(T::B_C + 2 * kr * T::LDB) * 8u, V + (size_t)h * p.ldv, (uint32_t)m * 16u,
                       full0 + 8u * s);
            } else if constexpr (MODE == 3 && !kProjSreg) {
              bulk_g2s(st + (uint32_t)(T::B_S + kr * T::LDBS) * 8u, vsum + (size_t)h * NP, (uint32_t)NP * 8u,
                       full0 + 8u * s);
            }
          }
        }
        if (gather) {
          const uint32_t stA = st + dA, stS = st + dS;
          const int kcut = pa >= 0 ? h_end - h0 : 0;  // columns kc < kcut hold data (zero-filled otherwise)
          auto elem = [&](auto j_c) {
            constexpr int j = decltype(j_c)::value;
            const int kc = kc0 + TPR * j;
            const int phc = __shfl_sync(0xffffffffu, ph, kc);
            const bool ok = kc < kcut;
            int idx = ok ? pa - phc : 0;
            PRONY_CHECK_INDEX(idx, 0, p.box);
            cp_async16_at<TPR * j * T::LDA * 16>(stA, grid + idx, ok ? 16 : 0);
            if constexpr (MODE == 3 && !kProjSreg) cp_async8_at<TPR * j * T::LDAS * 8>(stS, gsum + idx, ok ? 8 : 0);
          };
          static_for<KPT>(elem);
          mbar_arrive_cp_async(full0 + 8u * s);
        }
      }
      if (gather) cp_async_wait<0>();
    } else {
      if (pt < kGatherThreads) {
        // element-strided A gather over the kBK x BM tile: element e = pt + kGatherThreads * j -> (kc = e / BM,
        // ra = e % BM); P(k_ra) + shift from the shared row table sPA, P(h0 + kc) from lane kc (shfl)
        const double2* __restrict__ grid = p.grid;
        const double* __restrict__ gsum = p.gsum;
        // lane i < kBK holds P(h0 + i) of the stage being issued (prefetched one stage ahead)
        int ph_next = (plane < kBK && h_begin + plane < N) ? __ldg(ptab + h_begin + plane) : 0;
        for (int kt = 0; kt < KT; ++kt) {
          const int s = kt % kStages;
          const int h0 = h_begin + kt * kBK;
          const int ph = ph_next;
          const int hn = h0 + kBK + plane;
          ph_next = (plane < kBK && hn < N) ? __ldg(ptab + hn) : 0;
          if (kt >= kStages) mbar_wait(empty0 + 8u * s, (uint32_t)((kt / kStages) - 1) & 1u);
          const uint32_t st = sbase + (uint32_t)(s * T::STAGE) * 8u;
#pragma unroll 2
          for (int e = pt; e < kBK * BM; e += kGatherThreads) {
            const int kc = e / BM, ra = e % BM;
            const int phc = __shfl_sync(0xffffffffu, ph, kc);
            const int pa = sPA[ra];
            const bool ok = (pa >= 0) && (h0 + kc < h_end);
            int idx = ok ? pa - phc : 0;
            PRONY_CHECK_INDEX(idx, 0, p.box);
            cp_async16(st + (uint32_t)(T::A_C + 2 * (kc * T::LDA + ra)) * 8u, grid + idx, ok ? 16 : 0);
            if constexpr (MODE == 3 && !kProjSreg)
              cp_async8(st + (uint32_t)(T::A_S + kc * T::LDAS + ra) * 8u, gsum + idx, ok ? 8 : 0);
          }
          mbar_arrive_cp_async(full0 + 8u * s);
        }
        cp_async_wait<0>();
      } else {
        // B rows: one bulk copy per V row (lanes 0..15) and per Vsum row (lanes 16..31)
        const int kr = plane & (kBK - 1);
        const bool sum_plane = plane >= kBK;
        const double2* __restrict__ V = p.V;
        const double* __restrict__ vsum = p.vsum;
        for (int kt = 0; kt < KT; ++kt) {
          const int s = kt % kStages;
          const int h0 = h_begin + kt * kBK;
          if (kt >= kStages) mbar_wait(empty0 + 8u * s, (uint32_t)((kt / kStages) - 1) & 1u);
          const int nrows = min(kBK, h_end - h0);
          const uint32_t bytes_row = (uint32_t)m * 16u + (MODE == 3 && !kProjSreg ? (uint32_t)NP * 8u : 0u);
          if (plane == 0) mbar_arrive_expect_tx(full0 + 8u * s, bytes_row * (uint32_t)nrows);
          __syncwarp();
          const uint32_t st = sbase + (uint32_t)(s * T::STAGE) * 8u;
          if (plane < 2 * kBK && kr < nrows) {
            const int h = h0 + kr;
            if (!sum_plane) {
              bulk_g2s(st + (uint32_t)(T::B_C + 2 * kr * T::LDB) * 8u, V + (size_t)h * p.ldv, (uint32_t)m * 16u,
                       full0 + 8u * s);
            } else if constexpr (MODE == 3 && !kProjSreg) {
              bulk_g2s(st + (uint32_t)(T::B_S + kr * T::LDBS) * 8u, vsum + (size_t)h * NP, (uint32_t)NP * 8u,
                       full0 + 8u * s);
            }
          }
        }
      }
    }
    return;
  }

  // ==================================================================== consumer warpgroups
  setmaxnreg_inc<kConsumerRegs>();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int ntot = NP / 8;
  const int t0 = (ntot * wn) / WN;                    // first n-tile of this warp
  const int nt_active = (ntot * (wn + 1)) / WN - t0;  // <= NT

  double acc[3][NT][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;

  // the warp owning the last n-tile packs it when it holds <= 4 valid columns (3M only): 2 real products
  // instead of 3 on a half-empty tile (engine PK)
  const bool pk = MODE == 3 && (m % 8) != 0 && (m % 8) <= 4 && nt_active > 0 && t0 + nt_active == ntot;
  auto run = [&](auto na_c, auto pk_c) {
    constexpr int NA = decltype(na_c)::value;
    constexpr bool PK = decltype(pk_c)::value;
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % kStages;
      mbar_wait(full0 + 8u * s, (uint32_t)(kt / kStages) & 1u);
      if constexpr (NA > 0) {
        const double* st = smem + s * T::STAGE;
        const double2* Ac = reinterpret_cast<const double2*>(st + T::A_C) + wm * 16;
        const double* As = st + T::A_S + wm * 16;
        const double2* Bc = reinterpret_cast<const double2*>(st + T::B_C) + t0 * 8;
        const double* Bs = st + T::B_S + t0 * 8;
#pragma unroll kKkUnroll
        for (int kk = 0; kk < kBK / 4; ++kk)
          warp_cmma_k4<NT, NA, MODE, false, PK, kProjSreg>(acc, Ac + kk * 4 * T::LDA, As + kk * 4 * T::LDAS, T::LDA, T::LDAS,
                                                Bc + kk * 4 * T::LDB, Bs + kk * 4 * T::LDBS, T::LDB, T::LDBS, g, q);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8u * s);
    }
    // epilogue: Y[chunk][yoff_l + r][col], NP-wide rows (padding columns are zero). For NT <= 3 it runs here,
    // where NA and PK are compile-time (with the runtime form below, ptxas turns acc[.][nt_active-1] into a
    // dynamically indexed local-memory copy of acc for those shapes); for NT >= 4 after the dispatch
    // (measured: 28.45 vs 28.72 ms at cfg4 for the in-lambda form).
    if constexpr (NT <= 3) {
      const int r0 = rb0 + wm * 16 + g, r1 = r0 + 8;
      const size_t ybase = (size_t)chunk * p.R_tot + p.yoff[l];
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        double re[4], im[4];
        if constexpr (PK) {
          if (j == NA - 1) acc_packed_to_complex<NT>(acc, j, q, re, im);
          else acc_to_complex<NT, MODE>(acc, j, re, im);
        } else {
          acc_to_complex<NT, MODE>(acc, j, re, im);
        }
        const int col = (t0 + j) * 8 + 2 * q;
        if (r0 < rows) {
          double2* y = p.Y + (ybase + r0) * NP + col;
          y[0] = make_double2(re[0], im[0]);
          y[1] = make_double2(re[1], im[1]);
        }
        if (r1 < rows) {
          double2* y = p.Y + (ybase + r1) * NP + col;
          y[0] = make_double2(re[2], im[2]);
          y[1] = make_double2(re[3], im[3]);
        }
      }
    }
  };
  auto run_na = [&](auto na_c) {
    if (pk) run(na_c, std::true_type{});
    else run(na_c, std::false_type{});
  };
  if (nt_active == NT) {
    run_na(std::integral_constant<int, NT>{});
  } else if (nt_active == 0) {
    run(std::integral_constant<int, 0>{}, std::false_type{});
  } else if constexpr (NT > 1) {
    if (nt_active == NT - 1) {
      run_na(std::integral_constant<int, NT - 1>{});
    } else if constexpr (NT > 2) {
      if (nt_active == NT - 2) {
        run_na(std::integral_constant<int, NT - 2>{});
      } else if constexpr (NT > 3) {
        if (nt_active == NT - 3) run_na(std::integral_constant<int, NT - 3>{});
      }
    }
  }

  if constexpr (NT > 3) {
    const int r0 = rb0 + wm * 16 + g, r1 = r0 + 8;
    const size_t ybase = (size_t)chunk * p.R_tot + p.yoff[l];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j < nt_active) {
        double re[4], im[4];
        if (pk && j == nt_active - 1) acc_packed_to_complex<NT>(acc, j, q, re, im);
        else acc_to_complex<NT, MODE>(acc, j, re, im);
        const int col = (t0 + j) * 8 + 2 * q;
        if (r0 < rows) {
          double2* y = p.Y + (ybase + r0) * NP + col;
          y[0] = make_double2(re[0], im[0]);
          y[1] = make_double2(re[1], im[1]);
        }
        if (r1 < rows) {
          double2* y = p.Y + (ybase + r1) * NP + col;
          y[0] = make_double2(re[2], im[2]);
          y[1] = make_double2(re[3], im[3]);
        }
      }
    }
  }

  // split-K fixup: the last of the KC chunk CTAs of this row block sums the KC partial tiles in
  // fixed chunk order (deterministic whatever the arrival order) into chunk slot 0
  if (p.KC > 1) {
    constexpr int kCons = kConsumerWarps * 32;
    __threadfence();  // make this thread's partial-tile stores visible device-wide
    asm volatile("bar.sync 1, %0;\n" ::"r"(kCons) : "memory");
    int* flag = reinterpret_cast<int*>(smem + T::PAT) + BM;  // after the row table
    if (tid == 0) {
      const int old = atomicAdd(p.counters + l * p.nrb + blockIdx.x, 1);
      *flag = (old == p.KC - 1);
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(kCons) : "memory");
    if (*flag) {
      __threadfence();
      const int nr = min(BM, rows - rb0);
      const size_t cstride = (size_t)p.R_tot * NP;
      double2* y0 = p.Y + ((size_t)p.yoff[l] + rb0) * NP;
      for (int e = tid; e < nr * NP; e += kCons) {
        double2 s = __ldcg(y0 + e);
        for (int c = 1; c < p.KC; ++c) {
          const double2 v = __ldcg(y0 + c * cstride + e);
          s.x += v.x;
          s.y += v.y;
        }
        y0[e] = s;
      }
    }
  }
}

// ---------------------------------------------------------------------------- reduce
// grid (RP, d, ceil(NP/64)); CTA (p, l, jb) sums rows k in [rows*p/RP, rows*(p+1)/RP) of segment l,
// computed transposed so both operands stream as contiguous rows:
//   S_part[l][p][i][j] = sum_k conj(U[k][i]) Y[k][j]   <=>   S_part^T = Y^T conj(U)
// (Y = chunk slot 0, where k_project's last-arriving chunk CTA left the sum of the KC partials)
// A operand = Y_c rows (columns j in [64 jb, 64 jb + 64)), B operand = U rows under CONJB (conj).
// K loop over (16-row slab, chunk c) stages, kRedStages-deep cp.async ring; the 3M sum planes
// (Re+Im of Y, Re-Im of U) are formed in shared memory after each stage lands.
constexpr int kRedSlab = 16;
constexpr int kRedStages = 3;
template <int NT, int WN>
struct RedTile {
  static constexpr int WM = (kReduceThreads / 32) / WN;  // 4 (WN = 4) or 8 (WN = 2)
  static constexpr int BJ = 16 * WM;                      // rows j of S^T per CTA
  static constexpr int NPU = 8 * NT * WN;                 // capacity of the i dimension
  static constexpr int LDY = BJ + 2, LDYS = BJ + 4, LDU = NPU + 2, LDUS = NPU + 4;
  static constexpr int Y_C = 0, Y_S = Y_C + 2 * kRedSlab * LDY, U_C = Y_S + kRedSlab * LDYS,
                       U_S = U_C + 2 * kRedSlab * LDU, STAGE = U_S + kRedSlab * LDUS;
  static constexpr size_t SMEM = kRedStages * (size_t)STAGE * sizeof(double);
  static_assert(STAGE % 2 == 0 && Y_S % 2 == 0 && U_C % 2 == 0 && U_S % 2 == 0, "16-byte alignment");
};

template <int NT, int WN, int MODE>
__global__ void __launch_bounds__(kReduceThreads, 1) k_reduce(RedParams p) {
  using T = RedTile<NT, WN>;
  constexpr int WM = T::WM, BJ = T::BJ;
  extern __shared__ __align__(16) double rsm[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(rsm);
  const int l = blockIdx.y;
  const int P = blockIdx.x;
  const int j0 = blockIdx.z * BJ;
  const int rows = p.rows[l];
  const int rbeg = (int)((int64_t)rows * P / p.RP), rend = (int)((int64_t)rows * (P + 1) / p.RP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int m = p.m, NP = p.NP, KC = p.KC;
  const int ntot = (m + 7) / 8;  // n-tiles over i
  const int t0 = (ntot * wn) / WN;
  const int nt_active = (ntot * (wn + 1)) / WN - t0;
  const bool warp_rows = (j0 + wm * 16) < NP;
  const int nslab = (rend - rbeg + kRedSlab - 1) / kRedSlab;
  const int nstage = nslab * KC;

  auto issue = [&](int stg, int buf) {
    const int slab = stg / KC, c = stg % KC;
    const int r0 = rbeg + slab * kRedSlab;
    const uint32_t st = sbase + (uint32_t)(buf * T::STAGE) * 8u;
    for (int e = tid; e < kRedSlab * BJ; e += kReduceThreads) {
      const int r = e / BJ, jj = e % BJ;
      const int row = r0 + r, j = j0 + jj;
      const bool ok = row < rend && j < NP;
      const double2* src = p.Y + (ok ? ((size_t)c * p.R_tot + p.yoff[l] + row) * NP + j : 0);
      cp_async16(st + (uint32_t)(T::Y_C + 2 * (r * T::LDY + jj)) * 8u, src, ok ? 16 : 0);
    }
    // U rows: the row map is loaded for all of this thread's elements first (independent loads in
    // flight together), then the copies are issued
    constexpr int kUPer = (kRedSlab * T::NPU + kReduceThreads - 1) / kReduceThreads;
    int urows[kUPer];
#pragma unroll
    for (int u = 0; u < kUPer; ++u) {
      const int e = tid + u * kReduceThreads;
      const int row = r0 + e / T::NPU;
      int urow = p.kb[l] + row;
      if (p.umap && row < rend && e < kRedSlab * T::NPU) urow = __ldg(p.umap + (size_t)l * p.E + urow);  // -1: none
      urows[u] = urow;
    }
#pragma unroll
    for (int u = 0; u < kUPer; ++u) {
      const int e = tid + u * kReduceThreads;
      if (e < kRedSlab * T::NPU) {
        const int r = e / T::NPU, i = e % T::NPU;
        const int row = r0 + r;
        const bool ok = row < rend && i < m && urows[u] >= 0;
        const double2* src = p.U + (ok ? (size_t)urows[u] * m + i : 0);
        cp_async16(st + (uint32_t)(T::U_C + 2 * (r * T::LDU + i)) * 8u, src, ok ? 16 : 0);
      }
    }
    cp_async_commit();
  };

  double acc[3][NT][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;

#pragma unroll
  for (int s = 0; s < kRedStages - 1; ++s) {
    if (s < nstage) issue(s, s);
    else cp_async_commit();
  }
  for (int stg = 0; stg < nstage; ++stg) {
    const int buf = stg % kRedStages;
    cp_async_wait<kRedStages - 2>();
    __syncthreads();
    // refill the slot consumed in the previous iteration (all threads passed the barrier above)
    if (stg + kRedStages - 1 < nstage) issue(stg + kRedStages - 1, (stg + kRedStages - 1) % kRedStages);
    else cp_async_commit();
    double* sb = rsm + buf * T::STAGE;
    if constexpr (MODE == 3) {  // sum planes: Re+Im of Y, Re-Im of U (the B operand is conj(U))
      const double2* Yc = reinterpret_cast<const double2*>(sb + T::Y_C);
      const double2* Uc = reinterpret_cast<const double2*>(sb + T::U_C);
      for (int e = tid; e < kRedSlab * BJ; e += kReduceThreads) {
        const int r = e / BJ, jj = e % BJ;
        const double2 v = Yc[r * T::LDY + jj];
        sb[T::Y_S + r * T::LDYS + jj] = v.x + v.y;
      }
      for (int e = tid; e < kRedSlab * T::NPU; e += kReduceThreads) {
        const int r = e / T::NPU, i = e % T::NPU;
        const double2 v = Uc[r * T::LDU + i];
        sb[T::U_S + r * T::LDUS + i] = v.x - v.y;
      }
      __syncthreads();
    }
    if (warp_rows) {
      const double2* Ac = reinterpret_cast<const double2*>(sb + T::Y_C) + wm * 16;
      const double* As = sb + T::Y_S + wm * 16;
      const double2* Bc = reinterpret_cast<const double2*>(sb + T::U_C) + t0 * 8;
      const double* Bs = sb + T::U_S + t0 * 8;
#pragma unroll
      for (int kk = 0; kk < kRedSlab / 4; ++kk)
        warp_cmma_k4_n<NT, MODE, true>(nt_active, acc, Ac + kk * 4 * T::LDY, As + kk * 4 * T::LDYS, T::LDY,
                                       T::LDYS, Bc + kk * 4 * T::LDU, Bs + kk * 4 * T::LDUS, T::LDU, T::LDUS, g, q);
    }
  }
  // acc rows = j, columns = i  ->  S_part[i][j]
  double2* out = p.Spart + ((size_t)l * p.RP + P) * m * m;
  const int ja = j0 + wm * 16 + g, jb = ja + 8;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if (t < nt_active) {
      double re[4], im[4];
      acc_to_complex<NT, MODE>(acc, t, re, im);
      const int i = (t0 + t) * 8 + 2 * q;
      if (ja < m) {
        if (i < m) out[(size_t)i * m + ja] = make_double2(re[0], im[0]);
        if (i + 1 < m) out[(size_t)(i + 1) * m + ja] = make_double2(re[1], im[1]);
      }
      if (jb < m) {
        if (i < m) out[(size_t)i * m + jb] = make_double2(re[2], im[2]);
        if (i + 1 < m) out[(size_t)(i + 1) * m + jb] = make_double2(re[3], im[3]);
      }
    }
  }
}

// ---------------------------------------------------------------------------- warp-specialized reduce
// k_reduce_ws (3M, the default): the same S_part[l][P] = U[rows_P]^* Y[rows_P] (computed transposed,
// S^T = Y^T conj(U)) with 8 consumer warps of 232 registers (WM = 4 along j -> 64-row j-blocks, WN = 2 along
// i with up to 8 n-tiles per warp; the last n-tile packed when m % 8 <= 4) fed by ONE producer warp through a
// kRedWsStages-deep ring of 16-row slabs: lanes 0..15 move the slab's Y rows (columns [j0, j0 + BJ)) and
// lanes 16..31 its U rows (through the row map) with one bulk copy each, completing on the stage's "full"
// mbarrier (expect_tx); a U row with no data (no row of T_l, or past the partition) is zeroed in place
// first. The 3M sum operands are formed in the consumers' registers (warp_cmma_k4 SREG), so the producer
// does no arithmetic and nothing waits for a sum plane; consumers release slabs on "empty". Grid
// (RP, d, nj): every j-block takes the same row partitions (the U rows, which dominate the traffic, cost
// the same for each); rp_j[z] < RP would make the extra CTAs write zero partials.
constexpr int kRedWsStages = 4;
constexpr int kRwsCons = 8;                        // consumer warps: WM = 4 along j x WN = 2 along i
constexpr int kRwsThreads = 32 * (kRwsCons + 4);   // + the producer warpgroup (warp 0 of it copies)
constexpr int kRwsConsRegs = 232, kRwsProdRegs = 40;  // 256 x 232 + 128 x 40 = 64512 <= 65536
template <int NT, int WN>
struct RedWsTile {
  static constexpr int WM = kRwsCons / WN;
  static constexpr int BJ = 16 * WM;       // rows j of S^T per CTA
  static constexpr int NPU = 8 * NT * WN;  // capacity of the i dimension
  static constexpr int LDA = BJ + 2, LDB = NPU + 2;
  static constexpr int A_C = 0, B_C = A_C + 2 * kRedSlab * LDA, STAGE = B_C + 2 * kRedSlab * LDB;
  static constexpr int BAR = kRedWsStages * STAGE;  // 2 mbarriers per stage
  static constexpr size_t SMEM = (size_t)(BAR + 2 * kRedWsStages) * sizeof(double);
  static_assert(STAGE % 2 == 0 && B_C % 2 == 0, "16-byte alignment");
};

template <int NT, int WN>
__global__ void __launch_bounds__(kRwsThreads, 1) k_reduce_ws(RedParams p) {
  using T = RedWsTile<NT, WN>;
  constexpr int WM = T::WM, BJ = T::BJ;
  extern __shared__ __align__(16) double smem[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t full0 = sbase + (uint32_t)T::BAR * 8u, empty0 = full0 + (uint32_t)kRedWsStages * 8u;
  const int tid = threadIdx.x;
  const int l = blockIdx.y, P = blockIdx.x, jb = blockIdx.z;
  const int j0 = jb * BJ;
  const int m = p.m, NP = p.NP;
  const int RPj = p.rp_j[jb];
  double2* out = p.Spart + ((size_t)l * p.RP + P) * m * m;
  if (P >= RPj) {  // this j-block needs fewer partitions: its columns of this partial are zero
    for (int e = tid; e < m * BJ; e += kRwsThreads) {
      const int i = e / BJ, j = j0 + e % BJ;
      if (j < m) out[(size_t)i * m + j] = make_double2(0.0, 0.0);
    }
    return;
  }
  const int rows = p.rows[l];
  const int rbeg = (int)((int64_t)rows * P / RPj), rend = (int)((int64_t)rows * (P + 1) / RPj);
  const int nslab = (rend - rbeg + kRedSlab - 1) / kRedSlab;
  const int ny = min(BJ, NP - j0);  // Y columns this j-block reads

  // zero once: padding columns (i >= m, j >= ny) are never written by the copies
  for (int e = tid; e < kRedWsStages * T::STAGE; e += kRwsThreads) smem[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < kRedWsStages; ++s) {
      mbar_init(full0 + 8u * s, 1);
      mbar_init(empty0 + 8u * s, kRwsCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= kRwsCons * 32) {
    // ================================================================== producer warp
    setmaxnreg_dec<kRwsProdRegs>();
    if (tid >= kRwsCons * 32 + 32) return;
    const int lane = tid & 31;
    const int r = lane & (kRedSlab - 1);
    for (int st = 0; st < nslab; ++st) {
      const int s = st % kRedWsStages;
      if (st >= kRedWsStages) mbar_wait(empty0 + 8u * s, (uint32_t)((st / kRedWsStages) - 1) & 1u);
      const int row = rbeg + st * kRedSlab + r;
      uint32_t bytes = 0;
      const double2* src = nullptr;
      uint32_t dst = sbase + (uint32_t)(s * T::STAGE) * 8u;
      if (lane < kRedSlab) {  // Y row (a row past the partition keeps stale finite data: its U row is zero)
        if (row < rend) {
          bytes = (uint32_t)ny * 16u;
          src = p.Y + ((size_t)p.yoff[l] + row) * NP + j0;
        }
        dst += (uint32_t)(T::A_C + 2 * r * T::LDA) * 8u;
      } else {  // U row through the map
        int urow = -1;
        if (row < rend) {
          urow = p.kb[l] + row;
          if (p.umap) urow = __ldg(p.umap + (size_t)l * p.E + urow);  // -1: no row of T_l
        }
        double2* Urow = reinterpret_cast<double2*>(smem + s * T::STAGE + T::B_C) + r * T::LDB;
        if (urow >= 0) {
          bytes = (uint32_t)m * 16u;
          src = p.U + (size_t)urow * m;
        } else {
          for (int i = 0; i < m; ++i) Urow[i] = make_double2(0.0, 0.0);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // before later bulk writes of the row
        }
        dst += (uint32_t)(T::B_C + 2 * r * T::LDB) * 8u;
      }
      uint32_t tot = bytes;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
      __syncwarp();  // the zeroed rows are ordered before the release below
      if (lane == 0) mbar_arrive_expect_tx(full0 + 8u * s, tot);
      __syncwarp();
      if (bytes) bulk_g2s(dst, src, bytes, full0 + 8u * s);
    }
    return;
  }

  // ==================================================================== consumer warpgroups
  setmaxnreg_inc<kRwsConsRegs>();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int ntot = (m + 7) / 8;  // n-tiles over i
  const int t0 = (ntot * wn) / WN;
  const int nt_active = (ntot * (wn + 1)) / WN - t0;
  const bool warp_rows = (j0 + wm * 16) < NP;
  const bool pk = (m % 8) != 0 && (m % 8) <= 4 && nt_active > 0 && t0 + nt_active == ntot;

  double acc[3][NT][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;

  auto run = [&](auto na_c, auto pk_c) {
    constexpr int NA = decltype(na_c)::value;
    constexpr bool PK = decltype(pk_c)::value;
    for (int st = 0; st < nslab; ++st) {
      const int s = st % kRedWsStages;
      mbar_wait(full0 + 8u * s, (uint32_t)(st / kRedWsStages) & 1u);
      if constexpr (NA > 0) {
        const double* sp = smem + s * T::STAGE;
        const double2* Ac = reinterpret_cast<const double2*>(sp + T::A_C) + wm * 16;
        const double2* Bc = reinterpret_cast<const double2*>(sp + T::B_C) + t0 * 8;
#pragma unroll
        for (int kk = 0; kk < kRedSlab / 4; ++kk)
          warp_cmma_k4<NT, NA, 3, true, PK, true>(acc, Ac + kk * 4 * T::LDA, nullptr, T::LDA, 0,
                                                  Bc + kk * 4 * T::LDB, nullptr, T::LDB, 0, g, q);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8u * s);
    }
    // acc rows = j, columns = i  ->  S_part[i][j] (NA, PK compile-time: static accumulator indices)
    const int ja = j0 + wm * 16 + g, jb2 = ja + 8;
#pragma unroll
    for (int t = 0; t < NA; ++t) {
      double re[4], im[4];
      if constexpr (PK) {
        if (t == NA - 1) acc_packed_to_complex<NT, true>(acc, t, q, re, im);
        else acc_to_complex<NT, 3>(acc, t, re, im);
      } else {
        acc_to_complex<NT, 3>(acc, t, re, im);
      }
      const int i = (t0 + t) * 8 + 2 * q;
      if (ja < m) {
        if (i < m) out[(size_t)i * m + ja] = make_double2(re[0], im[0]);
        if (i + 1 < m) out[(size_t)(i + 1) * m + ja] = make_double2(re[1], im[1]);
      }
      if (jb2 < m) {
        if (i < m) out[(size_t)i * m + jb2] = make_double2(re[2], im[2]);
        if (i + 1 < m) out[(size_t)(i + 1) * m + jb2] = make_double2(re[3], im[3]);
      }
    }
  };
  auto run_na = [&](auto na_c) {
    if (pk) run(na_c, std::true_type{});
    else run(na_c, std::false_type{});
  };
  if (!warp_rows || nt_active == 0) {
    run(std::integral_constant<int, 0>{}, std::false_type{});
  } else if (nt_active == NT) {
    run_na(std::integral_constant<int, NT>{});
  } else if constexpr (NT > 1) {
    if (nt_active == NT - 1) {
      run_na(std::integral_constant<int, NT - 1>{});
    } else if constexpr (NT > 2) {
      if (nt_active == NT - 2) {
        run_na(std::integral_constant<int, NT - 2>{});
      } else if constexpr (NT > 3) {
        if (nt_active == NT - 3) run_na(std::integral_constant<int, NT - 3>{});
      }
    }
  }
}

// S[l][i][j] = (sum_{p < RP} S_part[l][p][i][j]) / sigma_j   (fixed order).
// Scale guard (SPEC compute_S "sigma_m below underflow guard"): a sigma that is not
// finite and positive, or below N eps_M sigma_max (the rank rule of P:581), reports PRONY_ERR_SINGULAR
// in the status word; S is still written.
__global__ void k_finalize(int d, int m, int RP, const double2* __restrict__ Spart, const double* __restrict__ sigma,
                           double2* __restrict__ S, int N, int32_t* __restrict__ status) {
  if (status && blockIdx.x == 0 && threadIdx.x == 0) {
    double smax = 0.0;
    bool bad = false;
    for (int j = 0; j < m; ++j) {
      const double sj = sigma[j];
      if (!(sj > 0.0) || !isfinite(sj)) bad = true;
      else smax = fmax(smax, sj);
    }
    for (int j = 0; j < m && !bad; ++j)
      if (sigma[j] <= (double)N * 2.220446049250313e-16 * smax) bad = true;
    if (bad) set_status(status, PRONY_ERR_SINGULAR);
  }
  // a group of kFinLanes lanes per output: lane l sums P = l, l + kFinLanes, ... in order, then a fixed
  // shuffle tree (deterministic; independent load streams instead of one chain of RP dependent loads)
  constexpr int kFinLanes = 8;
  const int sub = threadIdx.x & (kFinLanes - 1);
  const int64_t total = (int64_t)d * m * m;
  const int64_t groups = ((int64_t)gridDim.x * blockDim.x) / kFinLanes;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kFinLanes; e < total + groups - 1 - (total + groups - 1) % groups; e += groups) {
    const bool live = e < total;
    const int l = live ? (int)(e / ((int64_t)m * m)) : 0;
    const int ij = live ? (int)(e % ((int64_t)m * m)) : 0;
    double2 s = make_double2(0.0, 0.0);
    if (live)
      for (int P = sub; P < RP; P += kFinLanes) {
        const double2 v = __ldcg(Spart + ((size_t)l * RP + P) * m * m + ij);
        s.x += v.x;
        s.y += v.y;
      }
#pragma unroll
    for (int off = kFinLanes / 2; off > 0; off >>= 1) {
      s.x += __shfl_down_sync(0xffffffffu, s.x, off, kFinLanes);
      s.y += __shfl_down_sync(0xffffffffu, s.y, off, kFinLanes);
    }
    if (live && sub == 0) {
      const double inv = 1.0 / sigma[ij % m];
      S[e] = make_double2(s.x * inv, s.y * inv);
    }
  }
}

// ---------------------------------------------------------------------------- host side
// k_project: 12 consumer warps = WM x WN. For m <= 80 (<= 10 n-tiles) WN = 2, WM = 6: each warp carries
// ceil(ntot/2) <= 5 n-tiles (A-fragment reuse) and a CTA covers 96 rows per gathered column (measured:
// cfg5 m = 30 6.9 ms vs 8.6 ms with WN = 3, cfg2 m = 20 -12%). Above that WN = 3, WM = 4 puts all column
// parts of one 16-row m-tile on the same SM sub-partition (warp w -> SMSP w % 4 = wm), so every SMSP
// gets exactly ceil(m/8) n-tiles of DMMA work per k-step; NT <= 5 keeps the 3M accumulators within 160
// registers.
// k_reduce: 16 warps, WN column warps with <= 4 n-tiles (3M accumulators within 128 registers).
ProjShape proj_shape(int m) {
  ProjShape s;
  const int ntot = (m + 7) / 8;
  if (kConsumerWarps == 8) {
    s.WN = 2;  // WM = 4: warp w -> SMSP w % 4 = wm, balanced; NT <= 8 (3M accumulators in 240 regs)
  } else if (ntot <= 10) {
    s.WN = 2;  // WM = 6, BM = 96: more n-tiles per warp (A-fragment reuse) and more rows per gathered column
  } else if (ntot <= 15) {
    s.WN = 3;
  } else {
    s.WN = 4;
  }
  const char* ewn = getenv("PRONY_PROJ_WN");  // experiments: force the column-warp count (2, 3, 4)
  if (ewn && kConsumerWarps == 12 && ewn[0] >= '2' && ewn[0] <= '4') {
    const int wn = ewn[0] - '0';
    if ((ntot + wn - 1) / wn <= (wn == 4 ? 4 : 5)) s.WN = wn;
  }
  s.NT = (ntot + s.WN - 1) / s.WN;
  s.WM = kConsumerWarps / s.WN;  // k_project consumer warps along rows
  s.BM = 16 * s.WM;              // k_project rows per CTA
  s.rWN = ntot <= 8 ? 2 : 4;
  s.rNT = (ntot + s.rWN - 1) / s.rWN;
  s.BI = 16 * (kReduceThreads / 32) / s.rWN;  // k_reduce rows j of S^T per CTA
  s.NP = 8 * ntot;
  return s;
}

int project_plan(const ProjGeom& g, int sm_count, ProjPlan* pl) {
  const ProjShape sh = proj_shape(g.m);
  pl->shape = sh;
  int R_tot = 0, max_rows = 0, row_blocks = 0;
  if (g.shared) {  // one product over rows [e0, e1) of T_E serves every l
    R_tot = max_rows = g.e1 - g.e0;
    row_blocks = (R_tot + sh.BM - 1) / sh.BM;
    for (int l = 0; l < g.d; ++l) pl->yoff[l] = 0;
  } else {
    for (int l = 0; l < g.d; ++l) {
      pl->yoff[l] = R_tot;
      R_tot += g.rows[l];
      max_rows = std::max(max_rows, g.rows[l]);
      row_blocks += (g.rows[l] + sh.BM - 1) / sh.BM;
    }
  }
  pl->R_tot = R_tot;
  pl->max_rows = max_rows;
  // split-K: chunk count KC minimizing waves x (chunk columns + pipeline fill), subject to
  // KC * R_tot <= kYCap max(d N, |E|) (workspace bound) and chunks of >= 64 columns.
  const int64_t cap_rows = (int64_t)kYCap * std::max<int64_t>((int64_t)g.d * g.N, ext_rows(g.d, g.n));
  int kc_max = (int)std::min<int64_t>(64, std::max<int64_t>(1, cap_rows / std::max(R_tot, 1)));
  kc_max = std::max(1, std::min(kc_max, std::max(1, g.N / 64)));
  double best = 1e30;
  int best_kc = 1;
  for (int kc = 1; kc <= kc_max; ++kc) {
    const double ctas = (double)row_blocks * kc;
    const double waves = std::ceil(ctas / sm_count);
    const double cost = waves * ((double)g.N / kc + 4.0 * kBK);
    if (cost < best - 1e-9) {
      best = cost;
      best_kc = kc;
    }
  }
  const char* ekc = getenv("PRONY_KC");  // experiments: force the chunk count (1 .. kc_max)
  if (ekc && atoi(ekc) >= 1) best_kc = std::min(atoi(ekc), kc_max);
  int chunk_w = (g.N + best_kc - 1) / best_kc;
  chunk_w = (chunk_w + kBK - 1) / kBK * kBK;
  pl->chunk_w = chunk_w;
  pl->chunk0_w = chunk_w;
  pl->KC = (g.N + chunk_w - 1) / chunk_w;  // every chunk non-empty
  // reduce partition: about 1 CTA per SM in total
  const int slabs = std::max(1, (max_rows + 15) / 16);
  if (cmul_mode() == 3) {
    // k_reduce_ws: 64-row j-blocks, the same row partitions for each (about one CTA per SM in total)
    const int nj = (sh.NP + 63) / 64;
    const int rp = std::max(1, std::min(slabs, sm_count / std::max(1, g.d * nj)));
    int rpmax = rp;
    for (int z = 0; z < 4; ++z) pl->rp_j[z] = z < nj ? rp : 0;
    pl->nj = nj;
    pl->RP = rpmax;
    return 0;
  }
  const int ib = (sh.NP + sh.BI - 1) / sh.BI;  // j-blocks of k_reduce
  int RP = sm_count / std::max(1, g.d * ib);
  RP = std::max(1, std::min(RP, slabs));
  pl->RP = RP;
  pl->nj = 0;
  return 0;
}

int64_t ext_rows(int d, int n) { return ipow(n + 2, d); }

namespace {
struct WsLayout {
  size_t ptab, etab, umap, gsum, vsum, Y, Spart, counters, total;
};
WsLayout ws_layout(int d, int n, int N, int m, int sm_count) {
  const ProjShape sh = proj_shape(m);
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  WsLayout w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  const int64_t E = ext_rows(d, n);
  w.ptab = take((size_t)(N + kPtabPad) * sizeof(int32_t));
  w.etab = take((size_t)(E + kPtabPad) * sizeof(int32_t));
  w.umap = take((size_t)d * E * sizeof(int32_t));
  w.gsum = take((size_t)box * sizeof(double));
  w.vsum = take((size_t)N * sh.NP * sizeof(double));
  // Y partials: KC * R_tot <= kYCap * max(dN, |E|)
  w.Y = take((size_t)kYCap * std::max<int64_t>((int64_t)d * N, E) * sh.NP * sizeof(double2));
  const int RP = std::max(1, sm_count / std::max(1, d));  // >= the partitions of either reduce kernel
  w.Spart = take((size_t)d * RP * m * m * sizeof(double2));
  w.counters = take((size_t)d * ((std::max<int64_t>(N, E) + 15) / 16 + 1) * sizeof(int));  // split-K arrivals
  w.total = off;
  return w;
}
}  // namespace

void project_plan_lead(const ProjGeom& g, ProjPlan* pl) {
  if (pl->KC < 2) return;
  const int64_t cap_rows = (int64_t)kYCap * std::max<int64_t>((int64_t)g.d * g.N, ext_rows(g.d, g.n));
  if ((int64_t)(pl->KC + 1) * std::max(pl->R_tot, 1) > cap_rows) return;  // no Y slot for one more chunk
  const char* eld = getenv("PRONY_LEAD_DIV");  // experiments: lead chunk = chunk_w / div (default 8)
  const int div = eld && atoi(eld) >= 1 ? atoi(eld) : 8;
  const int w0 = (pl->chunk_w / div + kBK - 1) / kBK * kBK;
  if (w0 < kBK || w0 >= g.N) return;
  int w = (g.N - w0 + pl->KC - 1) / pl->KC;
  w = (w + kBK - 1) / kBK * kBK;
  pl->chunk0_w = w0;
  pl->chunk_w = w;
  pl->KC = 1 + (g.N - w0 + w - 1) / w;
}

size_t project_workspace_bytes(int d, int n, int N, int m, int sm_count) {
  return ws_layout(d, n, N, m, sm_count).total;
}

template <int NT, int WN>
static int launch_project_t(const ProjParams& p, dim3 grid, cudaStream_t st, int mode, prony_exec_info* info) {
  const size_t smem = ProjTile<NT, WN>::SMEM;
  auto kp = mode == 4 ? k_project<NT, WN, 4> : k_project<NT, WN, 3>;
  if (ensure_smem_attr(kp, smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  if (info && info->ev_main_begin) cudaEventRecord((cudaEvent_t)info->ev_main_begin, st);
  kp<<<grid, kThreads, smem, st>>>(p);
  if (info && info->ev_main_end) cudaEventRecord((cudaEvent_t)info->ev_main_end, st);
  return PRONY_OK;
}

template <int NT, int WN>
static int launch_reduce_t(const RedParams& r, dim3 rgrid, cudaStream_t st, int mode) {
  auto kr = mode == 4 ? k_reduce<NT, WN, 4> : k_reduce<NT, WN, 3>;
  const size_t smem = RedTile<NT, WN>::SMEM;
  if (ensure_smem_attr(kr, smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  rgrid.z = (r.NP + RedTile<NT, WN>::BJ - 1) / RedTile<NT, WN>::BJ;
  kr<<<rgrid, kReduceThreads, smem, st>>>(r);
  return PRONY_OK;
}

template <int NT, int WN>
static int launch_reduce_ws_t(const RedParams& r, dim3 rgrid, cudaStream_t st) {
  const size_t smem = RedWsTile<NT, WN>::SMEM;
  if (ensure_smem_attr(k_reduce_ws<NT, WN>, smem) != cudaSuccess) return PRONY_ERR_CUDA;
  k_reduce_ws<NT, WN><<<rgrid, kRwsThreads, smem, st>>>(r);
  return PRONY_OK;
}

int project_launch(const ProjGeom& g, const ProjPlan& pl, const double2* grid, const double2* U, const double2* V,
                   const double* sigma, double2* S, void* ws, int sm_count, cudaStream_t st,
                   prony_exec_info* info, cudaEvent_t wait_before_reduce, int ell_base, int32_t* dev_status,
                   const ProjSplit* sp, cudaEvent_t ev_prepped, bool reset_status) {
  const WsLayout wl = ws_layout(g.d, g.n, g.N, g.m, sm_count);
  char* w = (char*)ws;
  int32_t* ptab = (int32_t*)(w + wl.ptab);
  int32_t* etab = (int32_t*)(w + wl.etab);
  int32_t* umap = (int32_t*)(w + wl.umap);
  double* gsum = (double*)(w + wl.gsum);
  double* vsum = (double*)(w + wl.vsum);
  double2* Y = (double2*)(w + wl.Y);
  double2* Spart = (double2*)(w + wl.Spart);
  int* counters = (int*)(w + wl.counters);
  const int64_t E = ext_rows(g.d, g.n);
  const int pslots = g.shared ? 1 : g.d;  // k_project row segments

  if (info) {
    info->launches = 0;
    info->main_grid[0] = info->main_grid[1] = info->main_grid[2] = 0;
    info->main_block = 0;
    info->split_k = 0;
    info->main_flops = 0.0;
  }
  if (pl.R_tot == 0) {
    if (cudaMemsetAsync(S, 0, (size_t)g.d * g.m * g.m * sizeof(double2), st) != cudaSuccess) return PRONY_ERR_CUDA;
    if (reset_status && dev_status && cudaMemsetAsync(dev_status, 0, sizeof(int32_t), st) != cudaSuccess)
      return PRONY_ERR_CUDA;
    if (ev_prepped && cudaEventRecord(ev_prepped, st) != cudaSuccess) return PRONY_ERR_CUDA;
    return PRONY_OK;
  }
  int64_t box = 1;
  for (int i = 0; i < g.d; ++i) box *= (2 * (int64_t)g.n + 2);
  const int nrb = (pl.max_rows + pl.shape.BM - 1) / pl.shape.BM;
  const bool split = sp && pl.KC > 1;
  const int vrows0 = split ? std::min(pl.chunk0_w, g.N) : g.N;
  k_prep<<<8 * sm_count, 256, 0, st>>>(g.d, g.n, g.N, g.m, g.m, pl.shape.NP, box, grid, V, ptab, gsum, vsum,
                                       vrows0, E, g.shared ? etab : nullptr, umap, counters,
                                       pl.KC > 1 ? pslots * nrb : 0, reset_status ? dev_status : nullptr);
  if (ev_prepped && cudaEventRecord(ev_prepped, st) != cudaSuccess) return PRONY_ERR_CUDA;

  ProjParams p{};
  p.grid = grid;
  p.gsum = gsum;
  p.V = V;
  p.ldv = g.m;
  p.vsum = vsum;
  p.ptab = ptab;
  p.rtab = g.shared ? etab : ptab;
  p.Y = Y;
  p.N = g.N;
  p.m = g.m;
  p.NP = pl.shape.NP;
  p.chunk_w = pl.chunk_w;
  p.chunk0_w = pl.chunk0_w;
  p.R_tot = pl.R_tot;
  p.KC = pl.KC;
  p.nrb = nrb;
  p.counters = counters;
  p.box = (int)box;
  const int L = 2 * g.n + 2;
  int64_t C0 = 0, s = 1;
  for (int i = 0; i < g.d; ++i) {
    C0 += (int64_t)g.n * s;
    s *= L;
  }
  for (int l = 0; l < g.d; ++l) {
    p.kb[l] = g.kb[l];
    p.rows[l] = g.rows[l];
    p.yoff[l] = pl.yoff[l];
    const int ell = l + ell_base;  // segment l holds T_ell (ell_base 1: S_1..S_d; 0: segment 0 is T)
    p.shift[l] = (int)(C0 + (ell >= 1 ? ipow(L, g.d - ell) : 0));  // s_ell = L^(d-ell)
  }
  if (g.shared) {  // one segment: rows [e0, e1) of T_E = [f(k'-h)]
    p.kb[0] = g.e0;
    p.rows[0] = pl.R_tot;
    p.yoff[0] = 0;
    p.shift[0] = (int)C0;
  }
  RedParams r{};
  r.Y = Y;
  r.U = U;
  r.umap = g.shared ? umap : nullptr;
  r.E = (int)E;
  r.Spart = Spart;
  r.m = g.m;
  r.NP = pl.shape.NP;
  r.KC = 1;  // k_project's fixup left the summed tile in chunk slot 0
  r.R_tot = pl.R_tot;
  r.RP = pl.RP;
  for (int l = 0; l < g.d; ++l) {
    r.kb[l] = g.shared ? g.e0 : g.kb[l];
    r.rows[l] = g.shared ? pl.R_tot : g.rows[l];
    r.yoff[l] = pl.yoff[l];
  }
  for (int z = 0; z < 4; ++z) r.rp_j[z] = pl.rp_j[z];
  dim3 grd((pl.max_rows + pl.shape.BM - 1) / pl.shape.BM, pl.KC, pslots);
  dim3 rgrd(pl.RP, g.d, (pl.shape.NP + pl.shape.BI - 1) / pl.shape.BI);
  const int NT = pl.shape.NT, WN = pl.shape.WN;
  const int mode = cmul_mode();
  auto launch_main = [&](const ProjParams& pp, dim3 gg, cudaStream_t ss, prony_exec_info* inf) -> int {
    switch (WN * 16 + NT) {
#define PRONY_CASE(nt, wn) \
  case wn * 16 + nt:       \
    return launch_project_t<nt, wn>(pp, gg, ss, mode, inf);
#if PRONY_CONSUMER_WARPS == 12
      PRONY_CASE(1, 2) PRONY_CASE(2, 2) PRONY_CASE(3, 2) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(1, 3)
      PRONY_CASE(2, 3) PRONY_CASE(3, 3) PRONY_CASE(4, 3) PRONY_CASE(5, 3) PRONY_CASE(4, 4)
#else
      PRONY_CASE(1, 2) PRONY_CASE(2, 2) PRONY_CASE(3, 2) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(6, 2)
      PRONY_CASE(7, 2) PRONY_CASE(8, 2)
#endif
#undef PRONY_CASE
      default:
        return PRONY_ERR_RANGE;
    }
  };
  int lrc = PRONY_OK;
  if (split) {
    // chunk 0 (V rows [0, chunk0_w), already resident) on st; chunks 1..KC-1 in up to kSplitStreams groups, each
    // on its own stream once its V rows are in (the caller's copy events) and its Vsum rows are formed
    if (cudaEventRecord(sp->ev_a, st) != cudaSuccess) return PRONY_ERR_CUDA;
    lrc = launch_main(p, dim3(grd.x, 1, grd.z), st, info);
    if (lrc != PRONY_OK) return lrc;
    const int nrest = pl.KC - 1, ng = std::min(kSplitStreams, nrest);
    for (int gi = 0; gi < ng; ++gi) {
      const int c_lo = 1 + nrest * gi / ng, c_hi = 1 + nrest * (gi + 1) / ng;  // chunks [c_lo, c_hi)
      const int r0 = pl.chunk0_w + (c_lo - 1) * pl.chunk_w;
      const int r1 = std::min(pl.chunk0_w + (c_hi - 1) * pl.chunk_w, g.N);
      cudaStream_t ss = sp->s_rest[gi];
      if (cudaStreamWaitEvent(ss, sp->ev_a, 0) != cudaSuccess ||
          cudaStreamWaitEvent(ss, sp->ev_chunk[std::min(c_hi - 2, kMaxChunkEv - 1)], 0) != cudaSuccess)
        return PRONY_ERR_CUDA;
      k_vsum<<<8 * sm_count, 256, 0, ss>>>(r0, r1, g.m, g.m, pl.shape.NP, V, vsum);
      ProjParams pr = p;
      pr.chunk_base = c_lo;
      lrc = launch_main(pr, dim3(grd.x, c_hi - c_lo, grd.z), ss, nullptr);
      if (lrc != PRONY_OK) return lrc;
      if (cudaEventRecord(sp->ev_b[gi], ss) != cudaSuccess || cudaStreamWaitEvent(st, sp->ev_b[gi], 0) != cudaSuccess)
        return PRONY_ERR_CUDA;
    }
  } else {
    lrc = launch_main(p, grd, st, info);
  }
  if (lrc != PRONY_OK) return lrc;
  // U is first read by k_reduce: a caller may still be copying it on another stream
  if (wait_before_reduce && cudaStreamWaitEvent(st, wait_before_reduce, 0) != cudaSuccess) return PRONY_ERR_CUDA;
  if (pl.nj > 0) {
    const dim3 wgrd(pl.RP, g.d, pl.nj);
    switch ((pl.shape.NP / 8 + 1) / 2) {  // n-tiles per consumer warp (WN = 2)
#define PRONY_WCASE(nt) \
  case nt:              \
    lrc = launch_reduce_ws_t<nt, 2>(r, wgrd, st); \
    break;
      PRONY_WCASE(1) PRONY_WCASE(2) PRONY_WCASE(3) PRONY_WCASE(4) PRONY_WCASE(5) PRONY_WCASE(6) PRONY_WCASE(7)
      PRONY_WCASE(8)
#undef PRONY_WCASE
      default:
        return PRONY_ERR_RANGE;
    }
  } else {
  switch (pl.shape.rWN * 16 + pl.shape.rNT) {
#define PRONY_RCASE(nt, wn) \
  case wn * 16 + nt:        \
    lrc = launch_reduce_t<nt, wn>(r, rgrd, st, mode); \
    break;
    PRONY_RCASE(1, 2) PRONY_RCASE(2, 2) PRONY_RCASE(3, 2) PRONY_RCASE(4, 2) PRONY_RCASE(3, 4) PRONY_RCASE(4, 4)
#undef PRONY_RCASE
    default:
      return PRONY_ERR_RANGE;
  }
  }
  if (lrc != PRONY_OK) return lrc;
  const int64_t tot = (int64_t)g.d * g.m * g.m;
  k_finalize<<<(int)std::min<int64_t>((8 * tot + 255) / 256, 4096), 256, 0, st>>>(g.d, g.m, pl.RP, Spart, sigma, S,
                                                                                  g.N, dev_status);
  if (info) {
    info->launches = 4 + (split ? 2 * std::min(kSplitStreams, pl.KC - 1) : 0);  // k_prep
                      // (with the shared-row tables), k_project, k_reduce, k_finalize (+ per later chunk group: k_vsum,
                      // k_project)
    info->main_grid[0] = (int)grd.x;
    info->main_grid[1] = (int)grd.y;
    info->main_grid[2] = (int)grd.z;
    info->main_block = kThreads;
    info->split_k = pl.KC;
    info->main_flops = 8.0 * g.m * (double)g.N * (double)pl.R_tot;
  }
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

// ---------------------------------------------------------------------------- B_mu (NEXT-4)
// g_mu[x] = sum_l mu_l g[x + s_l]: B_mu = sum_l mu_l T_l is the Toeplitz operator
// [g_mu[P(k) - P(h) + C0]], so C_mu = U* B_mu V Sigma^-1 is ONE projection on the combined grid.
__global__ void k_combine_grid(int d, int n, int64_t box, const double2* __restrict__ grid,
                               const double2* __restrict__ mu, double2* __restrict__ out) {
  const int L = 2 * n + 2;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < box; x += (int64_t)gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    int64_t sl = 1;
    for (int l = d; l >= 1; --l) {  // s_l = L^(d-l)
      if (x + sl < box) s = cadd(s, cmul(mu[l - 1], grid[x + sl]));
      sl *= L;
    }
    out[x] = s;
  }
}

// ---------------------------------------------------------------------------- Toeplitz apply
// Y = T_l X (l = 1..d), Y = T X (l = 0) or Y = T^H X (l = 0, conj) for an N x r block X, with the
// k_project pipeline (the same implicit gather; NEXT-1 reuses it for the block power SVD).
// T^H[h][k] = conj(f(k-h)) = f'(h-k) with f'(v) = conj(f(-v)): the same Toeplitz form on the reflected,
// conjugated grid (built by k_reflect_conj; points whose reflection leaves the box are never read
// for l = 0 and are set to 0).
__global__ void k_reflect_conj(int d, int n, int64_t box, const double2* __restrict__ grid, double2* __restrict__ out) {
  const int L = 2 * n + 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < box; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e, idx = 0, s = 1;
    bool inside = true;
    for (int i = d - 1; i >= 0; --i) {
      const int v = (int)(r % L) - n;  // coordinate in {-n..n+1}
      r /= L;
      const int w = -v;                // reflected coordinate
      if (w < -n || w > n + 1) inside = false;
      idx += (int64_t)(w + n) * s;
      s *= L;
    }
    out[e] = inside ? cconj(grid[idx]) : make_double2(0.0, 0.0);
  }
}

__global__ void k_copy_cols(int N, int w, int NP, const double2* __restrict__ Y0, double2* __restrict__ Yout, int ldy,
                            int c0) {
  const int64_t tot = (int64_t)N * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / w;
    const int j = (int)(e % w);
    Yout[k * ldy + c0 + j] = Y0[k * NP + j];
  }
}

// ---------------------------------------------------------------------------- Toeplitz matvec (r = 1)
// The Lanczos recurrence (NEXT-3, Alg. 2) applies T and T^H to ONE vector per step. On the DMMA path
// that single column is padded to an 8-wide n-tile and the A gather (24 B per T element) bounds it
// (8.1 ms at cfg4). This DFMA kernel uses the multilevel Toeplitz structure instead. Split the
// multi-index into an outer prefix (first d - q coordinates) and an inner block (last q coordinates,
// A = (n+1)^q points): k = (k'', a), h = (h'', b) and
//   T[k, h] = g[L^q (P''(k'') - P''(h'')) + shift + Pin(a) - Pin(b)],   Pin(a) = sum_i a_i L^(q-1-i),
// so for one prefix pair the A x A block reads ONE window of 2 Pmax + 1 consecutive samples
// (Pmax = Pin(n,..,n)). CTA (k'', slice s of h'') stages window + x[h'', :] in shared memory
// (double-buffered cp.async); a thread owns 4 consecutive outputs inside one run of the last inner
// coordinate and walks each run of b with a sliding register window (1 window load + 1 broadcast load
// per 4 complex MACs). Partial sums per slice are reduced in fixed slice order (deterministic).
constexpr int kMvThreads = 256;
constexpr int kMvPerThread = 4;
constexpr int kMvMaxSlots = 4;  // output slots (4 outputs each) per thread
constexpr int kMvMaxSlices = 64;

__global__ void __launch_bounds__(kMvThreads) k_toeplitz_mv(int d, int n, int q, int Mp, int S,
                                                            const double2* __restrict__ g, int shift,
                                                            const double2* __restrict__ x, int ldx,
                                                            double2* __restrict__ ypart) {
  extern __shared__ __align__(16) double2 mvs[];
  const int n1 = n + 1, L = 2 * n + 2;
  int A = 1, Lq = 1, Pmax = 0;
  for (int i = 0; i < q; ++i) {
    A *= n1;
    Pmax = Pmax * L + n;
    Lq *= L;
  }
  const int runs = A / n1;             // runs of the last coordinate inside the inner block
  const int tpr = (n1 + kMvPerThread - 1) / kMvPerThread;  // threads (slots) per run
  const int nslot = runs * tpr;
  // window slot: logical w(-1 .. Wl+2) (1 pad in front, 3 behind) stored 4-way interleaved, element e at
  // ((e+1) % 4) Q + (e+1) / 4, so the 32 lanes of a warp (outputs 4 apart) read 32 consecutive 16-B words
  const int Wl = 2 * Pmax + 1, Q = (Wl + 4 + 3) / 4, WS = 4 * Q;
  const int slot = WS + A;
  const int kp = blockIdx.x, s = blockIdx.y, tid = threadIdx.x, nth = blockDim.x;
  auto Pdig = [&](int idx, int ndig) {  // linear box offset of an (ndig)-digit base-(n+1) index
    int P = 0, mul = 1;
    for (int i = 0; i < ndig; ++i) {
      P += (idx % n1) * mul;
      idx /= n1;
      mul *= L;
    }
    return P;
  };
  const int pk = Pdig(kp, d - q);
  const int hb = (int)((int64_t)Mp * s / S), he = (int)((int64_t)Mp * (s + 1) / S);
  for (int e = tid; e < 2 * slot; e += nth) mvs[e] = make_double2(0.0, 0.0);  // pads stay zero
  __syncthreads();
  auto issue = [&](int hp, int buf) {
    double2* w = mvs + buf * slot;
    const int wbase = Lq * (pk - Pdig(hp, d - q)) + shift - Pmax;
    const uint32_t sw = (uint32_t)__cvta_generic_to_shared(w);
    for (int j = tid; j < Wl; j += nth)
      cp_async16(sw + 16u * (((j + 1) & 3) * Q + ((j + 1) >> 2)), g + wbase + j, 16);
    const uint32_t sx = (uint32_t)__cvta_generic_to_shared(w + WS);
    for (int b = tid; b < A; b += nth) cp_async16(sx + 16u * b, x + ((size_t)hp * A + b) * ldx, 16);
    cp_async_commit();
  };
  double2 acc[kMvMaxSlots][kMvPerThread];
#pragma unroll
  for (int u = 0; u < kMvMaxSlots; ++u)
#pragma unroll
    for (int r = 0; r < kMvPerThread; ++r) acc[u][r] = make_double2(0.0, 0.0);
  if (hb < he) issue(hb, 0);
  for (int hp = hb; hp < he; ++hp) {
    const int buf = (hp - hb) & 1;
    if (hp + 1 < he) {
      issue(hp + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* wb = mvs + buf * slot;  // w(j) = g[wbase + j], j in [-1, Wl + 2] readable
    auto w = [&](int j) { return wb[((j + 1) & 3) * Q + ((j + 1) >> 2)]; };
    const double2* xs = mvs + buf * slot + WS;
#pragma unroll
    for (int u = 0; u < kMvMaxSlots; ++u) {
      const int sl = tid + u * nth;
      if (sl < nslot) {
        const int rho = sl / tpr, j0 = kMvPerThread * (sl % tpr);
        const int prho = L * Pdig(rho, q - 1);
        double2 c0 = acc[u][0], c1 = acc[u][1], c2 = acc[u][2], c3 = acc[u][3];
        auto step = [&](const double2& p0, const double2& p1, const double2& p2, const double2& p3, double2 xb) {
          c0.x = fma(p0.x, xb.x, fma(-p0.y, xb.y, c0.x));
          c0.y = fma(p0.x, xb.y, fma(p0.y, xb.x, c0.y));
          c1.x = fma(p1.x, xb.x, fma(-p1.y, xb.y, c1.x));
          c1.y = fma(p1.x, xb.y, fma(p1.y, xb.x, c1.y));
          c2.x = fma(p2.x, xb.x, fma(-p2.y, xb.y, c2.x));
          c2.y = fma(p2.x, xb.y, fma(p2.y, xb.x, c2.y));
          c3.x = fma(p3.x, xb.x, fma(-p3.y, xb.y, c3.x));
          c3.y = fma(p3.x, xb.y, fma(p3.y, xb.x, c3.y));
        };
        for (int beta = 0; beta < runs; ++beta) {
          // outputs (rho, j0 + r), inputs (beta, bl): window index c + r - bl
          const int c = prho - L * Pdig(beta, q - 1) + j0 + Pmax;
          const double2* xr = xs + beta * n1;
          double2 v0 = w(c), v1 = w(c + 1), v2 = w(c + 2), v3 = w(c + 3);
          int bl = 0;
          for (; bl + 4 <= n1; bl += 4) {
            const double2 x0 = xr[bl], x1 = xr[bl + 1], x2 = xr[bl + 2], x3 = xr[bl + 3];
            const double2 u0 = w(c - bl - 1), u1 = w(c - bl - 2), u2 = w(c - bl - 3), u3 = w(c - bl - 4);
            step(v0, v1, v2, v3, x0);
            step(u0, v0, v1, v2, x1);
            step(u1, u0, v0, v1, x2);
            step(u2, u1, u0, v0, x3);
            v3 = u0;
            v2 = u1;
            v1 = u2;
            v0 = u3;
          }
          for (; bl < n1; ++bl) {
            step(v0, v1, v2, v3, xr[bl]);
            v3 = v2;
            v2 = v1;
            v1 = v0;
            v0 = w(c - bl - 1);
          }
        }
        acc[u][0] = c0;
        acc[u][1] = c1;
        acc[u][2] = c2;
        acc[u][3] = c3;
      }
    }
    __syncthreads();  // the slot is refilled by the next iteration's issue
  }
  double2* yp = ypart + (size_t)s * Mp * A + (size_t)kp * A;
#pragma unroll
  for (int u = 0; u < kMvMaxSlots; ++u) {
    const int sl = tid + u * nth;
    if (sl < nslot) {
      const int rho = sl / tpr, j0 = kMvPerThread * (sl % tpr);
#pragma unroll
      for (int r = 0; r < kMvPerThread; ++r)
        if (j0 + r < n1) yp[rho * n1 + j0 + r] = acc[u][r];
    }
  }
}

// y[k * ldy] = sum_{s < S} ypart[s][k]   (fixed order)
__global__ void k_mv_reduce(int N, int S, const double2* __restrict__ ypart, double2* __restrict__ y, int ldy) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    double2 a = ypart[k];
    for (int s = 1; s < S; ++s) a = cadd(a, ypart[(size_t)s * N + k]);
    y[(size_t)k * ldy] = a;
  }
}

namespace {
constexpr int kApplyMaxW = 120;  // columns per k_project pass (NT <= 5 over WN = 3 warps)
struct ApplyLayout {
  size_t refl, ptab, gsum, vsum, Y, counters, total;
};
ApplyLayout apply_layout(int d, int n, int N) {
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  ApplyLayout a{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  a.refl = take((size_t)box * sizeof(double2));
  a.ptab = take((size_t)(N + kPtabPad) * sizeof(int32_t));
  a.gsum = take((size_t)box * sizeof(double));
  a.vsum = take((size_t)N * kApplyMaxW * sizeof(double));
  a.Y = take((size_t)kYCap * N * kApplyMaxW * sizeof(double2));
  a.counters = take((size_t)((N + 15) / 16 + 1) * sizeof(int));
  a.total = off;
  return a;
}
}  // namespace

size_t apply_workspace_bytes(int d, int n, int N) { return apply_layout(d, n, N).total; }

int toeplitz_apply_launch(int d, int n, int N, const double2* grid, int ell, int conj, const double2* X, int ldx, int r,
                          double2* Yout, int ldy, void* ws, int sm_count, cudaStream_t st) {
  const ApplyLayout al = apply_layout(d, n, N);
  char* w = (char*)ws;
  double2* refl = (double2*)(w + al.refl);
  int32_t* ptab = (int32_t*)(w + al.ptab);
  double* gsum = (double*)(w + al.gsum);
  double* vsum = (double*)(w + al.vsum);
  double2* Y = (double2*)(w + al.Y);
  int* counters = (int*)(w + al.counters);
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  const double2* g = grid;
  if (conj) {
    k_reflect_conj<<<2 * sm_count, 256, 0, st>>>(d, n, box, grid, refl);
    g = refl;
  }
  const int L = 2 * n + 2;
  int64_t C0 = 0, s = 1;
  for (int i = 0; i < d; ++i) {
    C0 += (int64_t)n * s;
    s *= L;
  }
  const int shift = (int)(C0 + (ell >= 1 ? ipow(L, d - ell) : 0));
  const char* emv = getenv("PRONY_APPLY");
  // single vector: DFMA Toeplitz matvec with q inner coordinates (q = 1 when a run has >= 64 points,
  // else 2 when d >= 3 and runs are short enough for one CTA's output slots)
  int q = 0;
  if (r == 1 && d >= 2 && !(emv && emv[0] == 'd')) {
    const int n1 = n + 1, tpr = (n1 + kMvPerThread - 1) / kMvPerThread;
    if (n1 >= 64 && tpr <= kMvMaxSlots * kMvThreads) q = 1;
    else if (d >= 3 && n1 * tpr <= kMvMaxSlots * kMvThreads && n1 * n1 >= 64) q = 2;
  }
  if (q) {
    int A = 1, Pmax = 0;
    for (int i = 0; i < q; ++i) {
      A *= (n + 1);
      Pmax = Pmax * L + n;
    }
    const int Mp = N / A;
    const int nslot = (A / (n + 1)) * ((n + 1 + kMvPerThread - 1) / kMvPerThread);
    const int nth = std::min(kMvThreads, std::max(32, (std::min(nslot, kMvThreads) + 31) / 32 * 32));
    const char* esl = getenv("PRONY_MV_SLICES");
    int S = std::max(1, std::min({kMvMaxSlices, Mp, (40 * sm_count + Mp - 1) / Mp}));
    if (esl) S = std::max(1, std::min({kMvMaxSlices, Mp, atoi(esl)}));
    const size_t smem = (size_t)2 * (4 * ((2 * Pmax + 1 + 4 + 3) / 4) + A) * sizeof(double2);
    if (smem > 227 * 1024) q = 0;
    if (q) {
      if (smem > 48 * 1024 &&
          ensure_smem_attr(k_toeplitz_mv, smem) != cudaSuccess)
        return PRONY_ERR_CUDA;
      k_toeplitz_mv<<<dim3(Mp, S), nth, smem, st>>>(d, n, q, Mp, S, g, shift, X, ldx, Y);
      k_mv_reduce<<<(N + 255) / 256, 256, 0, st>>>(N, S, Y, Yout, ldy);
      return cudaGetLastError() == cudaSuccess ? PRONY_OK : PRONY_ERR_CUDA;
    }
  }
  const int npass = (r + kApplyMaxW - 1) / kApplyMaxW;
  const int mode = cmul_mode();
  for (int ps = 0; ps < npass; ++ps) {
    const int c0 = (int)((int64_t)r * ps / npass), c1 = (int)((int64_t)r * (ps + 1) / npass);
    const int wcols = c1 - c0;
    ProjGeom gg{};
    gg.d = 1;
    gg.n = n;
    gg.m = wcols;
    gg.N = N;
    gg.kb[0] = 0;
    gg.rows[0] = N;
    ProjPlan pl{};
    project_plan(gg, sm_count, &pl);
    const int nrb = (pl.max_rows + pl.shape.BM - 1) / pl.shape.BM;
    if (pl.KC > 1 && cudaMemsetAsync(counters, 0, (size_t)nrb * sizeof(int), st) != cudaSuccess) return PRONY_ERR_CUDA;
    k_prep<<<8 * sm_count, 256, 0, st>>>(d, n, N, wcols, ldx, pl.shape.NP, box, g, X + c0, ptab, gsum, vsum, N, 0,
                                         nullptr, nullptr, nullptr, 0, nullptr);
    ProjParams p{};
    p.grid = g;
    p.gsum = gsum;
    p.V = X + c0;
    p.ldv = ldx;
    p.vsum = vsum;
    p.ptab = ptab;
    p.rtab = ptab;
    p.Y = Y;
    p.N = N;
    p.m = wcols;
    p.NP = pl.shape.NP;
    p.chunk_w = pl.chunk_w;
    p.chunk0_w = pl.chunk0_w;
    p.R_tot = pl.R_tot;
    p.KC = pl.KC;
    p.nrb = nrb;
    p.counters = counters;
    p.box = (int)box;
    p.kb[0] = 0;
    p.rows[0] = N;
    p.yoff[0] = 0;
    p.shift[0] = shift;
    dim3 grd(nrb, pl.KC, 1);
    int lrc = PRONY_OK;
    switch (pl.shape.WN * 16 + pl.shape.NT) {
#define PRONY_CASE(nt, wn) \
  case wn * 16 + nt:       \
    lrc = launch_project_t<nt, wn>(p, grd, st, mode, nullptr); \
    break;
#if PRONY_CONSUMER_WARPS == 12
      PRONY_CASE(1, 2) PRONY_CASE(2, 2) PRONY_CASE(3, 2) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(1, 3)
      PRONY_CASE(2, 3) PRONY_CASE(3, 3) PRONY_CASE(4, 3) PRONY_CASE(5, 3) PRONY_CASE(4, 4)
#else
      PRONY_CASE(1, 2) PRONY_CASE(2, 2) PRONY_CASE(3, 2) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(6, 2)
      PRONY_CASE(7, 2) PRONY_CASE(8, 2)
#endif
#undef PRONY_CASE
      default:
        return PRONY_ERR_RANGE;
    }
    if (lrc != PRONY_OK) return lrc;
    const int64_t tot = (int64_t)N * wcols;
    k_copy_cols<<<(int)std::min<int64_t>((tot + 255) / 256, 8 * sm_count), 256, 0, st>>>(N, wcols, pl.shape.NP, Y,
                                                                                        Yout, ldy, c0);
  }
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

}  // namespace prony

#ifdef PRONY_DEBUG
// debug builds only (not part of the ABI in prony.h): gather-index violations seen so far
extern "C" unsigned long long prony_debug_violations(void) {
  unsigned long long v = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&v, prony::g_prony_violations, sizeof(v));
  return v;
}
#endif
