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

#include "common.cuh"
#include "engine.cuh"
#include "project.cuh"

namespace prony {

// complex product formulation: 3 (Gauss/3M, default) or 4 (4M); env PRONY_CMUL=4m selects 4M
static int cmul_mode() {
  const char* e = getenv("PRONY_CMUL");
  return (e && (e[0] == '4')) ? 4 : 3;
}

// ---------------------------------------------------------------------------- prep
__global__ void k_prep(int d, int n, int N, int m, int NP, int64_t box, const double2* __restrict__ grid,
                       const double2* __restrict__ V, int32_t* __restrict__ ptab, double* __restrict__ gsum,
                       double* __restrict__ vsum) {
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
  const int64_t nv = (int64_t)N * NP;
  for (int64_t e = t0; e < nv; e += stride) {
    const int64_t h = e / NP;
    const int c = (int)(e % NP);
    double s = 0.0;
    if (c < m) {
      const double2 v = V[h * m + c];
      s = v.x + v.y;
    }
    vsum[e] = s;
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
constexpr int kProducerThreads = 128;
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
#ifndef PRONY_GATHER_UNROLL
#define PRONY_GATHER_UNROLL 2
#endif
constexpr int kKkUnroll = PRONY_KK_UNROLL;
constexpr int kGatherUnroll = PRONY_GATHER_UNROLL;
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
  static constexpr size_t SMEM = (size_t)PAT * sizeof(double) + (size_t)BM * sizeof(int);
  static_assert(STAGE % 2 == 0, "stage must keep 16-byte alignment");
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
  const int chunk = blockIdx.y;
  const int h_begin = chunk * p.chunk_w;
  const int h_end = min(h_begin + p.chunk_w, p.N);
  const int KT = (h_end - h_begin + kBK - 1) / kBK;
  const int m = p.m, N = p.N, NP = p.NP;

  // zero the B planes of every slot once: padding columns [m, NP) are never written by the bulk
  // copies, and rows past h_end of a partial last stage must not hold garbage (A is 0 there)
  for (int s = 0; s < kStages; ++s)
    for (int e = tid; e < kBK * (T::LDB * 2 + T::LDBS); e += kThreads) smem[s * T::STAGE + T::B_C + e] = 0.0;
  int* sPA = reinterpret_cast<int*>(smem + T::PAT);
  for (int r = tid; r < BM; r += kThreads)
    sPA[r] = (rb0 + r < rows) ? p.ptab[p.kb[l] + rb0 + r] + p.shift[l] : -1;  // -1: row outside
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8u * s, kGatherThreads + 1);  // A-gather cp.async arrivals + B expect_tx
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
    if (pt < kGatherThreads) {
      // A gather over the kBK x BM tile: element e = pt + kGatherThreads * j -> (kc = e / BM, ra = e % BM);
      // P(k_ra) + shift comes from the shared row table sPA, P(h0 + kc) from lane kc (shfl)
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
#pragma unroll kGatherUnroll
        for (int e = pt; e < kBK * BM; e += kGatherThreads) {
          const int kc = e / BM, ra = e % BM;
          const int phc = __shfl_sync(0xffffffffu, ph, kc);
          const int pa = sPA[ra];
          const bool ok = (pa >= 0) && (h0 + kc < h_end);
          const int idx = ok ? pa - phc : 0;
          cp_async16(st + (uint32_t)(T::A_C + 2 * (kc * T::LDA + ra)) * 8u, grid + idx, ok ? 16 : 0);
          if constexpr (MODE == 3)
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
        const uint32_t bytes_row = (uint32_t)m * 16u + (MODE == 3 ? (uint32_t)NP * 8u : 0u);
        if (plane == 0) mbar_arrive_expect_tx(full0 + 8u * s, bytes_row * (uint32_t)nrows);
        __syncwarp();
        const uint32_t st = sbase + (uint32_t)(s * T::STAGE) * 8u;
        if (kr < nrows) {
          const int h = h0 + kr;
          if (!sum_plane) {
            bulk_g2s(st + (uint32_t)(T::B_C + 2 * kr * T::LDB) * 8u, V + (size_t)h * m, (uint32_t)m * 16u,
                     full0 + 8u * s);
          } else if constexpr (MODE == 3) {
            bulk_g2s(st + (uint32_t)(T::B_S + kr * T::LDBS) * 8u, vsum + (size_t)h * NP, (uint32_t)NP * 8u,
                     full0 + 8u * s);
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

  auto run = [&](auto na_c) {
    constexpr int NA = decltype(na_c)::value;
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
          warp_cmma_k4<NT, NA, MODE>(acc, Ac + kk * 4 * T::LDA, As + kk * 4 * T::LDAS, T::LDA, T::LDAS,
                                     Bc + kk * 4 * T::LDB, Bs + kk * 4 * T::LDBS, T::LDB, T::LDBS, g, q);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8u * s);
    }
  };
  if (nt_active == NT) {
    run(std::integral_constant<int, NT>{});
  } else if (nt_active == 0) {
    run(std::integral_constant<int, 0>{});
  } else if constexpr (NT > 1) {
    if (nt_active == NT - 1) {
      run(std::integral_constant<int, NT - 1>{});
    } else if constexpr (NT > 2) {
      if (nt_active == NT - 2) {
        run(std::integral_constant<int, NT - 2>{});
      } else if constexpr (NT > 3) {
        if (nt_active == NT - 3) run(std::integral_constant<int, NT - 3>{});
      }
    }
  }

  // epilogue: Y[chunk][yoff_l + r][col], NP-wide rows (padding columns are zero)
  const int r0 = rb0 + wm * 16 + g, r1 = r0 + 8;
  const size_t ybase = (size_t)chunk * p.R_tot + p.yoff[l];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < nt_active) {
      double re[4], im[4];
      acc_to_complex<NT, MODE>(acc, j, re, im);
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

// ---------------------------------------------------------------------------- reduce
// grid (RP, d, ceil(m/BI)); CTA (p, l, ib) sums rows k in [rows*p/RP, rows*(p+1)/RP) of segment l:
//   S_part[l][p][i][j] = sum_k conj(U[k][i]) * sum_c Y_c[k][j],  i in [BI ib, BI ib + BI), j < m
// with the k_project warp engine (16 warps: WM x WN, BI = 16 WM): A = U^H staged as [k][i] planes
// (conj, conj-sum), B = sum_c Y_c staged as [k][j] planes; 8 rows k per slab, register-prefetched
// one slab ahead.
template <int NT, int WN, int MODE>
__global__ void __launch_bounds__(kReduceThreads, 1) k_reduce(RedParams p) {
  constexpr int WM = (kReduceThreads / 32) / WN, BI = 16 * WM, NPMAX = 8 * NT * WN;
  constexpr int LDA = BI + 2, LDAS = BI + 4, LDB = NPMAX + 2, LDBS = NPMAX + 4;
  constexpr int SL = 8;  // rows k per slab
  __shared__ __align__(16) double2 Ac[SL * LDA];
  __shared__ double As[SL * LDAS];
  __shared__ __align__(16) double2 Bc[SL * LDB];
  __shared__ double Bs[SL * LDBS];
  const int l = blockIdx.y;
  const int P = blockIdx.x;
  const int i0 = blockIdx.z * BI;
  const int rows = p.rows[l];
  const int rbeg = (int)((int64_t)rows * P / p.RP), rend = (int)((int64_t)rows * (P + 1) / p.RP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int m = p.m, NP = p.NP;
  const int ntot = NP / 8;
  const int t0 = (ntot * wn) / WN;
  const int nt_active = (ntot * (wn + 1)) / WN - t0;
  const bool warp_rows = (i0 + wm * 16) < m;

  double acc[3][NT][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;

  constexpr int NU = (SL * BI + kReduceThreads - 1) / kReduceThreads;
  constexpr int NY = (SL * NPMAX + kReduceThreads - 1) / kReduceThreads;
  double2 ru[NU], ry[NY];
  auto load_slab = [&](int s) {
#pragma unroll
    for (int x = 0; x < NU; ++x) {
      const int e = tid + kReduceThreads * x;
      const int r = e / BI, ii = e % BI;
      const int row = s + r, i = i0 + ii;
      ru[x] = (e < SL * BI && row < rend && i < m) ? ldg2(p.U + (size_t)(p.kb[l] + row) * m + i)
                                                     : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int y = 0; y < NY; ++y) {
      const int e = tid + kReduceThreads * y;
      double2 a2 = make_double2(0.0, 0.0);
      if (e < SL * NP) {
        const int r = e / NP, jj = e % NP;
        const int row = s + r;
        if (row < rend) {
          for (int c = 0; c < p.KC; ++c) {  // fixed chunk order
            const double2 v = ldg2(p.Y + ((size_t)c * p.R_tot + p.yoff[l] + row) * NP + jj);
            a2.x += v.x;
            a2.y += v.y;
          }
        }
      }
      ry[y] = a2;
    }
  };
  if (rbeg < rend) load_slab(rbeg);
  for (int s = rbeg; s < rend; s += SL) {
#pragma unroll
    for (int x = 0; x < NU; ++x) {
      const int e = tid + kReduceThreads * x;
      if (e < SL * BI) {
        const int r = e / BI, ii = e % BI;
        const double2 u = make_double2(ru[x].x, -ru[x].y);  // conj(U)
        Ac[r * LDA + ii] = u;
        As[r * LDAS + ii] = u.x + u.y;
      }
    }
#pragma unroll
    for (int y = 0; y < NY; ++y) {
      const int e = tid + kReduceThreads * y;
      if (e < SL * NP) {
        const int r = e / NP, jj = e % NP;
        Bc[r * LDB + jj] = ry[y];
        Bs[r * LDBS + jj] = ry[y].x + ry[y].y;
      }
    }
    __syncthreads();
    if (s + SL < rend) load_slab(s + SL);
    if (warp_rows) {
#pragma unroll
      for (int kk = 0; kk < SL / 4; ++kk)
        warp_cmma_k4_n<NT, MODE>(nt_active, acc, Ac + kk * 4 * LDA + wm * 16, As + kk * 4 * LDAS + wm * 16, LDA,
                                 LDAS, Bc + kk * 4 * LDB + t0 * 8, Bs + kk * 4 * LDBS + t0 * 8, LDB, LDBS, g, q);
    }
    __syncthreads();
  }
  double2* out = p.Spart + ((size_t)l * p.RP + P) * m * m;
  const int ia = i0 + wm * 16 + g, ib = ia + 8;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < nt_active) {
      double re[4], im[4];
      acc_to_complex<NT, MODE>(acc, j, re, im);
      const int col = (t0 + j) * 8 + 2 * q;
      if (ia < m) {
        if (col < m) out[(size_t)ia * m + col] = make_double2(re[0], im[0]);
        if (col + 1 < m) out[(size_t)ia * m + col + 1] = make_double2(re[1], im[1]);
      }
      if (ib < m) {
        if (col < m) out[(size_t)ib * m + col] = make_double2(re[2], im[2]);
        if (col + 1 < m) out[(size_t)ib * m + col + 1] = make_double2(re[3], im[3]);
      }
    }
  }
}

// S[l][i][j] = (sum_{p < RP} S_part[l][p][i][j]) / sigma_j   (fixed order)
__global__ void k_finalize(int d, int m, int RP, const double2* __restrict__ Spart, const double* __restrict__ sigma,
                           double2* __restrict__ S) {
  const int64_t total = (int64_t)d * m * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(e / ((int64_t)m * m));
    const int ij = (int)(e % ((int64_t)m * m));
    const int j = ij % m;
    double2 s = make_double2(0.0, 0.0);
    for (int P = 0; P < RP; ++P) {
      const double2 v = Spart[((size_t)l * RP + P) * m * m + ij];
      s.x += v.x;
      s.y += v.y;
    }
    const double inv = 1.0 / sigma[j];
    S[e] = make_double2(s.x * inv, s.y * inv);
  }
}

// ---------------------------------------------------------------------------- host side
// k_project: 12 consumer warps = WM x WN. WM = 4 puts all column parts of one 16-row m-tile on the
// same SM sub-partition (warp w -> SMSP w % 4 = wm), so every SMSP gets exactly ceil(m/8) n-tiles of
// DMMA work per k-step (balanced for any m); NT <= 5 keeps the 3M accumulators within 160 registers.
// k_reduce: 16 warps, WN column warps with <= 4 n-tiles (3M accumulators within 128 registers).
ProjShape proj_shape(int m) {
  ProjShape s;
  const int ntot = (m + 7) / 8;
  if (kConsumerWarps == 8) {
    s.WN = 2;  // WM = 4: warp w -> SMSP w % 4 = wm, balanced; NT <= 8 (3M accumulators in 240 regs)
  } else if (ntot <= 2) {
    s.WN = 2;
  } else if (ntot <= 15) {
    s.WN = 3;
  } else {
    s.WN = 4;
  }
  s.NT = (ntot + s.WN - 1) / s.WN;
  s.WM = kConsumerWarps / s.WN;  // k_project consumer warps along rows
  s.BM = 16 * s.WM;              // k_project rows per CTA
  s.rWN = ntot <= 8 ? 2 : 4;
  s.rNT = (ntot + s.rWN - 1) / s.rWN;
  s.BI = 16 * (kReduceThreads / 32) / s.rWN;  // k_reduce rows i per CTA
  s.NP = 8 * ntot;
  return s;
}

int project_plan(const ProjGeom& g, int sm_count, ProjPlan* pl) {
  const ProjShape sh = proj_shape(g.m);
  pl->shape = sh;
  int R_tot = 0, max_rows = 0, row_blocks = 0;
  for (int l = 0; l < g.d; ++l) {
    pl->yoff[l] = R_tot;
    R_tot += g.rows[l];
    max_rows = std::max(max_rows, g.rows[l]);
    row_blocks += (g.rows[l] + sh.BM - 1) / sh.BM;
  }
  pl->R_tot = R_tot;
  pl->max_rows = max_rows;
  // split-K: chunk count KC minimizing waves x (chunk columns + pipeline fill), subject to
  // KC * R_tot <= kYCap d N (workspace bound) and chunks of >= 64 columns.
  const int64_t cap_rows = (int64_t)kYCap * g.d * g.N;
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
  int chunk_w = (g.N + best_kc - 1) / best_kc;
  chunk_w = (chunk_w + kBK - 1) / kBK * kBK;
  pl->chunk_w = chunk_w;
  pl->KC = (g.N + chunk_w - 1) / chunk_w;  // every chunk non-empty
  // reduce partition: about 1 CTA per SM in total
  const int ib = (g.m + sh.BI - 1) / sh.BI;
  int RP = sm_count / std::max(1, g.d * ib);
  RP = std::max(1, std::min(RP, std::max(1, (max_rows + 7) / 8)));
  pl->RP = RP;
  return 0;
}

namespace {
struct WsLayout {
  size_t ptab, gsum, vsum, Y, Spart, total;
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
  w.ptab = take((size_t)(N + kPtabPad) * sizeof(int32_t));
  w.gsum = take((size_t)box * sizeof(double));
  w.vsum = take((size_t)N * sh.NP * sizeof(double));
  w.Y = take((size_t)kYCap * d * N * sh.NP * sizeof(double2));  // Y partials (KC*R_tot <= kYCap*dN)
  const int ib = (m + sh.BI - 1) / sh.BI;
  const int RP = std::max(1, sm_count / std::max(1, d * ib));
  w.Spart = take((size_t)d * RP * m * m * sizeof(double2));
  w.total = off;
  return w;
}
}  // namespace

size_t project_workspace_bytes(int d, int n, int N, int m, int sm_count) {
  return ws_layout(d, n, N, m, sm_count).total;
}

template <int NT, int WN>
static int launch_project_t(const ProjParams& p, dim3 grid, cudaStream_t st, int mode, prony_exec_info* info) {
  const size_t smem = ProjTile<NT, WN>::SMEM;
  auto kp = mode == 4 ? k_project<NT, WN, 4> : k_project<NT, WN, 3>;
  if (cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  if (info && info->ev_main_begin) cudaEventRecord((cudaEvent_t)info->ev_main_begin, st);
  kp<<<grid, kThreads, smem, st>>>(p);
  if (info && info->ev_main_end) cudaEventRecord((cudaEvent_t)info->ev_main_end, st);
  return PRONY_OK;
}

template <int NT, int WN>
static int launch_reduce_t(const RedParams& r, dim3 rgrid, cudaStream_t st, int mode) {
  auto kr = mode == 4 ? k_reduce<NT, WN, 4> : k_reduce<NT, WN, 3>;
  kr<<<rgrid, kReduceThreads, 0, st>>>(r);
  return PRONY_OK;
}

int project_launch(const ProjGeom& g, const ProjPlan& pl, const double2* grid, const double2* U, const double2* V,
                   const double* sigma, double2* S, void* ws, int sm_count, cudaStream_t st,
                   prony_exec_info* info) {
  const WsLayout wl = ws_layout(g.d, g.n, g.N, g.m, sm_count);
  char* w = (char*)ws;
  int32_t* ptab = (int32_t*)(w + wl.ptab);
  double* gsum = (double*)(w + wl.gsum);
  double* vsum = (double*)(w + wl.vsum);
  double2* Y = (double2*)(w + wl.Y);
  double2* Spart = (double2*)(w + wl.Spart);

  if (info) {
    info->launches = 0;
    info->main_grid[0] = info->main_grid[1] = info->main_grid[2] = 0;
    info->main_block = 0;
    info->split_k = 0;
    info->main_flops = 0.0;
  }
  if (pl.R_tot == 0) {
    if (cudaMemsetAsync(S, 0, (size_t)g.d * g.m * g.m * sizeof(double2), st) != cudaSuccess) return PRONY_ERR_CUDA;
    return PRONY_OK;
  }
  int64_t box = 1;
  for (int i = 0; i < g.d; ++i) box *= (2 * (int64_t)g.n + 2);
  k_prep<<<2 * sm_count, 256, 0, st>>>(g.d, g.n, g.N, g.m, pl.shape.NP, box, grid, V, ptab, gsum, vsum);

  ProjParams p{};
  p.grid = grid;
  p.gsum = gsum;
  p.V = V;
  p.vsum = vsum;
  p.ptab = ptab;
  p.Y = Y;
  p.N = g.N;
  p.m = g.m;
  p.NP = pl.shape.NP;
  p.chunk_w = pl.chunk_w;
  p.R_tot = pl.R_tot;
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
    p.shift[l] = (int)(ipow(L, g.d - 1 - l) + C0);  // s_l = L^(d-l) for l = 1..d
  }
  RedParams r{};
  r.Y = Y;
  r.U = U;
  r.Spart = Spart;
  r.m = g.m;
  r.NP = pl.shape.NP;
  r.KC = pl.KC;
  r.R_tot = pl.R_tot;
  r.RP = pl.RP;
  for (int l = 0; l < g.d; ++l) {
    r.kb[l] = g.kb[l];
    r.rows[l] = g.rows[l];
    r.yoff[l] = pl.yoff[l];
  }
  dim3 grd((pl.max_rows + pl.shape.BM - 1) / pl.shape.BM, pl.KC, g.d);
  dim3 rgrd(pl.RP, g.d, (g.m + pl.shape.BI - 1) / pl.shape.BI);
  const int NT = pl.shape.NT, WN = pl.shape.WN;
  const int mode = cmul_mode();
  int lrc = PRONY_OK;
  switch (WN * 16 + NT) {
#define PRONY_CASE(nt, wn) \
  case wn * 16 + nt:       \
    lrc = launch_project_t<nt, wn>(p, grd, st, mode, info); \
    break;
#if PRONY_CONSUMER_WARPS == 12
    PRONY_CASE(1, 2) PRONY_CASE(1, 3) PRONY_CASE(2, 3) PRONY_CASE(3, 3) PRONY_CASE(4, 3) PRONY_CASE(5, 3)
    PRONY_CASE(4, 4)
#else
    PRONY_CASE(1, 2) PRONY_CASE(2, 2) PRONY_CASE(3, 2) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(6, 2)
    PRONY_CASE(7, 2) PRONY_CASE(8, 2)
#endif
#undef PRONY_CASE
    default:
      return PRONY_ERR_RANGE;
  }
  if (lrc != PRONY_OK) return lrc;
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
  if (lrc != PRONY_OK) return lrc;
  const int64_t tot = (int64_t)g.d * g.m * g.m;
  k_finalize<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256, 0, st>>>(g.d, g.m, pl.RP, Spart, sigma, S);
  if (info) {
    info->launches = 4;
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

}  // namespace prony
