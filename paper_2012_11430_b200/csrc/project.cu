// project.cu — S_l = U* T_l V Sigma^-1 (eq_generateSl) on sm_100a.
//
// Three launches per call:
//   k_ptab      P(k) = sum_i k_i L^(d-1-i) for k in I_n (the linear box offset of k, so that
//               T_l[k,h] = grid[P(k) - P(h) + L^(d-l) + C0], C0 = n sum_i L^i; F5)
//   k_project   Y_c = T_l[rows, chunk c] * V[chunk c, :] — implicit-Toeplitz gather of T_l
//               straight from the L2-resident sample grid into DMMA fragments (T_l is never
//               written anywhere), complex FP64 4M on the FP64 tensor pipe (DMMA), split-K
//               over column chunks c for wave balance; writes Y partials (N x NP per chunk).
//   k_reduce    S_part[p] = U[rows_p]^* (sum_c Y_c[rows_p]) (fixed-order), then
//   k_finalize  S_l = (sum_p S_part[p]) diag(1/sigma) (fixed order -> deterministic).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "project.cuh"

namespace prony {

// complex product formulation of k_project: 3 (Gauss/3M, default) or 4 (4M); env PRONY_CMUL=4m
static int cmul_mode() {
  const char* e = getenv("PRONY_CMUL");
  return (e && (e[0] == '4')) ? 4 : 3;
}

// ---------------------------------------------------------------------------- P table
__global__ void k_ptab(int d, int n, int N, int32_t* __restrict__ ptab) {
  const int L = 2 * n + 2;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N + kPtabPad; k += gridDim.x * blockDim.x) {
    if (k >= N) {
      ptab[k] = 0;
      continue;
    }
    int r = k, P = 0, s = 1;
    for (int i = d - 1; i >= 0; --i) {  // last coordinate fastest, stride 1
      P += (r % (n + 1)) * s;
      r /= (n + 1);
      s *= L;
    }
    ptab[k] = P;
  }
}

// ---------------------------------------------------------------------------- projection
// CTA = 8 warps = WM (row) x WN (col) warps; CTA tile BM = 16*WM rows of T_l x NP = 8*NT*WN
// columns of V; warp tile 16 rows x 8*NT columns. The K loop (columns h of T_l, rows of V) runs
// in stages of BK = 16 through a kStages-deep cp.async ring in shared memory:
//   A tile  As[kc][r] = T_l[k_r][h0+kc] = grid[P(k_r) + s_l + C0 - P(h0+kc)]   (implicit Toeplitz
//           gather: one 16-byte cp.async per element straight from the L2/L1-resident grid)
//   B tile  Bs[kc][c] = V[h0+kc][c]  (zero-filled for c >= m and h >= h_end)
// Consumers read the DMMA fragments with conflict-free LDS.128 (row strides BM+2, NP+2 double2).
// Lane (g = lane>>2, q = lane&3): A frag rows g, g+8 at column q; B frag row q, column g.
// MODE 4: 4M  Re += Ar Br - Ai Bi, Im += Ar Bi + Ai Br              (4 DMMA m16n8k4 / n-tile)
// MODE 3: 3M  P1 += Ar Br, P2 += Ai Bi, P3 += (Ar+Ai)(Br+Bi);
//             Re = P1 - P2, Im = P3 - P1 - P2                       (3 DMMA m16n8k4 / n-tile)
constexpr int kBK = 16;
constexpr int kStages = 4;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_cg(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// non-volatile so ptxas may interleave independent MMAs
__device__ __forceinline__ void mma16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

template <int NT, int WN>
struct ProjTile {
  static constexpr int WM = 8 / WN;
  static constexpr int BM = 16 * WM;
  static constexpr int NP = 8 * NT * WN;
  static constexpr int AS = BM + 2;
  static constexpr int BS = NP + 2;
  static constexpr int STAGE = kBK * (AS + BS);  // double2 per stage
  static constexpr size_t SMEM = (size_t)kStages * STAGE * sizeof(double2);
  static constexpr int GA = kBK * BM / 256;      // A elements gathered per thread per stage
  static constexpr int KSTEP = 256 / BM;         // column stride between a thread's A elements
  static constexpr int GB = (kBK * NP + 255) / 256;
};

template <int NT, int WN, int MODE>
__global__ void __launch_bounds__(256, 1) k_project(ProjParams p) {
  using T = ProjTile<NT, WN>;
  constexpr int WM = T::WM, BM = T::BM, NP = T::NP, AS = T::AS, BS = T::BS, GA = T::GA, KSTEP = T::KSTEP,
                GB = T::GB;
  constexpr int NACC = MODE == 3 ? 3 : 2;
  extern __shared__ __align__(16) double2 smem[];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int l = blockIdx.z;
  const int rows = p.rows[l];
  const int rb0 = blockIdx.x * BM;
  if (rb0 >= rows) return;
  const int chunk = blockIdx.y;
  const int h_begin = chunk * p.chunk_w;
  const int h_end = min(h_begin + p.chunk_w, p.N);
  const int KT = (h_end - h_begin + kBK - 1) / kBK;
  const int32_t* __restrict__ ptab = p.ptab;
  const double2* __restrict__ grid = p.grid;
  const double2* __restrict__ V = p.V;
  const int m = p.m, N = p.N;

  // gather role: row ra of the tile, columns kc0 + KSTEP*x
  const int ra = tid % BM, kc0 = tid / BM;
  const bool va = rb0 + ra < rows;
  const int PA = va ? ptab[p.kb[l] + rb0 + ra] + p.shift[l] : 0;

  auto load_ph = [&](int h0, int (&ph)[GA]) {
#pragma unroll
    for (int x = 0; x < GA; ++x) {
      const int h = h0 + kc0 + KSTEP * x;
      ph[x] = h < N ? __ldg(ptab + h) : 0;
    }
  };
  auto load_stage = [&](int slot, int h0, const int (&ph)[GA]) {
    double2* As = smem + slot * T::STAGE;
    double2* Bs = As + kBK * AS;
#pragma unroll
    for (int x = 0; x < GA; ++x) {
      const int kc = kc0 + KSTEP * x;
      const bool ok = va && (h0 + kc < h_end);
      cp_async16(As + kc * AS + ra, grid + (ok ? PA - ph[x] : 0), ok ? 16 : 0);
    }
#pragma unroll
    for (int y = 0; y < GB; ++y) {
      const int e = tid + 256 * y;
      if (e < kBK * NP) {
        const int kr = e / NP, col = e % NP;
        const int h = h0 + kr;
        const bool ok = (h < h_end) && (col < m);
        cp_async16_cg(Bs + kr * BS + col, V + (ok ? (size_t)h * m + col : 0), ok ? 16 : 0);
      }
    }
  };

  double acc[NACC][NT][4];
#pragma unroll
  for (int a = 0; a < NACC; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;

  int ph[GA];
  load_ph(h_begin, ph);
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < KT) {
      load_stage(s, h_begin + s * kBK, ph);
      load_ph(h_begin + (s + 1) * kBK, ph);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nk = kt + kStages - 1;
    if (nk < KT) {
      load_stage(nk % kStages, h_begin + nk * kBK, ph);
      load_ph(h_begin + (nk + 1) * kBK, ph);
    }
    cp_async_commit();

    const double2* As = smem + (kt % kStages) * T::STAGE;
    const double2* Bs = As + kBK * AS;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const double2 a0 = As[(kk * 4 + q) * AS + wm * 16 + g];
      const double2 a1 = As[(kk * 4 + q) * AS + wm * 16 + g + 8];
      const double2* brow = Bs + (kk * 4 + q) * BS + wn * NT * 8 + g;
      if constexpr (MODE == 3) {
        const double s0 = a0.x + a0.y, s1 = a1.x + a1.y;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const double2 b = brow[8 * j];
          mma16x8x4(acc[0][j], a0.x, a1.x, b.x);
          mma16x8x4(acc[1][j], a0.y, a1.y, b.y);
          mma16x8x4(acc[2][j], s0, s1, b.x + b.y);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const double2 b = brow[8 * j];
          mma16x8x4(acc[0][j], a0.x, a1.x, b.x);
          mma16x8x4(acc[1][j], a0.x, a1.x, b.y);
          mma16x8x4(acc[0][j], -a0.y, -a1.y, b.y);
          mma16x8x4(acc[1][j], a0.y, a1.y, b.x);
        }
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: Y[chunk][yoff_l + r][col], NP-wide rows (all NP columns written)
  const int r0 = rb0 + wm * 16 + g, r1 = r0 + 8;
  const size_t ybase = (size_t)chunk * p.R_tot + p.yoff[l];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    double re[4], im[4];
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
    const int col = wn * NT * 8 + 8 * j + 2 * q;
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

// ---------------------------------------------------------------------------- reduce
// grid (RP, d, ceil(m/64)); CTA p of segment l sums rows [rows*p/RP, rows*(p+1)/RP):
//   S_part[l][p][i][j] = sum_k conj(U[k][i]) * sum_c Y_c[k][j],  i in [i0, i0+64), j < m.
// Thread (ti, tj) owns i = i0 + ti + 16a (a<4), j = tj + 16b (b<8). DFMA (0.25% of the flops).
__global__ void __launch_bounds__(256) k_reduce(RedParams p) {
  __shared__ double2 Us[16][64];
  __shared__ double2 Ys[16][kMaxNP];
  const int l = blockIdx.y;
  const int P = blockIdx.x;
  const int i0 = blockIdx.z * 64;
  const int rows = p.rows[l];
  const int rbeg = (int)((int64_t)rows * P / p.RP), rend = (int)((int64_t)rows * (P + 1) / p.RP);
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const int m = p.m, NP = p.NP;
  double2 acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = make_double2(0.0, 0.0);

  for (int s = rbeg; s < rend; s += 16) {
    for (int e = tid; e < 16 * 64; e += 256) {
      const int r = e >> 6, ii = e & 63;
      const int row = s + r, i = i0 + ii;
      double2 u = make_double2(0.0, 0.0);
      if (row < rend && i < m) u = cconj(ldg2(p.U + (size_t)(p.kb[l] + row) * m + i));
      Us[r][ii] = u;
    }
    for (int e = tid; e < 16 * kMaxNP; e += 256) {
      const int r = e / kMaxNP, jj = e % kMaxNP;
      const int row = s + r;
      double2 y = make_double2(0.0, 0.0);
      if (row < rend && jj < NP) {
        for (int c = 0; c < p.KC; ++c) {  // fixed chunk order
          const double2 v = ldg2(p.Y + ((size_t)c * p.R_tot + p.yoff[l] + row) * NP + jj);
          y.x += v.x;
          y.y += v.y;
        }
      }
      Ys[r][jj] = y;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < 16; ++r) {
      double2 u[4], y[8];
#pragma unroll
      for (int a = 0; a < 4; ++a) u[a] = Us[r][ti + 16 * a];
#pragma unroll
      for (int b = 0; b < 8; ++b) y[b] = Ys[r][tj + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          acc[a][b].x = fma(u[a].x, y[b].x, acc[a][b].x);
          acc[a][b].x = fma(-u[a].y, y[b].y, acc[a][b].x);
          acc[a][b].y = fma(u[a].x, y[b].y, acc[a][b].y);
          acc[a][b].y = fma(u[a].y, y[b].x, acc[a][b].y);
        }
    }
    __syncthreads();
  }
  double2* out = p.Spart + ((size_t)l * p.RP + P) * m * m;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + ti + 16 * a;
    if (i >= m) continue;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int j = tj + 16 * b;
      if (j < m) out[(size_t)i * m + j] = acc[a][b];
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
ProjShape proj_shape(int m) {
  ProjShape s;
  const int ntot = (m + 7) / 8;
  s.WN = (ntot + 6) / 7;  // <= 7 n-tiles per warp
  if (s.WN > 2) s.WN = 2;
  s.NT = (ntot + s.WN - 1) / s.WN;
  s.WM = 8 / s.WN;
  s.BM = 16 * s.WM;
  s.NP = 8 * s.NT * s.WN;
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
  // split-K: chunk count KC minimizing ceil(waves)/KC (time per CTA ~ 1/KC), subject to
  // KC * R_tot <= 2 d N (workspace bound) and chunks of >= 64 columns.
  const int64_t cap_rows = (int64_t)kYCap * g.d * g.N;
  int kc_max = (int)std::min<int64_t>(64, std::max<int64_t>(1, cap_rows / std::max(R_tot, 1)));
  kc_max = std::max(1, std::min(kc_max, std::max(1, g.N / 64)));
  double best = 1e30;
  int best_kc = 1;
  for (int kc = 1; kc <= kc_max; ++kc) {
    const double ctas = (double)row_blocks * kc;
    const double waves = std::ceil(ctas / sm_count);
    // time ~ waves x (chunk columns + pipeline fill/drain of ~4 stages)
    const double cost = waves * ((double)g.N / kc + 4.0 * kBK);
    if (cost < best - 1e-12) {
      best = cost;
      best_kc = kc;
    }
  }
  int chunk_w = (g.N + best_kc - 1) / best_kc;
  chunk_w = (chunk_w + 3) / 4 * 4;
  pl->chunk_w = chunk_w;
  pl->KC = (g.N + chunk_w - 1) / chunk_w;  // every chunk non-empty
  // reduce partition: about 2 CTAs per SM in total
  const int ib = (g.m + 63) / 64;
  int RP = (2 * sm_count) / std::max(1, g.d * ib);
  RP = std::max(1, std::min(RP, std::max(1, (max_rows + 15) / 16)));
  pl->RP = RP;
  return 0;
}

size_t project_workspace_bytes(int d, int N, int m, int sm_count) {
  const ProjShape sh = proj_shape(m);
  size_t bytes = align_up((size_t)(N + kPtabPad) * sizeof(int32_t), 256);
  bytes += align_up((size_t)kYCap * d * N * sh.NP * sizeof(double2), 256);  // Y partials (KC*R_tot <= kYCap*dN)
  const int ib = (m + 63) / 64;
  int RP = std::max(1, (2 * sm_count) / std::max(1, d * ib));
  bytes += align_up((size_t)d * RP * m * m * sizeof(double2), 256);
  return bytes;
}

template <int NT, int WN>
static int launch_project_t(const ProjParams& p, dim3 grid, cudaStream_t st, int mode) {
  const size_t smem = ProjTile<NT, WN>::SMEM;
  if (mode == 4) {
    if (cudaFuncSetAttribute(k_project<NT, WN, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return PRONY_ERR_CUDA;
    k_project<NT, WN, 4><<<grid, 256, smem, st>>>(p);
  } else {
    if (cudaFuncSetAttribute(k_project<NT, WN, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return PRONY_ERR_CUDA;
    k_project<NT, WN, 3><<<grid, 256, smem, st>>>(p);
  }
  return PRONY_OK;
}

int project_launch(const ProjGeom& g, const ProjPlan& pl, const double2* grid, const double2* U, const double2* V,
                   const double* sigma, double2* S, void* ws, cudaStream_t st, prony_exec_info* info) {
  char* w = (char*)ws;
  int32_t* ptab = (int32_t*)w;
  w += align_up((size_t)(g.N + kPtabPad) * sizeof(int32_t), 256);
  double2* Y = (double2*)w;
  w += align_up((size_t)kYCap * g.d * g.N * pl.shape.NP * sizeof(double2), 256);
  double2* Spart = (double2*)w;

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
  k_ptab<<<(g.N + kPtabPad + 255) / 256, 256, 0, st>>>(g.d, g.n, g.N, ptab);

  ProjParams p{};
  p.grid = grid;
  p.V = V;
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
  dim3 grd((pl.max_rows + pl.shape.BM - 1) / pl.shape.BM, pl.KC, g.d);
  const int NT = pl.shape.NT, WN = pl.shape.WN;
  if (info && info->ev_main_begin) cudaEventRecord((cudaEvent_t)info->ev_main_begin, st);
  const int mode = cmul_mode();
  int lrc = PRONY_OK;
  switch (WN * 16 + NT) {
#define PRONY_CASE(nt, wn) \
  case wn * 16 + nt:       \
    lrc = launch_project_t<nt, wn>(p, grd, st, mode); \
    break;
    PRONY_CASE(1, 1) PRONY_CASE(2, 1) PRONY_CASE(3, 1) PRONY_CASE(4, 1) PRONY_CASE(5, 1) PRONY_CASE(6, 1)
    PRONY_CASE(7, 1) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(6, 2) PRONY_CASE(7, 2) PRONY_CASE(8, 2)
#undef PRONY_CASE
    default:
      return PRONY_ERR_RANGE;
  }
  if (lrc != PRONY_OK) return lrc;
  if (info && info->ev_main_end) cudaEventRecord((cudaEvent_t)info->ev_main_end, st);

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
  k_reduce<<<dim3(pl.RP, g.d, (g.m + 63) / 64), 256, 0, st>>>(r);
  const int64_t tot = (int64_t)g.d * g.m * g.m;
  k_finalize<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256, 0, st>>>(g.d, g.m, pl.RP, Spart, sigma, S);
  if (info) {
    info->launches = 4;
    info->main_grid[0] = (int)grd.x;
    info->main_grid[1] = (int)grd.y;
    info->main_grid[2] = (int)grd.z;
    info->main_block = 256;
    info->split_k = pl.KC;
    info->main_flops = 8.0 * g.m * (double)g.N * (double)pl.R_tot;
  }
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

}  // namespace prony
