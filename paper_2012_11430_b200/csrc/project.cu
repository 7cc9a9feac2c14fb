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
#include <cstdio>

#include "common.cuh"
#include "project.cuh"

namespace prony {

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
// CTA = 8 warps = WM (row) x WN (col) warps; warp tile 16 rows x (8*NT) columns of Y.
// Lane (g = lane>>2, q = lane&3) owns rows g, g+8 of its warp tile for the A fragment and
// column g of each n-tile for the B fragment; per k-step of 4 columns h of T_l it loads
//   A: T_l[k_g][h0+q], T_l[k_{g+8}][h0+q]   = grid[P0 - P(h)], grid[P1 - P(h)]   (2 x LDG.128)
//   B: V[h0+q][col0 + 8j], j < NT                                                 (NT x LDG.128)
// one step ahead (register double buffer) and issues 4*NT DMMA m16n8k4.
template <int NT, int WN>
__global__ void __launch_bounds__(256, 1) k_project(ProjParams p) {
  constexpr int WM = 8 / WN;
  constexpr int BM = 16 * WM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int l = blockIdx.z;
  const int rows = p.rows[l];
  const int rb0 = blockIdx.x * BM;
  if (rb0 >= rows) return;
  const int chunk = blockIdx.y;
  const int h_begin = chunk * p.chunk_w;
  const int h_end = min(h_begin + p.chunk_w, p.N);

  const int r0 = rb0 + wm * 16 + g, r1 = r0 + 8;
  const bool v0 = r0 < rows, v1 = r1 < rows;
  const int32_t* __restrict__ ptab = p.ptab;
  const int P0 = ptab[p.kb[l] + (v0 ? r0 : 0)] + p.shift[l];
  const int P1 = ptab[p.kb[l] + (v1 ? r1 : 0)] + p.shift[l];
  const int colw = wn * NT * 8;
  const double2* __restrict__ grid = p.grid;
  const double2* __restrict__ V = p.V;
  const int m = p.m;
  const double2 zero = make_double2(0.0, 0.0);

  double acc_re[NT][4], acc_im[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc_re[j][e] = acc_im[j][e] = 0.0;

  double2 a0, a1, b[NT];
  auto load = [&](int h0, double2& x0, double2& x1, double2 (&y)[NT]) {
    const int h = h0 + q;
    const bool vh = h < h_end;
    const int Ph = ptab[h];  // padded table: h < N + kPtabPad always
    x0 = (v0 && vh) ? ldg2(grid + (P0 - Ph)) : zero;
    x1 = (v1 && vh) ? ldg2(grid + (P1 - Ph)) : zero;
    const double2* vrow = V + (size_t)h * m;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int col = colw + 8 * j + g;
      y[j] = (vh && col < m) ? ldg2(vrow + col) : zero;
    }
  };

  load(h_begin, a0, a1, b);
  for (int h0 = h_begin; h0 < h_end; h0 += 4) {
    double2 na0, na1, nb[NT];
    if (h0 + 4 < h_end) {
      load(h0 + 4, na0, na1, nb);
    } else {
      na0 = na1 = zero;
#pragma unroll
      for (int j = 0; j < NT; ++j) nb[j] = zero;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) cmma16x8x4_4m(acc_re[j], acc_im[j], a0, a1, b[j]);
    a0 = na0;
    a1 = na1;
#pragma unroll
    for (int j = 0; j < NT; ++j) b[j] = nb[j];
  }

  // epilogue: Y[chunk][yoff_l + r][col], NP-wide rows (all NP columns written)
  const size_t ybase = (size_t)chunk * p.R_tot + p.yoff[l];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int col = colw + 8 * j + 2 * q;
    if (v0) {
      double2* y = p.Y + (ybase + r0) * p.NP + col;
      y[0] = make_double2(acc_re[j][0], acc_im[j][0]);
      y[1] = make_double2(acc_re[j][1], acc_im[j][1]);
    }
    if (v1) {
      double2* y = p.Y + (ybase + r1) * p.NP + col;
      y[0] = make_double2(acc_re[j][2], acc_im[j][2]);
      y[1] = make_double2(acc_re[j][3], acc_im[j][3]);
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
  const int64_t cap_rows = 2LL * g.d * g.N;
  int kc_max = (int)std::min<int64_t>(64, std::max<int64_t>(1, cap_rows / std::max(R_tot, 1)));
  kc_max = std::max(1, std::min(kc_max, std::max(1, g.N / 64)));
  double best = 1e30;
  int best_kc = 1;
  for (int kc = 1; kc <= kc_max; ++kc) {
    const double ctas = (double)row_blocks * kc;
    const double waves = std::ceil(ctas / sm_count);
    const double cost = waves / kc * (1.0 + 0.002 * kc);  // small per-chunk overhead (Y traffic)
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
  bytes += align_up((size_t)2 * d * N * sh.NP * sizeof(double2), 256);  // Y partials (KC*R_tot <= 2dN)
  const int ib = (m + 63) / 64;
  int RP = std::max(1, (2 * sm_count) / std::max(1, d * ib));
  bytes += align_up((size_t)d * RP * m * m * sizeof(double2), 256);
  return bytes;
}

template <int NT, int WN>
static void launch_project_t(const ProjParams& p, dim3 grid, cudaStream_t st) {
  k_project<NT, WN><<<grid, 256, 0, st>>>(p);
}

int project_launch(const ProjGeom& g, const ProjPlan& pl, const double2* grid, const double2* U, const double2* V,
                   const double* sigma, double2* S, void* ws, cudaStream_t st, prony_exec_info* info) {
  char* w = (char*)ws;
  int32_t* ptab = (int32_t*)w;
  w += align_up((size_t)(g.N + kPtabPad) * sizeof(int32_t), 256);
  double2* Y = (double2*)w;
  w += align_up((size_t)2 * g.d * g.N * pl.shape.NP * sizeof(double2), 256);
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
  switch (WN * 16 + NT) {
#define PRONY_CASE(nt, wn) \
  case wn * 16 + nt:       \
    launch_project_t<nt, wn>(p, grd, st); \
    break;
    PRONY_CASE(1, 1) PRONY_CASE(2, 1) PRONY_CASE(3, 1) PRONY_CASE(4, 1) PRONY_CASE(5, 1) PRONY_CASE(6, 1)
    PRONY_CASE(7, 1) PRONY_CASE(4, 2) PRONY_CASE(5, 2) PRONY_CASE(6, 2) PRONY_CASE(7, 2) PRONY_CASE(8, 2)
#undef PRONY_CASE
    default:
      return PRONY_ERR_RANGE;
  }
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
