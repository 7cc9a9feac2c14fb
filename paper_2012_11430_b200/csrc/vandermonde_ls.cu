// vandermonde_ls.cu — A = [z_j^k], G = A conj(A)^T, b = A conj(f) (PAPER.md:59,
// normal equations of argmin ||A^T c - f||_2; R10), c = conj(G^-1 b), t.
//
//   k_powers     pwT[l][a][j] = z_j(l)^a, a = 0..n, by repeated multiplication (R9)
//   k_vls        per column block (16 warps): A tile (m x 16 columns) built in shared memory from
//                the power tables (A[j][k] = prod_l pwT[l][k_l][j]), double-buffered against the MMAs,
//                optional coalesced A write; the LOWER triangle of G_part += A_tile conj(A_tile)^T on the
//                DMMA warp engine (3M; G is Hermitian), b_part += A conj(f)
//   k_ls_reduce  fixed-order sum of the partials -> G (upper triangle mirrored), b
//   k_solve      one CTA, factor resident in shared memory: blocked right-looking Cholesky G = L L^H,
//                L y = b, L^H x = y, c = conj(x); t = (-arg z / 2 pi) mod 1 (R4)
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "engine.cuh"
#include "vandermonde_ls.cuh"

namespace prony {

// pwT[l][a][j] = z_j(l)^a, a = 0..n, by repeated multiplication (R9); the j index is fastest so that the A-tile
// build (consecutive threads = consecutive j) reads it coalesced
__global__ void k_powers(int d, int n, int m, const double2* __restrict__ z, double2* __restrict__ pw) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d * m) return;
  const int l = e / m, j = e % m;
  const double2 zz = z[(size_t)j * d + l];
  double2 p = make_double2(1.0, 0.0);
  double2* out = pw + (size_t)l * (n + 1) * m + j;
  for (int a = 0; a <= n; ++a) {
    out[(size_t)a * m] = p;
    p = cmul(p, zz);
  }
}

// grid (CB, ceil(units / 16)); CTA (cb, y) handles columns [cbeg, cend) of I_n in tiles of kTile. A "unit" is
// one warp's share of the LOWER triangle of G (G is Hermitian: only i >= j is computed, k_ls_reduce mirrors
// the rest): 16 rows i of m-tile r and up to NT n-tiles of 8 columns j <= 16 r + 15 (host table p.unit).
// Per tile, double-buffered in shared memory: the column info (multi-index digits of k, conj f(k)), and the
// A tile At[kk][j] = prod_l pwT[l][k_l][j] with its 3M planes Sp = Re+Im, Sm = Re-Im; warp (unit) MMAs of
// tile t overlap the build of tile t+1 by the other warps, one barrier per tile.
// G_part[i][j] += sum_k A[i][k] conj(A[j][k]) (B operand conj(A) rows, engine CONJB); b_part[i] += A[i][k]
// conj(f(k)) by threads i < m of CTA y = 0, which also writes the optional A columns.
template <int NT>
__global__ void __launch_bounds__(kVlsThreads, 1) k_vls(VlsParams p) {
  extern __shared__ __align__(16) double vsm[];
  const int cap = p.cap;  // row capacity of the smem planes (>= every row read)
  const int lda = cap + 2, lds = cap + 4;
  const int plane = 2 * kTile * lda + 2 * kTile * lds;  // doubles per buffer
  int* cinfo = reinterpret_cast<int*>(vsm + 2 * plane);  // [2][kTile][PRONY_MAX_D + 1]: digits, -1 = padding
  double2* Fs = reinterpret_cast<double2*>(vsm + 2 * plane + kTile * (PRONY_MAX_D + 1));  // [2][kTile] conj f

  const int cb = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int m = p.m, d = p.d, n = p.n;
  const int u = blockIdx.y * (kVlsThreads / 32) + warp;
  const bool has_unit = u < p.nunits;
  const int mt = has_unit ? p.unit[u][0] : 0, t0 = has_unit ? p.unit[u][1] : 0, nt_active = has_unit ? p.unit[u][2] : 0;
  const bool lead = blockIdx.y == 0;
  const int64_t W = p.col_end - p.col_begin;
  const int64_t cbeg = p.col_begin + W * cb / p.CB;
  const int64_t cend = p.col_begin + W * (cb + 1) / p.CB;
  const int ntiles = (int)((cend - cbeg + kTile - 1) / kTile);
  const int L = 2 * n + 2;
  const size_t pwl = (size_t)(n + 1) * m;  // stride of l in pwT

  // rows >= m of the planes stay zero (both buffers)
  for (int e = tid; e < 2 * plane; e += kVlsThreads) vsm[e] = 0.0;

  auto colinfo = [&](int tile, int buf) {  // threads < kTile: digits of k and conj f(k)
    if (tid < kTile) {
      const int64_t k = cbeg + (int64_t)tile * kTile + tid;
      int* ci = cinfo + (buf * kTile + tid) * (PRONY_MAX_D + 1);
      double2 f = make_double2(0.0, 0.0);
      if (k < cend) {
        int64_t r = k, idx = 0, sL = 1;
        for (int l = d - 1; l >= 0; --l) {  // digits of k, last coordinate fastest
          const int dg = (int)(r % (n + 1));
          r /= (n + 1);
          ci[l] = dg;
          idx += (int64_t)(dg + n) * sL;
          sL *= L;
        }
        ci[PRONY_MAX_D] = 1;
        f = cconj(ldg2(p.grid + idx));
      } else {
        ci[PRONY_MAX_D] = -1;
      }
      Fs[buf * kTile + tid] = f;
    }
  };
  auto build = [&](int tile, int buf) {  // A tile: A[j][k] = prod_l pwT[l][k_l][j], product in order l = 1..d (R9)
    double2* At = reinterpret_cast<double2*>(vsm + buf * plane);
    double* Sp = vsm + buf * plane + 2 * kTile * lda;
    double* Sm = Sp + kTile * lds;
    const int64_t c0 = cbeg + (int64_t)tile * kTile;
    for (int e = tid; e < m * kTile; e += kVlsThreads) {
      const int kk = e / m, j = e % m;
      const int* ci = cinfo + (buf * kTile + kk) * (PRONY_MAX_D + 1);
      double2 a = make_double2(0.0, 0.0);
      if (ci[PRONY_MAX_D] > 0) {
        a = ldg2(p.pw + (size_t)ci[0] * m + j);
        for (int l = 1; l < d; ++l) a = cmul(a, ldg2(p.pw + l * pwl + (size_t)ci[l] * m + j));
        if (p.A && lead) p.A[(size_t)j * W + (c0 + kk - p.col_begin)] = a;
      }
      At[kk * lda + j] = a;
      Sp[kk * lds + j] = a.x + a.y;
      Sm[kk * lds + j] = a.x - a.y;
    }
  };

  double acc[3][NT][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;
  double2 bacc = make_double2(0.0, 0.0);
  __syncthreads();
  if (ntiles > 0) colinfo(0, 0);
  if (ntiles > 1) colinfo(1, 1);
  __syncthreads();
  if (ntiles > 0) build(0, 0);
  __syncthreads();

  for (int tile = 0; tile < ntiles; ++tile) {
    const int buf = tile & 1;
    const double2* At = reinterpret_cast<const double2*>(vsm + buf * plane);
    const double* Sp = vsm + buf * plane + 2 * kTile * lda;
    const double* Sm = Sp + kTile * lds;
    if (has_unit) {
      const int i0 = mt * 16;
#pragma unroll
      for (int kk = 0; kk < kTile / 4; ++kk)
        warp_cmma_k4_n<NT, 3, true>(nt_active, acc, At + kk * 4 * lda + i0, Sp + kk * 4 * lds + i0, lda, lds,
                                    At + kk * 4 * lda + t0 * 8, Sm + kk * 4 * lds + t0 * 8, lda, lds, g, q);
    }
    if (lead && tid < m) {
      const double2* F = Fs + buf * kTile;
#pragma unroll 4
      for (int kk = 0; kk < kTile; ++kk) {
        const double2 a = At[kk * lda + tid], f = F[kk];
        bacc.x = fma(a.x, f.x, bacc.x);
        bacc.x = fma(-a.y, f.y, bacc.x);
        bacc.y = fma(a.x, f.y, bacc.y);
        bacc.y = fma(a.y, f.x, bacc.y);
      }
    }
    // the other buffer: its tile (tile - 1) was consumed before the previous barrier
    if (tile + 1 < ntiles) build(tile + 1, buf ^ 1);
    __syncthreads();
    // column info of tile + 2 into this buffer's slot (tile's build, its last reader, is done)
    if (tile + 2 < ntiles) colinfo(tile + 2, buf);
    __syncthreads();
  }
  double2* G = p.Gpart + (size_t)cb * m * m;
  const int ia = mt * 16 + g, ib = ia + 8;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (has_unit && j < nt_active) {
      double re[4], im[4];
      acc_to_complex<NT, 3>(acc, j, re, im);
      const int col = (t0 + j) * 8 + 2 * q;
      if (ia < m) {
        if (col < m) G[(size_t)ia * m + col] = make_double2(re[0], im[0]);
        if (col + 1 < m) G[(size_t)ia * m + col + 1] = make_double2(re[1], im[1]);
      }
      if (ib < m) {
        if (col < m) G[(size_t)ib * m + col] = make_double2(re[2], im[2]);
        if (col + 1 < m) G[(size_t)ib * m + col + 1] = make_double2(re[3], im[3]);
      }
    }
  }
  if (lead && tid < m) p.bpart[(size_t)cb * m + tid] = bacc;
}

// G[i][j] = sum_c G_part[c][i][j] for j <= i, G[j][i] = conj(G[i][j]); b likewise. One WARP per output: lane l
// sums the partials c = l, l + 32, ... in order, then a fixed shuffle tree (deterministic; 32 independent
// load streams per output instead of one serial chain of CB dependent loads)
__global__ void k_ls_reduce(int m, int CB, const double2* __restrict__ Gpart, const double2* __restrict__ bpart,
                            double2* __restrict__ G, double2* __restrict__ b) {
  const int lane = threadIdx.x & 31;
  const int tri = m * (m + 1) / 2;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < tri + m; o += nwarps) {
    const double2* src;
    size_t stride;
    int i = 0, j = 0;
    if (o < tri) {
      i = (int)((sqrt(8.0 * o + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > o) --i;
      while ((i + 1) * (i + 2) / 2 <= o) ++i;
      j = o - i * (i + 1) / 2;
      src = Gpart + (size_t)i * m + j;
      stride = (size_t)m * m;
    } else {
      src = bpart + (o - tri);
      stride = (size_t)m;
    }
    double2 s = make_double2(0.0, 0.0);
    for (int c = lane; c < CB; c += 32) s = cadd(s, __ldcg(src + (size_t)c * stride));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s.x += __shfl_down_sync(0xffffffffu, s.x, off);
      s.y += __shfl_down_sync(0xffffffffu, s.y, off);
    }
    if (lane == 0) {
      if (o < tri) {
        G[(size_t)i * m + j] = s;
        if (j != i) G[(size_t)j * m + i] = cconj(s);
      } else {
        b[o - tri] = s;
      }
    }
  }
}

// One CTA of kSolveThreads (16 warps). Blocked right-looking Cholesky G = L L^H, the lower triangle packed in
// shared memory (A[i][k] at i(i+1)/2 + k), in panels of kPanel columns [p0, p0 + pb):
//   1. warp 0 factors the diagonal block A11 = L11 L11^H (lane r owns row p0 + r; pivots and columns are
//      broadcast by shuffles; 1/L_jj by rsqrt, kept in dinv);
//   2. every thread solves its rows of L21 = A21 L11^{-H} (rows are independent: L11 is read as broadcasts);
//   3. all warps apply the rank-pb update A22 -= L21 L21^H (warp per row, lanes over columns).
// Three CTA barriers per panel. The substitutions L y = b and L^H x = y are blocked the same way: warp 0
// solves the pb x pb diagonal block with shuffles, then every thread updates its rows. c = conj(x) (R10),
// t = (-arg z / 2 pi) mod 1 (R4). A pivot that is not > 0 (G not HPD) sets PRONY_ERR_SINGULAR, c = NaN.
constexpr int kPanel = 8;
__global__ void __launch_bounds__(kSolveThreads) k_solve(int d, int m, const double2* __restrict__ G,
                                                         const double2* __restrict__ b,
                                                         const double2* __restrict__ z, double2* __restrict__ c,
                                                         double* __restrict__ t, int32_t* status) {
  extern __shared__ __align__(16) double2 As[];  // m(m+1)/2 packed lower triangle
  __shared__ double dinv[PRONY_MAX_M];            // 1 / L_jj (the substitutions never divide)
  __shared__ double2 ys[PRONY_MAX_M];             // right-hand side -> y -> x
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kSolveThreads / 32;
  auto at = [](int i, int k) { return i * (i + 1) / 2 + k; };
#ifdef PRONY_SOLVE_TIMING
  long long clk0 = clock64(), clk_panel = 0, clk_upd = 0, clk_tmp = 0;
#endif
  if (tid == 0) bad = 0;
  for (int i = warp; i < m; i += kWarps)
    for (int k = lane; k <= i; k += 32) As[at(i, k)] = G[(size_t)i * m + k];
  for (int i = tid; i < m; i += kSolveThreads) ys[i] = b[i];
  __syncthreads();
#ifdef PRONY_SOLVE_TIMING
  const long long clk_load = clock64() - clk0;
#endif

  for (int p0 = 0; p0 < m; p0 += kPanel) {
    const int pb = min(kPanel, m - p0);
#ifdef PRONY_SOLVE_TIMING
    clk_tmp = clock64();
#endif
    // 1. diagonal block
    if (warp == 0) {
      const int i = p0 + lane;
      double2 r[kPanel];
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj)
        r[jj] = (lane < pb && jj <= lane) ? As[at(i, p0 + jj)] : make_double2(0.0, 0.0);
      bool fail = false;
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj) {
        if (jj < pb) {
          const double djj = __shfl_sync(0xffffffffu, r[jj].x, jj);
          if (!(djj > 0.0)) fail = true;
          const double inv = rsqrt(djj), ljj = djj * inv;
          if (lane == 0) dinv[p0 + jj] = inv;
          if (lane == jj) r[jj] = make_double2(ljj, 0.0);
          else if (lane > jj) r[jj] = make_double2(r[jj].x * inv, r[jj].y * inv);
#pragma unroll
          for (int kk = 0; kk < kPanel; ++kk) {
            if (kk > jj && kk < pb) {
              const double lkx = __shfl_sync(0xffffffffu, r[jj].x, kk);  // L[p0 + kk][p0 + jj]
              const double lky = __shfl_sync(0xffffffffu, r[jj].y, kk);
              if (lane >= kk && lane < pb) {
                r[kk].x -= r[jj].x * lkx + r[jj].y * lky;
                r[kk].y -= r[jj].y * lkx - r[jj].x * lky;
              }
            }
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj)
        if (lane < pb && jj <= lane) As[at(i, p0 + jj)] = r[jj];
      if (fail && lane == 0) bad = 1;
    }
    __syncthreads();
    if (bad) break;
    // 2. L21 = A21 L11^{-H}, one row per thread
    const int t0 = p0 + pb;
    for (int i = t0 + tid; i < m; i += kSolveThreads) {
      double2 x[kPanel];
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj) x[jj] = jj < pb ? As[at(i, p0 + jj)] : make_double2(0.0, 0.0);
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj) {
        if (jj < pb) {
          double2 a = x[jj];
#pragma unroll
          for (int tt = 0; tt < kPanel; ++tt) {
            if (tt < jj) {  // a -= L[i][p0+tt] conj(L[p0+jj][p0+tt])
              const double2 l = As[at(p0 + jj, p0 + tt)];
              a.x -= x[tt].x * l.x + x[tt].y * l.y;
              a.y -= x[tt].y * l.x - x[tt].x * l.y;
            }
          }
          const double inv = dinv[p0 + jj];
          x[jj] = make_double2(a.x * inv, a.y * inv);
        }
      }
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj)
        if (jj < pb) As[at(i, p0 + jj)] = x[jj];
    }
    __syncthreads();
#ifdef PRONY_SOLVE_TIMING
    clk_panel += clock64() - clk_tmp;
    clk_tmp = clock64();
#endif
    // 3. trailing update of rows/columns >= t0
    for (int i = t0 + warp; i < m; i += kWarps) {
      double2 li[kPanel];
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj) li[jj] = jj < pb ? As[at(i, p0 + jj)] : make_double2(0.0, 0.0);
      for (int k = t0 + lane; k <= i; k += 32) {
        double2 a = As[at(i, k)];
#pragma unroll
        for (int jj = 0; jj < kPanel; ++jj) {
          if (jj < pb) {
            const double2 lk = As[at(k, p0 + jj)];
            a.x -= li[jj].x * lk.x + li[jj].y * lk.y;
            a.y -= li[jj].y * lk.x - li[jj].x * lk.y;
          }
        }
        As[at(i, k)] = a;
      }
    }
    __syncthreads();
#ifdef PRONY_SOLVE_TIMING
    clk_upd += clock64() - clk_tmp;
#endif
  }
#ifdef PRONY_SOLVE_TIMING
  const long long clk_fact = clock64();
#endif

  if (bad) {
    if (tid == 0) set_status(status, PRONY_ERR_SINGULAR);
    for (int i = tid; i < m; i += kSolveThreads) c[i] = make_double2(NAN, NAN);
  } else {
    // forward L y = b, blocked: warp 0 solves the diagonal block, then every thread updates its rows below
    for (int p0 = 0; p0 < m; p0 += kPanel) {
      const int pb = min(kPanel, m - p0);
      if (warp == 0) {
        double2 y = lane < pb ? ys[p0 + lane] : make_double2(0.0, 0.0);
#pragma unroll
        for (int jj = 0; jj < kPanel; ++jj) {
          if (jj < pb) {
            double yjx = __shfl_sync(0xffffffffu, y.x, jj), yjy = __shfl_sync(0xffffffffu, y.y, jj);
            const double inv = dinv[p0 + jj];
            yjx *= inv;
            yjy *= inv;
            if (lane == jj) y = make_double2(yjx, yjy);
            if (lane > jj && lane < pb) {
              const double2 l = As[at(p0 + lane, p0 + jj)];
              y.x -= l.x * yjx - l.y * yjy;
              y.y -= l.x * yjy + l.y * yjx;
            }
          }
        }
        if (lane < pb) ys[p0 + lane] = y;
      }
      __syncthreads();
      for (int i = p0 + pb + tid; i < m; i += kSolveThreads) {
        double2 a = ys[i];
#pragma unroll
        for (int jj = 0; jj < kPanel; ++jj) {
          if (jj < pb) {
            const double2 l = As[at(i, p0 + jj)], yj = ys[p0 + jj];
            a.x -= l.x * yj.x - l.y * yj.y;
            a.y -= l.x * yj.y + l.y * yj.x;
          }
        }
        ys[i] = a;
      }
      __syncthreads();
    }
    // backward L^H x = y, blocked from the last block: x_j = (y_j - sum_{i > j} conj(L_ij) x_i) / L_jj
    for (int p0 = ((m - 1) / kPanel) * kPanel; p0 >= 0; p0 -= kPanel) {
      const int pb = min(kPanel, m - p0);
      if (warp == 0) {
        double2 x = lane < pb ? ys[p0 + lane] : make_double2(0.0, 0.0);
#pragma unroll
        for (int jj = kPanel - 1; jj >= 0; --jj) {
          if (jj < pb) {
            double xjx = __shfl_sync(0xffffffffu, x.x, jj), xjy = __shfl_sync(0xffffffffu, x.y, jj);
            const double inv = dinv[p0 + jj];
            xjx *= inv;
            xjy *= inv;
            if (lane == jj) x = make_double2(xjx, xjy);
            if (lane < jj) {  // x_lane -= conj(L[p0+jj][p0+lane]) x_jj
              const double2 l = As[at(p0 + jj, p0 + lane)];
              x.x -= l.x * xjx + l.y * xjy;
              x.y -= l.x * xjy - l.y * xjx;
            }
          }
        }
        if (lane < pb) ys[p0 + lane] = x;
      }
      __syncthreads();
      for (int i = tid; i < p0; i += kSolveThreads) {
        double2 a = ys[i];
#pragma unroll
        for (int jj = 0; jj < kPanel; ++jj) {
          if (jj < pb) {
            const double2 l = As[at(p0 + jj, i)], xj = ys[p0 + jj];  // conj(L[p0+jj][i]) x_jj
            a.x -= l.x * xj.x + l.y * xj.y;
            a.y -= l.x * xj.y - l.y * xj.x;
          }
        }
        ys[i] = a;
      }
      __syncthreads();
    }
    for (int i = tid; i < m; i += kSolveThreads) c[i] = cconj(ys[i]);
#ifdef PRONY_SOLVE_TIMING
    if (tid == 0)
      printf("k_solve m=%d clocks: load %lld panels %lld updates %lld substitution %lld total %lld\n", m, clk_load,
             clk_panel, clk_upd, clock64() - clk_fact, clock64() - clk0);
#endif
  }
  if (t) {
    const double inv2pi = 0.15915494309189533577;  // 1 / (2 pi)
    for (int e = tid; e < m * d; e += kSolveThreads) {
      const double2 zz = z[e];
      double v = -atan2(zz.y, zz.x) * inv2pi;  // (-arg z / 2 pi) mod 1  (R4)
      v = v - floor(v);
      if (v >= 1.0) v = 0.0;
      t[e] = v;
    }
  }
}

// ---------------------------------------------------------------------------- host side
namespace {
constexpr int kVlsNT = 4;  // n-tiles per unit (3M accumulators: 48 doubles per thread)
// lower-triangle units: m-tile r (rows 16r..16r+15) needs n-tiles 0..ceil(min(16r+16, m)/8)-1, split into
// near-equal runs of <= kVlsNT
int vls_units(int m, int (*unit)[3]) {
  int cnt = 0;
  for (int r = 0; 16 * r < m; ++r) {
    const int nt = (std::min(16 * r + 16, m) + 7) / 8;
    const int parts = (nt + kVlsNT - 1) / kVlsNT;
    for (int pp = 0; pp < parts; ++pp) {
      const int a = nt * pp / parts, b = nt * (pp + 1) / parts;
      if (unit && cnt < kVlsMaxUnits) {
        unit[cnt][0] = r;
        unit[cnt][1] = a;
        unit[cnt][2] = b - a;
      }
      ++cnt;
    }
  }
  return cnt;
}
size_t vls_smem(int cap) {
  const int lda = cap + 2, lds = cap + 4;
  return (size_t)2 * (2 * kTile * lda + 2 * kTile * lds) * sizeof(double) +
         (size_t)kTile * (PRONY_MAX_D + 1) * sizeof(int) * 2 + 2 * kTile * sizeof(double2);
}
int vls_cb(int64_t W, int ctas_per_block, int sm_count) {
  const int64_t tiles = (W + kTile - 1) / kTile;
  int64_t cb = std::max<int64_t>(1, sm_count / std::max(1, ctas_per_block));
  cb = std::max<int64_t>(1, std::min<int64_t>(cb, tiles));
  return (int)cb;
}
size_t solve_smem(int m) { return (size_t)m * (m + 1) / 2 * sizeof(double2); }
}  // namespace

size_t ls_workspace_bytes(int d, int n, int m, int sm_count) {
  size_t bytes = align_up((size_t)d * m * (n + 1) * sizeof(double2), 256);  // power tables
  const int cbmax = std::max(1, sm_count);
  bytes += align_up((size_t)cbmax * m * m * sizeof(double2), 256);  // G partials
  bytes += align_up((size_t)cbmax * m * sizeof(double2), 256);      // b partials
  return bytes;
}

static int launch_vls(const VlsParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  if (ensure_smem_attr(k_vls<kVlsNT>, smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  k_vls<kVlsNT><<<grid, kVlsThreads, smem, st>>>(p);
  return PRONY_OK;
}

int ls_solve_launch(int d, int m, const double2* G, const double2* b, const double2* z, double2* c, double* t,
                    void* ws, int32_t* status, cudaStream_t st) {
  (void)ws;
  const size_t smem = solve_smem(m);
  if (ensure_smem_attr(k_solve, smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  k_solve<<<1, kSolveThreads, smem, st>>>(d, m, G, b, z, c, t, status);
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

int ls_launch(int d, int n, int m, int N, const double2* z, const double2* grid, int64_t col_begin, int64_t col_end,
              double2* A, double2* G, double2* b, double2* c, double* t, void* ws, int32_t* status, int sm_count,
              cudaStream_t st, prony_exec_info* info) {
  char* w = (char*)ws;
  double2* pw = (double2*)w;
  w += align_up((size_t)d * m * (n + 1) * sizeof(double2), 256);
  const int cbmax = std::max(1, sm_count);
  double2* Gpart = (double2*)w;
  w += align_up((size_t)cbmax * m * m * sizeof(double2), 256);
  double2* bpart = (double2*)w;

  const int64_t W = col_end - col_begin;
  if (info) {
    info->launches = 0;
    info->main_grid[0] = info->main_grid[1] = info->main_grid[2] = 0;
    info->main_block = 0;
    info->split_k = 0;
    info->main_flops = 0.0;
  }
  if (W <= 0) {
    if (cudaMemsetAsync(G, 0, (size_t)m * m * sizeof(double2), st) != cudaSuccess) return PRONY_ERR_CUDA;
    if (cudaMemsetAsync(b, 0, (size_t)m * sizeof(double2), st) != cudaSuccess) return PRONY_ERR_CUDA;
    return PRONY_OK;
  }
  k_powers<<<(d * m + 127) / 128, 128, 0, st>>>(d, n, m, z, pw);
  VlsParams p{};
  p.d = d;
  p.n = n;
  p.m = m;
  p.col_begin = col_begin;
  p.col_end = col_end;
  p.nunits = vls_units(m, p.unit);
  if (p.nunits > kVlsMaxUnits) return PRONY_ERR_RANGE;
  const int per_cta = kVlsThreads / 32;
  const int ny = (p.nunits + per_cta - 1) / per_cta;
  p.CB = vls_cb(W, ny, sm_count);
  p.cap = (m + 15) / 16 * 16;  // every A row (m-tiles) and B row (n-tiles <= the row's m-tile) read
  p.pw = pw;
  p.grid = grid;
  p.A = A;
  p.Gpart = Gpart;
  p.bpart = bpart;
  const dim3 vgrid(p.CB, ny);
  const size_t smem = vls_smem(p.cap);
  if (info && info->ev_main_begin) cudaEventRecord((cudaEvent_t)info->ev_main_begin, st);
  int rc = launch_vls(p, vgrid, smem, st);
  if (rc != PRONY_OK) return rc;
  if (info && info->ev_main_end) cudaEventRecord((cudaEvent_t)info->ev_main_end, st);
  int launches = 3;
  k_ls_reduce<<<std::max(1, std::min(2 * sm_count, (m * (m + 1) / 2 + m + 7) / 8)), 256, 0, st>>>(m, p.CB, Gpart,
                                                                                                   bpart, G, b);
  if (col_begin == 0 && col_end == N && (c || t)) {
    // only t requested: solve into the (now consumed) G partial buffer
    rc = ls_solve_launch(d, m, G, b, z, c ? c : Gpart, t, nullptr, status, st);
    if (rc != PRONY_OK) return rc;
    ++launches;
  }
  if (info) {
    info->launches = launches;
    info->main_grid[0] = p.CB;
    info->main_grid[1] = ny;
    info->main_grid[2] = 1;
    info->main_block = kVlsThreads;
    info->split_k = p.CB;
    // the LS products as defined (G = A conj(A)^T in full, b = A conj(f)), ZGEMM convention; the kernel
    // computes only the lower triangle of the Hermitian G
    info->main_flops = 8.0 * m * (double)m * (double)W + 8.0 * m * (double)W;
  }
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

}  // namespace prony
