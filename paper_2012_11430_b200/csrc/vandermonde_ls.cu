// vandermonde_ls.cu — A = [z_j^k], G = A conj(A)^T, b = A conj(f) (PAPER.md:59,
// normal equations of argmin ||A^T c - f||_2; R10), c = conj(G^-1 b), t.
//
//   k_powers     pw[l][j][a] = z_j(l)^a, a = 0..n, by repeated multiplication (R9)
//   k_vls        per column block: A tile (m x 32) in smem from the power tables
//                (A[j][k] = prod_l pw[l][j][k_l]), optional coalesced A write (HBM-bound),
//                G_part += A_tile A_tile^H and b_part += A_tile conj(f_tile) (DFMA)
//   k_ls_reduce  fixed-order sum of the partials -> G, b
//   k_solve      one CTA: Cholesky G = L L^H, L y = b, L^H x = y, c = conj(x); t = (-arg z/2pi) mod 1
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "vandermonde_ls.cuh"

namespace prony {

__global__ void k_powers(int d, int n, int m, const double2* __restrict__ z, double2* __restrict__ pw) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d * m) return;
  const int l = e / m, j = e % m;
  const double2 zz = z[(size_t)j * d + l];
  double2 p = make_double2(1.0, 0.0);
  double2* out = pw + (size_t)e * (n + 1);
  for (int a = 0; a <= n; ++a) {
    out[a] = p;
    p = cmul(p, zz);
  }
}

// grid (CB, ceil(m/64)); CTA cb handles columns [cbeg, cend) of I_n in tiles of kTile.
__global__ void __launch_bounds__(256) k_vls(VlsParams p) {
  __shared__ double2 As[kMaxM][kTile + 1];
  __shared__ double2 Fs[kTile];
  const int cb = blockIdx.x;
  const int i0 = blockIdx.y * 64;
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const int m = p.m, d = p.d, n = p.n;
  const int64_t W = p.col_end - p.col_begin;
  const int64_t cbeg = p.col_begin + W * cb / p.CB;
  const int64_t cend = p.col_begin + W * (cb + 1) / p.CB;
  const int L = 2 * n + 2;
  double2 acc[4][8];
  double2 bacc = make_double2(0.0, 0.0);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = make_double2(0.0, 0.0);

  for (int64_t c0 = cbeg; c0 < cend; c0 += kTile) {
    // A tile: As[j][kk] = prod_l pw[l][j][k_l], k = c0 + kk
    for (int e = tid; e < m * kTile; e += 256) {
      const int j = e / kTile, kk = e % kTile;
      const int64_t k = c0 + kk;
      double2 a = make_double2(0.0, 0.0);
      if (k < cend) {
        int digit[PRONY_MAX_D];
        int64_t r = k;
        for (int l = d - 1; l >= 0; --l) {
          digit[l] = (int)(r % (n + 1));
          r /= (n + 1);
        }
        a = p.pw[((size_t)0 * m + j) * (n + 1) + digit[0]];
        for (int l = 1; l < d; ++l) a = cmul(a, p.pw[((size_t)l * m + j) * (n + 1) + digit[l]]);
        if (p.A && blockIdx.y == 0) p.A[(size_t)j * W + (k - p.col_begin)] = a;
      }
      As[j][kk] = a;
    }
    if (tid < kTile) {
      const int64_t k = c0 + tid;
      double2 f = make_double2(0.0, 0.0);
      if (k < cend) {
        int64_t r = k, idx = 0, s = 1;
        for (int l = d - 1; l >= 0; --l) {
          idx += (r % (n + 1) + n) * s;
          r /= (n + 1);
          s *= L;
        }
        f = cconj(ldg2(p.grid + idx));
      }
      Fs[tid] = f;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kTile; ++kk) {
      double2 u[4], v[8];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = i0 + ti + 16 * a;
        u[a] = i < m ? As[i][kk] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int j = tj + 16 * b;
        v[b] = j < m ? cconj(As[j][kk]) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          acc[a][b].x = fma(u[a].x, v[b].x, acc[a][b].x);
          acc[a][b].x = fma(-u[a].y, v[b].y, acc[a][b].x);
          acc[a][b].y = fma(u[a].x, v[b].y, acc[a][b].y);
          acc[a][b].y = fma(u[a].y, v[b].x, acc[a][b].y);
        }
    }
    if (tid < 64 && i0 + tid < m) {
      const int i = i0 + tid;
      for (int kk = 0; kk < kTile; ++kk) {
        const double2 a = As[i][kk], f = Fs[kk];
        bacc.x = fma(a.x, f.x, bacc.x);
        bacc.x = fma(-a.y, f.y, bacc.x);
        bacc.y = fma(a.x, f.y, bacc.y);
        bacc.y = fma(a.y, f.x, bacc.y);
      }
    }
    __syncthreads();
  }
  double2* G = p.Gpart + (size_t)cb * m * m;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + ti + 16 * a;
    if (i >= m) continue;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int j = tj + 16 * b;
      if (j < m) G[(size_t)i * m + j] = acc[a][b];
    }
  }
  if (tid < 64 && i0 + tid < m) p.bpart[(size_t)cb * m + i0 + tid] = bacc;
}

__global__ void k_ls_reduce(int m, int CB, const double2* __restrict__ Gpart, const double2* __restrict__ bpart,
                            double2* __restrict__ G, double2* __restrict__ b) {
  const int tot = m * m + m;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    if (e < m * m) {
      for (int c = 0; c < CB; ++c) s = cadd(s, Gpart[(size_t)c * m * m + e]);
      G[e] = s;
    } else {
      const int i = e - m * m;
      for (int c = 0; c < CB; ++c) s = cadd(s, bpart[(size_t)c * m + i]);
      b[i] = s;
    }
  }
}

// One CTA (256 threads). Lw: m x m scratch (lower Cholesky factor), y: m scratch.
__global__ void __launch_bounds__(256) k_solve(int d, int m, const double2* __restrict__ G,
                                               const double2* __restrict__ b, const double2* __restrict__ z,
                                               double2* __restrict__ Lw, double2* __restrict__ y,
                                               double2* __restrict__ c, double* __restrict__ t, int32_t* status) {
  __shared__ int bad;
  __shared__ double ljj_s;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < m * m; e += blockDim.x) Lw[e] = G[e];
  __syncthreads();
  // left-looking Cholesky, column j: L[j][j] = sqrt(G[j][j] - sum_p |L[j][p]|^2),
  // L[i][j] = (G[i][j] - sum_{p<j} L[i][p] conj(L[j][p])) / L[j][j]   (i > j)
  for (int j = 0; j < m; ++j) {
    if (tid == 0) {
      double djj = Lw[(size_t)j * m + j].x;
      for (int q = 0; q < j; ++q) {
        const double2 v = Lw[(size_t)j * m + q];
        djj -= v.x * v.x + v.y * v.y;
      }
      if (!(djj > 0.0)) bad = 1;
      ljj_s = bad ? 1.0 : sqrt(djj);
      Lw[(size_t)j * m + j] = make_double2(ljj_s, 0.0);
    }
    __syncthreads();
    const double ljj = ljj_s;
    for (int i = j + 1 + tid; i < m; i += blockDim.x) {
      double2 s = Lw[(size_t)i * m + j];
      for (int q = 0; q < j; ++q) {
        const double2 a = Lw[(size_t)i * m + q], bb = cconj(Lw[(size_t)j * m + q]);
        s.x -= a.x * bb.x - a.y * bb.y;
        s.y -= a.x * bb.y + a.y * bb.x;
      }
      Lw[(size_t)i * m + j] = make_double2(s.x / ljj, s.y / ljj);
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) set_status(status, PRONY_ERR_SINGULAR);
    for (int i = tid; i < m; i += blockDim.x) c[i] = make_double2(NAN, NAN);
  } else if (tid < 32) {
    // forward: L y = b ; backward: L^H x = y  (one warp, lane-parallel dot products)
    const int lane = tid;
    for (int i = 0; i < m; ++i) {
      double2 s = make_double2(0.0, 0.0);
      for (int q = lane; q < i; q += 32) {
        const double2 a = Lw[(size_t)i * m + q], v = y[q];
        s.x += a.x * v.x - a.y * v.y;
        s.y += a.x * v.y + a.y * v.x;
      }
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) {
        const double2 bi = b[i];
        const double lii = Lw[(size_t)i * m + i].x;
        y[i] = make_double2((bi.x - s.x) / lii, (bi.y - s.y) / lii);
      }
      __syncwarp();
    }
    for (int i = m - 1; i >= 0; --i) {
      double2 s = make_double2(0.0, 0.0);
      for (int q = i + 1 + lane; q < m; q += 32) {
        const double2 a = cconj(Lw[(size_t)q * m + i]), v = y[q];
        s.x += a.x * v.x - a.y * v.y;
        s.y += a.x * v.y + a.y * v.x;
      }
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) {
        const double2 yi = y[i];
        const double lii = Lw[(size_t)i * m + i].x;
        y[i] = make_double2((yi.x - s.x) / lii, (yi.y - s.y) / lii);
      }
      __syncwarp();
    }
    for (int i = lane; i < m; i += 32) c[i] = cconj(y[i]);
  }
  if (t) {
    const double inv2pi = 0.15915494309189533577;  // 1 / (2 pi)
    for (int e = tid; e < m * d; e += blockDim.x) {
      const double2 zz = z[e];
      double v = -atan2(zz.y, zz.x) * inv2pi;  // (-arg z / 2 pi) mod 1  (R4)
      v = v - floor(v);
      if (v >= 1.0) v = 0.0;
      t[e] = v;
    }
  }
}

// ---------------------------------------------------------------------------- host side
static int vls_cb(int64_t W, int m, int sm_count) {
  const int ib = (m + 63) / 64;
  int64_t tiles = (W + kTile - 1) / kTile;
  int64_t cb = (2 * (int64_t)sm_count) / ib;
  cb = std::max<int64_t>(1, std::min<int64_t>(cb, tiles));
  return (int)cb;
}

size_t ls_workspace_bytes(int d, int n, int m, int sm_count) {
  size_t bytes = align_up((size_t)d * m * (n + 1) * sizeof(double2), 256);  // power tables
  const int ib = (m + 63) / 64;
  const int cbmax = std::max(1, (2 * sm_count) / ib);
  bytes += align_up((size_t)cbmax * m * m * sizeof(double2), 256);  // G partials
  bytes += align_up((size_t)cbmax * m * sizeof(double2), 256);      // b partials
  bytes += align_up((size_t)m * m * sizeof(double2), 256);          // Cholesky factor
  bytes += align_up((size_t)m * sizeof(double2), 256);              // y
  return bytes;
}

int ls_launch(int d, int n, int m, int N, const double2* z, const double2* grid, int64_t col_begin, int64_t col_end,
              double2* A, double2* G, double2* b, double2* c, double* t, void* ws, int32_t* status, int sm_count,
              cudaStream_t st, prony_exec_info* info) {
  char* w = (char*)ws;
  double2* pw = (double2*)w;
  w += align_up((size_t)d * m * (n + 1) * sizeof(double2), 256);
  const int ib = (m + 63) / 64;
  const int cbmax = std::max(1, (2 * sm_count) / ib);
  double2* Gpart = (double2*)w;
  w += align_up((size_t)cbmax * m * m * sizeof(double2), 256);
  double2* bpart = (double2*)w;
  w += align_up((size_t)cbmax * m * sizeof(double2), 256);
  double2* Lw = (double2*)w;
  w += align_up((size_t)m * m * sizeof(double2), 256);
  double2* yv = (double2*)w;

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
  p.CB = vls_cb(W, m, sm_count);
  p.pw = pw;
  p.grid = grid;
  p.A = A;
  p.Gpart = Gpart;
  p.bpart = bpart;
  if (info && info->ev_main_begin) cudaEventRecord((cudaEvent_t)info->ev_main_begin, st);
  k_vls<<<dim3(p.CB, ib), 256, 0, st>>>(p);
  if (info && info->ev_main_end) cudaEventRecord((cudaEvent_t)info->ev_main_end, st);
  int launches = 3;
  k_ls_reduce<<<(m * m + m + 255) / 256, 256, 0, st>>>(m, p.CB, Gpart, bpart, G, b);
  if (col_begin == 0 && col_end == N && (c || t)) {
    double2* cc = c ? c : yv;  // c is required by the solve; if only t is wanted, solve into scratch
    if (c) k_solve<<<1, 256, 0, st>>>(d, m, G, b, z, Lw, yv, cc, t, status);
    else k_solve<<<1, 256, 0, st>>>(d, m, G, b, z, Lw, yv, Lw, t, status);
    ++launches;
  }
  if (info) {
    info->launches = launches;
    info->main_grid[0] = p.CB;
    info->main_grid[1] = ib;
    info->main_grid[2] = 1;
    info->main_block = 256;
    info->split_k = p.CB;
    info->main_flops = 8.0 * m * (double)m * (double)W + 8.0 * m * (double)W;
  }
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

int ls_solve_launch(int d, int m, const double2* G, const double2* b, const double2* z, double2* c, double* t,
                    void* ws, int32_t* status, cudaStream_t st) {
  double2* Lw = (double2*)ws;
  double2* yv = (double2*)((char*)ws + align_up((size_t)m * m * sizeof(double2), 256));
  k_solve<<<1, 256, 0, st>>>(d, m, G, b, z, Lw, yv, c, t, status);
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

}  // namespace prony
