// vandermonde_ls.cu — A = [z_j^k], G = A conj(A)^T, b = A conj(f) (PAPER.md:59,
// normal equations of argmin ||A^T c - f||_2; R10), c = conj(G^-1 b), t.
//
//   k_powers     pw[l][j][a] = z_j(l)^a, a = 0..n, by repeated multiplication (R9)
//   k_vls        per column block (16 warps): A tile (m x 16 columns) built in shared memory from
//                the power tables (A[j][k] = prod_l pw[l][j][k_l]), optional coalesced A write,
//                G_part += A_tile conj(A_tile)^T on the DMMA warp engine (3M), b_part += A conj(f)
//   k_ls_reduce  fixed-order sum of the partials -> G, b
//   k_solve      one CTA, factor resident in shared memory: right-looking Cholesky G = L L^H,
//                L y = b, L^H x = y, c = conj(x); t = (-arg z / 2 pi) mod 1 (R4)
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "engine.cuh"
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

// grid (CB, ceil(m/BI)); CTA (cb, ib) handles columns [cbeg, cend) of I_n in tiles of kTile and
// rows i in [BI ib, BI ib + BI) of G. Shared memory (dynamic): At[kTile][cap] (A[j][k], double2),
// Sp[kTile][cap] (Re+Im), Sm[kTile][cap] (Re-Im), Fs[kTile] (conj f). A operand rows i, B operand
// conj(A) rows j (engine CONJB) -> G[i][j] = sum_k A[i][k] conj(A[j][k]).
template <int NT, int WN>
__global__ void __launch_bounds__(kVlsThreads, 1) k_vls(VlsParams p) {
  constexpr int WM = (kVlsThreads / 32) / WN, BI = 16 * WM;
  extern __shared__ __align__(16) double vsm[];
  const int cap = p.cap;  // row capacity of the smem planes (>= every row read)
  const int lda = cap + 2, lds = cap + 4;
  double2* At = reinterpret_cast<double2*>(vsm);
  double* Sp = vsm + 2 * kTile * lda;
  double* Sm = Sp + kTile * lds;
  double2* Fs = reinterpret_cast<double2*>(Sm + kTile * lds);

  const int cb = blockIdx.x;
  const int i0 = blockIdx.y * BI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q = lane & 3;
  const int m = p.m, d = p.d, n = p.n;
  const int ntot = (m + 7) / 8;
  const int t0 = (ntot * wn) / WN;
  const int nt_active = (ntot * (wn + 1)) / WN - t0;
  const bool warp_rows = (i0 + wm * 16) < m;
  const int64_t W = p.col_end - p.col_begin;
  const int64_t cbeg = p.col_begin + W * cb / p.CB;
  const int64_t cend = p.col_begin + W * (cb + 1) / p.CB;
  const int L = 2 * n + 2;

  // rows >= m of the planes stay zero
  for (int e = tid; e < kTile * lda; e += kVlsThreads) At[e] = make_double2(0.0, 0.0);
  for (int e = tid; e < kTile * lds; e += kVlsThreads) Sp[e] = Sm[e] = 0.0;

  double acc[3][NT][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][j][e] = 0.0;
  double2 bacc = make_double2(0.0, 0.0);
  __syncthreads();

  for (int64_t c0 = cbeg; c0 < cend; c0 += kTile) {
    // A tile: A[j][k] = prod_l pw[l][j][k_l], k = c0 + kk, product in order l = 1..d (R9)
    for (int e = tid; e < m * kTile; e += kVlsThreads) {
      const int j = e / kTile, kk = e % kTile;
      const int64_t k = c0 + kk;
      double2 a = make_double2(0.0, 0.0);
      if (k < cend) {
        int dig[PRONY_MAX_D];
        int64_t r = k;
        for (int l = d - 1; l >= 0; --l) {  // digits of k, last coordinate fastest
          dig[l] = (int)(r % (n + 1));
          r /= (n + 1);
        }
        a = p.pw[(size_t)j * (n + 1) + dig[0]];
        for (int l = 1; l < d; ++l) a = cmul(a, p.pw[((size_t)l * m + j) * (n + 1) + dig[l]]);
        if (p.A && blockIdx.y == 0) p.A[(size_t)j * W + (k - p.col_begin)] = a;
      }
      At[kk * lda + j] = a;
      Sp[kk * lds + j] = a.x + a.y;
      Sm[kk * lds + j] = a.x - a.y;
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
    if (warp_rows) {
#pragma unroll
      for (int kk = 0; kk < kTile / 4; ++kk)
        warp_cmma_k4_n<NT, 3, true>(nt_active, acc, At + kk * 4 * lda + i0 + wm * 16,
                                    Sp + kk * 4 * lds + i0 + wm * 16, lda, lds, At + kk * 4 * lda + t0 * 8,
                                    Sm + kk * 4 * lds + t0 * 8, lda, lds, g, q);
    }
    if (tid < BI && i0 + tid < m) {
      const int i = i0 + tid;
#pragma unroll 4
      for (int kk = 0; kk < kTile; ++kk) {
        const double2 a = At[kk * lda + i], f = Fs[kk];
        bacc.x = fma(a.x, f.x, bacc.x);
        bacc.x = fma(-a.y, f.y, bacc.x);
        bacc.y = fma(a.x, f.y, bacc.y);
        bacc.y = fma(a.y, f.x, bacc.y);
      }
    }
    __syncthreads();
  }
  double2* G = p.Gpart + (size_t)cb * m * m;
  const int ia = i0 + wm * 16 + g, ib = ia + 8;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < nt_active) {
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
  if (tid < BI && i0 + tid < m) p.bpart[(size_t)cb * m + i0 + tid] = bacc;
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

// One CTA of kSolveThreads. Right-looking Cholesky G = L L^H with lazily scaled columns: column j is
// never rescaled, L[i][j] = A[i][j] / sqrt(d_j) with d_j the pivot (inv[j] = 1/sqrt(d_j)). The lower
// triangle lives in registers (each thread owns <= kSolveOwn entries); per column the owners publish
// column j to a double-buffered shared vector, ONE barrier, and every owner of an entry right of it
// applies the rank-1 update. The factor is then stored packed (A[i][k] at i(i+1)/2 + k) for the
// substitutions.
// Forward / backward substitution run in one warp with the right-hand side in registers.
constexpr int kSolveMaxRowsPerLane = (PRONY_MAX_M + 31) / 32;
constexpr int kSolveOwn = (PRONY_MAX_M * (PRONY_MAX_M + 1) / 2 + kSolveThreads - 1) / kSolveThreads;
__global__ void __launch_bounds__(kSolveThreads) k_solve(int d, int m, const double2* __restrict__ G,
                                                         const double2* __restrict__ b,
                                                         const double2* __restrict__ z, double2* __restrict__ c,
                                                         double* __restrict__ t, int32_t* status) {
  extern __shared__ __align__(16) double2 As[];  // m(m+1)/2 packed
  __shared__ double inv[PRONY_MAX_M];
  __shared__ double2 colbuf[2][PRONY_MAX_M];  // the pivot column, double-buffered
  __shared__ int bad;
  const int tid = threadIdx.x;
  auto at = [](int i, int k) { return i * (i + 1) / 2 + k; };
  if (tid == 0) bad = 0;
  // each thread owns up to kSolveOwn entries of the lower triangle, kept in registers for the whole
  // factorization: entry e = tid + kSolveThreads s of the packed order
  const int T = m * (m + 1) / 2;
  double2 val[kSolveOwn];
  int oi[kSolveOwn], ok[kSolveOwn];
#pragma unroll
  for (int s = 0; s < kSolveOwn; ++s) {
    const int e = tid + kSolveThreads * s;
    oi[s] = -1;
    ok[s] = -1;
    val[s] = make_double2(0.0, 0.0);
    if (e < T) {
      int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > e) --i;
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      oi[s] = i;
      ok[s] = e - i * (i + 1) / 2;
      val[s] = G[(size_t)i * m + ok[s]];
    }
  }
  for (int j = 0; j < m; ++j) {
    double2* buf = colbuf[j & 1];
#pragma unroll
    for (int s = 0; s < kSolveOwn; ++s)
      if (ok[s] == j) buf[oi[s]] = val[s];  // publish column j (final: updated through column j-1)
    __syncthreads();
    const double dj = buf[j].x;  // uniform
    if (!(dj > 0.0)) {
      if (tid == 0) bad = 1;
      break;
    }
    const double invd = 1.0 / dj;  // L[i][j] conj(L[k][j]) = A[i][j] conj(A[k][j]) / d_j
    if (tid == 0) inv[j] = sqrt(invd);
#pragma unroll
    for (int s = 0; s < kSolveOwn; ++s) {
      if (ok[s] > j) {
        const double2 a = buf[oi[s]], bb = buf[ok[s]];
        val[s].x -= (a.x * bb.x + a.y * bb.y) * invd;
        val[s].y -= (a.y * bb.x - a.x * bb.y) * invd;
      }
    }
    // no second barrier: column j+1 goes to the other buffer, and this buffer is rewritten only after
    // the next iteration's barrier, which every thread reaches after its reads here
  }
#pragma unroll
  for (int s = 0; s < kSolveOwn; ++s)
    if (oi[s] >= 0) As[at(oi[s], ok[s])] = val[s];  // lazily scaled factor for the substitutions
  __syncthreads();
  if (bad) {
    if (tid == 0) set_status(status, PRONY_ERR_SINGULAR);
    for (int i = tid; i < m; i += kSolveThreads) c[i] = make_double2(NAN, NAN);
  } else if (tid < 32) {
    const int lane = tid;
    double2 y[kSolveMaxRowsPerLane];
#pragma unroll
    for (int q = 0; q < kSolveMaxRowsPerLane; ++q) {
      const int i = lane + 32 * q;
      y[q] = i < m ? b[i] : make_double2(0.0, 0.0);
    }
    // forward: L y = b, column oriented: y_j /= L_jj; y_i -= L_ij y_j (i > j)
    for (int j = 0; j < m; ++j) {
      const int qj = j >> 5, lj = j & 31;
      double2 yj = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kSolveMaxRowsPerLane; ++q)
        if (q == qj) yj = y[q];
      yj.x = __shfl_sync(0xffffffffu, yj.x, lj);
      yj.y = __shfl_sync(0xffffffffu, yj.y, lj);
      const double ij = inv[j];
      yj = make_double2(yj.x * ij, yj.y * ij);
#pragma unroll
      for (int q = 0; q < kSolveMaxRowsPerLane; ++q) {
        const int i = lane + 32 * q;
        if (i == j) y[q] = yj;
        if (i > j && i < m) {
          const double2 a = As[at(i, j)];
          const double2 l = make_double2(a.x * ij, a.y * ij);
          y[q].x -= l.x * yj.x - l.y * yj.y;
          y[q].y -= l.x * yj.y + l.y * yj.x;
        }
      }
    }
    // backward: L^H x = y: x_j = y_j / L_jj; y_i -= conj(L_ji) x_j (i < j)
    for (int j = m - 1; j >= 0; --j) {
      const int qj = j >> 5, lj = j & 31;
      double2 xj = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kSolveMaxRowsPerLane; ++q)
        if (q == qj) xj = y[q];
      xj.x = __shfl_sync(0xffffffffu, xj.x, lj);
      xj.y = __shfl_sync(0xffffffffu, xj.y, lj);
      const double ij = inv[j];
      xj = make_double2(xj.x * ij, xj.y * ij);
#pragma unroll
      for (int q = 0; q < kSolveMaxRowsPerLane; ++q) {
        const int i = lane + 32 * q;
        if (i == j) y[q] = xj;
        if (i < j) {
          const double2 a = As[at(j, i)];
          const double ii_ = inv[i];
          const double2 l = make_double2(a.x * ii_, -a.y * ii_);  // conj(L_ji)
          y[q].x -= l.x * xj.x - l.y * xj.y;
          y[q].y -= l.x * xj.y + l.y * xj.x;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kSolveMaxRowsPerLane; ++q) {
      const int i = lane + 32 * q;
      if (i < m) c[i] = cconj(y[q]);
    }
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
struct VlsShape {
  int NT, WN, BI, cap;
};
VlsShape vls_shape(int m) {
  VlsShape s;
  const int ntot = (m + 7) / 8;
  s.WN = ntot <= 8 ? 2 : 4;
  s.NT = (ntot + s.WN - 1) / s.WN;
  s.BI = 16 * ((kVlsThreads / 32) / s.WN);
  const int rows_a = (m + s.BI - 1) / s.BI * s.BI;  // A-operand rows read (whole i-blocks)
  const int rows_b = 8 * s.NT * s.WN;              // B-operand rows read
  s.cap = std::max(rows_a, rows_b);
  return s;
}
size_t vls_smem(int cap) {
  const int lda = cap + 2, lds = cap + 4;
  return (size_t)(2 * kTile * lda + 2 * kTile * lds) * sizeof(double) + kTile * sizeof(double2);
}
int vls_cb(int64_t W, int m, int sm_count) {
  const VlsShape s = vls_shape(m);
  const int ib = (m + s.BI - 1) / s.BI;
  const int64_t tiles = (W + kTile - 1) / kTile;
  int64_t cb = std::max<int64_t>(1, sm_count / ib);
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

template <int NT, int WN>
static int launch_vls_t(const VlsParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  if (cudaFuncSetAttribute(k_vls<NT, WN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  k_vls<NT, WN><<<grid, kVlsThreads, smem, st>>>(p);
  return PRONY_OK;
}

int ls_solve_launch(int d, int m, const double2* G, const double2* b, const double2* z, double2* c, double* t,
                    void* ws, int32_t* status, cudaStream_t st) {
  (void)ws;
  const size_t smem = solve_smem(m);
  if (cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
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
  const VlsShape sh = vls_shape(m);
  VlsParams p{};
  p.d = d;
  p.n = n;
  p.m = m;
  p.col_begin = col_begin;
  p.col_end = col_end;
  p.CB = vls_cb(W, m, sm_count);
  p.cap = sh.cap;
  p.pw = pw;
  p.grid = grid;
  p.A = A;
  p.Gpart = Gpart;
  p.bpart = bpart;
  const int ib = (m + sh.BI - 1) / sh.BI;
  const dim3 vgrid(p.CB, ib);
  const size_t smem = vls_smem(sh.cap);
  if (info && info->ev_main_begin) cudaEventRecord((cudaEvent_t)info->ev_main_begin, st);
  int rc = PRONY_OK;
  switch (sh.WN * 16 + sh.NT) {
#define PRONY_VCASE(nt, wn) \
  case wn * 16 + nt:        \
    rc = launch_vls_t<nt, wn>(p, vgrid, smem, st); \
    break;
    PRONY_VCASE(1, 2) PRONY_VCASE(2, 2) PRONY_VCASE(3, 2) PRONY_VCASE(4, 2) PRONY_VCASE(3, 4) PRONY_VCASE(4, 4)
#undef PRONY_VCASE
    default:
      return PRONY_ERR_RANGE;
  }
  if (rc != PRONY_OK) return rc;
  if (info && info->ev_main_end) cudaEventRecord((cudaEvent_t)info->ev_main_end, st);
  int launches = 3;
  k_ls_reduce<<<(m * m + m + 255) / 256, 256, 0, st>>>(m, p.CB, Gpart, bpart, G, b);
  if (col_begin == 0 && col_end == N && (c || t)) {
    // only t requested: solve into the (now consumed) G partial buffer
    rc = ls_solve_launch(d, m, G, b, z, c ? c : Gpart, t, nullptr, status, st);
    if (rc != PRONY_OK) return rc;
    ++launches;
  }
  if (info) {
    info->launches = launches;
    info->main_grid[0] = p.CB;
    info->main_grid[1] = ib;
    info->main_grid[2] = 1;
    info->main_block = kVlsThreads;
    info->split_k = p.CB;
    info->main_flops = 8.0 * m * (double)m * (double)W + 8.0 * m * (double)W;
  }
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  return PRONY_OK;
}

}  // namespace prony
