// dense.cu — the small dense linear algebra of Algorithm 1 that runs on the device outside the
// measured hot path (NEXT-1): tall-skinny Gram / Cholesky-QR with diagonal pivoting
// (rank determination of the block power method, Alg. 3), the SVD of the projected
// r x r matrix Q_k (one-sided Jacobi), the eigendecomposition of C_mu (Hessenberg reduction
// + shifted QR eigenvalues + inverse-iteration eigenvectors) and the simultaneous diagonalization
// W^-1 S_l W.
// Everything is FP64 complex; the N-sized products use all SMs, the r x r / m x m algorithms run in
// one CTA (or one warp) on L2-resident matrices. All matrices are row-major.
#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "common.cuh"
#include "dense.cuh"

namespace prony {

__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // c + a*b
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) { return make_double2(warp_sum(v.x), warp_sum(v.y)); }

// ---------------------------------------------------------------------------- random block
// Seeded complex Gaussian entries from a counter-based generator (splitmix64 of (seed, index)) +
// Box-Muller: the same block for the same seed on every GPU and run (R14: U0/V0 unspecified by P:181).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void k_fill_random(int64_t count, uint64_t seed, double2* __restrict__ out, int rows, int cols, int ld) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h1 = splitmix64(seed ^ (2 * (uint64_t)e));
    const uint64_t h2 = splitmix64(seed ^ (2 * (uint64_t)e + 1));
    const double u1 = ((h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = ((h2 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double rr = sqrt(-2.0 * log(u1));
    const int64_t r = e / cols, c = e % cols;
    if (r < rows) out[r * ld + c] = make_double2(rr * cospi(2.0 * u2), rr * sinpi(2.0 * u2));
  }
}

// ---------------------------------------------------------------------------- Gram
// Gp[z][i][j] = sum_{k in slice z} conj(X[k][i]) Y[k][j]  (ri x rj; 32 x 32 output tile per CTA, DFMA)
constexpr int kGT = 32;
__global__ void __launch_bounds__(256) k_gram(int N, int ri, int rj, const double2* __restrict__ X, int ldx,
                                             const double2* __restrict__ Y, int ldy, int KS,
                                             double2* __restrict__ Gp) {
  __shared__ double2 Xi[kGT][kGT + 1];
  __shared__ double2 Xj[kGT][kGT + 1];
  const int i0 = blockIdx.x * kGT, j0 = blockIdx.y * kGT, z = blockIdx.z;
  const int k_begin = (int)((int64_t)N * z / KS), k_end = (int)((int64_t)N * (z + 1) / KS);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double2 acc[2][2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) acc[a][b] = make_double2(0.0, 0.0);
  for (int k0 = k_begin; k0 < k_end; k0 += kGT) {
    for (int e = threadIdx.x; e < kGT * kGT; e += 256) {
      const int kk = e / kGT, c = e % kGT;
      const int k = k0 + kk;
      Xi[kk][c] = (k < k_end && i0 + c < ri) ? X[(size_t)k * ldx + i0 + c] : make_double2(0.0, 0.0);
      Xj[kk][c] = (k < k_end && j0 + c < rj) ? Y[(size_t)k * ldy + j0 + c] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kGT; ++kk) {
      const double2 u0 = Xi[kk][ty], u1 = Xi[kk][ty + 16];
      const double2 v0 = Xj[kk][tx], v1 = Xj[kk][tx + 16];
      acc[0][0] = cfma(cconj(u0), v0, acc[0][0]);
      acc[0][1] = cfma(cconj(u0), v1, acc[0][1]);
      acc[1][0] = cfma(cconj(u1), v0, acc[1][0]);
      acc[1][1] = cfma(cconj(u1), v1, acc[1][1]);
    }
    __syncthreads();
  }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i < ri && j < rj) Gp[((size_t)z * ri + i) * rj + j] = acc[a][b];
    }
}

// out[e] = sum_{z < KS} parts[z * count + e]   (fixed order)
__global__ void k_sum_parts(int64_t count, int KS, const double2* __restrict__ parts, double2* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int z = 0; z < KS; ++z) s = cadd(s, parts[(size_t)z * count + e]);
    out[e] = s;
  }
}

// ---------------------------------------------------------------------------- small GEMM
// Y[N x c] = alpha * X[N x r] M[r x c] + beta * Y   (64 x 32 output tile per CTA, DFMA)
__global__ void __launch_bounds__(256) k_gemm_nm(int N, int r, int c, const double2* __restrict__ X, int ldx,
                                                const double2* __restrict__ M, int ldm, double2* __restrict__ Y,
                                                int ldy, double alpha, double beta) {
  __shared__ double2 Xs[64][17];
  __shared__ double2 Ms[16][33];
  const int row0 = blockIdx.x * 64, col0 = blockIdx.y * 32;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 2 columns x 4 rows per thread
  double2 acc[4][2];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 2; ++b) acc[a][b] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < r; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int rr = e / 16, kk = e % 16;
      const int row = row0 + rr, k = k0 + kk;
      Xs[rr][kk] = (row < N && k < r) ? X[(size_t)row * ldx + k] : make_double2(0.0, 0.0);
    }
    for (int e = threadIdx.x; e < 16 * 32; e += 256) {
      const int kk = e / 32, cc = e % 32;
      const int k = k0 + kk, col = col0 + cc;
      Ms[kk][cc] = (k < r && col < c) ? M[(size_t)k * ldm + col] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const double2 m0 = Ms[kk][tx], m1 = Ms[kk][tx + 16];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double2 x = Xs[ty + 16 * a][kk];
        acc[a][0] = cfma(x, m0, acc[a][0]);
        acc[a][1] = cfma(x, m1, acc[a][1]);
      }
    }
    __syncthreads();
  }
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 2; ++b) {
      const int row = row0 + ty + 16 * a, col = col0 + tx + 16 * b;
      if (row < N && col < c) {
        double2* y = Y + (size_t)row * ldy + col;
        const double2 old = beta != 0.0 ? *y : make_double2(0.0, 0.0);
        *y = make_double2(alpha * acc[a][b].x + beta * old.x, alpha * acc[a][b].y + beta * old.y);
      }
    }
}

// ---------------------------------------------------------------------------- norms
// parts[blockIdx] = sum of |X[k][j]|^2 over the block's elements (then summed in fixed order)
__global__ void k_fro2_parts(int N, int c, const double2* __restrict__ X, int ldx, double* __restrict__ parts) {
  __shared__ double red[32];
  double s = 0.0;
  const int64_t tot = (int64_t)N * c;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
    s += cabs2(X[(e / c) * ldx + e % c]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) parts[blockIdx.x] = v;
  }
}
// ||T||_F^2 = sum over v in {-n..n}^d of |f(v)|^2 prod_i (n + 1 - |v_i|)   (T = [f(k-h)])
__global__ void k_normT2_parts(int d, int n, int64_t box, const double2* __restrict__ grid, double* __restrict__ parts) {
  __shared__ double red[32];
  const int L = 2 * n + 2;
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < box; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e;
    double mult = 1.0;
    for (int i = 0; i < d; ++i) {
      const int v = (int)(r % L) - n;
      r /= L;
      mult *= (v > n) ? 0.0 : (double)(n + 1 - abs(v));
    }
    if (mult > 0.0) s += mult * cabs2(grid[e]);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) parts[blockIdx.x] = v;
  }
}
__global__ void k_sum_doubles(int count, const double* __restrict__ parts, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += parts[i];
    *out = s;
  }
}

// ---------------------------------------------------------------------------- Householder QR (tall)
// Reduced QR of a tall N x r matrix X (row-major, ld ldx, r <= kHouseMaxCols) by Householder reflectors
// ("QR factorization implemented with Householder reflectors"), optionally with column pivoting
// (the column with the largest remaining norm first; the rank is the first k with
// ||R(k:, k:)||_F <= tol ||R||_F, P:193 / P:203, the rule of Alg. 3 line 10), and the explicit
// Q(:, :rank) = H_0 ... H_{rank-1} [I; 0] in logical (pivoted) column order.
// ONE cooperative launch: CTA c owns the rows [c rows_per_cta, (c+1) rows_per_cta); one pass over the
// trailing rows and one two-level grid reduction (two barriers) per factorization step and per Q step.
// The pass leaves per-CTA column partials (warp accumulators summed in a fixed warp order) in a
// column-major buffer; the columns are then summed over the CTAs in a fixed order by warps spread over
// the grid and broadcast back to every CTA, so the pivot choice and the rank decision are bitwise
// identical in all CTAs and the result is deterministic. The trailing norms are recomputed
// exactly at every step from the updated entries (the pivot of step k + 1 is chosen from them downdated by
// row k of R, so that step k's pass can already accumulate step k + 1's products). Pivoting is logical: a done[] flag
// per physical column, X is never permuted, so every row access stays coalesced.
// On exit X holds the reflector tails below the diagonal of the pivot columns (row k keeps its values before
// H_k: R itself is not needed by the callers).
namespace cg = cooperative_groups;
constexpr int kHqThreads = 512;
constexpr int kHqWarps = kHqThreads / 32;
constexpr int kHqT = kHouseMaxCols / 32;  // column chunks per lane

template <typename T>
__device__ __forceinline__ T hq_zero();
template <>
__device__ __forceinline__ double hq_zero<double>() { return 0.0; }
template <>
__device__ __forceinline__ double2 hq_zero<double2>() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double hq_add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 hq_add(double2 a, double2 b) { return cadd(a, b); }
__device__ __forceinline__ double hq_shfl(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ double2 hq_shfl(double2 v, int o) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}

// CTA column partials: part[j * G + blockIdx.x] = sum over the warps (fixed order) of acc[t] (j = lane + 32 t)
template <typename T>
__device__ __forceinline__ void hq_cta_part(const T (&acc)[kHqT], T* red, int r, int j0, T* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < kHqT; ++t) {
    const int j = lane + 32 * t;
    if (j < r) red[warp * r + j] = acc[t];
  }
  __syncthreads();
  for (int j = j0 + threadIdx.x; j < r; j += kHqThreads) {
    T s = red[j];
    for (int w = 1; w < kHqWarps; ++w) s = hq_add(s, red[w * r + j]);
    part[(size_t)j * gridDim.x + blockIdx.x] = s;
  }
  __syncthreads();
}

// Two-level grid reduction of the column partials, deterministic: phase A (after the barrier that published
// the partials) spreads the columns over the warps of the whole grid, fin[j] = sum_c part[j * G + c] in a
// fixed order (lanes over CTAs, then a fixed shuffle tree); phase B (after the next barrier) copies the
// finished columns into every CTA's shared memory. Both phases skip the columns flagged in skip[].
template <typename T>
__device__ __forceinline__ void hq_reduce_a(const T* part, T* fin, int r, int j0, const unsigned char* skip) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  for (int j = j0 + blockIdx.x * kHqWarps + warp; j < r; j += G * kHqWarps) {
    if (skip && skip[j]) continue;
    T s = hq_zero<T>();
    for (int c = lane; c < G; c += 32) s = hq_add(s, __ldcg(part + (size_t)j * G + c));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = hq_add(s, hq_shfl(s, o));
    if (lane == 0) fin[j] = s;
  }
}
template <typename T>
__device__ __forceinline__ void hq_reduce_b(const T* fin, int r, int j0, const unsigned char* skip, T* out) {
  for (int j = j0 + threadIdx.x; j < r; j += kHqThreads)
    if (!(skip && skip[j])) out[j] = __ldcg(fin + j);
  __syncthreads();
}

// argmax over the columns not done of val[] (ties: lowest column), warp 0 only; identical in every CTA
__device__ __forceinline__ int hq_argmax(const double* val, const unsigned char* done, int r, int skip) {
  const int lane = threadIdx.x & 31;
  double best = -1.0;
  int bj = r;
  for (int j = lane; j < r; j += 32) {
    if (done[j] || j == skip) continue;
    if (val[j] > best) {
      best = val[j];
      bj = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (ob > best || (ob == best && oj < bj)) {
      best = ob;
      bj = oj;
    }
  }
  return bj;
}

__global__ void __launch_bounds__(kHqThreads, 1) k_house_qr(HouseQrArgs a) {
  extern __shared__ double2 red2[];  // [kHqWarps][r] warp partials
  double* red1 = reinterpret_cast<double*>(red2);
  __shared__ double nrm[kHouseMaxCols];  // exact norms^2 of the remaining columns over rows >= k
  __shared__ double nd[kHouseMaxCols];   // the same, downdated by row k (next pivot choice)
  __shared__ double2 sv[kHouseMaxCols];  // s_j = x^H X(k:, j), x = X(k:, p_k)
  __shared__ double2 wv[kHouseMaxCols];  // w_j = v^H X(k:, j) (factorization) / y_c (Q accumulation)
  __shared__ double2 vh[kHouseMaxCols];  // v_k(k) = alpha - beta
  __shared__ double tau[kHouseMaxCols];
  __shared__ int perm[kHouseMaxCols];
  __shared__ unsigned char done[kHouseMaxCols];
  __shared__ int s_p, s_stop;
  __shared__ double s_tr;
  cg::grid_group grid = cg::this_grid();
  const int N = a.N, r = a.r, K = min(N, r);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int per = (N + G - 1) / G;
  const int lo = blockIdx.x * per, hi = min(N, lo + per);
  double2* X = a.X;
  const size_t ldx = a.ldx;
  for (int j = tid; j < r; j += kHqThreads) done[j] = 0;

  // exact column norms and ||X||_F^2 (= ||R||_F^2)
  {
    double an[kHqT];
#pragma unroll
    for (int t = 0; t < kHqT; ++t) an[t] = 0.0;
    for (int i = lo + warp; i < hi; i += kHqWarps) {
      const double2* row = X + (size_t)i * ldx;
#pragma unroll
      for (int t = 0; t < kHqT; ++t) {
        const int j = lane + 32 * t;
        if (j < r) an[t] += cabs2(row[j]);
      }
    }
    hq_cta_part<double>(an, red1, r, 0, a.npart);
    grid.sync();
    hq_reduce_a<double>(a.npart, a.nfin, r, 0, nullptr);
    grid.sync();
    hq_reduce_b<double>(a.nfin, r, 0, nullptr, nrm);
  }
  if (warp == 0) {
    double sum = 0.0;
    for (int j = lane; j < r; j += 32) sum += nrm[j];
    sum = warp_sum(sum);
    const int p0 = a.pivot ? hq_argmax(nrm, done, r, -1) : 0;
    if (lane == 0) {
      s_tr = sum;
      s_p = p0;
    }
  }
  __syncthreads();
  const double fro2 = s_tr;
  // s_j for the first pivot column
  {
    const int p = s_p;
    double2 as[kHqT];
#pragma unroll
    for (int t = 0; t < kHqT; ++t) as[t] = make_double2(0.0, 0.0);
    for (int i = lo + warp; i < hi; i += kHqWarps) {
      const double2* row = X + (size_t)i * ldx;
      const double2 xp = row[p];
#pragma unroll
      for (int t = 0; t < kHqT; ++t) {
        const int j = lane + 32 * t;
        if (j < r) as[t] = cfma(cconj(xp), row[j], as[t]);
      }
    }
    hq_cta_part<double2>(as, red2, r, 0, a.wpart);
    grid.sync();
    hq_reduce_a<double2>(a.wpart, a.wfin, r, 0, nullptr);
    grid.sync();
    hq_reduce_b<double2>(a.wfin, r, 0, nullptr, sv);
  }

  // Factorization: ONE pass over the trailing rows and one grid barrier per step. Step k applies H_k and,
  // in the same pass, accumulates the exact norms and s_j of step k + 1, whose pivot p_{k+1} is chosen
  // beforehand from the norms downdated by row k of R (exact norms are restored every step).
  int rank = K;
  for (int k = 0; k < K; ++k) {
    const int p = s_p;
    if (warp == 0) {
      double tr = 0.0;
      for (int j = lane; j < r; j += 32)
        if (!done[j]) tr += nrm[j];
      tr = warp_sum(tr);
      if (lane == 0) s_stop = a.pivot && !(tr > a.tol * a.tol * fro2);
    }
    __syncthreads();
    if (s_stop) {
      rank = k;
      break;
    }
    // the reflector of column p over rows k..N-1: H x = beta e_1 (oracle_householder_qr's convention)
    const double xn = sqrt(nrm[p]);
    const double2 alpha = __ldcg(X + (size_t)k * ldx + p);
    double tk = 0.0;
    double2 v0 = make_double2(0.0, 0.0);
    if (xn > 0.0) {
      const double aa = hypot(alpha.x, alpha.y);
      const double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
      v0 = make_double2(alpha.x + ph.x * xn, alpha.y + ph.y * xn);  // alpha - beta, beta = -ph xn
      tk = 1.0 / (xn * (xn + aa));                                  // 2 / v^H v
    }
    // w_j = v^H X(k:, j) = s_j + conj(v0 - alpha) X(k, j); R(k, j) = X(k, j) - tau v0 w_j; downdated norms
    const double2 dv = make_double2(v0.x - alpha.x, v0.y - alpha.y);
    for (int j = tid; j < r; j += kHqThreads) {
      if (done[j] || j == p) continue;
      const double2 xk = __ldcg(X + (size_t)k * ldx + j);
      const double2 w = cfma(cconj(dv), xk, sv[j]);
      wv[j] = w;
      const double2 tvw = make_double2(tk * (v0.x * w.x - v0.y * w.y), tk * (v0.x * w.y + v0.y * w.x));
      nd[j] = nrm[j] - cabs2(csub(xk, tvw));
    }
    __syncthreads();
    if (tid == 0) {
      done[p] = 1;
      perm[k] = p;
      vh[k] = v0;
      tau[k] = tk;
    }
    if (warp == 0) {
      int pn = -1;
      if (k + 1 < K) pn = a.pivot ? hq_argmax(nd, done, r, p) : k + 1;
      if (lane == 0) s_p = pn;
    }
    __syncthreads();
    const int pn = s_p;
    const double2 wpn = pn >= 0 ? wv[pn] : make_double2(0.0, 0.0);
    uint32_t act = 0;
#pragma unroll
    for (int t = 0; t < kHqT; ++t) {
      const int j = lane + 32 * t;
      if (j < r && !done[j]) act |= 1u << t;
    }
    double an[kHqT];
    double2 as[kHqT];
#pragma unroll
    for (int t = 0; t < kHqT; ++t) {
      an[t] = 0.0;
      as[t] = make_double2(0.0, 0.0);
    }
    // rows > k only: row k of R is never read again, and leaving X(k, :) untouched lets every CTA read it
    // (alpha, w_j above) while its owner has already moved on to this pass
    for (int i = lo + warp; i < hi; i += kHqWarps) {
      if (i <= k) continue;
      double2* row = X + (size_t)i * ldx;
      const double2 vi = row[p];
      const double2 tv = make_double2(tk * vi.x, tk * vi.y);
      double2 xpn = make_double2(0.0, 0.0);
      if (pn >= 0) {
        xpn = row[pn];
        xpn.x -= tv.x * wpn.x - tv.y * wpn.y;
        xpn.y -= tv.x * wpn.y + tv.y * wpn.x;
      }
      double2 x[kHqT];
#pragma unroll
      for (int t = 0; t < kHqT; ++t)
        if (act >> t & 1) x[t] = row[lane + 32 * t];
      __syncwarp();  // every lane has read row[pn] before its owner overwrites it
#pragma unroll
      for (int t = 0; t < kHqT; ++t) {
        if (act >> t & 1) {
          const double2 w = wv[lane + 32 * t];
          x[t].x -= tv.x * w.x - tv.y * w.y;
          x[t].y -= tv.x * w.y + tv.y * w.x;
          row[lane + 32 * t] = x[t];
          an[t] += cabs2(x[t]);
          as[t] = cfma(cconj(xpn), x[t], as[t]);
        }
      }
    }
    hq_cta_part<double>(an, red1, r, 0, a.npart);
    hq_cta_part<double2>(as, red2, r, 0, a.wpart);
    grid.sync();
    hq_reduce_a<double>(a.npart, a.nfin, r, 0, done);
    hq_reduce_a<double2>(a.wpart, a.wfin, r, 0, done);
    grid.sync();
    hq_reduce_b<double>(a.nfin, r, 0, done, nrm);
    hq_reduce_b<double2>(a.wfin, r, 0, done, sv);
  }
  if (blockIdx.x == 0) {
    for (int j = tid; j < rank; j += kHqThreads) a.perm[j] = perm[j];
    if (tid == 0) *a.rank = rank;
  }

  // Q(:, :rank) = H_0 ... H_{rank-1} [I; 0], accumulated backward: H_j acts on rows >= j and columns >= j
  // (columns < j are still e_c there). One pass per step applies H_j and accumulates y for H_{j-1}.
  double2* Q = a.Q;
  const size_t ldq = a.ldq;
  for (int i = lo + warp; i < hi; i += kHqWarps)
    for (int c = lane; c < rank; c += 32) Q[(size_t)i * ldq + c] = make_double2(i == c ? 1.0 : 0.0, 0.0);
  if (rank > 0) {  // y for H_{rank-1} on [I; 0]: y_c = conj(v(c)), c >= rank - 1
    const int j = rank - 1;
    if (tid == 0) wv[j] = cconj(vh[j]);
    for (int c = j + 1 + tid; c < rank; c += kHqThreads) wv[c] = cconj(__ldcg(X + (size_t)c * ldx + perm[j]));
  }
  __syncthreads();
  for (int j = rank - 1; j >= 0; --j) {
    const int p = perm[j];
    const double2 v0 = vh[j];
    const double tj = tau[j];
    const int pm = j > 0 ? perm[j - 1] : 0;
    double2 ay[kHqT];
#pragma unroll
    for (int t = 0; t < kHqT; ++t) ay[t] = make_double2(0.0, 0.0);
    for (int i = lo + warp; i < hi; i += kHqWarps) {
      if (i < j) continue;
      double2* qrow = Q + (size_t)i * ldq;
      const double2 vi = (i == j) ? v0 : X[(size_t)i * ldx + p];
      const double2 tv = make_double2(tj * vi.x, tj * vi.y);
      const double2 vm = j > 0 ? X[(size_t)i * ldx + pm] : make_double2(0.0, 0.0);  // v_{j-1}(i), i >= j
#pragma unroll
      for (int t = 0; t < kHqT; ++t) {
        const int c = lane + 32 * t;
        if (c >= j && c < rank) {
          const double2 y = wv[c];
          double2 q = qrow[c];
          q.x -= tv.x * y.x - tv.y * y.y;
          q.y -= tv.x * y.y + tv.y * y.x;
          qrow[c] = q;
          ay[t] = cfma(cconj(vm), q, ay[t]);
        }
      }
    }
    if (j == 0) break;
    hq_cta_part<double2>(ay, red2, r, j, a.wpart);
    grid.sync();
    hq_reduce_a<double2>(a.wpart, a.wfin, rank, j, nullptr);
    grid.sync();
    hq_reduce_b<double2>(a.wfin, rank, j, nullptr, wv);
    // row j-1 of Q is still e_{j-1}: it adds conj(v_{j-1}(j-1)) to y_{j-1} (rows >= j hold 0 in column j-1)
    if (tid == 0) wv[j - 1] = cconj(vh[j - 1]);
    __syncthreads();
  }
}

size_t house_qr_workspace_bytes(int r) {
  return align_up((size_t)r * kHouseMaxGrid * sizeof(double2), 256) +
         align_up((size_t)r * kHouseMaxGrid * sizeof(double), 256) + align_up((size_t)r * sizeof(double2), 256) +
         (size_t)r * sizeof(double);
}

int house_qr_launch(int N, int r, double2* X, int ldx, int pivot, double tol, double2* Q, int ldq, int* perm,
                    int* rank_dev, void* ws, int sm_count, cudaStream_t st) {
  if (N < 1 || r < 1 || r > kHouseMaxCols) return PRONY_ERR_INVALID;
  HouseQrArgs a{};
  a.N = N;
  a.r = r;
  a.X = X;
  a.ldx = ldx;
  a.pivot = pivot;
  a.tol = tol;
  a.Q = Q;
  a.ldq = ldq;
  a.perm = perm;
  a.rank = rank_dev;
  char* w = (char*)ws;
  a.wpart = (double2*)w;
  w += align_up((size_t)r * kHouseMaxGrid * sizeof(double2), 256);
  a.npart = (double*)w;
  w += align_up((size_t)r * kHouseMaxGrid * sizeof(double), 256);
  a.wfin = (double2*)w;
  w += align_up((size_t)r * sizeof(double2), 256);
  a.nfin = (double*)w;
  const size_t smem = (size_t)kHqWarps * r * sizeof(double2);
  if (ensure_smem_attr(k_house_qr, smem) != cudaSuccess)
    return PRONY_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_house_qr, kHqThreads, smem) != cudaSuccess || per_sm < 1)
    return PRONY_ERR_CUDA;
  // at least ~32 rows per CTA; never more CTAs than can be co-resident (cooperative launch)
  const int G = std::max(1, std::min({sm_count * per_sm, kHouseMaxGrid, (N + 31) / 32}));
  void* args[] = {&a};
  if (cudaLaunchCooperativeKernel((const void*)k_house_qr, dim3(G), dim3(kHqThreads), args, smem, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  return PRONY_OK;
}

// ---------------------------------------------------------------------------- one-sided Jacobi SVD
// One CTA. A (rows x cols, ld cols, rows >= cols; overwritten by U) is rotated into A V = U Sigma; V
// (cols x cols) accumulates the rotations. Round-robin column pairs (one warp per pair), sweeps until every pair
// satisfies |a_p^H a_q| <= eps * ||a_p|| ||a_q||. Then sigma_j = ||a_j||, U = a_j / sigma_j, sorted
// descending (perm applied to U and V columns). Used for Q_k = U_Q Sigma V_Q^H (Alg. 3).
__global__ void __launch_bounds__(1024) k_jacobi_svd(int rows, int cols, double2* __restrict__ A,
                                                     double2* __restrict__ Vm, double* __restrict__ sigma,
                                                     double2* __restrict__ Uout, double2* __restrict__ Vout,
                                                     int* __restrict__ order, int max_sweeps) {
  // The sweeps run on column-major copies (At = A^T in Uout, Vt in Vm: column p contiguous), so a warp's
  // lanes read consecutive entries of a column (coalesced) instead of one row-strided element each; the
  // arithmetic and its order are unchanged. A (row-major) is the input and scratch for the final U.
  __shared__ int s_rot;
  __shared__ int pairs[2][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int cp = cols + (cols & 1);  // even number of players (a virtual zero column if odd)
  double2* At = Uout;
  double2* Vt = Vm;
  for (int e = tid; e < rows * cols; e += blockDim.x) {
    const int i = e / cols, j = e % cols;
    At[(size_t)j * rows + i] = A[e];
  }
  for (int e = tid; e < cols * cols; e += blockDim.x) Vt[e] = make_double2((e / cols) == (e % cols) ? 1.0 : 0.0, 0.0);
  __syncthreads();
  const double eps = 1e-15;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < cp - 1; ++round) {
      // tournament pairing: player 0 fixed, others rotate
      for (int k = tid; k < cp / 2; k += blockDim.x) {
        int a = (k == 0) ? 0 : 1 + (k - 1 + round) % (cp - 1);
        int b = 1 + (cp - 2 - k + round) % (cp - 1);
        pairs[0][k] = min(a, b);
        pairs[1][k] = max(a, b);
      }
      __syncthreads();
      for (int k = warp; k < cp / 2; k += nw) {
        const int p = pairs[0][k], q = pairs[1][k];
        if (q >= cols) continue;  // virtual column
        double2* ap = At + (size_t)p * rows;
        double2* aq = At + (size_t)q * rows;
        double al = 0.0, be = 0.0;
        double2 ga = make_double2(0.0, 0.0);
        for (int i = lane; i < rows; i += 32) {
          const double2 x = ap[i], y = aq[i];
          al += cabs2(x);
          be += cabs2(y);
          ga = cadd(ga, cmulc(x, y));  // conj(a_p) a_q
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum2(ga);
        const double ag = sqrt(cabs2(ga));
        if (ag <= eps * sqrt(al * be) || ag == 0.0) continue;
        if (lane == 0) s_rot = 1;
        // rotation: [a_p a_q] <- [a_p a_q] J, J = [[c, -s e], [s conj(e), c]]... zeroing conj(a_p') a_q'
        const double zeta = (be - al) / (2.0 * ag);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        const double2 ph = make_double2(ga.x / ag, ga.y / ag);  // e^{i phi}, ga = |ga| e^{i phi}
        const double2 phc = cconj(ph);
        // a_p' = c a_p - s conj(ph) a_q ; a_q' = s ph a_p + c a_q
        for (int i = lane; i < rows; i += 32) {
          const double2 x = ap[i], y = aq[i];
          ap[i] = csub(cscale(x, c), cscale(cmul(phc, y), s));
          aq[i] = cadd(cscale(cmul(ph, x), s), cscale(y, c));
        }
        double2* vp = Vt + (size_t)p * cols;
        double2* vq = Vt + (size_t)q * cols;
        for (int i = lane; i < cols; i += 32) {
          const double2 x = vp[i], y = vq[i];
          vp[i] = csub(cscale(x, c), cscale(cmul(phc, y), s));
          vq[i] = cadd(cscale(cmul(ph, x), s), cscale(y, c));
        }
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
  // singular values and sort (descending, stable), U = A V columns normalized
  for (int j = warp; j < cols; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < rows; i += 32) s2 += cabs2(At[(size_t)j * rows + i]);
    s2 = warp_sum(s2);
    if (lane == 0) sigma[j] = sqrt(s2);
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < cols; ++j) order[j] = j;
    for (int a = 1; a < cols; ++a) {  // insertion sort on indices
      const int key = order[a];
      int b = a - 1;
      while (b >= 0 && sigma[order[b]] < sigma[key]) {
        order[b + 1] = order[b];
        --b;
      }
      order[b + 1] = key;
    }
  }
  __syncthreads();
  // U (row-major) into A, then back into Uout (which held At)
  for (int e = tid; e < rows * cols; e += blockDim.x) {
    const int i = e / cols, j = e % cols;
    const int src = order[j];
    const double sv = sigma[src];
    const double2 a = At[(size_t)src * rows + i];
    A[e] = sv > 0.0 ? cscale(a, 1.0 / sv) : make_double2(0.0, 0.0);
  }
  for (int e = tid; e < cols * cols; e += blockDim.x) {
    const int i = e / cols, j = e % cols;
    Vout[(size_t)i * cols + j] = Vt[(size_t)order[j] * cols + i];
  }
  __syncthreads();
  for (int e = tid; e < rows * cols; e += blockDim.x) Uout[e] = A[e];
}

// sigma_sorted[j] = sigma[order[j]]
__global__ void k_permute_sigma(int cols, const double* __restrict__ sigma, const int* __restrict__ order,
                                double* __restrict__ out) {
  for (int j = threadIdx.x; j < cols; j += blockDim.x) out[j] = sigma[order[j]];
}

// ---------------------------------------------------------------------------- eig, parallel form
// The eigendecomposition of C_mu in four steps that keep every sequential chain short:
//   k_hess       one CTA: Householder reduction C = Q H Q^H to upper Hessenberg form, the left update one
//                thread per column, the right update one thread per row (H and the unit reflectors v_k kept
//                in global memory, L1-resident);
//   k_hqr_vals   one warp: complex single-shift QR with Wilkinson shifts on a copy of H, eigenvalues only
//                (updates restricted to the active block, no Schur vectors);
//   k_inv_iter   one warp per eigenvalue: inverse iteration (H - lambda_j I) y = b on the Hessenberg matrix
//                (LU with partial pivoting between consecutive rows: O(m^2)), two solves from b = 1, then
//                w_j = Q y = H_0 H_1 ... H_{m-3} y, normalized (R23);
// and the simultaneous diagonalization: k_lu (one CTA, LU with partial pivoting of W), then
// k_diag_z with one warp per (l, j): x = W^-1 (S_l w_j) by the LU solves, z_j(l) = x_j, t (R4).
__global__ void __launch_bounds__(256) k_hess(int m, double2* __restrict__ H, double2* __restrict__ Vh) {
  __shared__ double red[256];
  __shared__ double2 sv0;
  __shared__ double sxn, svn;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < m * m; e += nt) Vh[e] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int k = 0; k + 2 < m; ++k) {
    double part = 0.0;
    for (int i = k + 1 + tid; i < m; i += nt) part += cabs2(H[(size_t)i * m + k]);
    red[tid] = part;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (tid < o) red[tid] += red[tid + o];
      __syncthreads();
    }
    if (tid == 0) {
      const double xn2 = red[0], xn = sqrt(xn2);
      const double2 alpha = H[(size_t)(k + 1) * m + k];
      const double aa = sqrt(cabs2(alpha));
      const double2 ph = aa > 0.0 ? make_double2(alpha.x / aa, alpha.y / aa) : make_double2(1.0, 0.0);
      sxn = xn;
      sv0 = make_double2(alpha.x + ph.x * xn, alpha.y + ph.y * xn);  // v = x - beta e1, beta = -ph ||x||
      svn = sqrt(xn2 - cabs2(alpha) + cabs2(sv0));
    }
    __syncthreads();
    const double xn = sxn, vn = svn;
    if (xn == 0.0 || vn == 0.0) continue;  // column already reduced (uniform)
    const double inv = 1.0 / vn;
    for (int i = k + 1 + tid; i < m; i += nt) {
      const double2 x = i == k + 1 ? sv0 : H[(size_t)i * m + k];
      Vh[(size_t)i * m + k] = cscale(x, inv);
    }
    __syncthreads();
    // left: H[k+1:, j] -= 2 v (v^H H[k+1:, j]), j > k (one thread per column)
    for (int j = k + 1 + tid; j < m; j += nt) {
      double2 sacc = make_double2(0.0, 0.0);
      for (int i = k + 1; i < m; ++i) sacc = cadd(sacc, cmulc(Vh[(size_t)i * m + k], H[(size_t)i * m + j]));
      sacc = cscale(sacc, 2.0);
      for (int i = k + 1; i < m; ++i) H[(size_t)i * m + j] = csub(H[(size_t)i * m + j], cmul(Vh[(size_t)i * m + k], sacc));
    }
    __syncthreads();
    // right: H[i, k+1:] -= 2 (H[i, k+1:] v) v^H, every row (one thread per row)
    for (int i = tid; i < m; i += nt) {
      double2 sacc = make_double2(0.0, 0.0);
      for (int j = k + 1; j < m; ++j) sacc = cadd(sacc, cmul(H[(size_t)i * m + j], Vh[(size_t)j * m + k]));
      sacc = cscale(sacc, 2.0);
      for (int j = k + 1; j < m; ++j)
        H[(size_t)i * m + j] = csub(H[(size_t)i * m + j], cmul(sacc, cconj(Vh[(size_t)j * m + k])));
    }
    __syncthreads();
    // column k: beta = -ph ||x|| on the subdiagonal (ph = the phase of alpha = the phase of v0), zeros below
    for (int i = k + 1 + tid; i < m; i += nt) {
      double2 val = make_double2(0.0, 0.0);
      if (i == k + 1) {
        const double av0 = sqrt(cabs2(sv0));
        const double2 ph = av0 > 0.0 ? make_double2(sv0.x / av0, sv0.y / av0) : make_double2(1.0, 0.0);
        val = make_double2(-ph.x * xn, -ph.y * xn);
      }
      H[(size_t)i * m + k] = val;
    }
    __syncthreads();
  }
}

// eigenvalues of the upper Hessenberg H (m x m, overwritten) by single-shift QR; one warp. For m <= 119 the
// matrix is staged in shared memory (<= 226.6 KB); the deflation test runs lane-parallel over the subdiagonal
// (ballot), without square roots (|h_{l,l-1}|^2 <= eps^2 (|h_{l-1,l-1}|^2 + |h_{l,l}|^2)); the rotations use
// reciprocal square roots only; updates are restricted to the active block (eigenvalues only).
constexpr int kHqrSmemMaxM = 119;  // 119^2 x 16 B = 226.6 KB <= 227 KB
__global__ void __launch_bounds__(32) k_hqr_vals(int m, double2* __restrict__ Hg, double2* __restrict__ lam,
                                                 int* __restrict__ status, int max_iter_per_eig) {
  extern __shared__ __align__(16) double2 Hs[];
  const int lane = threadIdx.x;
  const bool in_smem = m <= kHqrSmemMaxM;
  double2* H = in_smem ? Hs : Hg;
  if (in_smem) {
    for (int e = lane; e < m * m; e += 32) Hs[e] = Hg[e];
    __syncwarp();
  }
  auto h = [&](int i, int j) -> double2& { return H[(size_t)i * m + j]; };
  double anorm2 = 0.0;
  for (int e = lane; e < m * m; e += 32) anorm2 += cabs2(H[e]);
  anorm2 = warp_sum(anorm2);
  const double ulp = 2.220446049250313e-16, ulp2 = ulp * ulp;
  int hi = m - 1, iter = 0, total = 0;
  while (hi > 0) {
    // lo = the largest l in [1, hi] with a negligible subdiagonal h(l, l-1), else 0 (lane-parallel scan down
    // from hi in chunks of 32)
    int lo = 0;
    for (int top = hi; top >= 1; top -= 32) {
      const int l = top - lane;
      bool neg = false;
      if (l >= 1) {
        const double sd = cabs2(h(l - 1, l - 1)) + cabs2(h(l, l));
        neg = cabs2(h(l, l - 1)) <= ulp2 * (sd > 0.0 ? sd : anorm2);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, neg);
      if (bal) {
        lo = top - (__ffs(bal) - 1);  // the lowest lane = the largest l
        break;
      }
    }
    __syncwarp();
    if (lo > 0 && lane == 0) h(lo, lo - 1) = make_double2(0.0, 0.0);
    __syncwarp();
    if (lo == hi) {
      --hi;
      iter = 0;
      continue;
    }
    if (++iter > max_iter_per_eig || ++total > 30 * m * max_iter_per_eig) {
      if (lane == 0) set_status(status, PRONY_ERR_NOT_CONVERGED);
      break;
    }
    const double2 a = h(hi - 1, hi - 1), b = h(hi - 1, hi), c = h(hi, hi - 1), dd = h(hi, hi);
    double2 mu;
    if (iter % 10 == 0) {
      mu = cadd(dd, make_double2(0.75 * sqrt(cabs2(c)), 0.0));
    } else {
      const double2 tr2 = cscale(cadd(a, dd), 0.5);
      const double2 diff = cscale(csub(a, dd), 0.5);
      const double2 disc = cadd(cmul(diff, diff), cmul(b, c));
      const double r = sqrt(sqrt(cabs2(disc)));
      const double th = 0.5 * atan2(disc.y, disc.x);
      const double2 sq = make_double2(r * cos(th), r * sin(th));
      const double2 m1 = cadd(tr2, sq), m2 = csub(tr2, sq);
      mu = (cabs2(csub(m1, dd)) < cabs2(csub(m2, dd))) ? m1 : m2;
    }
    for (int k = lo; k < hi; ++k) {
      double2 x, y;
      if (k == lo) {
        x = csub(h(lo, lo), mu);
        y = h(lo + 1, lo);
      } else {
        x = h(k, k - 1);
        y = h(k + 1, k - 1);
      }
      const double x2 = cabs2(x), y2 = cabs2(y);
      if (x2 + y2 == 0.0) continue;
      double cc;
      double2 sg;
      if (x2 == 0.0) {
        cc = 0.0;
        sg = cscale(cconj(y), rsqrt(y2));
      } else {
        const double rx = rsqrt(x2), rn = rsqrt(x2 + y2);
        cc = x2 * rx * rn;                        // |x| / ||(x, y)||
        sg = cscale(cmul(x, cconj(y)), rx * rn);  // (x/|x|) conj(y) / ||(x, y)||
      }
      __syncwarp();
      for (int j = max(lo, k - 1) + lane; j <= hi; j += 32) {
        const double2 u = h(k, j), v = h(k + 1, j);
        h(k, j) = cadd(cscale(u, cc), cmul(sg, v));
        h(k + 1, j) = csub(cscale(v, cc), cmul(cconj(sg), u));
      }
      __syncwarp();
      const int rmax = min(k + 2, hi);
      for (int i = lo + lane; i <= rmax; i += 32) {
        const double2 u = h(i, k), v = h(i, k + 1);
        h(i, k) = cadd(cscale(u, cc), cmul(cconj(sg), v));
        h(i, k + 1) = csub(cscale(v, cc), cmul(sg, u));
      }
      __syncwarp();
      if (k > lo && lane == 0) h(k + 1, k - 1) = make_double2(0.0, 0.0);
      __syncwarp();
    }
  }
  __syncwarp();
  for (int i = lane; i < m; i += 32) lam[i] = h(i, i);
}

// one warp per eigenvalue j: y = (Hh - lam_j I)^-1 b twice (b = 1, then the normalized y), Hessenberg LU with
// row pivoting between consecutive rows; U rows and the elimination record in the per-warp scratch; then
// w_j = Q y (reflectors v_{m-3} .. v_0 of k_hess applied in reverse), unit 2-norm, into column j of W
constexpr int kInvRowsPerLane = (PRONY_MAX_M + 31) / 32;
__global__ void __launch_bounds__(256) k_inv_iter(int m, const double2* __restrict__ Hh, const double2* __restrict__ lam,
                                                  const double2* __restrict__ Vh, double2* __restrict__ W,
                                                  double2* __restrict__ scratch, double anorm_hint) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= m) return;
  double2* U = scratch + (size_t)j * (m * m + 2 * m);  // U rows (m x m), multipliers (m), swap flags (m, as re)
  double2* fm = U + (size_t)m * m;
  double2* sw = fm + m;
  const double2 lj = lam[j];
  double anorm = 0.0;
  for (int e = lane; e < m * m; e += 32) anorm += cabs2(Hh[e]);
  anorm = sqrt(warp_sum(anorm));
  if (!(anorm > 0.0)) anorm = anorm_hint > 0.0 ? anorm_hint : 1.0;
  const double small = 2.220446049250313e-16 * anorm;
  // factorization: cur = row 0 of (Hh - lj I)
  double2 cur[kInvRowsPerLane];
#pragma unroll
  for (int q = 0; q < kInvRowsPerLane; ++q) {
    const int c = lane + 32 * q;
    double2 v = c < m ? Hh[c] : make_double2(0.0, 0.0);
    if (c == 0) v = csub(v, lj);
    cur[q] = v;
  }
  for (int k = 0; k < m - 1; ++k) {
    double2 nxt[kInvRowsPerLane];
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int c = lane + 32 * q;
      double2 v = (c < m && c >= k) ? Hh[(size_t)(k + 1) * m + c] : make_double2(0.0, 0.0);
      if (c == k + 1) v = csub(v, lj);
      nxt[q] = v;
    }
    // the column-k entries of both rows (lane k % 32, q = k / 32)
    const int qk = k >> 5, lk = k & 31;
    double2 ck = make_double2(0.0, 0.0), nk = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q)
      if (q == qk) {
        ck = cur[q];
        nk = nxt[q];
      }
    ck = make_double2(__shfl_sync(0xffffffffu, ck.x, lk), __shfl_sync(0xffffffffu, ck.y, lk));
    nk = make_double2(__shfl_sync(0xffffffffu, nk.x, lk), __shfl_sync(0xffffffffu, nk.y, lk));
    const bool swap = cabs2(nk) > cabs2(ck);
    if (swap) {
#pragma unroll
      for (int q = 0; q < kInvRowsPerLane; ++q) {
        const double2 tmp = cur[q];
        cur[q] = nxt[q];
        nxt[q] = tmp;
      }
      const double2 tmp = ck;
      ck = nk;
      nk = tmp;
    }
    if (sqrt(cabs2(ck)) < small) ck = make_double2(small, 0.0);
    const double2 f = cdiv(nk, ck);
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int c = lane + 32 * q;
      if (c < m) {
        if (c == k) U[(size_t)k * m + c] = ck;
        else U[(size_t)k * m + c] = cur[q];
        if (c > k) nxt[q] = csub(nxt[q], cmul(f, cur[q]));
      }
      cur[q] = nxt[q];
    }
    if (lane == 0) {
      fm[k] = f;
      sw[k] = make_double2(swap ? 1.0 : 0.0, 0.0);
    }
  }
  {
    const int qk = (m - 1) >> 5, lk = (m - 1) & 31;
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int c = lane + 32 * q;
      if (c < m) {
        double2 v = cur[q];
        if (c == m - 1 && sqrt(cabs2(v)) < small) v = make_double2(small, 0.0);
        U[(size_t)(m - 1) * m + c] = v;
      }
    }
    (void)qk;
    (void)lk;
  }
  __syncwarp();
  // two solves: rhs b (in registers, element i on lane i % 32, slot i / 32)
  double2 y[kInvRowsPerLane];
#pragma unroll
  for (int q = 0; q < kInvRowsPerLane; ++q) y[q] = make_double2(lane + 32 * q < m ? 1.0 : 0.0, 0.0);
  for (int it = 0; it < 2; ++it) {
    // apply the elimination record: for k: (swap rows k, k+1 of the rhs), rhs[k+1] -= f_k rhs[k]
    for (int k = 0; k < m - 1; ++k) {
      const int q0 = k >> 5, l0 = k & 31, q1 = (k + 1) >> 5, l1 = (k + 1) & 31;
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kInvRowsPerLane; ++q) {
        if (q == q0) a0 = y[q];
        if (q == q1) a1 = y[q];
      }
      a0 = make_double2(__shfl_sync(0xffffffffu, a0.x, l0), __shfl_sync(0xffffffffu, a0.y, l0));
      a1 = make_double2(__shfl_sync(0xffffffffu, a1.x, l1), __shfl_sync(0xffffffffu, a1.y, l1));
      if (sw[k].x != 0.0) {
        const double2 tmp = a0;
        a0 = a1;
        a1 = tmp;
      }
      a1 = csub(a1, cmul(fm[k], a0));
#pragma unroll
      for (int q = 0; q < kInvRowsPerLane; ++q) {
        if (q == q0 && lane == l0) y[q] = a0;
        if (q == q1 && lane == l1) y[q] = a1;
      }
    }
    // back substitution with U (upper triangular)
    for (int i = m - 1; i >= 0; --i) {
      double2 sacc = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kInvRowsPerLane; ++q) {
        const int c = lane + 32 * q;
        if (c > i && c < m) sacc = cadd(sacc, cmul(U[(size_t)i * m + c], y[q]));
      }
      sacc = warp_sum2(sacc);
      const int qi = i >> 5, li = i & 31;
#pragma unroll
      for (int q = 0; q < kInvRowsPerLane; ++q)
        if (q == qi && lane == li) y[q] = cdiv(csub(y[q], sacc), U[(size_t)i * m + i]);
    }
    // normalize (unit max-modulus keeps the second solve's scale sane)
    double nn = 0.0;
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) nn += cabs2(y[q]);
    nn = sqrt(warp_sum(nn));
    const double inv = nn > 0.0 ? 1.0 / nn : 0.0;
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) y[q] = cscale(y[q], inv);
  }
  // w = Q y = H_0 H_1 ... H_{m-3} y, H_k = I - 2 v_k v_k^H
  for (int k = m - 3; k >= 0; --k) {
    double2 sacc = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int c = lane + 32 * q;
      if (c > k && c < m) sacc = cadd(sacc, cmulc(Vh[(size_t)c * m + k], y[q]));
    }
    sacc = cscale(warp_sum2(sacc), 2.0);
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int c = lane + 32 * q;
      if (c > k && c < m) y[q] = csub(y[q], cmul(Vh[(size_t)c * m + k], sacc));
    }
  }
  double nn = 0.0;
#pragma unroll
  for (int q = 0; q < kInvRowsPerLane; ++q) nn += cabs2(y[q]);
  nn = sqrt(warp_sum(nn));
  const double inv = nn > 0.0 ? 1.0 / nn : 0.0;
#pragma unroll
  for (int q = 0; q < kInvRowsPerLane; ++q) {
    const int c = lane + 32 * q;
    if (c < m) W[(size_t)c * m + j] = cscale(y[q], inv);
  }
}

// LU with partial pivoting of W (one CTA): LU (m x m) and the row permutation pv; status SINGULAR on a zero pivot
__global__ void __launch_bounds__(256) k_lu(int m, const double2* __restrict__ W, double2* __restrict__ LU,
                                           int* __restrict__ pv, int* __restrict__ status) {
  __shared__ double sval[256];
  __shared__ int sidx[256];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < m * m; e += nt) LU[e] = W[e];
  for (int i = tid; i < m; i += nt) pv[i] = i;
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    double best = -1.0;
    int bi = j;
    for (int i = j + tid; i < m; i += nt) {
      const double v = cabs2(LU[(size_t)i * m + j]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    sval[tid] = best;
    sidx[tid] = bi;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (tid < o && sval[tid + o] > sval[tid]) {
        sval[tid] = sval[tid + o];
        sidx[tid] = sidx[tid + o];
      }
      __syncthreads();
    }
    const int p = sidx[0];
    if (!(sval[0] > 0.0)) {
      if (tid == 0) set_status(status, PRONY_ERR_SINGULAR);
      return;
    }
    __syncthreads();
    if (p != j) {
      for (int c = tid; c < m; c += nt) {
        const double2 x = LU[(size_t)j * m + c];
        LU[(size_t)j * m + c] = LU[(size_t)p * m + c];
        LU[(size_t)p * m + c] = x;
      }
      if (tid == 0) {
        const int x = pv[j];
        pv[j] = pv[p];
        pv[p] = x;
      }
    }
    __syncthreads();
    const double2 piv = LU[(size_t)j * m + j];
    for (int i = j + 1 + tid; i < m; i += nt) LU[(size_t)i * m + j] = cdiv(LU[(size_t)i * m + j], piv);
    __syncthreads();
    const int w = m - j - 1;
    for (int e = tid; e < w * w; e += nt) {
      const int i = j + 1 + e / w, k = j + 1 + e % w;
      LU[(size_t)i * m + k] = csub(LU[(size_t)i * m + k], cmul(LU[(size_t)i * m + j], LU[(size_t)j * m + k]));
    }
    __syncthreads();
  }
}

// one warp per (l, jj): x = P S_l w_jj, L u = x, U v = u down to row jj, z[jj][l] = v[jj], t (R4)
__global__ void __launch_bounds__(256) k_diag_z(int d, int m, const double2* __restrict__ LU,
                                               const int* __restrict__ pv, const double2* __restrict__ W,
                                               const double2* __restrict__ S, double2* __restrict__ z,
                                               double* __restrict__ t, const int* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= d * m) return;
  if (status && *status == PRONY_ERR_SINGULAR) return;
  const int l = wid / m, jj = wid % m;
  double2 x[kInvRowsPerLane];
#pragma unroll
  for (int q = 0; q < kInvRowsPerLane; ++q) {
    const int i = lane + 32 * q;
    double2 sacc = make_double2(0.0, 0.0);
    if (i < m) {
      const int src = pv[i];
      for (int k = 0; k < m; ++k)
        sacc = cadd(sacc, cmul(S[((size_t)l * m + src) * m + k], W[(size_t)k * m + jj]));
    }
    x[q] = sacc;
  }
  // forward: unit lower L
  for (int i = 1; i < m; ++i) {
    double2 sacc = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int k = lane + 32 * q;
      if (k < i) sacc = cadd(sacc, cmul(LU[(size_t)i * m + k], x[q]));
    }
    sacc = warp_sum2(sacc);
    const int qi = i >> 5, li = i & 31;
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q)
      if (q == qi && lane == li) x[q] = csub(x[q], sacc);
  }
  // backward: U, rows m-1 .. jj
  for (int i = m - 1; i >= jj; --i) {
    double2 sacc = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q) {
      const int k = lane + 32 * q;
      if (k > i && k < m) sacc = cadd(sacc, cmul(LU[(size_t)i * m + k], x[q]));
    }
    sacc = warp_sum2(sacc);
    const int qi = i >> 5, li = i & 31;
#pragma unroll
    for (int q = 0; q < kInvRowsPerLane; ++q)
      if (q == qi && lane == li) x[q] = cdiv(csub(x[q], sacc), LU[(size_t)i * m + i]);
  }
  const int qj = jj >> 5, lj = jj & 31;
  double2 zz = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < kInvRowsPerLane; ++q)
    if (q == qj) zz = x[q];
  zz = make_double2(__shfl_sync(0xffffffffu, zz.x, lj), __shfl_sync(0xffffffffu, zz.y, lj));
  if (lane == 0) {
    z[(size_t)jj * d + l] = zz;
    if (t) {
      double v = -atan2(zz.y, zz.x) * 0.15915494309189533577;
      v = v - floor(v);
      if (v >= 1.0) v = 0.0;
      t[(size_t)jj * d + l] = v;
    }
  }
}

// C = sum_l mu_l S_l
__global__ void k_combine(int d, int m, const double2* __restrict__ mu, const double2* __restrict__ S,
                          double2* __restrict__ C) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int l = 0; l < d; ++l) s = cadd(s, cmul(mu[l], S[(size_t)l * m * m + e]));
    C[e] = s;
  }
}

}  // namespace prony
