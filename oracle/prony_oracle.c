/*
 * prony_oracle.c — plain, slow, obviously-correct CPU reference of the hot path of
 * the multivariate matrix-pencil Prony method (arXiv 2012.11430, PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2012_11430_b200/) never links, loads or calls it, and shares no code with it.
 *
 * Arithmetic: IEEE binary64 complex (C99 double complex), naive loops in the order of
 * the definitions, no blocking, no BLAS. OpenMP only splits independent output rows
 * (the result of every output element is computed by exactly one thread in the plain
 * summation order, so the thread count does not change any value).
 *
 * Conventions (readings R1, R2):
 *   grid : f~(k) for k in the box {-n..n+1}^d, L = 2n+2 values per axis, lexicographic
 *          with the LAST coordinate fastest: box index of k = sum_i (k_i+n) L^(d-1-i).
 *   I_n  : {0..n}^d, same lexicographic order; row r <-> multi-index digits of r base n+1.
 *   U, V : N x m row-major complex (row r = element r of I_n).
 *   z    : m x d row-major complex nodes.
 *
 * Functions and the passages they follow:
 *   oracle_T_entry / oracle_build_T   T = [f(k-h)], T_l = [f(k-h+e_l)]
 *   oracle_project_rows               S_l = U* T_l V Sigma^-1            PAPER.md:27-29 (eq_generateSl)
 *   oracle_project_columns            selected columns of the same S_l
 *   oracle_vandermonde                A = [z_j^k], z_j^k = prod_l z_j(l)^(k_l)
 *   oracle_ls_products                G = A conj(A)^T, b = A conj(f)     PAPER.md:39-43, 59 (normal
 *                                     equations of argmin ||A^T c - f||_2; R10)
 *   oracle_cholesky_solve             c = conj(G^-1 b)                   PAPER.md:59; R10
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle_common.h"

int oracle_abi_version(void) { return 1; }

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* T_l[k,h] = f(k - h + e_l) for l in 1..d, T[k,h] = f(k - h) for l = 0 */
static cplx T_entry(int d, int n, const cplx* grid, const int* k, const int* h, int ell) {
  int v[16];
  for (int i = 0; i < d; ++i) v[i] = k[i] - h[i];
  if (ell >= 1) v[ell - 1] += 1;
  int64_t idx = box_index(d, n, v);
  return idx >= 0 ? grid[idx] : NAN;
}

int oracle_T_entry(int d, int n, const cplx* grid, int64_t row, int64_t col, int ell, cplx* out) {
  if (d < 1 || d > 16 || n < 1 || ell < 0 || ell > d) return 1;
  int k[16], h[16];
  index_of(d, n, row, k);
  index_of(d, n, col, h);
  *out = T_entry(d, n, grid, k, h, ell);
  return 0;
}

/* dense N x N T (ell = 0) or T_ell (ell = 1..d) — desk scale only */
int oracle_build_T(int d, int n, int ell, const cplx* grid, cplx* out) {
  if (d < 1 || d > 16 || n < 1 || ell < 0 || ell > d) return 1;
  int64_t N = 1;
  for (int i = 0; i < d; ++i) N *= (n + 1);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < N; ++r) {
    int k[16], h[16];
    index_of(d, n, r, k);
    for (int64_t c = 0; c < N; ++c) {
      index_of(d, n, c, h);
      out[r * N + c] = T_entry(d, n, grid, k, h, ell);
    }
  }
  return 0;
}

/*
 * Partial pencil over the rows k in [k_begin, k_end) of T_ell:
 *   S_part[i][j] = sum_{k in range} conj(U[k][i]) * (sum_h T_ell[k][h] V[h][j]) / sigma[j]
 * With the full range [0, N) this is S_ell = U* T_ell V Sigma^-1 (eq_generateSl);
 * Sigma^-1 is the column scale 1/sigma_j (R11).
 * Step 1: Y = T_ell V for the rows in range (naive triple loop over h, j).
 * Step 2: S = U* Y, then column scale.
 */
int oracle_project_rows(int d, int n, int m, const cplx* grid, const cplx* U, const cplx* V,
                        const double* sigma, int ell, int64_t k_begin, int64_t k_end, cplx* S_part) {
  if (d < 1 || d > 16 || n < 1 || m < 1 || ell < 1 || ell > d) return 1;
  int64_t N = 1;
  for (int i = 0; i < d; ++i) N *= (n + 1);
  if (k_begin < 0 || k_end > N || k_begin > k_end) return 2;
  int64_t R = k_end - k_begin;
  cplx* Y = (cplx*)calloc((size_t)(R > 0 ? R : 1) * m, sizeof(cplx));
  if (!Y) return 3;
  /* Step 1: Y[k][j] = sum_h T_ell[k][h] V[h][j] */
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t r = 0; r < R; ++r) {
    int k[16], h[16];
    index_of(d, n, k_begin + r, k);
    cplx* y = Y + r * m;
    for (int64_t c = 0; c < N; ++c) {
      index_of(d, n, c, h);
      cplx t = T_entry(d, n, grid, k, h, ell);
      const cplx* v = V + c * m;
      for (int j = 0; j < m; ++j) y[j] += t * v[j];
    }
  }
  /* Step 2: S[i][j] = sum_k conj(U[k][i]) Y[k][j], then / sigma_j */
#pragma omp parallel for schedule(static)
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j < m; ++j) {
      cplx s = 0;
      for (int64_t r = 0; r < R; ++r) s += conj(U[(k_begin + r) * m + i]) * Y[r * m + j];
      S_part[i * m + j] = s / sigma[j];
    }
  }
  free(Y);
  return 0;
}

/*
 * Selected columns j in cols[0..ncols) of S_ell (all rows i):
 *   out[i][q] = (u_i^* (T_ell v_j)) / sigma_j,  j = cols[q]
 * Same definition as oracle_project_rows, one column at a time (full-size sampled parity).
 */
int oracle_project_columns(int d, int n, int m, const cplx* grid, const cplx* U, const cplx* V,
                           const double* sigma, int ell, int ncols, const int* cols, cplx* out) {
  if (d < 1 || d > 16 || n < 1 || m < 1 || ell < 1 || ell > d) return 1;
  int64_t N = 1;
  for (int i = 0; i < d; ++i) N *= (n + 1);
  cplx* y = (cplx*)malloc((size_t)N * sizeof(cplx));
  if (!y) return 3;
  for (int q = 0; q < ncols; ++q) {
    int j = cols[q];
    if (j < 0 || j >= m) { free(y); return 2; }
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < N; ++r) {
      int k[16], h[16];
      index_of(d, n, r, k);
      cplx s = 0;
      for (int64_t c = 0; c < N; ++c) {
        index_of(d, n, c, h);
        s += T_entry(d, n, grid, k, h, ell) * V[c * m + j];
      }
      y[r] = s;
    }
    for (int i = 0; i < m; ++i) {
      cplx s = 0;
      for (int64_t r = 0; r < N; ++r) s += conj(U[r * m + i]) * y[r];
      out[i * ncols + q] = s / sigma[j];
    }
  }
  free(y);
  return 0;
}

/*
 * A[j][k] = z_j^k = prod_{l=1..d} z_j(l)^{k_l}  (Ã from z̃)
 * for the columns k in [col_begin, col_end) of I_n; A is m x (col_end-col_begin) row-major.
 * Powers by repeated multiplication z^a = (((1*z)*z)...*z), the product over l in order
 * l = 1..d starting from 1 ("k-fold multiplication", no pow()).
 */
int oracle_vandermonde(int d, int n, int m, const cplx* z, int64_t col_begin, int64_t col_end, cplx* A) {
  if (d < 1 || d > 16 || n < 1 || m < 1) return 1;
  int64_t N = 1;
  for (int i = 0; i < d; ++i) N *= (n + 1);
  if (col_begin < 0 || col_end > N || col_begin > col_end) return 2;
  int64_t W = col_end - col_begin;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < m; ++j) {
    int k[16];
    for (int64_t c = 0; c < W; ++c) {
      index_of(d, n, col_begin + c, k);
      cplx a = 1.0;
      for (int l = 0; l < d; ++l) {
        cplx p = 1.0;
        for (int e = 0; e < k[l]; ++e) p = p * z[j * d + l];
        a = a * p;
      }
      A[j * W + c] = a;
    }
  }
  return 0;
}

/*
 * LS products over the columns k in [col_begin, col_end) (A holds exactly those columns):
 *   G[i][j] = sum_k A[i][k] conj(A[j][k])     (G = A conj(A)^T = A A^H)
 *   b[i]    = sum_k A[i][k] conj(f(k))        (b = A conj(f)), f(k) = grid at k in I_n
 * The normal equations of argmin ||A^T c - f||_2 are G conj(c) = b (R10).
 */
int oracle_ls_products(int d, int n, int m, const cplx* A, const cplx* grid, int64_t col_begin,
                       int64_t col_end, cplx* G, cplx* b) {
  if (d < 1 || d > 16 || n < 1 || m < 1) return 1;
  int64_t N = 1;
  for (int i = 0; i < d; ++i) N *= (n + 1);
  if (col_begin < 0 || col_end > N || col_begin > col_end) return 2;
  int64_t W = col_end - col_begin;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j < m; ++j) {
      cplx s = 0;
      for (int64_t c = 0; c < W; ++c) s += A[i * W + c] * conj(A[j * W + c]);
      G[i * m + j] = s;
    }
    cplx s = 0;
    int k[16];
    for (int64_t c = 0; c < W; ++c) {
      index_of(d, n, col_begin + c, k);
      s += A[i * W + c] * conj(grid[box_index(d, n, k)]);
    }
    b[i] = s;
  }
  return 0;
}

/*
 * c = conj(G^-1 b) for Hermitian positive definite G (m x m): G = L L^H (Cholesky,
 * textbook column order), L y = b, L^H x = y, c = conj(x).  Returns 4 if G is not HPD.
 */
int oracle_cholesky_solve(int m, const cplx* G, const cplx* b, cplx* c) {
  cplx* Lm = (cplx*)calloc((size_t)m * m, sizeof(cplx));
  cplx* y = (cplx*)malloc((size_t)m * sizeof(cplx));
  if (!Lm || !y) { free(Lm); free(y); return 3; }
  for (int j = 0; j < m; ++j) {
    double djj = creal(G[j * m + j]);
    for (int p = 0; p < j; ++p) djj -= creal(Lm[j * m + p] * conj(Lm[j * m + p]));
    if (!(djj > 0.0)) { free(Lm); free(y); return 4; }
    double ljj = sqrt(djj);
    Lm[j * m + j] = ljj;
    for (int i = j + 1; i < m; ++i) {
      cplx s = G[i * m + j];
      for (int p = 0; p < j; ++p) s -= Lm[i * m + p] * conj(Lm[j * m + p]);
      Lm[i * m + j] = s / ljj;
    }
  }
  for (int i = 0; i < m; ++i) {
    cplx s = b[i];
    for (int p = 0; p < i; ++p) s -= Lm[i * m + p] * y[p];
    y[i] = s / Lm[i * m + i];
  }
  for (int i = m - 1; i >= 0; --i) {
    cplx s = y[i];
    for (int p = i + 1; p < m; ++p) s -= conj(Lm[p * m + i]) * y[p];
    y[i] = s / Lm[i * m + i];
  }
  for (int i = 0; i < m; ++i) c[i] = conj(y[i]);
  free(Lm);
  free(y);
  return 0;
}
