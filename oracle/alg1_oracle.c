/*
 * alg1_oracle.c — plain CPU reference of the steps of Algorithm 1 that surround the
 * hot path: the reduced SVD of T (line 2), the eigendecomposition of C_mu (line 4), the simultaneous
 * diagonalization (line 5), t from z (line 6) and the least-squares solve (line 7).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so. The product path (paper_2012_11430_b200/) never
 * links, loads or calls it, and shares no code with it.
 *
 * Everything here is a textbook algorithm written out in plain C99 complex FP64 loops — no BLAS,
 * no LAPACK, no blocking. OpenMP only splits independent output rows of the Toeplitz apply (every
 * output element is still summed by one thread in the plain order).
 *
 * Functions and the passages they follow:
 *   oracle_householder_qr   reduced QR, optionally with column pivoting (largest remaining column
 *                           norm first), by Householder reflectors. P:191-193 (Alg. 3 lines 7, 9),
 *                           P:203 ("QR factorization implemented with Householder reflectors")
 *   oracle_jacobi_svd       one-sided (Hestenes) Jacobi SVD of a dense complex matrix: the dense
 *                           reduced SVD of eq_T_svd P:22-26 at desk scale and the SVD of Q_k,
 *                           Alg. 3 line 14; SPEC S:201 admits one-sided Jacobi
 *   oracle_toeplitz_apply   Y = T_l X or T_l^H X with T_l[k,h] = f(k-h+e_l) generated entry by
 *                           entry; l = 0 is T
 *   oracle_T_fro            ||T||_F by summing |f(k-h)|^2 over all (k,h) (Alg. 3 line 4)
 *   oracle_block_power_svd  Algorithm 3: block power method with the rank determined by
 *                           the pivoted QR of the first iteration only, R14
 *   oracle_eig              eigenvalues/vectors of a general complex m x m matrix: Householder
 *                           reduction to Hessenberg form, complex single-shift QR iteration (Wilkinson
 *                           shift) to Schur form, eigenvectors by back substitution (R23)
 *   oracle_lu_solve         A X = B by LU with partial pivoting
 *   oracle_diagonalize      C_mu = sum_l mu_l S_l, W from eig(C_mu),
 *                           z_tau(j)(l) = (W^-1 S_l W)_jj (eq_diagonalizeSl)
 *   oracle_t_from_z         t = (-arg z / 2 pi) mod 1 (reading R4)
 *   oracle_lstsq_qr         argmin_c ||A^T c - f||_2 by Householder QR of A^T
 *
 * Storage: every matrix is row-major, element (i, j) at X[i * ld + j].
 */
#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_common.h"

#define EPS_M DBL_EPSILON

static double cabs2(cplx a) { return creal(a) * creal(a) + cimag(a) * cimag(a); }

/* ------------------------------------------------------------------------------------------------
 * Householder QR.  A (M x C, lda) -> Q (M x K, ldq) with orthonormal columns, R (K x C, ldr) upper
 * trapezoidal, K = min(M, C); with pivot != 0, perm[j] = the column of A that sits in column j of
 * Q R (the column with the largest remaining norm is moved to the front at every step).
 * Reflector k: x = W[k:, k], beta = -(alpha/|alpha|) ||x||, v = x - beta e_1, H_k = I - 2 v v^H / v^H v,
 * so H_k x = beta e_1.  Q = H_0 H_1 ... H_{K-1} [I_K; 0].
 */
int oracle_householder_qr(int64_t M, int C, const cplx* A, int64_t lda, int pivot, cplx* Q, int64_t ldq, cplx* R,
                          int ldr, int* perm) {
  if (M < 1 || C < 1) return 1;
  const int K = (int)(M < C ? M : C);
  cplx* W = (cplx*)malloc((size_t)M * C * sizeof(cplx));
  cplx* Vh = (cplx*)calloc((size_t)M * K, sizeof(cplx)); /* column k: unit Householder vector u_k */
  int* pv = (int*)malloc((size_t)C * sizeof(int));
  if (!W || !Vh || !pv) { free(W); free(Vh); free(pv); return 3; }
  for (int64_t i = 0; i < M; ++i)
    for (int j = 0; j < C; ++j) W[i * C + j] = A[i * lda + j];
  for (int j = 0; j < C; ++j) pv[j] = j;

  for (int k = 0; k < K; ++k) {
    if (pivot) {
      int best = k;
      double bestn = -1.0;
      for (int j = k; j < C; ++j) {
        double s = 0.0;
        for (int64_t i = k; i < M; ++i) s += cabs2(W[i * C + j]);
        if (s > bestn) { bestn = s; best = j; }
      }
      if (best != k) {
        for (int64_t i = 0; i < M; ++i) {
          cplx tmp = W[i * C + k];
          W[i * C + k] = W[i * C + best];
          W[i * C + best] = tmp;
        }
        int tp = pv[k]; pv[k] = pv[best]; pv[best] = tp;
      }
    }
    double xn2 = 0.0;
    for (int64_t i = k; i < M; ++i) xn2 += cabs2(W[i * C + k]);
    const double xnorm = sqrt(xn2);
    if (xnorm == 0.0) continue; /* H_k = I, u_k = 0 */
    const cplx alpha = W[k * C + k];
    const double aa = cabs(alpha);
    const cplx phase = aa > 0.0 ? alpha / aa : 1.0;
    const cplx beta = -phase * xnorm;
    /* v = x - beta e_1 */
    double vn2 = 0.0;
    for (int64_t i = k; i < M; ++i) {
      cplx v = (i == k) ? alpha - beta : W[i * C + k];
      Vh[i * K + k] = v;
      vn2 += cabs2(v);
    }
    const double vn = sqrt(vn2);
    for (int64_t i = k; i < M; ++i) Vh[i * K + k] /= vn;
    /* W[k:, j] -= 2 u (u^H W[k:, j]) for the columns j > k; column k becomes beta e_1 */
    for (int j = k + 1; j < C; ++j) {
      cplx s = 0.0;
      for (int64_t i = k; i < M; ++i) s += conj(Vh[i * K + k]) * W[i * C + j];
      s *= 2.0;
      for (int64_t i = k; i < M; ++i) W[i * C + j] -= s * Vh[i * K + k];
    }
    W[k * C + k] = beta;
    for (int64_t i = k + 1; i < M; ++i) W[i * C + k] = 0.0;
  }
  if (R) {
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < C; ++j) R[(int64_t)i * ldr + j] = (j >= i) ? W[(int64_t)i * C + j] : 0.0;
  }
  if (Q) {
    for (int64_t i = 0; i < M; ++i)
      for (int j = 0; j < K; ++j) Q[i * ldq + j] = (i == j) ? 1.0 : 0.0;
    for (int k = K - 1; k >= 0; --k) {
      for (int j = k; j < K; ++j) {
        cplx s = 0.0;
        for (int64_t i = k; i < M; ++i) s += conj(Vh[i * K + k]) * Q[i * ldq + j];
        s *= 2.0;
        for (int64_t i = k; i < M; ++i) Q[i * ldq + j] -= s * Vh[i * K + k];
      }
    }
  }
  if (perm)
    for (int j = 0; j < C; ++j) perm[j] = pv[j];
  free(W);
  free(Vh);
  free(pv);
  return 0;
}

/* ------------------------------------------------------------------------------------------------
 * One-sided Jacobi SVD (Hestenes).  A (M x C, lda) = U diag(sigma) V^H with V (C x C, ldv) unitary,
 * U (M x C, ldu) = A V diag(1/sigma) (a zero column where sigma_j = 0), sigma nonincreasing.
 * Columns p < q of W = A V are rotated in cyclic order until every pair is orthogonal to
 * |w_p^H w_q| <= sqrt(M) eps_M ||w_p|| ||w_q|| (pairs with a column of norm <= sqrt(M) eps_M ||A||_F are
 * not rotated).  With gamma = w_p^H w_q = |gamma| e^{i phi}, the pair
 * (w_p, e^{-i phi} w_q) has a real inner product and the real Jacobi rotation
 *   zeta = (||w_q||^2 - ||w_p||^2) / (2 |gamma|),  t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
 *   c = 1 / sqrt(1 + t^2), s = c t,   w_p <- c w_p - s e^{-i phi} w_q,  w_q <- s w_p + c e^{-i phi} w_q
 * makes it orthogonal; V receives the same column operations.
 */
int oracle_jacobi_svd(int64_t M, int C, const cplx* A, int64_t lda, double* sigma, cplx* U, int64_t ldu, cplx* V,
                      int ldv, int max_sweeps, int* sweeps_out) {
  if (M < 1 || C < 1) return 1;
  /* column-major working copies: column j of W at Wc + j * M (storage only, same arithmetic) */
  cplx* Wc = (cplx*)malloc((size_t)M * C * sizeof(cplx));
  cplx* Vc = (cplx*)calloc((size_t)C * C, sizeof(cplx));
  int* ord = (int*)malloc((size_t)C * sizeof(int));
  double* nrm = (double*)malloc((size_t)C * sizeof(double));
  if (!Wc || !Vc || !ord || !nrm) { free(Wc); free(Vc); free(ord); free(nrm); return 3; }
  for (int j = 0; j < C; ++j) {
    for (int64_t i = 0; i < M; ++i) Wc[(int64_t)j * M + i] = A[i * lda + j];
    Vc[(int64_t)j * C + j] = 1.0;
  }
  const double tol = sqrt((double)M) * EPS_M;
  /* columns of norm <= sqrt(M) eps_M ||A||_F are rounding noise (a rank-deficient A leaves C - rank of them):
     they are not rotated, so that the sweep terminates; skipping a pair with such a column changes the
     other singular values by O(M (eps_M ||A||_F)^2 / sigma) */
  double a2 = 0.0;
  for (int64_t e = 0; e < M * C; ++e) a2 += cabs2(Wc[e]);
  const double small2 = (double)M * EPS_M * EPS_M * a2;
  int sweep = 0, converged = 0;
  for (sweep = 1; sweep <= max_sweeps; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < C - 1; ++p) {
      for (int q = p + 1; q < C; ++q) {
        cplx* wp = Wc + (int64_t)p * M;
        cplx* wq = Wc + (int64_t)q * M;
        double al = 0.0, be = 0.0;
        cplx ga = 0.0;
        for (int64_t i = 0; i < M; ++i) {
          al += cabs2(wp[i]);
          be += cabs2(wq[i]);
          ga += conj(wp[i]) * wq[i];
        }
        const double g = cabs(ga);
        if (al <= small2 || be <= small2 || g <= tol * sqrt(al) * sqrt(be)) continue;
        rotated = 1;
        const cplx eph = conj(ga / g); /* e^{-i phi} */
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int64_t i = 0; i < M; ++i) {
          const cplx xp = wp[i], xq = eph * wq[i];
          wp[i] = c * xp - s * xq;
          wq[i] = s * xp + c * xq;
        }
        cplx* vp = Vc + (int64_t)p * C;
        cplx* vq = Vc + (int64_t)q * C;
        for (int i = 0; i < C; ++i) {
          const cplx xp = vp[i], xq = eph * vq[i];
          vp[i] = c * xp - s * xq;
          vq[i] = s * xp + c * xq;
        }
      }
    }
    if (!rotated) { converged = 1; break; }
  }
  if (sweeps_out) *sweeps_out = converged ? sweep : -max_sweeps;
  for (int j = 0; j < C; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < M; ++i) s += cabs2(Wc[(int64_t)j * M + i]);
    nrm[j] = sqrt(s);
    ord[j] = j;
  }
  /* sort by nonincreasing norm (insertion sort, stable) */
  for (int a = 1; a < C; ++a) {
    int o = ord[a];
    int b = a - 1;
    while (b >= 0 && nrm[ord[b]] < nrm[o]) { ord[b + 1] = ord[b]; --b; }
    ord[b + 1] = o;
  }
  for (int j = 0; j < C; ++j) {
    const int o = ord[j];
    sigma[j] = nrm[o];
    if (U)
      for (int64_t i = 0; i < M; ++i) U[i * ldu + j] = nrm[o] > 0.0 ? Wc[(int64_t)o * M + i] / nrm[o] : 0.0;
    if (V)
      for (int i = 0; i < C; ++i) V[(int64_t)i * ldv + j] = Vc[(int64_t)o * C + i];
  }
  free(Wc);
  free(Vc);
  free(ord);
  free(nrm);
  return converged ? 0 : 5;
}

/* ------------------------------------------------------------------------------------------------
 * Toeplitz apply with the entries generated from the samples:
 *   adjoint = 0:  Y[k][j] = sum_h T_l[k][h] X[h][j]
 *   adjoint = 1:  Y[h][j] = sum_k conj(T_l[k][h]) X[k][j]
 * T_l[k][h] = f(k - h + e_l) (l = 1..d), T[k][h] = f(k - h) (l = 0). X, Y: N x r row-major.
 */
int oracle_toeplitz_apply(int d, int n, const cplx* grid, int ell, int adjoint, int r, const cplx* X, cplx* Y) {
  if (d < 1 || d > ORACLE_MAX_D || n < 1 || ell < 0 || ell > d || r < 1) return 1;
  const int64_t N = count_N(d, n);
  int* mi = (int*)malloc((size_t)N * d * sizeof(int)); /* multi-indices of I_n (index cache only) */
  if (!mi) return 3;
  for (int64_t q = 0; q < N; ++q) index_of(d, n, q, mi + q * d);
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t a = 0; a < N; ++a) {
    cplx* y = Y + a * r;
    for (int j = 0; j < r; ++j) y[j] = 0.0;
    int v[ORACLE_MAX_D];
    for (int64_t b = 0; b < N; ++b) {
      /* (k, h) = (a, b) for T_l X; (k, h) = (b, a) for T_l^H X */
      const int* k = adjoint ? mi + b * d : mi + a * d;
      const int* h = adjoint ? mi + a * d : mi + b * d;
      for (int i = 0; i < d; ++i) v[i] = k[i] - h[i];
      if (ell >= 1) v[ell - 1] += 1;
      const cplx t = grid[box_index(d, n, v)];
      const cplx te = adjoint ? conj(t) : t;
      const cplx* x = X + b * r;
      for (int j = 0; j < r; ++j) y[j] += te * x[j];
    }
  }
  free(mi);
  return 0;
}

/* ||T||_F = sqrt(sum_{k,h} |f(k-h)|^2) (Alg. 3 line 4 needs ||A||_F) */
double oracle_T_fro(int d, int n, const cplx* grid) {
  const int64_t N = count_N(d, n);
  double s = 0.0;
  int k[ORACLE_MAX_D], h[ORACLE_MAX_D], v[ORACLE_MAX_D];
  for (int64_t a = 0; a < N; ++a) {
    index_of(d, n, a, k);
    for (int64_t b = 0; b < N; ++b) {
      index_of(d, n, b, h);
      for (int i = 0; i < d; ++i) v[i] = k[i] - h[i];
      s += cabs2(grid[box_index(d, n, v)]);
    }
  }
  return sqrt(s);
}

/* Y (rows x c) = X^H Z for X (rows x a), Z (rows x c) */
static void mat_hmul(int64_t rows, int a, int c, const cplx* X, int64_t ldx, const cplx* Z, int64_t ldz, cplx* Y,
                     int ldy) {
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < c; ++j) {
      cplx s = 0.0;
      for (int64_t k = 0; k < rows; ++k) s += conj(X[k * ldx + i]) * Z[k * ldz + j];
      Y[(int64_t)i * ldy + j] = s;
    }
}

/* Y (rows x c) = X Z for X (rows x a), Z (a x c) */
static void mat_mul(int64_t rows, int a, int c, const cplx* X, int64_t ldx, const cplx* Z, int64_t ldz, cplx* Y,
                    int64_t ldy) {
  for (int64_t i = 0; i < rows; ++i)
    for (int j = 0; j < c; ++j) {
      cplx s = 0.0;
      for (int k = 0; k < a; ++k) s += X[i * ldx + k] * Z[(int64_t)k * ldz + j];
      Y[i * ldy + j] = s;
    }
}

/* ------------------------------------------------------------------------------------------------
 * Algorithm 3, A = T (N x N), in the paper's line order:
 *   1-2  Q_0 = U_0^* A V_0,  R_0 = A V_0 - U_0 Q_0
 *   4    while ||R_k||_F > tol ||A||_F   (and k < max_iter):
 *   6-7    Ubar_k = A V_{k-1} = U_k R_{U_k}                        (Householder QR)
 *   8      Vbar_k = A^* U_k
 *   9-11   k = 1: Vbar_1 P = V_1 R_{V_1} (pivoted QR); r_1 = first i with
 *                 ||R_{V_1}(i:, i:)||_F <= tol ||R_{V_1}||_F, minus one; V_1 = V_1(:, 1:r_1)
 *          k > 1: Vbar_k = V_k R_{V_k} (plain QR, "only once in the first step")
 *   12     R_k = A V_k - U_k Q_k with Q_k = U_k^* A V_k recomputed (reading R14)
 *   14-15  Q_k = U_Q Sigma V_Q^* (one-sided Jacobi); U = U_k U_Q, V = V_k V_Q
 * Inputs U0, V0 (N x r0, orthonormal columns; the seeded draws of reading R14 are passed in).
 * Outputs U, V (N x r0 buffers, ld r0; the first *rank columns are valid), sigma (r0, first *rank).
 * Returns 0, 4 if the detected rank is 0, 5 if not converged within max_iter (outputs still written).
 */
int oracle_block_power_svd(int d, int n, const cplx* grid, int r0, const cplx* U0, const cplx* V0, double tol,
                           int max_iter, cplx* U, cplx* V, double* sigma, int* rank_out, int* iters_out,
                           double* resid_out) {
  const int64_t N = count_N(d, n);
  if (r0 < 1 || r0 > N) return 1;
  const size_t nr = (size_t)N * r0;
  cplx* Vk = (cplx*)malloc(nr * sizeof(cplx));
  cplx* Uk = (cplx*)malloc(nr * sizeof(cplx));
  cplx* AV = (cplx*)malloc(nr * sizeof(cplx));
  cplx* Vb = (cplx*)malloc(nr * sizeof(cplx));
  cplx* Qm = (cplx*)malloc((size_t)r0 * r0 * sizeof(cplx));
  cplx* Rm = (cplx*)malloc((size_t)r0 * r0 * sizeof(cplx));
  cplx* Uq = (cplx*)malloc((size_t)r0 * r0 * sizeof(cplx));
  cplx* Vq = (cplx*)malloc((size_t)r0 * r0 * sizeof(cplx));
  int* perm = (int*)malloc((size_t)r0 * sizeof(int));
  int rc = 0;
  if (!Vk || !Uk || !AV || !Vb || !Qm || !Rm || !Uq || !Vq || !perm) { rc = 3; goto done; }

  const double normA = oracle_T_fro(d, n, grid);
  int ru = r0, rv = r0;
  memcpy(Vk, V0, nr * sizeof(cplx));
  memcpy(Uk, U0, nr * sizeof(cplx));
  /* lines 1-2 */
  oracle_toeplitz_apply(d, n, grid, 0, 0, rv, Vk, AV);
  mat_hmul(N, ru, rv, Uk, r0, AV, r0, Qm, r0);
  double res2 = 0.0;
  for (int64_t i = 0; i < N; ++i)
    for (int j = 0; j < rv; ++j) {
      cplx s = AV[i * r0 + j];
      for (int q = 0; q < ru; ++q) s -= Uk[i * r0 + q] * Qm[(int64_t)q * r0 + j];
      res2 += cabs2(s);
    }
  double resid = sqrt(res2) / normA;
  int k = 0;
  while (resid > tol && k < max_iter) {
    ++k;
    /* lines 6-7: U_k = Q factor of Ubar_k = A V_{k-1} (N x rv) */
    cplx* Qf = (cplx*)malloc((size_t)N * rv * sizeof(cplx));
    if (!Qf) { rc = 3; goto done; }
    oracle_householder_qr(N, rv, AV, r0, 0, Qf, rv, NULL, 0, NULL);
    ru = rv;
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < ru; ++j) Uk[i * r0 + j] = Qf[i * rv + j];
    free(Qf);
    /* line 8: Vbar_k = A^* U_k (N x ru) */
    cplx* Ucmp = (cplx*)malloc((size_t)N * ru * sizeof(cplx));
    cplx* Vbc = (cplx*)malloc((size_t)N * ru * sizeof(cplx));
    cplx* Vf = (cplx*)malloc((size_t)N * ru * sizeof(cplx));
    if (!Ucmp || !Vbc || !Vf) { free(Ucmp); free(Vbc); free(Vf); rc = 3; goto done; }
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < ru; ++j) Ucmp[i * ru + j] = Uk[i * r0 + j];
    oracle_toeplitz_apply(d, n, grid, 0, 1, ru, Ucmp, Vbc);
    /* lines 9-11 */
    if (k == 1) {
      oracle_householder_qr(N, ru, Vbc, ru, 1, Vf, ru, Rm, r0, perm);
      double rn2 = 0.0;
      for (int i = 0; i < ru; ++i)
        for (int j = i; j < ru; ++j) rn2 += cabs2(Rm[(int64_t)i * r0 + j]);
      const double rnorm = sqrt(rn2);
      int r1 = ru;
      for (int i = 0; i < ru; ++i) { /* 0-based i = paper's i - 1 */
        double t2 = 0.0;
        for (int a = i; a < ru; ++a)
          for (int b = a; b < ru; ++b) t2 += cabs2(Rm[(int64_t)a * r0 + b]);
        if (sqrt(t2) <= tol * rnorm) { r1 = i; break; }
      }
      rv = r1;
    } else {
      oracle_householder_qr(N, ru, Vbc, ru, 0, Vf, ru, NULL, 0, NULL);
      rv = ru;
    }
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < rv; ++j) Vk[i * r0 + j] = Vf[i * ru + j];
    free(Ucmp);
    free(Vbc);
    free(Vf);
    if (rv < 1) { rc = 4; goto done; }
    /* line 12: R_k = A V_k - U_k Q_k, Q_k = U_k^* A V_k */
    cplx* Vcmp = (cplx*)malloc((size_t)N * rv * sizeof(cplx));
    cplx* AVc = (cplx*)malloc((size_t)N * rv * sizeof(cplx));
    if (!Vcmp || !AVc) { free(Vcmp); free(AVc); rc = 3; goto done; }
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < rv; ++j) Vcmp[i * rv + j] = Vk[i * r0 + j];
    oracle_toeplitz_apply(d, n, grid, 0, 0, rv, Vcmp, AVc);
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < rv; ++j) AV[i * r0 + j] = AVc[i * rv + j];
    free(Vcmp);
    free(AVc);
    mat_hmul(N, ru, rv, Uk, r0, AV, r0, Qm, r0);
    res2 = 0.0;
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < rv; ++j) {
        cplx s = AV[i * r0 + j];
        for (int q = 0; q < ru; ++q) s -= Uk[i * r0 + q] * Qm[(int64_t)q * r0 + j];
        res2 += cabs2(s);
      }
    resid = sqrt(res2) / normA;
  }
  /* lines 14-15: SVD of Q_k (ru x rv) */
  {
    double* sq = (double*)malloc((size_t)rv * sizeof(double));
    if (!sq) { rc = 3; goto done; }
    oracle_jacobi_svd(ru, rv, Qm, r0, sq, Uq, r0, Vq, r0, 100, NULL);
    mat_mul(N, ru, rv, Uk, r0, Uq, r0, U, r0);
    mat_mul(N, rv, rv, Vk, r0, Vq, r0, V, r0);
    for (int j = 0; j < r0; ++j) sigma[j] = j < rv ? sq[j] : 0.0;
    free(sq);
  }
  if (rank_out) *rank_out = rv;
  if (iters_out) *iters_out = k;
  if (resid_out) *resid_out = resid;
  if (resid > tol) rc = 5;
done:
  free(Vk); free(Uk); free(AV); free(Vb); free(Qm); free(Rm); free(Uq); free(Vq); free(perm);
  return rc;
}

/* ------------------------------------------------------------------------------------------------
 * Eigen decomposition of a general complex m x m matrix A (row-major): A W = W diag(lambda),
 * unit-norm columns of W.
 *   1. Householder reduction H = Z^* A Z to upper Hessenberg form.
 *   2. Complex single-shift QR iteration on H (Wilkinson shift: the eigenvalue of the trailing 2 x 2
 *      block closer to its last diagonal entry; an exceptional shift every 10 iterations without
 *      deflation), one QR step = Givens rotations G_k zeroing the subdiagonal of H - mu I, then
 *      H <- R Q + mu I; deflation when |h_{i,i-1}| <= eps_M (|h_{i-1,i-1}| + |h_{i,i}|).
 *      The rotations act on the whole matrix and are accumulated into Z: A = Z T Z^*, T upper
 *      triangular (Schur form).
 *   3. Eigenvectors of T by back substitution: x_k = 1, x_i = -(sum_{j=i+1..k} T_ij x_j)/(T_ii - T_kk)
 *      for i < k (a zero denominator is replaced by eps_M ||T||_F); w_k = Z x / ||Z x||.
 * Returns 0, or 5 if the QR iteration did not converge within 30 m iterations per eigenvalue.
 */
int oracle_eig(int m, const cplx* A, cplx* lambda, cplx* W, int* iters_out) {
  if (m < 1) return 1;
  cplx* H = (cplx*)malloc((size_t)m * m * sizeof(cplx));
  cplx* Z = (cplx*)malloc((size_t)m * m * sizeof(cplx));
  cplx* v = (cplx*)malloc((size_t)m * sizeof(cplx));
  cplx* gc = (cplx*)malloc((size_t)m * sizeof(cplx));
  cplx* gs = (cplx*)malloc((size_t)m * sizeof(cplx));
  cplx* x = (cplx*)malloc((size_t)m * sizeof(cplx));
  if (!H || !Z || !v || !gc || !gs || !x) { free(H); free(Z); free(v); free(gc); free(gs); free(x); return 3; }
  memcpy(H, A, (size_t)m * m * sizeof(cplx));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) Z[i * m + j] = (i == j) ? 1.0 : 0.0;

  /* 1. Hessenberg reduction: reflector P_k on rows/columns k+1..m-1 zeroes H[k+2:, k] */
  for (int k = 0; k < m - 2; ++k) {
    double xn2 = 0.0;
    for (int i = k + 1; i < m; ++i) xn2 += cabs2(H[i * m + k]);
    const double xnorm = sqrt(xn2);
    if (xnorm == 0.0) continue;
    const cplx alpha = H[(k + 1) * m + k];
    const double aa = cabs(alpha);
    const cplx phase = aa > 0.0 ? alpha / aa : 1.0;
    const cplx beta = -phase * xnorm;
    double vn2 = 0.0;
    for (int i = k + 1; i < m; ++i) {
      v[i] = (i == k + 1) ? alpha - beta : H[i * m + k];
      vn2 += cabs2(v[i]);
    }
    const double vn = sqrt(vn2);
    for (int i = k + 1; i < m; ++i) v[i] /= vn;
    /* H <- P H: rows k+1.. , every column */
    for (int j = 0; j < m; ++j) {
      cplx s = 0.0;
      for (int i = k + 1; i < m; ++i) s += conj(v[i]) * H[i * m + j];
      s *= 2.0;
      for (int i = k + 1; i < m; ++i) H[i * m + j] -= s * v[i];
    }
    /* H <- H P, Z <- Z P: columns k+1.., every row */
    for (int i = 0; i < m; ++i) {
      cplx s = 0.0, t = 0.0;
      for (int j = k + 1; j < m; ++j) {
        s += H[i * m + j] * v[j];
        t += Z[i * m + j] * v[j];
      }
      s *= 2.0;
      t *= 2.0;
      for (int j = k + 1; j < m; ++j) {
        H[i * m + j] -= s * conj(v[j]);
        Z[i * m + j] -= t * conj(v[j]);
      }
    }
    for (int i = k + 2; i < m; ++i) H[i * m + k] = 0.0;
  }

  /* 2. shifted QR iteration */
  int hi = m - 1, its = 0, total = 0, rc = 0;
  const int max_total = 30 * m;
  while (hi > 0) {
    int l = hi;
    while (l > 0) {
      const double sub = cabs(H[l * m + l - 1]);
      if (sub <= EPS_M * (cabs(H[(l - 1) * m + l - 1]) + cabs(H[l * m + l]))) {
        H[l * m + l - 1] = 0.0;
        break;
      }
      --l;
    }
    if (l == hi) { /* H[hi][hi] is an eigenvalue */
      --hi;
      its = 0;
      continue;
    }
    if (total >= max_total) { rc = 5; break; }
    ++its;
    ++total;
    cplx mu;
    if (its % 10 == 0) { /* exceptional shift */
      mu = H[hi * m + hi] + cabs(creal(H[hi * m + hi - 1])) + (hi >= 2 ? cabs(creal(H[(hi - 1) * m + hi - 2])) : 0.0);
    } else { /* Wilkinson: eigenvalue of [[a b][c e]] closer to e */
      const cplx a = H[(hi - 1) * m + hi - 1], b = H[(hi - 1) * m + hi];
      const cplx c = H[hi * m + hi - 1], e = H[hi * m + hi];
      const cplx hd = 0.5 * (a - e);
      const cplx disc = csqrt(hd * hd + b * c);
      const cplx l1 = 0.5 * (a + e) + disc, l2 = 0.5 * (a + e) - disc;
      mu = cabs(l1 - e) <= cabs(l2 - e) ? l1 : l2;
    }
    /* QR step on the active block l..hi of H - mu I */
    for (int i = l; i <= hi; ++i) H[i * m + i] -= mu;
    for (int k = l; k < hi; ++k) {
      const cplx a = H[k * m + k], b = H[(k + 1) * m + k];
      const double r = sqrt(cabs2(a) + cabs2(b));
      cplx c = 1.0, s = 0.0;
      if (r > 0.0) { c = a / r; s = b / r; }
      gc[k] = c;
      gs[k] = s;
      /* rows k, k+1 <- [[conj c, conj s], [-s, c]] rows k, k+1 (columns k..m-1) */
      for (int j = k; j < m; ++j) {
        const cplx p = H[k * m + j], q = H[(k + 1) * m + j];
        H[k * m + j] = conj(c) * p + conj(s) * q;
        H[(k + 1) * m + j] = -s * p + c * q;
      }
    }
    for (int k = l; k < hi; ++k) {
      const cplx c = gc[k], s = gs[k];
      /* columns k, k+1 <- columns k, k+1 times [[c, -conj s], [s, conj c]] (rows 0..min(k+2, hi)) */
      const int top = (k + 2 < hi) ? k + 2 : hi;
      for (int i = 0; i <= top; ++i) {
        const cplx p = H[i * m + k], q = H[i * m + k + 1];
        H[i * m + k] = p * c + q * s;
        H[i * m + k + 1] = -p * conj(s) + q * conj(c);
      }
      for (int i = 0; i < m; ++i) {
        const cplx p = Z[i * m + k], q = Z[i * m + k + 1];
        Z[i * m + k] = p * c + q * s;
        Z[i * m + k + 1] = -p * conj(s) + q * conj(c);
      }
    }
    for (int i = l; i <= hi; ++i) H[i * m + i] += mu;
  }
  if (iters_out) *iters_out = total;

  /* 3. eigenvectors of the Schur form by back substitution */
  double tn2 = 0.0;
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) tn2 += cabs2(H[i * m + j]);
  const double small = EPS_M * sqrt(tn2);
  for (int k = 0; k < m; ++k) {
    lambda[k] = H[k * m + k];
    for (int i = 0; i < m; ++i) x[i] = 0.0;
    x[k] = 1.0;
    for (int i = k - 1; i >= 0; --i) {
      cplx s = 0.0;
      for (int j = i + 1; j <= k; ++j) s += H[i * m + j] * x[j];
      cplx den = H[i * m + i] - H[k * m + k];
      if (cabs(den) < small) den = small;
      x[i] = -s / den;
    }
    double wn2 = 0.0;
    for (int i = 0; i < m; ++i) {
      cplx s = 0.0;
      for (int j = 0; j <= k; ++j) s += Z[i * m + j] * x[j];
      W[i * m + k] = s;
      wn2 += cabs2(s);
    }
    const double wn = sqrt(wn2);
    for (int i = 0; i < m; ++i) W[i * m + k] /= wn;
  }
  free(H); free(Z); free(v); free(gc); free(gs); free(x);
  return rc;
}

/* A X = B (A m x m, B and X m x nrhs) by LU with partial pivoting (Doolittle, row interchanges).
 * Returns 4 if A is exactly singular. */
int oracle_lu_solve(int m, const cplx* A, int nrhs, const cplx* B, cplx* X) {
  cplx* LU = (cplx*)malloc((size_t)m * m * sizeof(cplx));
  int* piv = (int*)malloc((size_t)m * sizeof(int));
  if (!LU || !piv) { free(LU); free(piv); return 3; }
  memcpy(LU, A, (size_t)m * m * sizeof(cplx));
  int rc = 0;
  for (int i = 0; i < m; ++i) piv[i] = i;
  for (int k = 0; k < m; ++k) {
    int p = k;
    double best = cabs(LU[k * m + k]);
    for (int i = k + 1; i < m; ++i)
      if (cabs(LU[i * m + k]) > best) { best = cabs(LU[i * m + k]); p = i; }
    if (best == 0.0) { rc = 4; break; }
    if (p != k) {
      for (int j = 0; j < m; ++j) {
        cplx t = LU[k * m + j]; LU[k * m + j] = LU[p * m + j]; LU[p * m + j] = t;
      }
      int t = piv[k]; piv[k] = piv[p]; piv[p] = t;
    }
    for (int i = k + 1; i < m; ++i) {
      const cplx f = LU[i * m + k] / LU[k * m + k];
      LU[i * m + k] = f;
      for (int j = k + 1; j < m; ++j) LU[i * m + j] -= f * LU[k * m + j];
    }
  }
  if (rc == 0) {
    for (int c = 0; c < nrhs; ++c) {
      /* forward: L y = P b; backward: U x = y */
      for (int i = 0; i < m; ++i) {
        cplx s = B[(int64_t)piv[i] * nrhs + c];
        for (int j = 0; j < i; ++j) s -= LU[i * m + j] * X[(int64_t)j * nrhs + c];
        X[(int64_t)i * nrhs + c] = s;
      }
      for (int i = m - 1; i >= 0; --i) {
        cplx s = X[(int64_t)i * nrhs + c];
        for (int j = i + 1; j < m; ++j) s -= LU[i * m + j] * X[(int64_t)j * nrhs + c];
        X[(int64_t)i * nrhs + c] = s / LU[i * m + i];
      }
    }
  }
  free(LU);
  free(piv);
  return rc;
}

/* Algorithm 1 lines 4-5: C_mu = sum_l mu_l S_l, W from eig(C_mu), D_l = W^-1 (S_l W) by LU
 * (P:34-37), z[j][l] = D_l[j][j].  S: d x m x m; z: m x d; W: m x m; offdiag[l] =
 * ||D_l - diag(D_l)||_F / ||D_l||_F. */
int oracle_diagonalize(int d, int m, const cplx* S, const cplx* mu, cplx* z, cplx* W, double* offdiag) {
  const size_t mm = (size_t)m * m;
  cplx* Cm = (cplx*)calloc(mm, sizeof(cplx));
  cplx* lam = (cplx*)malloc((size_t)m * sizeof(cplx));
  cplx* SW = (cplx*)malloc(mm * sizeof(cplx));
  cplx* D = (cplx*)malloc(mm * sizeof(cplx));
  if (!Cm || !lam || !SW || !D) { free(Cm); free(lam); free(SW); free(D); return 3; }
  for (int l = 0; l < d; ++l)
    for (size_t e = 0; e < mm; ++e) Cm[e] += mu[l] * S[l * mm + e];
  int rc = oracle_eig(m, Cm, lam, W, NULL);
  for (int l = 0; l < d && rc == 0; ++l) {
    const cplx* Sl = S + l * mm;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        cplx s = 0.0;
        for (int k = 0; k < m; ++k) s += Sl[i * m + k] * W[k * m + j];
        SW[i * m + j] = s;
      }
    rc = oracle_lu_solve(m, W, m, SW, D);
    double off2 = 0.0, all2 = 0.0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        all2 += cabs2(D[i * m + j]);
        if (i != j) off2 += cabs2(D[i * m + j]);
      }
    for (int j = 0; j < m; ++j) z[j * d + l] = D[j * m + j];
    if (offdiag) offdiag[l] = sqrt(off2) / sqrt(all2);
  }
  free(Cm); free(lam); free(SW); free(D);
  return rc;
}

/* t = (-arg z / 2 pi) mod 1, in [0, 1) (reading R4) */
int oracle_t_from_z(int64_t count, const cplx* z, double* t) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < count; ++i) {
    double v = fmod(-carg(z[i]) / two_pi, 1.0);
    if (v < 0.0) v += 1.0;
    if (v >= 1.0) v = 0.0;
    t[i] = v;
  }
  return 0;
}

/* argmin_c ||A^T c - f||_2, f = [f(k)]_{k in I_n} read from the box: Householder QR
 * A^T = Q R (N x m, m x m), c = R^{-1} Q^* f, and the relative residual ||A^T c - f|| / ||f||.
 * A: m x N row-major. Returns 4 if R has a zero diagonal entry (rank-deficient A^T). */
int oracle_lstsq_qr(int d, int n, int m, const cplx* A, const cplx* grid, cplx* c, double* resid) {
  const int64_t N = count_N(d, n);
  if (m < 1 || m > N) return 1;
  cplx* At = (cplx*)malloc((size_t)N * m * sizeof(cplx));
  cplx* Q = (cplx*)malloc((size_t)N * m * sizeof(cplx));
  cplx* R = (cplx*)malloc((size_t)m * m * sizeof(cplx));
  cplx* f = (cplx*)malloc((size_t)N * sizeof(cplx));
  cplx* y = (cplx*)malloc((size_t)m * sizeof(cplx));
  if (!At || !Q || !R || !f || !y) { free(At); free(Q); free(R); free(f); free(y); return 3; }
  int k[ORACLE_MAX_D];
  for (int64_t i = 0; i < N; ++i) {
    index_of(d, n, i, k);
    f[i] = grid[box_index(d, n, k)];
    for (int j = 0; j < m; ++j) At[i * m + j] = A[(int64_t)j * N + i];
  }
  int rc = oracle_householder_qr(N, m, At, m, 0, Q, m, R, m, NULL);
  if (rc == 0) {
    for (int j = 0; j < m; ++j) {
      cplx s = 0.0;
      for (int64_t i = 0; i < N; ++i) s += conj(Q[i * m + j]) * f[i];
      y[j] = s;
    }
    for (int i = m - 1; i >= 0; --i) {
      cplx s = y[i];
      for (int j = i + 1; j < m; ++j) s -= R[i * m + j] * c[j];
      if (R[i * m + i] == 0.0) { rc = 4; break; }
      c[i] = s / R[i * m + i];
    }
  }
  if (rc == 0 && resid) {
    double r2 = 0.0, f2 = 0.0;
    for (int64_t i = 0; i < N; ++i) {
      cplx s = -f[i];
      for (int j = 0; j < m; ++j) s += At[i * m + j] * c[j];
      r2 += cabs2(s);
      f2 += cabs2(f[i]);
    }
    *resid = sqrt(r2) / sqrt(f2);
  }
  free(At); free(Q); free(R); free(f); free(y);
  return rc;
}
