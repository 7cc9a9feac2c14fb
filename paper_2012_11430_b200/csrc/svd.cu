// svd.cu — NEXT-1 drivers (outside the measured hot path; north_star: "the rank-m SVD of T and the
// m x m eigendecomposition of C_mu run on the device ... and reuse the implicit-Toeplitz apply"):
//
//   block_power_svd     reduced SVD T = U Sigma V* by the block power method of Alg. 3
//                       (P:179-201), with T V and T^H U from toeplitz_apply (the k_project gather),
//                       Cholesky-QR (Gram on all SMs, factor in one CTA) for the QR steps and
//                       diagonal-pivoted Cholesky of the Gram for the pivoted-QR rank determination
//                       (R22), one-sided Jacobi SVD of Q_k.
//   diagonalize_launch  C_mu = sum mu_l S_l, W from eig(C_mu), z_j(l) = (W^-1 S_l W)_jj
//                       (P:34-37, 57), t = (-arg z / 2 pi) mod 1 (R4).
//
// The block power loop needs the detected rank and the residual on the host (it decides the
// next launch shapes), so block_power_svd synchronizes the stream once per iteration.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "dense.cuh"
#include "project.cuh"

namespace prony {

namespace {

constexpr int kGramKS = 32;  // K splits of the Gram products

struct SvdLayout {
  size_t V0, A1, A2, A3, A4, Gp, G, Rinv, Q, Jv, Ju, Jvv, piv, ints, dparts, dscal, sig, apply, total;
};

SvdLayout svd_layout(int d, int n, int N, int m) {
  const int r0 = std::min(2 * m, N);
  SvdLayout s{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  const size_t nr = (size_t)N * r0 * sizeof(double2);
  s.V0 = take(nr);
  s.A1 = take(nr);
  s.A2 = take(nr);
  s.A3 = take(nr);
  s.A4 = take(nr);
  s.Gp = take((size_t)kGramKS * r0 * r0 * sizeof(double2));
  s.G = take((size_t)r0 * r0 * sizeof(double2));
  s.Rinv = take((size_t)r0 * r0 * sizeof(double2));
  s.Q = take((size_t)r0 * r0 * sizeof(double2));
  s.Jv = take((size_t)r0 * r0 * sizeof(double2));
  s.Ju = take((size_t)r0 * r0 * sizeof(double2));
  s.Jvv = take((size_t)r0 * r0 * sizeof(double2));
  s.piv = take((size_t)(r0 + 8) * sizeof(int));
  s.ints = take(64 * sizeof(int));
  s.dparts = take(4096 * sizeof(double));
  s.dscal = take(64 * sizeof(double));
  s.sig = take((size_t)(r0 + 8) * sizeof(double));
  s.apply = take(apply_workspace_bytes(d, n, N));
  s.total = off;
  return s;
}

struct Ctx {
  int N, sms;
  cudaStream_t st;
  SvdLayout L;
  char* w;
  double2* P(size_t off) const { return (double2*)(w + off); }
};

int grid1(int64_t work, int sms) { return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8 * sms)); }

// G (ri x rj) = X^H Y over the N rows (fixed-order K split)
void gram(const Ctx& c, const double2* X, int ldx, int ri, const double2* Y, int ldy, int rj, double2* G) {
  dim3 g((ri + 31) / 32, (rj + 31) / 32, kGramKS);
  k_gram<<<g, 256, 0, c.st>>>(c.N, ri, rj, X, ldx, Y, ldy, kGramKS, c.P(c.L.Gp));
  k_sum_parts<<<grid1((int64_t)ri * rj, c.sms), 256, 0, c.st>>>((int64_t)ri * rj, kGramKS, c.P(c.L.Gp), G);
}

// ||X||_F^2 (N x cols) -> device scalar
void fro2(const Ctx& c, const double2* X, int ldx, int cols, double* out) {
  const int nb = std::min(4096, 2 * c.sms);
  k_fro2_parts<<<nb, 256, 0, c.st>>>(c.N, cols, X, ldx, (double*)(c.w + c.L.dparts));
  k_sum_doubles<<<1, 32, 0, c.st>>>(nb, (double*)(c.w + c.L.dparts), out);
}

// Orthonormal basis of the range of X (N x r): diagonal-pivoted Cholesky of X^H X (rank by the
// trailing-trace criterion when pivot = 1), Xout = X(:, piv(1:rank)) R11^-1. Returns rank (host).
int chol_basis(const Ctx& c, const double2* X, int ldx, int r, int pivot, double tol, double2* Xout, int ldout,
               int* rank_host) {
  double2* G = c.P(c.L.G);
  gram(c, X, ldx, r, X, ldx, r, G);
  int* piv = (int*)(c.w + c.L.piv);
  int* rk = (int*)(c.w + c.L.ints);
  k_chol_piv<<<1, 512, 0, c.st>>>(r, G, pivot, tol, piv, rk);
  int rank = 0;
  if (cudaMemcpyAsync(&rank, rk, sizeof(int), cudaMemcpyDeviceToHost, c.st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(c.st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (rank < 1) return PRONY_ERR_RANK;
  double2* Rinv = c.P(c.L.Rinv);
  k_trinv_from_lower<<<(rank + 127) / 128, 128, 0, c.st>>>(r, rank, G, Rinv, rank);
  // Xp = X(:, piv(1:rank)) into Xout, then Xout = Xp Rinv needs a separate buffer: use A4
  double2* Xp = c.P(c.L.A4);
  k_gather_cols<<<grid1((int64_t)c.N * rank, c.sms), 256, 0, c.st>>>(c.N, rank, piv, X, ldx, Xp, rank);
  dim3 g((c.N + 63) / 64, (rank + 31) / 32);
  k_gemm_nm<<<g, 256, 0, c.st>>>(c.N, rank, rank, Xp, rank, Rinv, rank, Xout, ldout, 1.0, 0.0);
  *rank_host = rank;
  return cudaGetLastError() == cudaSuccess ? PRONY_OK : PRONY_ERR_CUDA;
}

// CholeskyQR2 of a full-rank X (N x r) into Xout (the second pass restores orthogonality)
int cholqr2(const Ctx& c, const double2* X, int ldx, int r, double2* Xout, int ldout, double2* tmp) {
  int rank = 0;
  int rc = chol_basis(c, X, ldx, r, 0, 0.0, tmp, r, &rank);
  if (rc) return rc;
  if (rank != r) return PRONY_ERR_RANK;
  rc = chol_basis(c, tmp, r, r, 0, 0.0, Xout, ldout, &rank);
  if (rc) return rc;
  return rank == r ? PRONY_OK : PRONY_ERR_RANK;
}

}  // namespace

size_t svd_workspace_bytes(int d, int n, int N, int m) { return svd_layout(d, n, N, m).total; }

int block_power_svd(int d, int n, int N, const double2* grid, int m, double tol, int max_iter, uint64_t seed,
                    double2* U, double2* V, double* sigma, int* rank_out, int* iters_out, double* resid_out, void* ws,
                    int sm_count, cudaStream_t st) {
  Ctx c{};
  c.N = N;
  c.sms = sm_count;
  c.st = st;
  c.L = svd_layout(d, n, N, m);
  c.w = (char*)ws;
  const int r0 = std::min(2 * m, N);  // starting column dimension 2m
  void* aws = c.w + c.L.apply;
  double2 *Vk = c.P(c.L.V0), *A1 = c.P(c.L.A1), *A2 = c.P(c.L.A2), *A3 = c.P(c.L.A3);
  double* dscal = (double*)(c.w + c.L.dscal);
  // the Gram-based trailing norm resolves ||R(i:,i:)|| / ||R|| only down to ~sqrt(eps_M) (R22)
  const double rank_tol = std::max(tol, 1e-7);
  const double res_tol = std::max(tol, 1e-12);

  // ||T||_F^2 from the grid
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  const int nb = std::min(4096, 2 * sm_count);
  k_normT2_parts<<<nb, 256, 0, st>>>(d, n, box, grid, (double*)(c.w + c.L.dparts));
  k_sum_doubles<<<1, 32, 0, st>>>(nb, (double*)(c.w + c.L.dparts), dscal);
  // V0: seeded complex Gaussian, orthonormalized (R14)
  k_fill_random<<<grid1((int64_t)N * r0, sm_count), 256, 0, st>>>((int64_t)N * r0, seed, A1, N, r0, r0);
  int rv = 0, ru = 0, rc;
  rc = chol_basis(c, A1, r0, r0, 1, rank_tol, Vk, r0, &rv);  // (also guards a rank-deficient random block)
  if (rc) return rc;
  double normT2 = 0.0;
  if (cudaMemcpyAsync(&normT2, dscal, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
  const double normT = sqrt(normT2);

  // Ubar_1 = T V0
  rc = toeplitz_apply_launch(d, n, N, grid, 0, 0, Vk, r0, rv, A1, r0, aws, sm_count, st);
  if (rc) return rc;
  double resid = -1.0;
  int it = 0;
  for (it = 1; it <= max_iter; ++it) {
    // U_k = basis of T V_{k-1} (A1 -> A2)
    if (it == 1) rc = chol_basis(c, A1, r0, rv, 1, rank_tol, A2, r0, &ru);
    else {
      rc = cholqr2(c, A1, r0, rv, A2, r0, A3);
      ru = rv;
    }
    if (rc) return rc;
    // Vbar_k = T^H U_k (A2 -> A3)
    rc = toeplitz_apply_launch(d, n, N, grid, 0, 1, A2, r0, ru, A3, r0, aws, sm_count, st);
    if (rc) return rc;
    // V_k = pivoted (first iteration, rank determination P:203) or plain QR basis (A3 -> Vk)
    if (it == 1) rc = chol_basis(c, A3, r0, ru, 1, rank_tol, Vk, r0, &rv);
    else {
      rc = cholqr2(c, A3, r0, ru, Vk, r0, A1);
      rv = ru;
    }
    if (rc) return rc;
    // T V_k (Vk -> A1): next Ubar and the residual
    rc = toeplitz_apply_launch(d, n, N, grid, 0, 0, Vk, r0, rv, A1, r0, aws, sm_count, st);
    if (rc) return rc;
    // Q_k = U_k^H T V_k (ru x rv);  R_k = T V_k - U_k Q_k
    double2* Q = c.P(c.L.Q);
    gram(c, A2, r0, ru, A1, r0, rv, Q);
    // A4 = T V_k - U_k Q_k  (copy of T V_k, then beta = 1, alpha = -1)
    if (cudaMemcpy2DAsync(c.P(c.L.A4), (size_t)r0 * sizeof(double2), A1, (size_t)r0 * sizeof(double2),
                          (size_t)rv * sizeof(double2), N, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return PRONY_ERR_CUDA;
    k_gemm_nm<<<dim3((N + 63) / 64, (rv + 31) / 32), 256, 0, st>>>(N, ru, rv, A2, r0, Q, rv, c.P(c.L.A4), r0, -1.0,
                                                                 1.0);
    fro2(c, c.P(c.L.A4), r0, rv, dscal + 1);
    double res2 = 0.0;
    if (cudaMemcpyAsync(&res2, dscal + 1, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return PRONY_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
    resid = sqrt(res2) / (normT > 0 ? normT : 1.0);
    if (resid <= res_tol) break;
  }
  if (iters_out) *iters_out = std::min(it, max_iter);
  if (resid_out) *resid_out = resid;
  // SVD of Q (ru x rv, ru >= rv): Q = Uq Sigma Vq^H (one-sided Jacobi), U = U_k Uq, V = V_k Vq
  if (ru < rv) return PRONY_ERR_RANK;
  double2* Q = c.P(c.L.Q);
  double2 *Jv = c.P(c.L.Jv), *Ju = c.P(c.L.Ju), *Jvv = c.P(c.L.Jvv);
  double* sig = (double*)(c.w + c.L.sig);
  int* order = (int*)(c.w + c.L.piv);
  // Jacobi works on a copy of Q (A4 scratch is free)
  double2* Qa = c.P(c.L.A4);
  if (cudaMemcpyAsync(Qa, Q, (size_t)ru * rv * sizeof(double2), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  k_jacobi_svd<<<1, 1024, 0, st>>>(ru, rv, Qa, Jv, sig, Ju, Jvv, order, 60);
  const int k = std::min(m, rv);
  k_permute_sigma<<<1, 256, 0, st>>>(k, sig, order, sigma);
  // U = U_k (N x ru) * Uq (ru x rv)[:, :k];  V = V_k (N x rv) * Vq (rv x rv)[:, :k]
  k_gemm_nm<<<dim3((N + 63) / 64, (k + 31) / 32), 256, 0, st>>>(N, ru, k, A2, r0, Ju, rv, U, m, 1.0, 0.0);
  k_gemm_nm<<<dim3((N + 63) / 64, (k + 31) / 32), 256, 0, st>>>(N, rv, k, Vk, r0, Jvv, rv, V, m, 1.0, 0.0);
  *rank_out = rv;
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (rv < m) return PRONY_ERR_RANK;
  return (resid <= res_tol) ? PRONY_OK : PRONY_ERR_NOT_CONVERGED;
}

// ---------------------------------------------------------------------------- diagonalization
namespace {
struct DiagLayout {
  size_t C, Z, lam, LU, pv, col, total;
};
DiagLayout diag_layout(int d, int m) {
  (void)d;
  DiagLayout s{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  s.C = take((size_t)m * m * sizeof(double2));
  s.Z = take((size_t)m * m * sizeof(double2));
  s.lam = take((size_t)m * sizeof(double2));
  s.LU = take((size_t)m * m * sizeof(double2));
  s.pv = take((size_t)m * sizeof(int));
  s.col = take((size_t)m * sizeof(double2));
  s.total = off;
  return s;
}
}  // namespace

size_t diag_workspace_bytes(int d, int m) { return diag_layout(d, m).total; }

int diagonalize_launch(int d, int m, const double2* S, const double2* mu, double2* z, double* t, double2* W,
                       void* ws, int32_t* status, cudaStream_t st) {
  const DiagLayout L = diag_layout(d, m);
  char* w = (char*)ws;
  double2* C = (double2*)(w + L.C);
  k_combine<<<(m * m + 255) / 256, 256, 0, st>>>(d, m, mu, S, C);
  k_eig<<<1, 32, 0, st>>>(m, C, (double2*)(w + L.Z), (double2*)(w + L.lam), W, status, 60);
  k_diag_pencil<<<1, 256, 0, st>>>(d, m, W, S, (double2*)(w + L.LU), (int*)(w + L.pv), (double2*)(w + L.col), z, t,
                                   status);
  return cudaGetLastError() == cudaSuccess ? PRONY_OK : PRONY_ERR_CUDA;
}

}  // namespace prony
