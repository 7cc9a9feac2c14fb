// svd.cu — NEXT-1 drivers (outside the measured hot path; north_star: "the rank-m SVD of T and the
// m x m eigendecomposition of C_mu run on the device ... and reuse the implicit-Toeplitz apply"):
//
//   block_power_svd     reduced SVD T = U Sigma V* by the block power method of Alg. 3
//                       (P:179-201), with T V and T^H U from toeplitz_apply (the k_project gather),
//                       Householder QR of the tall blocks in one cooperative launch (k_house_qr,
//                       P:203), column-pivoted in the first iteration for the rank (
//                       DESIGN.md R22), one-sided Jacobi SVD of Q_k.
//   diagonalize_launch  C_mu = sum mu_l S_l, W from eig(C_mu), z_j(l) = (W^-1 S_l W)_jj
//                       (P:34-37, 57), t = (-arg z / 2 pi) mod 1 (R4).
//
// The block power loop needs the detected rank and the residual on the host (it decides the
// next launch shapes), so block_power_svd synchronizes the stream once per iteration.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "project.cuh"

namespace prony {

namespace {

constexpr int kGramKS = 32;  // K splits of the Gram products

struct SvdLayout {
  size_t V0, A1, A2, A3, A4, Gp, Q, Jv, Ju, Jvv, piv, ints, dparts, dscal, sig, hq, apply, total;
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
  s.Q = take((size_t)r0 * r0 * sizeof(double2));
  s.Jv = take((size_t)r0 * r0 * sizeof(double2));
  s.Ju = take((size_t)r0 * r0 * sizeof(double2));
  s.Jvv = take((size_t)r0 * r0 * sizeof(double2));
  s.piv = take((size_t)(r0 + 8) * sizeof(int));
  s.ints = take(64 * sizeof(int));
  s.dparts = take(4096 * sizeof(double));
  s.dscal = take(64 * sizeof(double));
  s.sig = take((size_t)(r0 + 8) * sizeof(double));
  s.hq = take(house_qr_workspace_bytes(r0));
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

// Orthonormal basis of the range of X (N x r) into Xout: Q(:, :rank) of the Householder QR (X is
// overwritten); with pivot = 1 the rank is the first k with ||R(k:, k:)||_F <= tol ||R||_F,
// otherwise rank = r. Returns the rank on the host.
int house_basis(const Ctx& c, double2* X, int ldx, int r, int pivot, double tol, double2* Xout, int ldout,
                int* rank_host) {
  int* piv = (int*)(c.w + c.L.piv);
  int* rk = (int*)(c.w + c.L.ints);
  int rc = house_qr_launch(c.N, r, X, ldx, pivot, tol, Xout, ldout, piv, rk, c.w + c.L.hq, c.sms, c.st);
  if (rc) return rc;
  int rank = 0;
  if (cudaMemcpyAsync(&rank, rk, sizeof(int), cudaMemcpyDeviceToHost, c.st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(c.st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (rank < 1) return PRONY_ERR_RANK;
  *rank_host = rank;
  return PRONY_OK;
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
  const double res_tol = std::max(tol, 1e-12);

  // ||T||_F^2 from the grid
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  const int nb = std::min(4096, 2 * sm_count);
  k_normT2_parts<<<nb, 256, 0, st>>>(d, n, box, grid, (double*)(c.w + c.L.dparts));
  k_sum_doubles<<<1, 32, 0, st>>>(nb, (double*)(c.w + c.L.dparts), dscal);
  // V0: seeded complex Gaussian, orthonormalized by Householder QR (R14)
  k_fill_random<<<grid1((int64_t)N * r0, sm_count), 256, 0, st>>>((int64_t)N * r0, seed, A1, N, r0, r0);
  int rv = 0, ru = 0, rc;
  rc = house_basis(c, A1, r0, r0, 0, 0.0, Vk, r0, &rv);
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
    // U_k = Q factor of Ubar_k = T V_{k-1} (A1 -> A2; Alg. 3 line 7: plain QR, rank-deficient blocks allowed)
    rc = house_basis(c, A1, r0, rv, 0, 0.0, A2, r0, &ru);
    if (rc) return rc;
    // Vbar_k = T^H U_k (A2 -> A3)
    rc = toeplitz_apply_launch(d, n, N, grid, 0, 1, A2, r0, ru, A3, r0, aws, sm_count, st);
    if (rc) return rc;
    // V_k = Q factor of Vbar_k, column-pivoted in the first iteration (rank determination)
    rc = house_basis(c, A3, r0, ru, it == 1 ? 1 : 0, tol, Vk, r0, &rv);
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
  size_t C, Hh, Vh, lam, LU, pv, scratch, total;
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
  s.Hh = take((size_t)m * m * sizeof(double2));
  s.Vh = take((size_t)m * m * sizeof(double2));
  s.lam = take((size_t)m * sizeof(double2));
  s.LU = take((size_t)m * m * sizeof(double2));
  s.pv = take((size_t)m * sizeof(int));
  s.scratch = take((size_t)m * ((size_t)m * m + 2 * m) * sizeof(double2));  // per-eigenvalue inverse iteration
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
  double2* Hh = (double2*)(w + L.Hh);
  double2* Vh = (double2*)(w + L.Vh);
  double2* lam = (double2*)(w + L.lam);
  k_hess<<<1, 256, 0, st>>>(m, C, Vh);  // C <- Hessenberg H (in place)
  if (cudaMemcpyAsync(Hh, C, (size_t)m * m * sizeof(double2), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  {
    const size_t hsm = m <= 119 ? (size_t)m * m * sizeof(double2) : 0;  // kHqrSmemMaxM (dense.cu)
    if (hsm && ensure_smem_attr(k_hqr_vals, hsm) != cudaSuccess)
      return PRONY_ERR_CUDA;
    k_hqr_vals<<<1, 32, hsm, st>>>(m, C, lam, status, 60);  // eigenvalues (C overwritten)
  }
  k_inv_iter<<<(m + 7) / 8, 256, 0, st>>>(m, Hh, lam, Vh, W, (double2*)(w + L.scratch), 0.0);
  k_lu<<<1, 256, 0, st>>>(m, W, (double2*)(w + L.LU), (int*)(w + L.pv), status);
  k_diag_z<<<(d * m + 7) / 8, 256, 0, st>>>(d, m, (double2*)(w + L.LU), (int*)(w + L.pv), W, S, z, t, status);
  return cudaGetLastError() == cudaSuccess ? PRONY_OK : PRONY_ERR_CUDA;
}

// ---------------------------------------------------------------------------- Lanczos (NEXT-3)
// Golub-Kahan-Lanczos bidiagonalization of T (Alg. 2) with full reorthogonalization
// (twice-is-enough classical Gram-Schmidt against all previous u / v), stopping criteria
// alpha_i <= tol ||T||_F or beta_i <= tol ||T||_F, the early-stop check of P:168 (a random
// vector orthogonal to the current basis that T or T^H does not annihilate restarts the recurrence),
// and the SVD of the bidiagonal factor -> rank, U, V, sigma without knowing m.
namespace {

__global__ void k_scale_vec(int N, double2* __restrict__ x, int ldx, double s) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x)
    x[(size_t)k * ldx] = make_double2(x[(size_t)k * ldx].x * s, x[(size_t)k * ldx].y * s);
}
__global__ void k_axpy_vec(int N, double a, const double2* __restrict__ x, int ldx, double2* __restrict__ y, int ldy) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    const double2 xv = x[(size_t)k * ldx];
    double2 yv = y[(size_t)k * ldy];
    yv.x += a * xv.x;
    yv.y += a * xv.y;
    y[(size_t)k * ldy] = yv;
  }
}

struct LanczosLayout {
  size_t Ub, Vb, c, tmp, Bt, Ju, Jv, Jvv, sig, sigs, ord, dparts, dscal, Gp, apply, total;
};
LanczosLayout lanczos_layout(int d, int n, int N, int kmax) {
  LanczosLayout s{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  s.Ub = take((size_t)N * (kmax + 1) * sizeof(double2));
  s.Vb = take((size_t)N * (kmax + 1) * sizeof(double2));
  s.c = take((size_t)(kmax + 2) * sizeof(double2));
  s.tmp = take((size_t)N * sizeof(double2));
  s.Bt = take((size_t)(kmax + 1) * kmax * sizeof(double2));
  s.Ju = take((size_t)(kmax + 1) * kmax * sizeof(double2));
  s.Jv = take((size_t)kmax * kmax * sizeof(double2));
  s.Jvv = take((size_t)kmax * kmax * sizeof(double2));
  s.sig = take((size_t)(kmax + 1) * sizeof(double));
  s.sigs = take((size_t)(kmax + 1) * sizeof(double));
  s.ord = take((size_t)(kmax + 1) * sizeof(int));
  s.dparts = take(4096 * sizeof(double));
  s.dscal = take(64 * sizeof(double));
  s.Gp = take((size_t)kGramKS * (kmax + 2) * sizeof(double2));
  s.apply = take(apply_workspace_bytes(d, n, N));
  s.total = off;
  return s;
}

}  // namespace

size_t lanczos_workspace_bytes(int d, int n, int N, int kmax) { return lanczos_layout(d, n, N, kmax).total; }

int lanczos_svd(int d, int n, int N, const double2* grid, int kmax, double tol, uint64_t seed, double2* U, double2* V,
                double* sigma, int ldo, int* rank_out, int* steps_out, void* ws, int sm_count, cudaStream_t st) {
  const LanczosLayout L = lanczos_layout(d, n, N, kmax);
  char* w = (char*)ws;
  double2* Ub = (double2*)(w + L.Ub);  // N x (kmax+1) row-major: u_j = column j
  double2* Vb = (double2*)(w + L.Vb);
  double2* cvec = (double2*)(w + L.c);
  double2* tmp = (double2*)(w + L.tmp);
  double* dparts = (double*)(w + L.dparts);
  double* dscal = (double*)(w + L.dscal);
  double2* Gp = (double2*)(w + L.Gp);
  void* aws = w + L.apply;
  const int ld = kmax + 1;
  const int gb = grid1(N, sm_count);
  const int nb = std::min(4096, 2 * sm_count);
  auto norm2 = [&](const double2* x, int ldx, double* host) -> int {
    k_fro2_parts<<<nb, 256, 0, st>>>(N, 1, x, ldx, dparts);
    k_sum_doubles<<<1, 32, 0, st>>>(nb, dparts, dscal);
    if (cudaMemcpyAsync(host, dscal, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess) return PRONY_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
    *host = sqrt(*host);
    return PRONY_OK;
  };
  // x (column of a row-major block, stride ldx) -= B(:, 0:k) B(:, 0:k)^H x, twice
  auto reorth = [&](const double2* B, int k, double2* x, int ldx) {
    if (k <= 0) return;
    for (int pass = 0; pass < 2; ++pass) {
      dim3 g((k + 31) / 32, 1, kGramKS);
      k_gram<<<g, 256, 0, st>>>(N, k, 1, B, ld, x, ldx, kGramKS, Gp);
      k_sum_parts<<<grid1(k, sm_count), 256, 0, st>>>(k, kGramKS, Gp, cvec);
      k_gemm_nm<<<dim3((N + 63) / 64, 1), 256, 0, st>>>(N, k, 1, B, ld, cvec, 1, x, ldx, -1.0, 1.0);
    }
  };
  // ||T||_F for the absolute tolerance
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  k_normT2_parts<<<nb, 256, 0, st>>>(d, n, box, grid, dparts);
  k_sum_doubles<<<1, 32, 0, st>>>(nb, dparts, dscal);
  double normT2 = 0.0;
  if (cudaMemcpyAsync(&normT2, dscal, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess) return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
  // rank / stopping tolerance: tol ||T||_F, floored at 1e-10 ||T||_F (reading R24: rounding in the
  // reorthogonalized basis leaves residuals ~1e-13 ||T||_F that N eps would count as rank)
  const double tol_abs = std::max(tol, kLanczosTolFloor) * sqrt(normT2);

  std::vector<double> alpha, beta;  // beta[0] = beta_1 of the paper
  // p_1 random, v_1 = p_1 / ||p_1||
  k_fill_random<<<gb, 256, 0, st>>>(N, seed, Vb, N, 1, ld);
  double b = 0.0;
  int rc = norm2(Vb, ld, &b);
  if (rc) return rc;
  k_scale_vec<<<gb, 256, 0, st>>>(N, Vb, ld, 1.0 / b);
  beta.push_back(b);
  int k = 0;             // vectors u_0..u_{k-1} accepted
  bool alpha_stop = false, stopped = false;
  uint64_t restart_seed = seed ^ 0x5DEECE66Dull;
  int steps = 0;
  for (;;) {
    if (k >= N) {  // the basis spans C^N: nothing left to find
      stopped = true;
      break;
    }
    if (k >= kmax) break;
    ++steps;
    // r = T v_k - beta_k u_{k-1}  -> stored in Ub column k
    rc = toeplitz_apply_launch(d, n, N, grid, 0, 0, Vb + k, ld, 1, Ub + k, ld, aws, sm_count, st);
    if (rc) return rc;
    if (k > 0) k_axpy_vec<<<gb, 256, 0, st>>>(N, -beta[k], Ub + (k - 1), ld, Ub + k, ld);
    reorth(Ub, k, Ub + k, ld);
    double a = 0.0;
    if ((rc = norm2(Ub + k, ld, &a))) return rc;
    if (a <= tol_abs) {
      // early-stop check: random y orthogonal to u_0..u_{k-1}; if T^H y = 0 we are done
      k_fill_random<<<gb, 256, 0, st>>>(N, restart_seed++, Ub + k, N, 1, ld);
      reorth(Ub, k, Ub + k, ld);
      double yn = 0.0;
      if ((rc = norm2(Ub + k, ld, &yn))) return rc;
      rc = toeplitz_apply_launch(d, n, N, grid, 0, 1, Ub + k, ld, 1, tmp, 1, aws, sm_count, st);
      if (rc) return rc;
      double zn = 0.0;
      if ((rc = norm2(tmp, 1, &zn))) return rc;
      if (yn == 0.0 || zn <= tol_abs * yn) {
        alpha_stop = stopped = true;
        break;
      }
      k_scale_vec<<<gb, 256, 0, st>>>(N, Ub + k, ld, 1.0 / yn);
      a = 0.0;  // continue with u_k = y / ||y|| and alpha_k = 0
    } else {
      k_scale_vec<<<gb, 256, 0, st>>>(N, Ub + k, ld, 1.0 / a);
    }
    alpha.push_back(a);
    ++k;
    // p = T^H u_{k-1} - alpha_{k-1} v_{k-1} -> Vb column k
    rc = toeplitz_apply_launch(d, n, N, grid, 0, 1, Ub + (k - 1), ld, 1, Vb + k, ld, aws, sm_count, st);
    if (rc) return rc;
    k_axpy_vec<<<gb, 256, 0, st>>>(N, -alpha[k - 1], Vb + (k - 1), ld, Vb + k, ld);
    reorth(Vb, k, Vb + k, ld);
    double bb = 0.0;
    if ((rc = norm2(Vb + k, ld, &bb))) return rc;
    if (bb <= tol_abs && k >= N) {
      stopped = true;  // V_k spans C^N (beta stop, B_k square)
      beta.push_back(0.0);
      break;
    }
    if (bb <= tol_abs) {
      // early-stop check: random w orthogonal to v_0..v_{k-1}; if T w = 0 we are done
      k_fill_random<<<gb, 256, 0, st>>>(N, restart_seed++, Vb + k, N, 1, ld);
      reorth(Vb, k, Vb + k, ld);
      double wn = 0.0;
      if ((rc = norm2(Vb + k, ld, &wn))) return rc;
      rc = toeplitz_apply_launch(d, n, N, grid, 0, 0, Vb + k, ld, 1, tmp, 1, aws, sm_count, st);
      if (rc) return rc;
      double zn = 0.0;
      if ((rc = norm2(tmp, 1, &zn))) return rc;
      if (wn == 0.0 || zn <= tol_abs * wn) {
        beta.push_back(0.0);
        stopped = true;
        break;  // beta stop: rank k, B_k square
      }
      k_scale_vec<<<gb, 256, 0, st>>>(N, Vb + k, ld, 1.0 / wn);
      bb = 0.0;
    } else {
      k_scale_vec<<<gb, 256, 0, st>>>(N, Vb + k, ld, 1.0 / bb);
    }
    beta.push_back(bb);
  }
  const int rank = k;  // dimension of the bidiagonal factor
  *rank_out = rank;
  if (steps_out) *steps_out = steps;
  if (rank == 0) return PRONY_ERR_RANK;
  if (k >= N && !alpha_stop) beta.push_back(0.0);
  // B^T (rows x rank): B has alpha_j on the diagonal and beta_{j+1} (beta[j+1]) on the superdiagonal;
  // alpha stop -> B_{k,k+1} (rows = k+1), otherwise B_k (rows = k)
  const int rows = (alpha_stop && rank < kmax) ? rank + 1 : rank;
  std::vector<double2> Bt((size_t)rows * rank, make_double2(0.0, 0.0));
  for (int j = 0; j < rank; ++j) {
    Bt[(size_t)j * rank + j] = make_double2(alpha[j], 0.0);               // B[j][j]
    if (j + 1 < rows) Bt[(size_t)(j + 1) * rank + j] = make_double2(beta[j + 1], 0.0);  // B[j][j+1]
  }
  double2* dBt = (double2*)(w + L.Bt);
  if (cudaMemcpyAsync(dBt, Bt.data(), Bt.size() * sizeof(double2), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  double2 *Ju = (double2*)(w + L.Ju), *Jv = (double2*)(w + L.Jv), *Jvv = (double2*)(w + L.Jvv);
  double* sg = (double*)(w + L.sig);
  int* ord = (int*)(w + L.ord);
  // B^T = (V_B) Sigma (U_B)^T: Jacobi on B^T gives Ju = V_B (rows x rank), Jvv = U_B (rank x rank)
  k_jacobi_svd<<<1, 1024, 0, st>>>(rows, rank, dBt, Jv, sg, Ju, Jvv, ord, 60);
  // rank = number of singular values of B above the tolerance ("catch the drop of singular
  // values"; with rounding the factor can carry one extra tiny singular value, reading R24)
  double* sgs = (double*)(w + L.sigs);
  k_permute_sigma<<<1, 256, 0, st>>>(rank, sg, ord, sgs);
  std::vector<double> sh(rank);
  if (cudaMemcpyAsync(sh.data(), sgs, rank * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
  int r_eff = 0;
  while (r_eff < rank && sh[r_eff] > tol_abs) ++r_eff;
  *rank_out = r_eff;
  if (r_eff == 0) return PRONY_ERR_RANK;
  const int kout = std::min(r_eff, ldo);
  if (cudaMemcpyAsync(sigma, sgs, kout * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  // U = U_k U_B (N x rank)(rank x kout), V = V_rows V_B (N x rows)(rows x kout)
  k_gemm_nm<<<dim3((N + 63) / 64, (kout + 31) / 32), 256, 0, st>>>(N, rank, kout, Ub, ld, Jvv, rank, U, ldo, 1.0, 0.0);
  k_gemm_nm<<<dim3((N + 63) / 64, (kout + 31) / 32), 256, 0, st>>>(N, rows, kout, Vb, ld, Ju, rank, V, ldo, 1.0, 0.0);
  if (cudaGetLastError() != cudaSuccess) return PRONY_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
  return stopped ? PRONY_OK : PRONY_ERR_NOT_CONVERGED;
}

}  // namespace prony
