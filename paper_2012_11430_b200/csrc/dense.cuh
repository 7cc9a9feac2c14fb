// dense.cuh — small dense linear algebra kernels of NEXT-1 (dense.cu) and the block-power SVD /
// diagonalization drivers (svd.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace prony {

__global__ void k_fill_random(int64_t count, uint64_t seed, double2* out, int rows, int cols, int ld);
__global__ void k_gram(int N, int ri, int rj, const double2* X, int ldx, const double2* Y, int ldy, int KS,
                       double2* Gp);
__global__ void k_sum_parts(int64_t count, int KS, const double2* parts, double2* out);
__global__ void k_gemm_nm(int N, int r, int c, const double2* X, int ldx, const double2* M, int ldm, double2* Y,
                          int ldy, double alpha, double beta);
__global__ void k_fro2_parts(int N, int c, const double2* X, int ldx, double* parts);
__global__ void k_normT2_parts(int d, int n, int64_t box, const double2* grid, double* parts);
__global__ void k_sum_doubles(int count, const double* parts, double* out);

// Householder QR of a tall N x r matrix in one cooperative launch (dense.cu, k_house_qr)
constexpr int kHouseMaxCols = 256;  // r0 = 2m <= 256 (m <= kMaxM = 128)
constexpr int kHouseMaxGrid = 256;  // CTAs of the cooperative launch (partial buffers are sized for it)
struct HouseQrArgs {
  int N, r, pivot;
  double tol;
  double2* X;  // N x r, ld ldx: overwritten (reflector tails / R)
  int ldx;
  double2* Q;  // out: N x rank, ld ldq, orthonormal columns in pivoted order
  int ldq;
  int* perm;   // out: perm[k] = column of X in column k of Q R (k < rank)
  int* rank;   // out: rank (pivot) or min(N, r)
  double2* wpart;  // [r][G] per-CTA column partials
  double* npart;
  double2* wfin;   // [r] reduced columns
  double* nfin;
};
__global__ void k_house_qr(HouseQrArgs a);
size_t house_qr_workspace_bytes(int r);
int house_qr_launch(int N, int r, double2* X, int ldx, int pivot, double tol, double2* Q, int ldq, int* perm,
                    int* rank_dev, void* ws, int sm_count, cudaStream_t st);
__global__ void k_jacobi_svd(int rows, int cols, double2* A, double2* Vm, double* sigma, double2* Uout, double2* Vout,
                             int* order, int max_sweeps);
__global__ void k_permute_sigma(int cols, const double* sigma, const int* order, double* out);
__global__ void k_combine(int d, int m, const double2* mu, const double2* S, double2* C);
__global__ void k_hess(int m, double2* H, double2* Vh);
__global__ void k_hqr_vals(int m, double2* H, double2* lam, int* status, int max_iter_per_eig);
__global__ void k_inv_iter(int m, const double2* Hh, const double2* lam, const double2* Vh, double2* W,
                           double2* scratch, double anorm_hint);
__global__ void k_lu(int m, const double2* W, double2* LU, int* pv, int* status);
__global__ void k_diag_z(int d, int m, const double2* LU, const int* pv, const double2* W, const double2* S,
                         double2* z, double* t, const int* status);

size_t svd_workspace_bytes(int d, int n, int N, int m);
int block_power_svd(int d, int n, int N, const double2* grid, int m, double tol, int max_iter, uint64_t seed,
                    double2* U, double2* V, double* sigma, int* rank_out, int* iters_out, double* resid_out, void* ws,
                    int sm_count, cudaStream_t st);
size_t diag_workspace_bytes(int d, int m);
constexpr int kLanczosMaxRank = 255;     // Jacobi pair table of the bidiagonal SVD
constexpr double kLanczosTolFloor = 1e-10;  // relative rank tolerance floor (R24)
size_t lanczos_workspace_bytes(int d, int n, int N, int kmax);
int lanczos_svd(int d, int n, int N, const double2* grid, int kmax, double tol, uint64_t seed, double2* U, double2* V,
                double* sigma, int ldo, int* rank_out, int* steps_out, void* ws, int sm_count, cudaStream_t st);
int diagonalize_launch(int d, int m, const double2* S, const double2* mu, double2* z, double* t, double2* W,
                       void* ws, int32_t* status, cudaStream_t st);

}  // namespace prony
