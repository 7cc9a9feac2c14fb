/*
 * prony.h — C ABI of the B200 (sm_100a) hot path of the multivariate matrix-pencil
 * Prony method (arXiv 2012.11430; citations "P:<line>" are lines of PAPER.md).
 *
 * Problem (Algorithm 1): samples f(k) of f(k) = sum_{j=1..m} c_j e^{-2 pi i <t_j,k>}
 * -> parameters t_j and coefficients c_j. This library implements the
 * data-parallel steps of that algorithm that the paper puts on the GPU:
 *
 *   prony_project        S_l = U* T_l V Sigma^-1,  T_l = [f(k-h+e_l)]_{k,h in I_n}
 *                        (P:21, P:27-29 eq_generateSl), T_l generated implicitly from the
 *                        sample grid (never materialized), complex FP64 on the DMMA pipe.
 *   prony_vandermonde_ls A = [z_j^k]_{j, k in I_n}, the normal-equation products
 *                        G = A conj(A)^T, b = A conj(f) of argmin_c ||A^T c - f||_2,
 *                        and, over the full column range, c = conj(G^-1 b) and
 *                        t_j = (-arg z_j / 2 pi) mod 1 (reading R4).
 *   prony_pencil_host    both of the above from HOST buffers (copies in, results out);
 *                        prony_pencil_host_part: one rank's partial share (multi-GPU end to end).
 *   prony_build_pencil   reduced SVD of T (block power method Alg. 3) on the
 *                        device, then prony_project (Algorithm 1 lines 1-3).
 *   prony_diagonalize    C_mu, its eigenvectors W, z = diag(W^-1 S_l W), t (Algorithm 1 lines 4-6).
 *   prony_toeplitz_apply T_l X, T X, T^H X with the implicit gather (the operator of the SVD).
 *   prony_lanczos_svd    rank-revealing reduced SVD of T by Lanczos bidiagonalization with full
 *                        reorthogonalization (Alg. 2) when m is unknown.
 *
 * Layout conventions (readings R1, R2):
 *   - complex numbers are prony_c128 {re, im} (== cuDoubleComplex == torch.complex128).
 *   - I_n = {0..n}^d in lexicographic order, LAST coordinate fastest;
 *     N = (n+1)^d. Row r of U, V and column r of A is element r of I_n.
 *   - grid: f(k) for k in the box {-n..n+1}^d (L = 2n+2 points per axis, L^d values),
 *     lexicographic, last coordinate fastest: value of k at index sum_i (k_i+n) L^(d-1-i).
 *     (Algorithm 1's input "f(k), k in I" must cover k-h+e_l, hence the box, R1.)
 *   - U, V: N x m row-major (leading dimension m); z: m x d row-major; sigma: m doubles.
 *   - S: d x m x m row-major (S[l-1][i][j]); G: m x m row-major; b, c: m; t: m x d.
 *
 * Ownership and execution:
 *   - Every pointer argument of prony_project / prony_vandermonde_ls is a DEVICE pointer
 *     owned by the caller (e.g. a torch tensor); the library never allocates, frees or
 *     retains memory. Scratch comes only from the caller's `workspace` (device, 256-byte
 *     aligned, size >= prony_workspace_size(...)). No global mutable state beyond
 *     idempotent, thread-safe memoization of device facts (the SM count per device, each
 *     kernel's shared-memory opt-in): calls are reentrant and CUDA-graph capturable.
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t; 0 = legacy
 *     default stream). Argument validation is synchronous, BEFORE any launch.
 *   - `dev_status` (device int32, caller-owned, nullable) receives numerical failures
 *     found on the device (first error wins); the caller must zero it beforehand (except for
 *     prony_pencil, which zeroes it itself) and read it after synchronizing. The return value covers validation and launch errors only.
 *
 * Error behaviour (return values):
 *   PRONY_OK                 launched (or nothing to do for an empty range)
 *   PRONY_ERR_INVALID        null / misaligned pointer, d,n,m out of range, bad unit_order
 *   PRONY_ERR_RANGE          (2n+2)^d >= 2^31, m > PRONY_MAX_M, m > N, range outside [0, limit]
 *   PRONY_ERR_SINGULAR       (dev_status) G not Hermitian positive definite in the Cholesky, a sigma below
 *                            the scale guard (prony_project), W singular (prony_diagonalize)
 *   PRONY_ERR_RANK           detected rank below m (prony_build_pencil) or T = 0 (prony_lanczos_svd)
 *   PRONY_ERR_NOT_CONVERGED  iteration cap reached (block power, Lanczos, QR eigensolver); outputs written
 *   PRONY_ERR_CUDA           a CUDA launch / copy failed (cudaGetLastError() is left set)
 *   PRONY_ERR_UNIMPLEMENTED  reserved (every entry point of this header is implemented)
 *   PRONY_ERR_WORKSPACE      workspace_bytes smaller than prony_workspace_size(...)
 *
 * Implementation limits (this build): 1 <= d <= PRONY_MAX_D, 1 <= m <= PRONY_MAX_M,
 * m <= N, (2n+2)^d < 2^31, N * 8 ceil(m/8) < 2^31.
 */
#ifndef PRONY_H
#define PRONY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRONY_ABI_VERSION 6  /* 2: PRONY_UNITS_SHARED, prony_lanczos_svd, PRONY_WS_LANCZOS; 3: prony_pencil_host_part;
                                 4: prony_host_context, prony_pencil_host_ctx, prony_pencil_host_part_ctx;
                                 5: prony_pencil, PRONY_WS_PENCIL;
                                 6: prony_exec_info.ev_wait_u (prony_project_ex) */
#define PRONY_MAX_D 8
#define PRONY_MAX_M 128

typedef struct prony_c128 {
  double re;
  double im;
} prony_c128;

/* cudaStream_t without including the CUDA headers */
typedef struct CUstream_st* prony_stream_t;
/* opaque: the side streams and events of the host-input pencil, created once (prony_host_context_create) */
typedef struct prony_host_context_s* prony_host_context;

typedef enum prony_status {
  PRONY_OK = 0,
  PRONY_ERR_INVALID = 1,
  PRONY_ERR_RANGE = 2,
  PRONY_ERR_SINGULAR = 3,
  PRONY_ERR_RANK = 4,
  PRONY_ERR_NOT_CONVERGED = 5,
  PRONY_ERR_CUDA = 6,
  PRONY_ERR_UNIMPLEMENTED = 7,
  PRONY_ERR_WORKSPACE = 8
} prony_status;

/* which workspace (prony_workspace_size) */
typedef enum prony_workspace_kind {
  PRONY_WS_PROJECT = 0,      /* prony_project, any unit range */
  PRONY_WS_LS = 1,           /* prony_vandermonde_ls, any column range */
  PRONY_WS_PENCIL_HOST = 2,  /* prony_pencil_host: device copies of inputs/outputs + both above */
  PRONY_WS_BUILD = 3,        /* prony_build_pencil */
  PRONY_WS_APPLY = 4,        /* prony_toeplitz_apply, any r */
  PRONY_WS_DIAG = 5,         /* prony_diagonalize */
  PRONY_WS_PROJECT_MU = 6,   /* prony_project_mu */
  PRONY_WS_LANCZOS = 7,      /* prony_lanczos_svd; the m argument is max_rank (<= 255) */
  PRONY_WS_PENCIL = 8        /* prony_pencil: the scratch of prony_project and prony_vandermonde_ls side by side */
} prony_workspace_kind;

/* unit orders of prony_project. L_MAJOR / ROW_MAJOR: units u in [0, d*N), one row k
 * of one T_l each. SHARED: units u in [0, (n+2)^d), one row k' of the extended Toeplitz block
 * T_E = [f(k'-h)]_{k' in {0..n+1}^d, h in I_n} each; since T_l[k,:] = T_E[k+e_l,:] (F8)
 * one product T_E V serves all d pencils ((n+2)^d instead of d(n+1)^d rows of work). */
typedef enum prony_unit_order {
  PRONY_UNITS_L_MAJOR = 0,    /* u = (l-1)*N + k  (l-sharding when ranks divide d) */
  PRONY_UNITS_ROW_MAJOR = 1,  /* u = k*d + (l-1)  (row-block sharding, all l per rank) */
  PRONY_UNITS_SHARED = 2      /* u = index of k' in {0..n+1}^d (lexicographic, last fastest) */
} prony_unit_order;

/*
 * Optional per-call execution record (the *_ex entry points). Nothing is retained after the
 * call returns. The events, when non-null, are cudaEvent_t created by the caller; they are
 * recorded on `stream` immediately before / after the call's dominant kernel (k_project for
 * prony_project_ex, k_vls for prony_vandermonde_ls_ex), so the caller can time that kernel.
 */
typedef struct prony_exec_info {
  void* ev_main_begin;    /* in, nullable: cudaEvent_t */
  void* ev_main_end;      /* in, nullable: cudaEvent_t */
  int32_t launches;       /* out: kernels launched by the call */
  int32_t main_grid[3];   /* out: grid of the dominant kernel */
  int32_t main_block;     /* out: threads per CTA of the dominant kernel */
  int32_t split_k;        /* out: column chunks of T_l (prony_project) / column blocks (LS) */
  double main_flops;      /* out: algorithmic FP64 flops of the dominant kernel (8 real flops per
                             complex multiply-add): 8 m N * rows for k_project, 8 m^2 W for k_vls */
  void* ev_wait_u;        /* in, nullable (prony_project_ex only): cudaEvent_t the stream waits on right
                             before the reduction, the first kernel that reads U — lets a caller still
                             copying U (another stream) overlap that copy with the projection */
} prony_exec_info;

/* ABI version (== PRONY_ABI_VERSION of the built library). */
int prony_abi_version(void);

/* Static description of a status code; never NULL. */
const char* prony_status_string(int status);

/* Number of SMs / compute capability of the current device, for diagnostics.
   Returns PRONY_ERR_CUDA if no device is usable. */
int prony_device_info(int* sm_count, int* cc_major, int* cc_minor);

/*
 * Workspace bytes for `kind` at (d, n, m) on the current device; an upper bound valid for
 * every unit / column range. Writes *bytes. Validates (d, n, m) as the calls do.
 */
int prony_workspace_size(int kind, int d, int n, int m, size_t* bytes);

/*
 * prony_project — the pencil S_l = U* T_l V Sigma^-1, partial over a unit range.
 *
 *   grid        device, L^d prony_c128: samples on the box {-n..n+1}^d (see layout above).
 *   U, V        device, N x m prony_c128 row-major: left / right singular vectors of T
 *               (eq_T_svd); any N x m inputs are accepted (the pencil is linear in
 *               them); identical inputs give bit-identical outputs (fixed-order reductions).
 *   sigma       device, m doubles > 0: Sigma^-1 is applied as the column scale 1/sigma_j (R11).
 *   unit_begin, unit_end, unit_order
 *               the call contributes the rows k of T_l for the units u in [unit_begin,
 *               unit_end) of [0, U) (order: prony_unit_order; U = d*N for L_MAJOR / ROW_MAJOR,
 *               (n+2)^d for SHARED). [0, U) gives the complete S_1..S_d; a partition of [0, U)
 *               over ranks gives partial pencils whose SUM is S (Sigma^-1 already applied),
 *               i.e. one all-reduce completes the pencil. SHARED is the fast order (the
 *               library's own full-pencil calls use it).
 *   S           device, d x m x m prony_c128, OVERWRITTEN with this call's partial sum
 *               (rows of S_l with no unit in range are zero).
 *   workspace   device scratch of workspace_bytes >= prony_workspace_size(PRONY_WS_PROJECT).
 *   dev_status  nullable device int32: PRONY_ERR_SINGULAR when a sigma_j is not finite and positive or
 *               sigma_min <= N eps_M sigma_max (the scale guard of SURVEY §8(b) / P:581); S is still
 *               written (the column scale 1/sigma_j is applied regardless).
 *   stream      CUDA stream for all launches.
 */
int prony_project(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                  const double* sigma, int64_t unit_begin, int64_t unit_end, int unit_order, prony_c128* S,
                  void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream);

/* prony_project + execution record (info nullable; same semantics otherwise). */
int prony_project_ex(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                     const double* sigma, int64_t unit_begin, int64_t unit_end, int unit_order, prony_c128* S,
                     void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream,
                     prony_exec_info* info);

/*
 * prony_vandermonde_ls — A = [z_j^k], G = A conj(A)^T and b = A conj(f) (P:59,
 * DESIGN.md R10) over the columns k in [col_begin, col_end) of I_n.
 *
 *   z           device, m x d prony_c128 nodes (computed z~ need not have unit modulus);
 *               powers z^a are formed by repeated multiplication (R9).
 *   grid        device, the same sample box as prony_project; f(k) is read at k in I_n.
 *   A           nullable device m x (col_end-col_begin) prony_c128 row-major: if non-null the
 *               Vandermonde block of the range is written (A[j][k-col_begin]).
 *   G, b        device m x m / m prony_c128, OVERWRITTEN with the range's partial sums.
 *   c, t        nullable device m prony_c128 / m x d doubles: written only when the range is
 *               the full [0, N): c = conj(G^-1 b) via Cholesky (G conj(c) = b, R10) and
 *               t = (-arg z / 2 pi) mod 1 (R4). If G is not HPD, *dev_status =
 *               PRONY_ERR_SINGULAR and c is left NaN.
 *   workspace   >= prony_workspace_size(PRONY_WS_LS).
 */
int prony_vandermonde_ls(int d, int n, int m, const prony_c128* z, const prony_c128* grid, int64_t col_begin,
                         int64_t col_end, prony_c128* A, prony_c128* G, prony_c128* b, prony_c128* c, double* t,
                         void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream);

/* prony_vandermonde_ls + execution record (info nullable; same semantics otherwise). */
int prony_vandermonde_ls_ex(int d, int n, int m, const prony_c128* z, const prony_c128* grid, int64_t col_begin,
                            int64_t col_end, prony_c128* A, prony_c128* G, prony_c128* b, prony_c128* c, double* t,
                            void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream,
                            prony_exec_info* info);

/*
 * prony_ls_solve — c = conj(G^-1 b) by Cholesky (G conj(c) = b, R10) and, if t is
 * non-null, t = (-arg z / 2 pi) mod 1 (R4), for G, b already summed over all
 * columns (e.g. after the all-reduce of per-rank prony_vandermonde_ls partials).
 *   G, b, z     device m x m, m, m x d prony_c128;  c device m prony_c128;  t nullable m x d doubles.
 *   workspace   unused (nullable; the factor lives in shared memory), kept for ABI stability.
 *   dev_status  PRONY_ERR_SINGULAR if G is not Hermitian positive definite (c is then NaN).
 */
int prony_ls_solve(int d, int m, const prony_c128* G, const prony_c128* b, const prony_c128* z, prony_c128* c,
                   double* t, void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream);

/*
 * prony_project_mu — C_mu = U* B_mu V Sigma^-1 with B_mu = sum_l mu_l T_l (the paper's B_mu
 * preprocessing; NEXT-4): B_mu is itself the Toeplitz operator of the combined grid
 * g_mu[x] = sum_l mu_l grid[x + L^(d-l)], so C_mu costs one projection instead of d. Equal to
 * sum_l mu_l S_l in exact arithmetic (R8).
 *   mu         device d prony_c128;  C device m x m (overwritten)
 *   workspace  >= prony_workspace_size(PRONY_WS_PROJECT_MU)
 */
int prony_project_mu(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                     const double* sigma, const prony_c128* mu, prony_c128* C, void* workspace, size_t workspace_bytes,
                     int32_t* dev_status, prony_stream_t stream);

/*
 * prony_toeplitz_apply — Y = T_l X (l = 1..d), Y = T X (l = 0) or, with conj = 1 and l = 0,
 * Y = T^H X, for an N x r block X; T = [f(k-h)], T_l = [f(k-h+e_l)] generated implicitly
 * from the grid exactly as in prony_project (never materialized). This is the operator the block
 * power SVD of T (Alg. 3) applies; any r >= 1 (processed in column passes).
 *   X           device N x r prony_c128, row stride ldx (elements, >= r)
 *   Y           device N x r prony_c128, row stride ldy (>= r), overwritten
 *   workspace   >= prony_workspace_size(PRONY_WS_APPLY)   (m argument ignored for this kind)
 * Errors: PRONY_ERR_INVALID for conj with l != 0, l out of [0, d], null/misaligned pointers.
 */
int prony_toeplitz_apply(int d, int n, const prony_c128* grid, int ell, int conj, const prony_c128* X, int ldx, int r,
                         prony_c128* Y, int ldy, void* workspace, size_t workspace_bytes, prony_stream_t stream);

/*
 * prony_pencil_host — one full pencil (prony_project over all SHARED units + prony_vandermonde_ls over
 * [0, N), c and t included) from HOST inputs to HOST outputs, synchronizing `stream` at the end. Only
 * the grid and the V rows of split-K chunk 0 are copied before the first DMMA: three side streams
 * (created and destroyed by the call, or taken from a prony_host_context, ordered after prior work on
 * `stream`) carry the rest of V with the remaining chunks of the projection, U after V on its own
 * stream (first needed by the final reduction), and z with the LS step. Host buffers should be page-locked for full PCIe bandwidth (not required).
 *   host inputs : grid (L^d), U, V (N x m), sigma (m), z (m x d)
 *   host outputs: S (d x m x m), G (m x m), b (m), c (m), t (m x d); any output may be NULL
 *   workspace   : DEVICE scratch >= prony_workspace_size(PRONY_WS_PENCIL_HOST)
 *   *status_out : (nullable host int32) the device status word after the call
 * Returns PRONY_OK, a validation error, or PRONY_ERR_CUDA.
 */
int prony_pencil_host(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                      const double* sigma, const prony_c128* z, prony_c128* S, prony_c128* G, prony_c128* b,
                      prony_c128* c, double* t, void* workspace, size_t workspace_bytes, int32_t* status_out,
                      prony_stream_t stream);

/*
 * prony_host_context_create / _destroy — an explicit context for the host-input pencil: the three side
 * streams and eight events prony_pencil_host* would otherwise create and destroy on every call (tens of
 * microseconds of host time, visible on small pencils). Owned by the caller; bound to the device current
 * at creation (a call on another device returns PRONY_ERR_INVALID); one context serves one call at a time
 * (calls sharing a context must be ordered on the same `stream`). _destroy synchronizes its streams.
 * Returns PRONY_OK, PRONY_ERR_INVALID (null out / ctx) or PRONY_ERR_CUDA.
 */
int prony_host_context_create(prony_host_context* ctx_out);
int prony_host_context_destroy(prony_host_context ctx);

/*
 * prony_pencil_host_ctx / prony_pencil_host_part_ctx — prony_pencil_host / prony_pencil_host_part with the
 * side streams and events taken from `ctx` (NULL: created for the call, as the plain entry points do).
 * Same arguments, results and errors otherwise.
 */
int prony_pencil_host_ctx(prony_host_context ctx, int d, int n, int m, const prony_c128* grid, const prony_c128* U,
                          const prony_c128* V, const double* sigma, const prony_c128* z, prony_c128* S, prony_c128* G,
                          prony_c128* b, prony_c128* c, double* t, void* workspace, size_t workspace_bytes,
                          int32_t* status_out, prony_stream_t stream);
int prony_pencil_host_part_ctx(prony_host_context ctx, int d, int n, int m, const prony_c128* grid,
                               const prony_c128* U, const prony_c128* V, const double* sigma, const prony_c128* z,
                               int64_t unit_begin, int64_t unit_end, int64_t col_begin, int64_t col_end, prony_c128* S,
                               prony_c128* G, prony_c128* b, void* workspace, size_t workspace_bytes,
                               int32_t* dev_status, prony_stream_t stream);

/*
 * prony_pencil — one full pencil on DEVICE buffers in ONE call: prony_project over all SHARED units on
 * `stream` and, concurrently on the context's side stream, prony_vandermonde_ls over [0, N) with c and t
 * (PAPER.md:27-29, 39, 58-59); `stream` is ordered after both on return (asynchronous). The launch path for
 * small, launch-bound pencils: one C call instead of the two entry points plus the stream fork/join.
 *   ctx          side stream + events (prony_host_context_create); NULL: created and destroyed by the call
 *   grid, U, V, sigma, z   device inputs as prony_project / prony_vandermonde_ls
 *   S, G, b, c, t          device outputs (d x m x m, m x m, m, m, m x d)
 *   workspace    device scratch >= prony_workspace_size(PRONY_WS_PENCIL)
 *   dev_status   nullable device int32, ZEROED BY THE CALL (in its first kernel, stream-ordered), then as
 *                prony_project / prony_vandermonde_ls: after `stream` completes it holds this pencil's first
 *                numerical failure or 0 (the launch path of small pencils saves the caller's separate reset)
 *   info_project, info_ls  nullable prony_exec_info of the two halves (events recorded on their streams)
 * Returns PRONY_OK, a validation error (as prony_project), PRONY_ERR_WORKSPACE or PRONY_ERR_CUDA.
 */
int prony_pencil(prony_host_context ctx, int d, int n, int m, const prony_c128* grid, const prony_c128* U,
                 const prony_c128* V, const double* sigma, const prony_c128* z, prony_c128* S, prony_c128* G,
                 prony_c128* b, prony_c128* c, double* t, void* workspace, size_t workspace_bytes,
                 int32_t* dev_status, prony_stream_t stream, prony_exec_info* info_project,
                 prony_exec_info* info_ls);

/*
 * prony_pencil_host_part — one rank's share of a pencil from HOST inputs (multi-GPU end to end, P:259-267
 * offload per rank): copies the grid, V, sigma, z and only the rows of U its SHARED unit range pairs
 * with, runs prony_project over units [unit_begin, unit_end) of [0, (n+2)^d) and the LS products over
 * columns [col_begin, col_end) of [0, N) (no solve), with the same copy/compute overlap as
 * prony_pencil_host, and leaves the partial S (d x m x m), G (m x m), b (m) in DEVICE memory for the
 * caller's all-reduce (then prony_ls_solve). Asynchronous and stream-ordered: host buffers must stay
 * valid (and be page-locked for overlap) until `stream` reaches the end of the call's work.
 *   workspace >= prony_workspace_size(PRONY_WS_PENCIL_HOST);  dev_status: as prony_project
 */
int prony_pencil_host_part(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                           const double* sigma, const prony_c128* z, int64_t unit_begin, int64_t unit_end,
                           int64_t col_begin, int64_t col_end, prony_c128* S, prony_c128* G, prony_c128* b,
                           void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream);

/*
 * prony_build_pencil — Algorithm 1 lines 1-3 on the device: the reduced SVD T = U Sigma V*
 * (eq_T_svd) by the block power method of Alg. 3 with starting dimension 2m
 * (P:595), T V and T^H U applied by the implicit-Toeplitz gather of prony_project, Householder QR of
 * every block, column-pivoted for Vbar_1 with rank = the first k with ||R(k:,k:)||_F <= tol ||R||_F
 * (R22), and the SVD of Q_k by one-sided Jacobi; then S_1..S_d = U* T_l V Sigma^-1 over all units (prony_project).
 * SYNCHRONOUS: the stream is synchronized once per power iteration (the rank and the residual steer it).
 *   grid            device L^d samples (as prony_project)
 *   seed            seeds the random starting block V_0 (counter-based generator, R14)
 *   tol             rank / convergence tolerance (P:581 noise-free N*eps_M; P:627 the noise level)
 *   max_iter        power iterations (>= 1)
 *   S               device d x m x m;  U, V device N x m;  sigma device m (nonincreasing)
 *   rank_out        host int32: detected rank r_1 (PRONY_ERR_RANK if < m)
 *   resid_out       nullable host double: ||T V_k - U_k Q_k||_F / ||T||_F at exit
 *   workspace       >= prony_workspace_size(PRONY_WS_BUILD)
 * Returns PRONY_OK, PRONY_ERR_RANK (rank below m), PRONY_ERR_NOT_CONVERGED (residual above tol after
 * max_iter; outputs are still written), or validation / CUDA errors.
 */
int prony_build_pencil(int d, int n, int m, const prony_c128* grid, uint64_t seed, double tol, int max_iter,
                       prony_c128* S, prony_c128* U, prony_c128* V, double* sigma, int32_t* rank_out,
                       double* resid_out, void* workspace, size_t workspace_bytes, int32_t* dev_status,
                       prony_stream_t stream);

/*
 * prony_diagonalize — Algorithm 1 lines 4-6: C_mu = sum_l mu_l S_l, W from the
 * eigendecomposition of C_mu (Hessenberg + shifted QR + back substitution; unit columns), the
 * simultaneous diagonalization z_tau(j)(l) = (W^-1 S_l W)_jj (by LU with partial pivoting)
 * and t = (-arg z / 2 pi) mod 1 (R4). One small CTA; asynchronous.
 *   S   device d x m x m;  mu device d (unit norm);  z device m x d;  t nullable device m x d;
 *   W   device m x m (eigenvectors, columns);  workspace >= prony_workspace_size(PRONY_WS_DIAG)
 *   dev_status: PRONY_ERR_NOT_CONVERGED (QR iteration cap) or PRONY_ERR_SINGULAR (W singular)
 */
int prony_diagonalize(int d, int m, const prony_c128* S, const prony_c128* mu, prony_c128* z, double* t, prony_c128* W,
                      void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream);

/*
 * prony_lanczos_svd — Algorithm 2: Lanczos bidiagonalization T V_i = U_i B_i,
 * T^H U_i = V_{i+1} B_{i,i+1}^T (eq_lanc_rec1/2) from a random p_1, with full
 * reorthogonalization of every u_i / v_i against all previous ones (two classical Gram-Schmidt passes,
 * P:170), stopping tests alpha <= tol_abs and beta <= tol_abs with tol_abs = tol * ||T||_F (P:172,
 * reading R24: ||T||_F bounds ||T||_2 and has a closed form in the samples), the early-stop check of
 * P:168 (a random vector orthogonalized against the basis that T^H resp. T does not annihilate
 * restarts the recurrence with alpha resp. beta = 0), and the SVD of the bidiagonal factor: alpha stop
 * -> B_{r,r+1} = Ubar_B [Sigma_B 0] Vbar_B^T, U = U_r Ubar_B, V = V_{r+1} Vbar_B(:,1:r);
 * beta stop -> B_r = U_B Sigma_B V_B^T, U = U_r U_B, V = V_r V_B. The rank r is the
 * dimension of the bidiagonal factor: no knowledge of m is needed.
 * SYNCHRONOUS (the stopping tests read alpha_i, beta_i on the host every step).
 *   grid        device L^d samples (as prony_project)
 *   max_rank    1 <= max_rank <= 255, max_rank <= N: the basis buffers; the iteration stops there
 *   tol         relative tolerance (>= 0): P:172 u ||T||_2 noise-free, the noise level for noisy data
 *   seed        seeds p_1 and the early-stop test vectors (counter-based generator, R14)
 *   ldo         columns of the outputs (1 <= ldo <= max_rank); the first min(r, ldo) are written
 *   U, V        device N x ldo (row-major): leading left / right singular vectors
 *   sigma       device ldo doubles, nonincreasing
 *   rank_out    host int32: r;  steps_out nullable host int32: Lanczos steps taken
 *   workspace   >= prony_workspace_size(PRONY_WS_LANCZOS, d, n, max_rank)
 * Returns PRONY_OK, PRONY_ERR_NOT_CONVERGED (max_rank steps without a stop: outputs hold the
 * rank-max_rank Lanczos approximation), PRONY_ERR_RANK (T = 0), or validation / CUDA errors.
 */
int prony_lanczos_svd(int d, int n, const prony_c128* grid, int max_rank, double tol, uint64_t seed, int ldo,
                      prony_c128* U, prony_c128* V, double* sigma, int32_t* rank_out, int32_t* steps_out,
                      void* workspace, size_t workspace_bytes, prony_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PRONY_H */
