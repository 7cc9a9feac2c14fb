"""CPU oracle of the multivariate matrix-pencil Prony method (arXiv 2012.11430).

TEST INFRASTRUCTURE ONLY — only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product path
(paper_2012_11430_b200/) never imports it and shares no code with it.

Layers:
  * liboracle.so (prony_oracle.c): plain C loops for everything O(N^2) or O(Nm):
    T/T_l entries, the pencil S_l = U* T_l V Sigma^-1, the Vandermonde A, the LS
    products G = A conj(A)^T and b = A conj(f), and c = conj(G^-1 b) by Cholesky.
  * alg1_oracle.c: plain C loops (no BLAS / LAPACK) for the rest of Algorithm 1:
    Householder QR (with column pivoting), one-sided Jacobi SVD (O4 at desk scale), the Toeplitz apply
    and Algorithm 3 block power (O4 at large N), Hessenberg + shifted-QR eig (O7), LU diagonalization
    (O8), t from z (O9), least squares by Householder QR (O11).
  * this module: ctypes marshalling and the rank rule (a comparison loop). No np.linalg call on any
    Algorithm-1 step; the random draws (mu, the Gaussian starting blocks of Alg. 3) come from the
    input generator workload.py.

Parity status per function (DESIGN.md §4 lists the pins):
  project / project_columns / vandermonde / ls_products / cholesky_solve / T_dense:
      pinned (tests/test_oracle_pins.py)
  householder_qr, jacobi_svd, svd_reduced, toeplitz_apply, T_fro, block_power_svd, eig, lu_solve,
      diagonalize, t_from_z, lstsq_qr, algorithm1: pinned (same file; LAPACK / closed forms / SPEC
      examples / the paper's table)
  project_units / _shared_runs (unit orders 0, 1, 2): pinned (unit-range linearity in
      test_oracle_pins.py; order 2 covers every row of every T_l exactly once, test_sharding.py)
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, f) for f in ("prony_oracle.c", "alg1_oracle.c")]
_HDRS = [os.path.join(_HERE, "oracle_common.h")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-fcx-limited-range", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (called by __graft_entry__.build() and tests)."""
    stale = not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(f)
                                                  for f in _SRCS + _HDRS)
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64, dp = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        L.oracle_T_entry.argtypes = [i32, i32, vp, i64, i64, i32, vp]
        L.oracle_build_T.argtypes = [i32, i32, i32, vp, vp]
        L.oracle_project_rows.argtypes = [i32, i32, i32, vp, vp, vp, dp, i32, i64, i64, vp]
        L.oracle_project_columns.argtypes = [i32, i32, i32, vp, vp, vp, dp, i32, i32, vp, vp]
        L.oracle_vandermonde.argtypes = [i32, i32, i32, vp, i64, i64, vp]
        L.oracle_ls_products.argtypes = [i32, i32, i32, vp, vp, i64, i64, vp, vp]
        L.oracle_cholesky_solve.argtypes = [i32, vp, vp, vp]
        L.oracle_set_num_threads.argtypes = [i32]
        L.oracle_householder_qr.argtypes = [i64, i32, vp, i64, i32, vp, i64, vp, i32, vp]
        L.oracle_jacobi_svd.argtypes = [i64, i32, vp, i64, vp, vp, i64, vp, i32, i32, vp]
        L.oracle_toeplitz_apply.argtypes = [i32, i32, vp, i32, i32, i32, vp, vp]
        L.oracle_T_fro.argtypes = [i32, i32, vp]
        L.oracle_T_fro.restype = ctypes.c_double
        L.oracle_block_power_svd.argtypes = [i32, i32, vp, i32, vp, vp, ctypes.c_double, i32, vp, vp, vp, vp, vp, vp]
        L.oracle_eig.argtypes = [i32, vp, vp, vp, vp]
        L.oracle_lu_solve.argtypes = [i32, vp, i32, vp, vp]
        L.oracle_diagonalize.argtypes = [i32, i32, vp, vp, vp, vp, vp]
        L.oracle_t_from_z.argtypes = [i64, vp, vp]
        L.oracle_lstsq_qr.argtypes = [i32, i32, i32, vp, vp, vp, vp]
        for f in ("oracle_T_entry", "oracle_build_T", "oracle_project_rows", "oracle_project_columns",
                  "oracle_vandermonde", "oracle_ls_products", "oracle_cholesky_solve",
                  "oracle_num_threads", "oracle_abi_version", "oracle_householder_qr", "oracle_jacobi_svd",
                  "oracle_toeplitz_apply", "oracle_block_power_svd", "oracle_eig", "oracle_lu_solve",
                  "oracle_diagonalize", "oracle_t_from_z", "oracle_lstsq_qr"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(t: int) -> None:
    lib().oracle_set_num_threads(int(t))


def _c(a, dtype=np.complex128):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with status {rc}")


def N_of(d, n):
    return (n + 1) ** d


# ---------------------------------------------------------------- O3: T, T_l
def T_entry(grid, d, n, row, col, ell):
    """T_l[row, col] (ell = 1..d) or T[row, col] (ell = 0) — PAPER.md:21."""
    g = _c(grid)
    out = np.zeros(1, np.complex128)
    _check(lib().oracle_T_entry(d, n, _p(g), row, col, ell, _p(out)), "T_entry")
    return out[0]


def T_dense(grid, d, n, ell):
    """Dense N x N T (ell=0) or T_ell (ell=1..d) — PAPER.md:21 (desk scale)."""
    N = N_of(d, n)
    g = _c(grid)
    out = np.empty((N, N), np.complex128)
    _check(lib().oracle_build_T(d, n, ell, _p(g), _p(out)), "build_T")
    return out


# ---------------------------------------------------------------- O5: S_l
def project_rows(grid, U, V, sigma, d, n, ell, k_begin=0, k_end=None):
    """Partial S_l over rows [k_begin, k_end) of T_l; full range = S_l."""
    N = N_of(d, n)
    m = U.shape[1]
    if k_end is None:
        k_end = N
    g, U_, V_ = _c(grid), _c(U), _c(V)
    s = _c(sigma, np.float64)
    S = np.zeros((m, m), np.complex128)
    _check(lib().oracle_project_rows(d, n, m, _p(g), _p(U_), _p(V_), _p(s), ell, k_begin, k_end, _p(S)),
           "project_rows")
    return S


def project(grid, U, V, sigma, d, n):
    """S_1..S_d, shape (d, m, m) — eq_generateSl."""
    return np.stack([project_rows(grid, U, V, sigma, d, n, ell) for ell in range(1, d + 1)])


def _shared_runs(d, n, ell, unit_begin, unit_end):
    """Unit order 2 (SHARED): unit u is the point k' of E = {0..n+1}^d with index u (lexicographic,
    last coordinate fastest); it stands for row k = k' - e_l of T_l whenever that k lies in I_n
    (F8). Returns the rows k of T_l covered by [unit_begin, unit_end) as (kb, ke) runs."""
    runs = []
    for u in range(unit_begin, unit_end):
        c = []
        r = u
        for _ in range(d):
            c.append(r % (n + 2))
            r //= n + 2
        c = c[::-1]                      # c[0] is the slowest coordinate (e_1 direction)
        c[ell - 1] -= 1
        if min(c) < 0 or max(c) > n:
            continue
        k = 0
        for ci in c:
            k = k * (n + 1) + ci
        if runs and runs[-1][1] == k:
            runs[-1][1] = k + 1
        else:
            runs.append([k, k + 1])
    return runs


def project_units(grid, U, V, sigma, d, n, unit_begin, unit_end, unit_order=0):
    """Partial pencil over a unit sub-range (DESIGN.md §6 sharding): unit_order 0: u = (l-1) N + k,
    1: u = k d + (l-1) (units in [0, dN)); 2: u = a point of {0..n+1}^d standing for row k' - e_l of
    every T_l (units in [0, (n+2)^d)). Each row is computed directly from T_l. Returns (d, m, m)."""
    N = N_of(d, n)
    m = U.shape[1]
    out = np.zeros((d, m, m), np.complex128)
    if unit_order == 2:
        for ell in range(1, d + 1):
            for kb, ke in _shared_runs(d, n, ell, unit_begin, unit_end):
                out[ell - 1] += project_rows(grid, U, V, sigma, d, n, ell, kb, ke)
        return out
    for ell in range(1, d + 1):
        if unit_order == 0:
            kb = min(max(unit_begin - (ell - 1) * N, 0), N)
            ke = min(max(unit_end - (ell - 1) * N, 0), N)
        else:
            kb = min(max(-(-(unit_begin - (ell - 1)) // d), 0), N)
            ke = min(max(-(-(unit_end - (ell - 1)) // d), 0), N)
        if ke > kb:
            out[ell - 1] = project_rows(grid, U, V, sigma, d, n, ell, kb, ke)
    return out


def project_columns(grid, U, V, sigma, d, n, ell, cols):
    """Columns `cols` of S_l (all m rows), one column at a time — full-size sampled parity."""
    m = U.shape[1]
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    g, U_, V_ = _c(grid), _c(U), _c(V)
    s = _c(sigma, np.float64)
    out = np.zeros((m, len(cols)), np.complex128)
    _check(lib().oracle_project_columns(d, n, m, _p(g), _p(U_), _p(V_), _p(s), ell, len(cols), _p(cols),
                                        _p(out)), "project_columns")
    return out


# ---------------------------------------------------------------- O10/O11: A, G, b, c
def vandermonde(z, d, n, col_begin=0, col_end=None):
    """A = [z_j^k], m x (col_end-col_begin) — PAPER.md:33, 39."""
    z_ = _c(z)
    m = z_.shape[0]
    if col_end is None:
        col_end = N_of(d, n)
    A = np.empty((m, col_end - col_begin), np.complex128)
    _check(lib().oracle_vandermonde(d, n, m, _p(z_), col_begin, col_end, _p(A)), "vandermonde")
    return A


def ls_products(A, grid, d, n, col_begin=0, col_end=None):
    """G = A conj(A)^T, b = A conj(f) over columns [col_begin, col_end) (R10)."""
    A_ = _c(A)
    m = A_.shape[0]
    if col_end is None:
        col_end = col_begin + A_.shape[1]
    g = _c(grid)
    G = np.zeros((m, m), np.complex128)
    b = np.zeros(m, np.complex128)
    _check(lib().oracle_ls_products(d, n, m, _p(A_), _p(g), col_begin, col_end, _p(G), _p(b)), "ls_products")
    return G, b


def cholesky_solve(G, b):
    """c = conj(G^-1 b) (normal equations G conj(c) = b of argmin ||A^T c - f||, R10)."""
    G_, b_ = _c(G), _c(b)
    m = b_.shape[0]
    c = np.zeros(m, np.complex128)
    _check(lib().oracle_cholesky_solve(m, _p(G_), _p(b_), _p(c)), "cholesky_solve")
    return c


def f_vector(grid, d, n):
    """f = [f(k)]_{k in I_n} read from the box."""
    L = 2 * n + 2
    N = N_of(d, n)
    idx = np.zeros(N, np.int64)
    r = np.arange(N, dtype=np.int64)
    for i in range(d - 1, -1, -1):
        digit = r % (n + 1)
        r = r // (n + 1)
        idx += (digit + n) * (L ** (d - 1 - i))
    return np.asarray(grid)[idx]


def lstsq_qr(A, grid, d, n):
    """argmin_c ||A^T c - f||_2 (Algorithm 1 line 7) by Householder QR of A^T (plain C,
    alg1_oracle.c), f = grid on I_n. Returns (c, relative residual ||A^T c - f|| / ||f||)."""
    A_ = _c(A)
    m = A_.shape[0]
    g = _c(grid)
    c = np.zeros(m, np.complex128)
    r = ctypes.c_double(0.0)
    _check(lib().oracle_lstsq_qr(d, n, m, _p(A_), _p(g), _p(c), ctypes.byref(r)), "lstsq_qr")
    return c, r.value


def t_from_z(z):
    """t = (-arg z / 2 pi) mod 1 (reading R4 corrects the sign of P:495)."""
    z_ = _c(z)
    t = np.empty(z_.shape, np.float64)
    _check(lib().oracle_t_from_z(z_.size, _p(z_), _p(t)), "t_from_z")
    return t


# ---------------------------------------------------------------- O4, O6-O9: plain C (alg1_oracle.c)
def householder_qr(A, pivot=False):
    """Reduced QR (optionally column-pivoted) by Householder reflectors: A[:, perm] = Q R."""
    A_ = _c(A)
    M, C = A_.shape
    K = min(M, C)
    Q = np.empty((M, K), np.complex128)
    R = np.empty((K, C), np.complex128)
    perm = np.empty(C, np.int32)
    _check(lib().oracle_householder_qr(M, C, _p(A_), C, int(bool(pivot)), _p(Q), K, _p(R), C, _p(perm)),
           "householder_qr")
    return Q, R, perm.astype(np.int64)


def jacobi_svd(A, max_sweeps=60):
    """One-sided Jacobi SVD A = U diag(s) V^H (s nonincreasing, V C x C unitary). Returns (U, s, V, sweeps)."""
    A_ = _c(A)
    M, C = A_.shape
    s = np.empty(C, np.float64)
    U = np.empty((M, C), np.complex128)
    V = np.empty((C, C), np.complex128)
    sw = ctypes.c_int(0)
    _check(lib().oracle_jacobi_svd(M, C, _p(A_), C, _p(s), _p(U), C, _p(V), C, max_sweeps, ctypes.byref(sw)),
           "jacobi_svd")
    return U, s, V, sw.value


def toeplitz_apply(grid, d, n, X, ell=0, adjoint=False):
    """T_l X (or T_l^H X) with T_l generated entry by entry from the samples."""
    X_ = _c(X)
    if X_.ndim == 1:
        X_ = X_[:, None]
    g = _c(grid)
    Y = np.empty_like(X_)
    _check(lib().oracle_toeplitz_apply(d, n, _p(g), ell, int(bool(adjoint)), X_.shape[1], _p(X_), _p(Y)),
           "toeplitz_apply")
    return Y


def T_fro(grid, d, n):
    """||T||_F from all N^2 entries f(k-h)."""
    return lib().oracle_T_fro(d, n, _p(_c(grid)))


def rank_rule(s, tol):
    """Numerical rank: the first i with sigma_i < tol sigma_1 gives rank i (PAPER.md:581 with
    tol = N eps_M; PAPER.md:627 with tol = eps)."""
    r = 0
    while r < len(s) and s[r] >= tol * s[0]:
        r += 1
    return r


def svd_reduced(T, tol=None, rank=None):
    """Reduced SVD T = U Sigma V* (eq_T_svd) of a dense desk-scale T by the one-sided
    Jacobi SVD (plain C); rank by rank_rule (tol defaults to N eps_M).
    Returns (U (N x r), V (N x r), sigma (r,), all singular values)."""
    U, s, V, _ = jacobi_svd(T)
    if rank is None:
        if tol is None:
            tol = T.shape[0] * np.finfo(np.float64).eps
        rank = rank_rule(s, tol)
    return np.ascontiguousarray(U[:, :rank]), np.ascontiguousarray(V[:, :rank]), s[:rank].copy(), s


def block_power_svd(grid, d, n, r0, G_U, G_V, tol, max_iter=100):
    """Algorithm 3 on T generated from the samples, plain C. G_U, G_V: the seeded
    complex Gaussian N x r0 draws (workload.gaussian_block); U_0, V_0 are their Householder Q factors
    (reading R14). Returns dict(U, V (N x rank), sigma (rank,), rank, iters, resid, status)."""
    N = (n + 1) ** d
    U0, _, _ = householder_qr(G_U)
    V0, _, _ = householder_qr(G_V)
    U0, V0 = _c(U0), _c(V0)
    U = np.zeros((N, r0), np.complex128)
    V = np.zeros((N, r0), np.complex128)
    s = np.zeros(r0, np.float64)
    rank, iters, resid = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_double(0.0)
    rc = lib().oracle_block_power_svd(d, n, _p(_c(grid)), r0, _p(U0), _p(V0), float(tol), int(max_iter), _p(U),
                                      _p(V), _p(s), ctypes.byref(rank), ctypes.byref(iters), ctypes.byref(resid))
    if rc not in (0, 5):
        _check(rc, "block_power_svd")
    r = rank.value
    return dict(U=np.ascontiguousarray(U[:, :r]), V=np.ascontiguousarray(V[:, :r]), sigma=s[:r].copy(), rank=r,
                iters=iters.value, resid=resid.value, status=rc)


def eig(C):
    """Eigenvalues and unit eigenvectors of a general complex matrix: Hessenberg + shifted QR + back
    substitution (reading R23). Returns (lam, W) with C W = W diag(lam)."""
    C_ = _c(C)
    m = C_.shape[0]
    lam = np.empty(m, np.complex128)
    W = np.empty((m, m), np.complex128)
    it = ctypes.c_int(0)
    _check(lib().oracle_eig(m, _p(C_), _p(lam), _p(W), ctypes.byref(it)), "eig")
    return lam, W


def lu_solve(A, B):
    """X = A^-1 B by LU with partial pivoting."""
    A_, B_ = _c(A), _c(B)
    one = B_.ndim == 1
    if one:
        B_ = B_[:, None].copy()
    X = np.empty_like(B_)
    _check(lib().oracle_lu_solve(A_.shape[0], _p(A_), B_.shape[1], _p(B_), _p(X)), "lu_solve")
    return X[:, 0] if one else X


def diagonalize(S, mu):
    """C_mu = sum_l mu_l S_l; W from eig(C_mu);
    z_tau(j)(l) = (W^-1 S_l W)[j, j] via LU solves. Returns (z (m,d), W, offdiag)."""
    S_ = _c(S)
    d, m, _ = S_.shape
    mu_ = _c(mu)
    z = np.empty((m, d), np.complex128)
    W = np.empty((m, m), np.complex128)
    off = np.empty(d, np.float64)
    _check(lib().oracle_diagonalize(d, m, _p(S_), _p(mu_), _p(z), _p(W), _p(off)), "diagonalize")
    return z, W, off


def random_mu(d, seed):
    """The random mu of PAPER.md:56 (reading R7), drawn by the input generator (workload.random_mu)."""
    import workload
    return workload.random_mu(d, seed)


def match_nodes(t_rec, t_true):
    """Optimal assignment of recovered to planted t on the torus inf-norm (reading R13).
    Returns perm with t_rec[perm[j]] matched to t_true[j]."""
    from scipy.optimize import linear_sum_assignment
    diff = np.abs(t_true[:, None, :] - t_rec[None, :, :]) % 1.0
    cost = np.max(np.minimum(diff, 1.0 - diff), axis=2)
    r, c = linear_sum_assignment(cost)
    perm = np.empty(len(t_true), np.int64)
    perm[r] = c
    return perm


def algorithm1(grid, d, n, tol=None, seed=0, rank=None, svd="jacobi", m_hint=None, mu=None, max_iter=100):
    """Algorithm 1 end to end, every step plain C:
    line 1-2  T and its reduced SVD: svd="jacobi" -> dense T (O3) + one-sided Jacobi SVD (desk scale,
              N up to ~500); svd="power" -> Algorithm 3 with r0 = 2 m_hint on the
              generated T (any N the CPU affords)
    line 3    S_l = U* T_l V Sigma^-1 (O5)
    line 4-5  mu (input draw, reading R7), C_mu, W by Hessenberg-QR eig, z = diag(W^-1 S_l W) (O6-O8)
    line 6    t = (-arg z / 2 pi) mod 1 (O9)
    line 7    A (O10); c by Householder QR of A^T and c_ne = conj(G^-1 b) by Cholesky (O11)
    tol: rank tolerance (N eps_M by default; eps for noisy data)."""
    import workload
    N = (n + 1) ** d
    if tol is None:
        tol = N * np.finfo(np.float64).eps
    extra = {}
    if svd == "jacobi":
        T = T_dense(grid, d, n, 0)
        U, V, s, s_all = svd_reduced(T, tol=tol, rank=rank)
        extra["sigma_all"] = s_all
    elif svd == "power":
        r0 = min(2 * m_hint, N)
        G_U, G_V = workload.gaussian_block(N, r0, seed, 0), workload.gaussian_block(N, r0, seed, 1)
        bp = block_power_svd(grid, d, n, r0, G_U, G_V, tol, max_iter=max_iter)
        U, V, s = bp["U"], bp["V"], bp["sigma"]
        extra.update(iters=bp["iters"], power_resid=bp["resid"], power_status=bp["status"])
    else:
        raise ValueError(svd)
    S = project(grid, U, V, s, d, n)
    if mu is None:
        mu = random_mu(d, seed)
    z, W, off = diagonalize(S, mu)
    t = t_from_z(z)
    A = vandermonde(z, d, n)
    G, b = ls_products(A, grid, d, n)
    c_ne = cholesky_solve(G, b)
    c_qr, resid = lstsq_qr(A, grid, d, n)
    return dict(U=U, V=V, sigma=s, rank=len(s), S=S, mu=mu, W=W, offdiag=off, z=z, t=t,
                A=A, G=G, b=b, c=c_qr, c_ne=c_ne, resid=resid, **extra)
