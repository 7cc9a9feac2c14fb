"""CPU oracle of the multivariate matrix-pencil Prony method (arXiv 2012.11430).

TEST INFRASTRUCTURE ONLY — only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product path
(paper_2012_11430_b200/) never imports it and shares no code with it.

Layers:
  * liboracle.so (prony_oracle.c): plain C loops for everything O(N^2) or O(Nm):
    T/T_l entries, the pencil S_l = U* T_l V Sigma^-1, the Vandermonde A, the LS
    products G = A conj(A)^T and b = A conj(f), and c = conj(G^-1 b) by Cholesky.
  * this module: ctypes marshalling, plus the m x m / desk-scale steps of Algorithm 1
     that use numpy LAPACK routines as library primitives:
    reduced SVD (O4, np.linalg.svd), rank rule, random mu and C_mu (O6), eig (O7),
    simultaneous diagonalization (O8), t from z (O9), LS by Householder QR (O11).

Parity status per function (DESIGN.md §4 lists the pins):
  project / project_columns / vandermonde / ls_products / cholesky_solve / T_dense:
      pinned (tests/test_oracle_pins.py)
  svd_reduced, eig, diagonalize, t_from_z, lstsq_qr, algorithm1: pinned (same file)
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
_SRC = os.path.join(_HERE, "prony_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-fcx-limited-range", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (called by __graft_entry__.build() and tests)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB_PATH, _SRC, "-lm"])
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
        for f in ("oracle_T_entry", "oracle_build_T", "oracle_project_rows", "oracle_project_columns",
                  "oracle_vandermonde", "oracle_ls_products", "oracle_cholesky_solve",
                  "oracle_num_threads", "oracle_abi_version"):
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


def lstsq_qr(A, f):
    """argmin_c ||A^T c - f||_2 by Householder QR of A^T (numpy/LAPACK)."""
    Q, R = np.linalg.qr(A.T)
    return np.linalg.solve(R, Q.conj().T @ f)


def t_from_z(z):
    """t = (-arg z / 2 pi) mod 1 (reading R4 corrects the sign of P:495)."""
    t = (-np.angle(z) / (2 * np.pi)) % 1.0
    return np.where(t >= 1.0, 0.0, t)


# ---------------------------------------------------------------- O4, O6-O9 (desk scale)
def svd_reduced(T, tol=None, rank=None):
    """Reduced SVD T = U Sigma V* (eq_T_svd) via LAPACK; rank = first i with
    sigma_i < tol * sigma_1 (PAPER.md:581 uses tol = N eps_M, PAPER.md:627 tol = eps)."""
    Uf, s, Vh = np.linalg.svd(T)
    if rank is None:
        if tol is None:
            tol = T.shape[0] * np.finfo(np.float64).eps
        rank = int(np.sum(s >= tol * s[0]))
    return np.ascontiguousarray(Uf[:, :rank]), np.ascontiguousarray(Vh[:rank].conj().T), s[:rank].copy(), s


def random_mu(d, seed):
    """mu ~ complex Gaussian, normalized to ||mu||_2 = 1 (reading R7)."""
    rng = np.random.default_rng([seed, 11])
    mu = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    return mu / np.linalg.norm(mu)


def diagonalize(S, mu):
    """C_mu = sum_l mu_l S_l; W from eig(C_mu);
    z_tau(j)(l) = (W^-1 S_l W)[j, j] via LU solves. Returns (z (m,d), W, offdiag)."""
    d, m, _ = S.shape
    C = np.tensordot(mu, S, axes=1)
    _, W = np.linalg.eig(C)
    z = np.empty((m, d), np.complex128)
    off = np.empty(d)
    for l in range(d):
        D = np.linalg.solve(W, S[l] @ W)
        z[:, l] = np.diag(D)
        off[l] = np.linalg.norm(D - np.diag(np.diag(D))) / np.linalg.norm(D)
    return z, W, off


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


def algorithm1(grid, d, n, tol=None, seed=0, rank=None):
    """Algorithm 1 end to end at desk scale (N up to ~2000):
    T (O3) -> reduced SVD (O4) -> S_l (O5) -> mu, C_mu, W (O6-O7) -> z (O8) -> t (O9)
    -> A (O10) -> c (O11, Cholesky on the normal equations and Householder QR)."""
    T = T_dense(grid, d, n, 0)
    U, V, s, s_all = svd_reduced(T, tol=tol, rank=rank)
    S = project(grid, U, V, s, d, n)
    mu = random_mu(d, seed)
    z, W, off = diagonalize(S, mu)
    t = t_from_z(z)
    A = vandermonde(z, d, n)
    G, b = ls_products(A, grid, d, n)
    c_ne = cholesky_solve(G, b)
    f = f_vector(grid, d, n)
    c_qr = lstsq_qr(A, f)
    resid = np.linalg.norm(A.T @ c_qr - f) / np.linalg.norm(f)
    return dict(U=U, V=V, sigma=s, sigma_all=s_all, rank=len(s), S=S, mu=mu, W=W, offdiag=off, z=z, t=t,
                A=A, G=G, b=b, c=c_qr, c_ne=c_ne, resid=resid)
