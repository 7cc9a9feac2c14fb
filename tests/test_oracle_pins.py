"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics fix.

None of these tests re-types the oracle's formula: each compares the oracle with an
independent route (a printed value, a closed form, a factorization, an FFT convolution,
an invariant, brute force) chosen so that a dropped term, a wrong sign / conjugate /
index or a transposed operand in the oracle fails at least one of them.
"""
import json
import math
import os

import numpy as np

from f7_fft import fft_apply  # noqa: E402  (tests/f7_fft.py, shared with the full-size GPU check)
import pytest

import workload as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def cplx(v):
    return complex(v[0], v[1])


def exp_matrix(t, d, n):
    """B[k, j] = exp(-2 pi i <t_j, k>) for k in I_n (independent of the oracle)."""
    k = W.index_set(d, n).astype(np.float64)
    ph = k @ t.T
    return np.exp(-2j * np.pi * (ph - np.floor(ph)))


def small_problem(d, n, m, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    t = W.planted_nodes(d, m, n, rng)
    c = W.planted_coeffs(m, rng)
    grid = W.sample_grid(t, c, n, noise, seed)
    return t, c, grid, rng


# ------------------------------------------------------------------ golden, paper-printed
def test_paper_family_golden():
    gold = json.load(open(os.path.join(GOLD, "paper_family.json")))
    for case in gold["cases"]:
        t, c = W.paper_family(case["d"], case["m"])
        j = case["j"] - 1
        if "t" in case:
            np.testing.assert_allclose(t[j], case["t"], rtol=0, atol=1e-15)
        if "c" in case:
            assert c[j] == cplx(case["c"])
    for d, n, N in gold["index_set_sizes"]["cases"]:
        assert W.index_set(d, n).shape == (N, d)
        assert W.Config("x", d, n, 1, 0.0, 0).N == N


def test_signal_examples_golden():
    gold = json.load(open(os.path.join(GOLD, "analytic_examples.json")))
    for ex in gold["f"]:
        v = W.evaluate(np.array([ex["t"]]), np.array([cplx(ex["c"])]), np.array([ex["k"]]))[0]
        assert abs(v - cplx(ex["f"])) < 1e-15


def test_signal_periodic_and_bounded():
    rng = np.random.default_rng(3)
    t = rng.random((4, 2))
    c = W.planted_coeffs(4, rng)
    k = W.box_coords(2, 5)
    f0 = W.evaluate(t, c, k)
    f1 = W.evaluate(t + 1.0, c, k)          # 1-periodicity in t
    assert np.max(np.abs(f0 - f1)) < 1e-13
    assert np.max(np.abs(f0)) <= np.sum(np.abs(c)) + 1e-12   # |f| <= sum |c|


def test_noise_model_bound_and_determinism():
    t, c, _, _ = small_problem(2, 6, 3, 1)
    g0 = W.sample_grid(t, c, 6, 0.0, 5)
    g1 = W.sample_grid(t, c, 6, 1e-6, 5)
    g2 = W.sample_grid(t, c, 6, 1e-6, 5)
    assert np.array_equal(g1, g2)
    r = np.abs(g1 - g0) / np.abs(g0)
    assert r.max() < 6e-6 and r.max() > 1e-7            # Gaussian: |delta| ~ sigma, injected


# ------------------------------------------------------------------ O3: T, T_l
def test_T_d1_n1_golden(oracle_mod):
    gold = json.load(open(os.path.join(GOLD, "analytic_examples.json")))
    for ex in gold["T_d1_n1"]:
        grid = W.sample_grid(np.array([ex["t"]]), np.array([1.0 + 0j]), 1)
        T = oracle_mod.T_dense(grid, 1, 1, 0)
        T1 = oracle_mod.T_dense(grid, 1, 1, 1)
        np.testing.assert_allclose(T, np.array(ex["T"], dtype=complex), atol=1e-15)
        np.testing.assert_allclose(T1, np.array(ex["T1"], dtype=complex), atol=1e-15)


@pytest.mark.parametrize("d,n,m", [(2, 4, 3), (3, 2, 4), (1, 7, 2)])
def test_T_entries_direct_evaluation(oracle_mod, d, n, m):
    """T_l[k,h] equals f evaluated directly at the lattice point k-h+e_l."""
    t, c, grid, rng = small_problem(d, n, m, 11)
    idx = W.index_set(d, n)
    N = idx.shape[0]
    for _ in range(40):
        r, q = rng.integers(0, N, 2)
        for ell in range(0, d + 1):
            p = idx[r] - idx[q]
            if ell:
                p = p.copy(); p[ell - 1] += 1
            want = W.evaluate(t, c, p[None, :])[0]
            assert abs(oracle_mod.T_entry(grid, d, n, int(r), int(q), ell) - want) < 1e-13


@pytest.mark.parametrize("d,n,m", [(2, 6, 3), (3, 3, 4)])
def test_T_factorization_F1(oracle_mod, d, n, m):
    """F1: T = B diag(c) B^H and T_l = B diag(c z_l) B^H, B[k,j] = z_j^k (noise-free)."""
    t, c, grid, _ = small_problem(d, n, m, 21)
    B = exp_matrix(t, d, n)
    z = W.node_vectors(t)
    assert rel(oracle_mod.T_dense(grid, d, n, 0), (B * c) @ B.conj().T) < 1e-13
    for ell in range(1, d + 1):
        want = (B * (c * z[:, ell - 1])) @ B.conj().T
        assert rel(oracle_mod.T_dense(grid, d, n, ell), want) < 1e-13


# ------------------------------------------------------------------ O5: S_l
@pytest.mark.parametrize("d,n,m", [(2, 6, 3), (3, 3, 5), (2, 9, 7), (4, 2, 3)])
def test_S_closed_form_any_UV(oracle_mod, d, n, m):
    """F1 consequence: for ANY U, V, sigma, U* T_l V Sigma^-1 = (U* B) diag(c z_l) (B^H V) Sigma^-1."""
    t, c, grid, rng = small_problem(d, n, m, 31)
    N = (n + 1) ** d
    U = W.random_orthonormal(N, m, rng)
    V = W.random_orthonormal(N, m, rng)
    sigma = np.sort(rng.random(m) + 0.5)[::-1]
    B = exp_matrix(t, d, n)
    z = W.node_vectors(t)
    S = oracle_mod.project(grid, U, V, sigma, d, n)
    for ell in range(d):
        want = ((U.conj().T @ B) * (c * z[:, ell])) @ (B.conj().T @ V) / sigma[None, :]
        assert rel(S[ell], want) < 1e-12


def test_S_spectrum_F2(oracle_mod):
    """F2 / PAPER.md:34-37: with the SVD of T, eig(S_l) = {z_j(l)} (simultaneously diagonalizable)."""
    d, n, m = 2, 8, 4
    t, c, grid, _ = small_problem(d, n, m, 41)
    T = oracle_mod.T_dense(grid, d, n, 0)
    U, V, s, _ = oracle_mod.svd_reduced(T)
    assert len(s) == m                                   # rank(T) = m
    S = oracle_mod.project(grid, U, V, s, d, n)
    z = W.node_vectors(t)
    for ell in range(d):
        ev = np.linalg.eigvals(S[ell])
        # multiset match
        for zj in z[:, ell]:
            assert np.min(np.abs(ev - zj)) < 1e-10


def test_S_m1_equals_node(oracle_mod):
    """m = 1: T = c z^k conj(z^h), rank 1, S_l = z(l) for any rank-1 SVD."""
    d, n = 3, 3
    t = np.array([[0.11, 0.62, 0.37]])
    c = np.array([1.3 - 0.4j])
    grid = W.sample_grid(t, c, n)
    T = oracle_mod.T_dense(grid, d, n, 0)
    U, V, s, _ = oracle_mod.svd_reduced(T)
    assert len(s) == 1
    S = oracle_mod.project(grid, U, V, s, d, n)
    z = W.node_vectors(t)[0]
    np.testing.assert_allclose(S[:, 0, 0], z, atol=1e-13)


def test_S_d1_n1_golden(oracle_mod):
    gold = json.load(open(os.path.join(GOLD, "analytic_examples.json")))
    for ex in gold["T_d1_n1"]:
        grid = W.sample_grid(np.array([ex["t"]]), np.array([1.0 + 0j]), 1)
        U = V = np.array([[1.0], [1.0]], dtype=complex) / math.sqrt(2)
        if ex["t"][0] == 0.5:
            V = np.array([[1.0], [-1.0]], dtype=complex) / math.sqrt(2)
            U = V
        S = oracle_mod.project(grid, U, V, np.array([2.0]), 1, 1)
        assert abs(S[0, 0, 0] - ex["S1"]) < 1e-15


@pytest.mark.parametrize("d,n,m,noise", [(2, 20, 6, 1e-6), (3, 6, 5, 1e-3), (2, 31, 8, 0.0)])
def test_S_noisy_fft_convolution_F7(oracle_mod, d, n, m, noise):
    """Noisy samples have no closed form; F7 computes U* (T~_l V) Sigma^-1 by FFT convolution."""
    t, c, grid, rng = small_problem(d, n, m, 51, noise)
    N = (n + 1) ** d
    U = W.random_orthonormal(N, m, rng)
    V = W.random_orthonormal(N, m, rng)
    sigma = rng.random(m) + 0.5
    S = oracle_mod.project(grid, U, V, sigma, d, n)
    for ell in range(1, d + 1):
        want = U.conj().T @ fft_apply(grid, d, n, ell, V) / sigma[None, :]
        assert rel(S[ell - 1], want) < 1e-12


def test_project_units_linearity(oracle_mod):
    """Sharding: partial pencils over a partition of units sum to S."""
    d, n, m = 3, 3, 4
    t, c, grid, rng = small_problem(d, n, m, 61, 1e-6)
    N = (n + 1) ** d
    U = W.random_orthonormal(N, m, rng)
    V = W.random_orthonormal(N, m, rng)
    sigma = rng.random(m) + 0.5
    full = oracle_mod.project(grid, U, V, sigma, d, n)
    for order in (0, 1):
        cuts = [0, 7, 50, 51, d * N - 3, d * N]
        acc = sum(oracle_mod.project_units(grid, U, V, sigma, d, n, a, b, order) for a, b in zip(cuts, cuts[1:]))
        assert rel(acc, full) < 1e-13


def test_project_columns_matches_full(oracle_mod):
    d, n, m = 2, 7, 5
    t, c, grid, rng = small_problem(d, n, m, 71, 1e-6)
    N = (n + 1) ** d
    U = W.random_orthonormal(N, m, rng)
    V = W.random_orthonormal(N, m, rng)
    sigma = rng.random(m) + 0.5
    S = oracle_mod.project(grid, U, V, sigma, d, n)
    cols = [4, 0, 2]
    Sc = oracle_mod.project_columns(grid, U, V, sigma, d, n, 2, cols)
    assert rel(Sc, S[1][:, cols]) < 1e-13


# ------------------------------------------------------------------ O10/O11: A, G, b, c
def test_vandermonde_golden(oracle_mod):
    gold = json.load(open(os.path.join(GOLD, "analytic_examples.json")))
    for ex in gold["A_d1_n2"]:
        A = oracle_mod.vandermonde(np.array([[cplx(ex["z"])]]), 1, 2)
        np.testing.assert_allclose(A[0], np.array(ex["row"], dtype=complex), atol=0)


@pytest.mark.parametrize("d,n,m", [(2, 10, 3), (3, 5, 6), (4, 3, 4)])
def test_vandermonde_exp_and_reproduces_f(oracle_mod, d, n, m):
    """A[j,k] = exp(-2 pi i <t_j,k>) for unit nodes, and f = A^T c (eq_ls_probl)."""
    t, c, grid, _ = small_problem(d, n, m, 81)
    A = oracle_mod.vandermonde(W.node_vectors(t), d, n)
    assert rel(A, exp_matrix(t, d, n).T) < 1e-13
    f = oracle_mod.f_vector(grid, d, n)
    assert rel(A.T @ c, f) < 1e-13
    # f_vector reads the box at k in I_n: compare with direct evaluation
    assert rel(f, W.evaluate(t, c, W.index_set(d, n))) < 1e-14


@pytest.mark.parametrize("unit", [True, False])
def test_gram_separable_F4(oracle_mod, unit):
    """F4: G[i,j] = prod_l sum_{a=0..n} (z_i(l) conj z_j(l))^a (any complex nodes)."""
    d, n, m = 3, 6, 5
    rng = np.random.default_rng(91)
    z = W.node_vectors(rng.random((m, d)))
    if not unit:
        z = z * (1.0 + 0.05 * (rng.random((m, d)) - 0.5))
    A = oracle_mod.vandermonde(z, d, n)
    grid = W.sample_grid(rng.random((2, d)), np.array([1.0, 2.0j]), n)
    G, _ = oracle_mod.ls_products(A, grid, d, n)
    want = np.ones((m, m), complex)
    for ell in range(d):
        q = z[:, None, ell] * z[None, :, ell].conj()
        want *= sum(q ** a for a in range(n + 1))
    assert rel(G, want) < 1e-13
    assert rel(G, G.conj().T) < 1e-15


def test_b_and_c_noise_free_F3(oracle_mod):
    """F3: noise-free b = G conj(c); c = conj(G^-1 b) recovers the planted c; QR agrees."""
    d, n, m = 2, 12, 6
    t, c, grid, _ = small_problem(d, n, m, 101)
    A = oracle_mod.vandermonde(W.node_vectors(t), d, n)
    G, b = oracle_mod.ls_products(A, grid, d, n)
    assert rel(b, G @ c.conj()) < 1e-13
    c_ne = oracle_mod.cholesky_solve(G, b)
    assert rel(c_ne, c) < 1e-12
    c_qr, resid = oracle_mod.lstsq_qr(A, grid, d, n)
    assert rel(c_qr, c) < 1e-12 and resid < 1e-13


def test_ls_products_partition(oracle_mod):
    d, n, m = 2, 9, 4
    t, c, grid, _ = small_problem(d, n, m, 111, 1e-6)
    z = W.node_vectors(t)
    N = (n + 1) ** d
    A = oracle_mod.vandermonde(z, d, n)
    G, b = oracle_mod.ls_products(A, grid, d, n)
    Gs = np.zeros_like(G); bs = np.zeros_like(b)
    for a, e in [(0, 13), (13, 60), (60, N)]:
        Ap = oracle_mod.vandermonde(z, d, n, a, e)
        assert np.array_equal(Ap, A[:, a:e])
        g_, b_ = oracle_mod.ls_products(Ap, grid, d, n, a, e)
        Gs += g_; bs += b_
    assert rel(Gs, G) < 1e-14 and rel(bs, b) < 1e-14


def test_cholesky_rejects_non_hpd(oracle_mod):
    G = np.array([[1, 2], [2, 1]], dtype=complex)
    with pytest.raises(RuntimeError):
        oracle_mod.cholesky_solve(G, np.ones(2, complex))


def test_t_from_z_golden(oracle_mod):
    gold = json.load(open(os.path.join(GOLD, "analytic_examples.json")))
    for ex in gold["t_from_z"]:
        z = np.exp(2j * np.pi * ex["z_angle_turns"])
        assert abs(oracle_mod.t_from_z(np.array([z]))[0] - ex["t"]) < 1e-15
    t = np.random.default_rng(1).random((50, 3))
    d = np.abs(oracle_mod.t_from_z(W.node_vectors(t)) - t)
    assert np.max(np.minimum(d, 1 - d)) < 1e-15


# ------------------------------------------------------------------ input synthesis pins
def test_planted_svd_is_svd_of_T(oracle_mod):
    d, n, m = 2, 7, 4
    t, c, grid, _ = small_problem(d, n, m, 121)
    U, V, s = W.planted_svd(t, c, n)
    T = oracle_mod.T_dense(grid, d, n, 0)
    assert rel(U @ np.diag(s) @ V.conj().T, T) < 1e-13
    np.testing.assert_allclose(U.conj().T @ U, np.eye(m), atol=1e-14)
    np.testing.assert_allclose(V.conj().T @ V, np.eye(m), atol=1e-14)
    _, _, s_or, _ = oracle_mod.svd_reduced(T)
    np.testing.assert_allclose(s, s_or, rtol=1e-12)


# ------------------------------------------------------------------ Algorithm 1 end to end
def test_algorithm1_noise_free_recovery(oracle_mod):
    d, n, m = 2, 12, 5
    t, c, grid, _ = small_problem(d, n, m, 131)
    out = oracle_mod.algorithm1(grid, d, n, seed=3)
    assert out["rank"] == m
    perm = oracle_mod.match_nodes(out["t"], t)
    terr = W.torus_dist_inf(out["t"][perm], t).max()
    assert terr < 1e-12
    assert rel(out["c"][perm], c) < 1e-11
    assert rel(out["c_ne"][perm], c) < 1e-10
    assert out["resid"] < 1e-13
    assert np.max(out["offdiag"]) < 1e-10


def test_algorithm1_paper_family_ranks(oracle_mod):
    """at d=2, n=20 the detected rank is below m for m = 15, 20 (sample too small);
    m = 5, 10 are recovered with full rank."""
    n, d = 20, 2
    ranks = {}
    for m in (5, 10, 15, 20):
        t, c = W.paper_family(d, m)
        grid = W.sample_grid(t, c, n)
        T = oracle_mod.T_dense(grid, d, n, 0)
        _, _, s, _ = oracle_mod.svd_reduced(T)
        ranks[m] = len(s)
    assert ranks[5] == 5 and ranks[10] == 10
    assert ranks[15] < 15 and ranks[20] < 20


def test_algorithm1_error_linear_in_eps_desk(oracle_mod):
    """PAPER.md:647 / 571: forward errors proportional to eps (Jacobi route, desk scale d=2, n=20, m=5 of the
    paper family, rank by tol = eps). The table itself is pinned at its own configuration
    d=3, n=20, m=5 in test_oracle_alg1_pins.py."""
    d, n, m = 2, 20, 5
    t, c = W.paper_family(d, m)
    errs = {}
    for eps in (0.0, 1e-9, 1e-6):
        grid = W.sample_grid(t, c, n, eps, 7, noise_model="disk")
        tol = eps if eps > 0 else None
        out = oracle_mod.algorithm1(grid, d, n, tol=tol, seed=5)
        assert out["rank"] == m
        perm = oracle_mod.match_nodes(out["t"], t)
        errs[eps] = (out["resid"], W.torus_dist_inf(out["t"][perm], t).max(), rel(out["c"][perm], c))
    assert errs[0.0][1] < 1e-13 and errs[0.0][2] < 1e-11
    for i in range(3):    # linear in eps: one pattern scaled by eps (R5b) gives a ratio of 1e3
        r = errs[1e-6][i] / errs[1e-9][i]
        assert 900 < r < 1100
