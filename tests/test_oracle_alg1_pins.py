"""Pins of the plain-C Algorithm-1 oracle (oracle/alg1_oracle.c): Householder QR, one-sided Jacobi SVD,
the generated Toeplitz apply, Algorithm 3 block power, Hessenberg-QR eig, LU diagonalization and the QR
least-squares solve.

Each is compared with something other than itself: an independent library routine (numpy/LAPACK — used
here ONLY as a pin, never inside the oracle), a closed form, a worked example (tests/golden/
linalg_examples.json, with citations), an invariant, or the paper's printed accuracy table
(tests/golden/accuracy_table.json) at the paper's own configuration d=3, n=20, m=5.
"""
import json
import math
import os

import numpy as np
import pytest

import workload as W
from f7_fft import fft_apply

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS = np.finfo(np.float64).eps


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def cmat(rows):
    return np.array([[complex(x[0], x[1]) for x in r] for r in rows])


def rand_c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def projector(X):
    return X @ X.conj().T


# ------------------------------------------------------------------ Householder QR
@pytest.mark.parametrize("M,C,pivot", [(30, 7, False), (30, 7, True), (5, 9, False), (64, 64, True)])
def test_householder_qr_vs_lapack(oracle_mod, M, C, pivot):
    rng = np.random.default_rng(M * 100 + C)
    A = rand_c(rng, M, C)
    Q, R, perm = oracle_mod.householder_qr(A, pivot)
    K = min(M, C)
    assert Q.shape == (M, K) and R.shape == (K, C)
    assert rel(Q @ R, A[:, perm]) < 1e-14
    assert np.abs(Q.conj().T @ Q - np.eye(K)).max() < 1e-14
    assert np.abs(np.tril(R, -1)).max() == 0.0
    _, R_l = np.linalg.qr(A[:, perm])                     # LAPACK on the same column order
    np.testing.assert_allclose(np.abs(np.diag(R)), np.abs(np.diag(R_l)), rtol=1e-12)
    if pivot:
        dg = np.abs(np.diag(R))
        assert np.all(dg[:-1] >= dg[1:] * (1 - 1e-12))    # pivoting makes |R_ii| nonincreasing
        assert sorted(perm.tolist()) == list(range(C))
    else:
        assert perm.tolist() == list(range(C))


def test_pivoted_qr_spec_examples(oracle_mod):
    gold = json.load(open(os.path.join(GOLD, "linalg_examples.json")))["pivoted_qr"]
    I = np.eye(gold[0]["n"], dtype=complex)
    Q, R, perm = oracle_mod.householder_qr(I, True)
    assert perm.tolist() == list(range(gold[0]["n"]))
    np.testing.assert_allclose(np.abs(R), np.eye(gold[0]["n"]), atol=1e-15)
    np.testing.assert_allclose(Q @ R, I, atol=1e-15)
    rng = np.random.default_rng(5)
    a = rand_c(rng, gold[1]["rows"], 1)
    A = np.hstack([a, a])
    _, R, _ = oracle_mod.householder_qr(A, True)
    assert abs(R[1, 1]) <= gold[1]["rows"] * EPS * np.linalg.norm(A)
    g = gold[2]
    A = rand_c(rng, g["rows"], g["rank"]) @ rand_c(rng, g["rank"], g["cols"])
    _, R, _ = oracle_mod.householder_qr(A, True)
    tails = [np.linalg.norm(R[i:, i:]) for i in range(g["cols"])]
    cut = next(i for i, x in enumerate(tails) if x <= g["tol"] * np.linalg.norm(R))
    assert cut == g["rank"]


# ------------------------------------------------------------------ one-sided Jacobi SVD
@pytest.mark.parametrize("M,C", [(40, 9), (9, 9), (6, 11), (120, 30)])
def test_jacobi_svd_vs_lapack(oracle_mod, M, C):
    rng = np.random.default_rng(M + 7 * C)
    A = rand_c(rng, M, C)
    U, s, V, sweeps = oracle_mod.jacobi_svd(A)
    assert sweeps > 0
    s_l = np.linalg.svd(A, compute_uv=False)
    k = min(M, C)
    np.testing.assert_allclose(s[:k], s_l, rtol=1e-12, atol=1e-13 * s_l[0])
    assert np.all(np.abs(s[k:]) < 1e-12 * s_l[0])
    assert rel((U * s) @ V.conj().T, A) < 1e-13
    assert np.abs(V.conj().T @ V - np.eye(C)).max() < 1e-13
    Uk = U[:, :k]
    assert np.abs(Uk.conj().T @ Uk - np.eye(k)).max() < 1e-12


def test_jacobi_svd_spec_examples(oracle_mod):
    for ex in json.load(open(os.path.join(GOLD, "linalg_examples.json")))["svd"]:
        A = np.array(ex["A"], dtype=complex)
        U, V, s, s_all = oracle_mod.svd_reduced(A, tol=ex["tol"])
        np.testing.assert_allclose(s_all, ex["sigma"], rtol=1e-14, atol=1e-15)
        assert len(s) == ex["rank"], ex["cite"]


def test_jacobi_svd_low_rank_subspaces(oracle_mod):
    """rank-r product: r nonzero singular values; the left/right singular subspaces are the factors' ranges."""
    rng = np.random.default_rng(9)
    X, Y = rand_c(rng, 50, 4), rand_c(rng, 4, 35)
    A = X @ Y
    U, V, s, s_all = oracle_mod.svd_reduced(A, tol=1e-12)
    assert len(s) == 4
    Qx, _ = np.linalg.qr(X)
    Qy, _ = np.linalg.qr(Y.conj().T)
    assert np.abs(projector(U) - projector(Qx)).max() < 1e-12
    assert np.abs(projector(V) - projector(Qy)).max() < 1e-12


# ------------------------------------------------------------------ Toeplitz apply, ||T||_F
@pytest.mark.parametrize("d,n,noise", [(2, 6, 0.0), (3, 3, 1e-3), (1, 9, 1e-6)])
def test_toeplitz_apply_vs_dense_and_fft(oracle_mod, d, n, noise):
    rng = np.random.default_rng(d * 10 + n)
    t = W.planted_nodes(d, 3, n, rng)
    c = W.planted_coeffs(3, rng)
    grid = W.sample_grid(t, c, n, noise, 3)
    N = (n + 1) ** d
    X = rand_c(rng, N, 4)
    for ell in range(0, d + 1):
        Tl = oracle_mod.T_dense(grid, d, n, ell)
        assert rel(oracle_mod.toeplitz_apply(grid, d, n, X, ell), Tl @ X) < 1e-14
        assert rel(oracle_mod.toeplitz_apply(grid, d, n, X, ell, adjoint=True), Tl.conj().T @ X) < 1e-14
        if ell:
            assert rel(oracle_mod.toeplitz_apply(grid, d, n, X, ell), fft_apply(grid, d, n, ell, X)) < 1e-12


@pytest.mark.parametrize("d,n", [(2, 5), (3, 3)])
def test_T_fro_closed_form(oracle_mod, d, n):
    """||T||_F^2 = sum over v in {-n..n}^d of |f(v)|^2 prod_i (n + 1 - |v_i|) (multiplicity of k - h = v)."""
    rng = np.random.default_rng(4)
    t = W.planted_nodes(d, 3, n, rng)
    grid = W.sample_grid(t, W.planted_coeffs(3, rng), n, 1e-3, 2)
    box = W.box_coords(d, n)
    keep = np.all(box <= n, axis=1)
    mult = np.prod(n + 1 - np.abs(box[keep]), axis=1)
    want = math.sqrt(float(np.sum(np.abs(grid[keep]) ** 2 * mult)))
    assert abs(oracle_mod.T_fro(grid, d, n) - want) < 1e-13 * want


# ------------------------------------------------------------------ Algorithm 3 block power
def test_block_power_paper_family_d2(oracle_mod):
    """SPEC S:221 / PAPER.md:595, 603: the paper family d=2, n=20 with r0 = 2m: ranks 5, 10, 14, 17 for
    m = 5, 10, 15, 20 (the sample is too small for m = 15, 20), the same ranks as the dense Jacobi SVD,
    and singular values equal to LAPACK's SVD of the dense T to 1e-10 relative."""
    d, n = 2, 20
    N = (n + 1) ** d
    tol = N * EPS
    want = {5: 5, 10: 10, 15: 14, 20: 17}
    for m, r in want.items():
        t, c = W.paper_family(d, m)
        grid = W.sample_grid(t, c, n)
        bp = oracle_mod.block_power_svd(grid, d, n, 2 * m, W.gaussian_block(N, 2 * m, m, 0),
                                        W.gaussian_block(N, 2 * m, m, 1), tol)
        assert bp["status"] == 0 and bp["rank"] == r, (m, bp["rank"])
        T = oracle_mod.T_dense(grid, d, n, 0)
        U_l, s_l, Vh_l = np.linalg.svd(T)
        # relative 1e-10; small sigma_i carry an absolute error ~ eps_M sigma_1 in any FP64 SVD
        np.testing.assert_allclose(bp["sigma"], s_l[:r], rtol=1e-10, atol=1e-13 * s_l[0])
        if m == 5:   # well separated: the singular subspaces themselves agree
            assert np.abs(projector(bp["U"]) - projector(U_l[:, :r])).max() < 1e-10
            assert np.abs(projector(bp["V"]) - projector(Vh_l[:r].conj().T)).max() < 1e-10
        if m in (5, 15):   # "all three algorithms determined the same rank"
            _, _, s_j, _ = oracle_mod.svd_reduced(T, tol=tol)
            assert len(s_j) == r


def test_block_power_reconstructs_T(oracle_mod):
    """noise-free planted input: U Sigma V^* = T and U^* U = V^* V = I (eq_T_svd)."""
    d, n, m = 3, 4, 6
    rng = np.random.default_rng(77)
    t = W.planted_nodes(d, m, n, rng)
    grid = W.sample_grid(t, W.planted_coeffs(m, rng), n)
    N = (n + 1) ** d
    bp = oracle_mod.block_power_svd(grid, d, n, 2 * m, W.gaussian_block(N, 2 * m, 1, 0),
                                    W.gaussian_block(N, 2 * m, 1, 1), N * EPS)
    assert bp["rank"] == m and bp["status"] == 0 and bp["iters"] >= 1
    T = oracle_mod.T_dense(grid, d, n, 0)
    assert rel((bp["U"] * bp["sigma"]) @ bp["V"].conj().T, T) < 1e-12
    assert np.abs(bp["U"].conj().T @ bp["U"] - np.eye(m)).max() < 1e-13
    assert np.abs(bp["V"].conj().T @ bp["V"] - np.eye(m)).max() < 1e-13


# ------------------------------------------------------------------ eig, LU, diagonalization
def test_eig_spec_examples(oracle_mod):
    for ex in json.load(open(os.path.join(GOLD, "linalg_examples.json")))["eig"]:
        C = cmat(ex["C"])
        lam, Wm = oracle_mod.eig(C)
        want = np.array([complex(*v) for v in ex["eigvals"]])
        assert sorted(np.round(lam, 13).tolist(), key=lambda z: (z.real, z.imag)) == \
            sorted(np.round(want, 13).tolist(), key=lambda z: (z.real, z.imag))
        np.testing.assert_allclose(np.linalg.norm(Wm, axis=0), 1.0, atol=1e-15)
        if "vectors" in ex:
            for j in range(len(lam)):
                v = Wm[:, j]
                best = max(abs(np.vdot(np.array(w, dtype=complex), v)) for w in ex["vectors"])
                assert abs(best - 1.0) < 1e-14
        else:   # diagonal: W = permutation of identity columns (up to unit phases)
            assert np.allclose(np.sort(np.abs(Wm), axis=None)[-len(lam):], 1.0, atol=1e-15)


@pytest.mark.parametrize("m", [1, 2, 5, 20, 64])
def test_eig_vs_lapack_and_residual(oracle_mod, m):
    rng = np.random.default_rng(m)
    C = rand_c(rng, m, m)
    lam, Wm = oracle_mod.eig(C)
    lam_l = np.linalg.eigvals(C)
    for x in lam_l:                                            # multiset match
        assert np.min(np.abs(lam - x)) < 1e-11 * np.linalg.norm(C)
    res = np.linalg.norm(C @ Wm - Wm * lam, axis=0)
    assert res.max() <= 1e-10 * np.linalg.norm(C)              # S:306 residual contract


def test_eig_upper_triangular_and_defective_safe(oracle_mod):
    """A triangular matrix is its own Schur form: eigenvalues are its diagonal."""
    rng = np.random.default_rng(3)
    T = np.triu(rand_c(rng, 7, 7))
    lam, _ = oracle_mod.eig(T)
    for x in np.diag(T):
        assert np.min(np.abs(lam - x)) < 1e-12


def test_lu_solve(oracle_mod):
    rng = np.random.default_rng(8)
    A, B = rand_c(rng, 12, 12), rand_c(rng, 12, 5)
    X = oracle_mod.lu_solve(A, B)
    assert rel(A @ X, B) < 1e-13
    assert rel(X, np.linalg.solve(A, B)) < 1e-12
    P = np.eye(4)[[2, 0, 3, 1]].astype(complex)               # needs pivoting (zero leading entry)
    assert rel(oracle_mod.lu_solve(P, np.eye(4)), P.T) < 1e-15


def test_diagonalize_known_pencil(oracle_mod):
    """S_l = X diag(z(:,l)) X^-1 for a known X: the eigenvalues of C_mu are sum_l mu_l z_j(l) and
    W^-1 S_l W recovers z up to one common permutation (eq_diagonalizeSl)."""
    rng = np.random.default_rng(21)
    d, m = 3, 6
    z = W.node_vectors(rng.random((m, d)))
    X = rand_c(rng, m, m)
    Xi = np.linalg.inv(X)
    S = np.stack([X @ np.diag(z[:, l]) @ Xi for l in range(d)])
    mu = W.random_mu(d, 4)
    lam, _ = oracle_mod.eig(np.tensordot(mu, S, axes=1))
    for x in z @ mu:
        assert np.min(np.abs(lam - x)) < 1e-11
    zz, Wm, off = oracle_mod.diagonalize(S, mu)
    assert off.max() < 1e-11
    for j in range(m):                                          # one common tau for every l
        i = int(np.argmin(np.abs(zz[:, 0] - z[j, 0]) + np.abs(zz[:, 1] - z[j, 1])))
        assert np.abs(zz[i] - z[j]).max() < 1e-11


def test_random_mu_unit(oracle_mod):
    for d in (1, 2, 5):
        mu = W.random_mu(d, 3)
        assert abs(np.linalg.norm(mu) - 1.0) < 1e-15
    assert not np.allclose(W.random_mu(3, 1), W.random_mu(3, 2))


# ------------------------------------------------------------------ least squares
def test_lstsq_qr_spec_and_lapack(oracle_mod):
    ex = json.load(open(os.path.join(GOLD, "linalg_examples.json")))["lstsq"][0]
    z = np.array([[complex(*ex["z"])]])
    grid = np.full((2 * ex["n"] + 2) ** ex["d"], complex(*ex["f_value"]))
    A = oracle_mod.vandermonde(z, ex["d"], ex["n"])
    c, r = oracle_mod.lstsq_qr(A, grid, ex["d"], ex["n"])
    assert abs(c[0] - complex(*ex["c"])) < 1e-15 and r < 1e-15
    d, n, m = 2, 9, 5
    rng = np.random.default_rng(12)
    zr = W.node_vectors(rng.random((m, d))) * (1 + 0.01 * rng.random((m, d)))
    grid = W.sample_grid(rng.random((3, d)), W.planted_coeffs(3, rng), n, 1e-3, 1)
    A = oracle_mod.vandermonde(zr, d, n)
    f = oracle_mod.f_vector(grid, d, n)
    c, r = oracle_mod.lstsq_qr(A, grid, d, n)
    c_l = np.linalg.lstsq(A.T, f, rcond=None)[0]
    assert rel(c, c_l) < 1e-12
    assert abs(r - np.linalg.norm(A.T @ c_l - f) / np.linalg.norm(f)) < 1e-12


# ------------------------------------------------------------------ noise model
def test_disk_noise_bound(oracle_mod):
    """|delta_k| <= eps exactly, one pattern reused across eps (R5b)."""
    t, c = W.paper_family(2, 3)
    g0 = W.sample_grid(t, c, 6)
    for eps in (1e-9, 1e-3):
        g = W.sample_grid(t, c, 6, eps, 7, noise_model="disk")
        r = np.abs(g / g0 - 1.0)
        assert r.max() <= eps * (1 + 1e-6) and r.max() > 0.9 * eps
    big = np.abs(g0) > 1e-3 * np.abs(g0).max()
    d9 = (W.sample_grid(t, c, 6, 1e-9, 7, "disk") - g0)[big]
    d6 = (W.sample_grid(t, c, 6, 1e-6, 7, "disk") - g0)[big]
    assert np.abs(d6 / d9 / 1000.0 - 1.0).max() < 1e-4


# ------------------------------------------------------------------ Algorithm 1 at the paper's table configuration
@pytest.fixture(scope="module")
def table_runs(oracle_mod):
    """Algorithm 1 (block power, r0 = 2m, plain C throughout) on the paper family d=3, n=20, m=5 with the
    paper's bounded noise, tol per table row; plus the tol = eps = 1e-3 run."""
    d, n, m = 3, 20, 5
    N = (n + 1) ** d
    t, c = W.paper_family(d, m)
    gold = json.load(open(os.path.join(GOLD, "accuracy_table.json")))
    runs = {}
    for row in gold["rows"]:
        eps = row[0]
        tol = N * EPS if row[1] == "N*eps_M" else row[1]
        grid = W.sample_grid(t, c, n, eps, 7, noise_model="disk")
        runs[eps] = (row, oracle_mod.algorithm1(grid, d, n, tol=tol, seed=5, svd="power", m_hint=m))
    grid = W.sample_grid(t, c, n, 1e-3, 7, noise_model="disk")
    runs["anomaly"] = oracle_mod.algorithm1(grid, d, n, tol=1e-3, seed=5, svd="power", m_hint=m)
    return t, c, runs


def _errors(oracle_mod, out, t, c):
    perm = oracle_mod.match_nodes(out["t"], t)
    return (out["resid"], W.torus_dist_inf(out["t"][perm], t).max(),
            np.linalg.norm(out["c"][perm] - c) / np.linalg.norm(c))


def test_algorithm1_accuracy_table(oracle_mod, table_runs):
    """Noisy rows (eps = 1e-9, 1e-6, 1e-3): residual, t error and c error within x5 of the printed values.
    Noise-free row: roundoff, bounded above only (t and c below x5 of the printed values; the residual below
    x20 — it is the amplification of the ~5e-15 node error through the powers z^k, |k| up to d n = 60)."""
    t, c, runs = table_runs
    for eps in (0.0, 1e-9, 1e-6, 1e-3):
        row, out = runs[eps]
        assert out["rank"] == 5 and out["power_status"] == 0
        got = _errors(oracle_mod, out, t, c)
        bands = (20.0, 5.0, 5.0) if eps == 0.0 else (5.0, 5.0, 5.0)
        for g, p, b in zip(got, row[2:], bands):
            assert g < p * b, (eps, got, row)
            if eps > 0:                    # the noise-free row is roundoff: bounded above only
                assert p / b < g, (eps, got, row)
        assert np.max(out["offdiag"]) < (1e-10 if eps == 0 else 100 * eps)


def test_algorithm1_linear_in_eps_and_same_mantissa(oracle_mod, table_runs):
    """errors proportional to eps; the printed 1e-9 and 1e-6 rows share their mantissas
    (3.00100e-10 / 3.00100e-07) — one noise pattern scaled by eps (R5b): ours do too, to 1e-3."""
    t, c, runs = table_runs
    e9 = _errors(oracle_mod, runs[1e-9][1], t, c)
    e6 = _errors(oracle_mod, runs[1e-6][1], t, c)
    for a, b in zip(e9, e6):
        assert abs(b / a / 1000.0 - 1.0) < 1e-3


def test_algorithm1_rank_anomaly(oracle_mod, table_runs):
    """with tol = eps = 1e-3 the detected numerical rank is 4."""
    _, _, runs = table_runs
    assert runs["anomaly"]["rank"] == 4


def test_algorithm1_jacobi_and_power_agree(oracle_mod):
    """Both SVD routes of the oracle give the same rank, nodes and coefficients."""
    d, n, m = 2, 12, 5
    rng = np.random.default_rng(131)
    t = W.planted_nodes(d, m, n, rng)
    c = W.planted_coeffs(m, rng)
    grid = W.sample_grid(t, c, n, 1e-6, 2, noise_model="disk")
    a = oracle_mod.algorithm1(grid, d, n, tol=1e-6, seed=3, svd="jacobi")
    b = oracle_mod.algorithm1(grid, d, n, tol=1e-6, seed=3, svd="power", m_hint=m)
    assert a["rank"] == b["rank"] == m
    pa, pb = oracle_mod.match_nodes(a["t"], t), oracle_mod.match_nodes(b["t"], t)
    assert W.torus_dist_inf(a["t"][pa], b["t"][pb]).max() < 1e-12
    assert rel(a["c"][pa], b["c"][pb]) < 1e-10


def test_perturbation_bounds_hoffman_wielandt_and_tail(oracle_mod):
    """for T~ = T + dT built from samples f(1+delta), |delta| <= eps,
    sqrt(sum_i |sigma~_i - sigma_i|^2) <= ||dT||_F <= eps ||T||_F (Hoffman-Wielandt) and the tail
    sqrt(sum_{i>m} sigma~_i^2) <= eps ||T||_F — checked on the oracle's own Jacobi SVDs of both matrices."""
    d, n, m = 2, 9, 4
    t, c = W.paper_family(d, m)
    eps = 1e-3
    g0 = W.sample_grid(t, c, n)
    g1 = W.sample_grid(t, c, n, eps, 3, noise_model="disk")
    T0, T1 = oracle_mod.T_dense(g0, d, n, 0), oracle_mod.T_dense(g1, d, n, 0)
    _, s0, _, _ = oracle_mod.jacobi_svd(T0)
    _, s1, _, _ = oracle_mod.jacobi_svd(T1)
    nT = oracle_mod.T_fro(g0, d, n)
    hw = math.sqrt(float(np.sum((s1 - s0) ** 2)))
    assert hw <= np.linalg.norm(T1 - T0) * (1 + 1e-12) <= eps * nT * (1 + 1e-12)
    assert hw > 0.01 * eps * nT * 1e-3               # the noise is really there
    tail = math.sqrt(float(np.sum(s1[m:] ** 2)))
    assert tail <= eps * nT
    assert s0[m] <= 1e-12 * s0[0]                    # noise-free T has rank m exactly


@pytest.mark.parametrize("d,n,m", [(2, 8, 3), (3, 4, 4)])
def test_pencil_forward_error_eq_deltaSl(oracle_mod, d, n, m):
    """PAPER.md:413-418 (eq_deltaSl): with samples f(1 + delta_k), |delta_k| <= eps, the pencil S~_l built from the
    noisy T's rank-m SVD, compared with S_l of the noise-free T in the gauge of P:332-334 (each column of U scaled
    by the phase that makes U(:,i)^* U~(:,i) real positive, the same scalars on V), obeys the first-order bound
    ||S~_l - S_l||_F <= eps ||T_l||_F / sigma~_m (1 + (1 + 4 sqrt2 + (2 + g) sqrt(2m)) ||T||_F / delta_min),
    delta_i = min{min_{j != i} |sigma_i - sigma~_j|, sigma_i}, with g = 8 (SPEC's default for the
    paper's unnamed constant) — all from the oracle's own Jacobi SVDs; and the error is linear in eps."""
    rng = np.random.default_rng(11 + d)
    t = W.planted_nodes(d, m, n, rng)
    c = W.planted_coeffs(m, rng)
    g0 = W.sample_grid(t, c, n)
    U0, s0, V0, _ = oracle_mod.jacobi_svd(oracle_mod.T_dense(g0, d, n, 0))
    U, V, sig = U0[:, :m], V0[:, :m], s0[:m]
    nT = oracle_mod.T_fro(g0, d, n)
    nTl = [np.linalg.norm(oracle_mod.T_dense(g0, d, n, ell)) for ell in range(1, d + 1)]
    worst = []
    for eps in (1e-8, 1e-6):
        g1 = W.sample_grid(t, c, n, eps, 5, noise_model="disk")
        U1f, s1, V1f, _ = oracle_mod.jacobi_svd(oracle_mod.T_dense(g1, d, n, 0))
        U1, V1, sig1 = U1f[:, :m], V1f[:, :m], s1[:m]
        ph = np.exp(1j * np.angle(np.sum(U.conj() * U1, axis=0)))  # gauge of P:332-334
        S0 = oracle_mod.project(g0, U * ph, V * ph, sig, d, n)
        S1 = oracle_mod.project(g1, U1, V1, sig1, d, n)
        delta_min = min(min(np.min(np.abs(np.delete(s1, i) - sig[i])), sig[i]) for i in range(m))
        k = (1 + 4 * math.sqrt(2) + 10 * math.sqrt(2 * m)) * nT / delta_min
        ratios = []
        for ell in range(d):
            err = np.linalg.norm(S1[ell] - S0[ell])
            bound = eps * nTl[ell] / sig1[-1] * (1 + k)
            assert err <= bound, (eps, ell, err, bound)
            ratios.append(err / (eps * nTl[ell] / sig1[-1]))
        worst.append(max(np.linalg.norm(S1[ell] - S0[ell]) for ell in range(d)))
    assert 50.0 < worst[1] / worst[0] < 200.0  # first order: 100x the noise, 100x the error
