"""NEXT-3: Lanczos bidiagonalization SVD (Alg. 2) on the device vs the oracle.

The device result is compared with the oracle's LAPACK SVD of the dense T (oracle.svd_reduced) at
small sizes, and with the planted closed-form SVD (workload.planted_svd, T = B diag(c) B^H) at the
full cfg4/cfg5 sizes: singular values, gauge-invariant subspace projectors, orthonormality, and
the rank detected without knowing m (the point of Alg. 2)."""
import numpy as np
import pytest
import torch

import workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2012_11430_b200 as pb
    return pb


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _proj(U):
    return U @ U.conj().T


def _problem(d, n, m, seed, noise=0.0):
    return W.make_problem(W.custom_config(d, n, m, noise, seed), with_svd=False)


@pytest.mark.parametrize("d,n,m,noise", [(2, 12, 5, 0.0), (3, 5, 6, 0.0), (2, 14, 7, 1e-6), (1, 40, 9, 0.0),
                                         (4, 3, 10, 0.0), (2, 20, 40, 0.0)])
def test_lanczos_vs_oracle_svd(pb, orc, d, n, m, noise):
    """alpha stop (random p_1 has a null-space component): rank == m, sigma and subspaces."""
    prob = _problem(d, n, m, 1300 + d + n + m, noise)
    tol = 1e-6 if noise else None
    out = pb.lanczos_svd(dev(prob.grid), d, n, max_rank=2 * m + 5, tol=tol, seed=7)
    assert out["status"] == pb.PRONY_OK, out["status"]
    assert out["rank"] == m
    T = orc.T_dense(prob.grid, d, n, 0)
    U_or, V_or, s_or, _ = orc.svd_reduced(T, rank=m)
    s = out["sigma"].cpu().numpy()[:m]
    assert np.max(np.abs(s - s_or) / s_or[0]) <= (1e-10 if noise == 0.0 else 1e-8)
    U = out["U"].cpu().numpy()[:, :m]
    V = out["V"].cpu().numpy()[:, :m]
    sub_tol = 1e-8 if noise == 0.0 else 1e-4
    assert np.linalg.norm(_proj(U) - _proj(U_or)) <= sub_tol
    assert np.linalg.norm(_proj(V) - _proj(V_or)) <= sub_tol
    np.testing.assert_allclose(U.conj().T @ U, np.eye(m), atol=1e-12)
    np.testing.assert_allclose(V.conj().T @ V, np.eye(m), atol=1e-12)
    # the triplets themselves: T V = U Sigma (gauge fixed by the pairing of U and V)
    assert np.linalg.norm(T @ V - U * s[None, :]) <= (1e-10 if noise == 0.0 else 1e-6) * s_or[0] * np.sqrt(m)
    assert np.all(np.diff(s) <= 0)


def test_lanczos_full_rank_beta_stop(pb, orc):
    """T of full rank N (d = 1, m = N nodes): v_1 lies in R(T^H) = C^N, so the recurrence ends with
    beta = 0 at i = r = N, the square B_r branch."""
    d, n, m = 1, 5, 6
    prob = _problem(d, n, m, 77)
    out = pb.lanczos_svd(dev(prob.grid), d, n, max_rank=6, seed=3)
    assert out["status"] == pb.PRONY_OK
    assert out["rank"] == 6
    T = orc.T_dense(prob.grid, d, n, 0)
    s_or = np.linalg.svd(T, compute_uv=False)
    s = out["sigma"].cpu().numpy()
    assert np.max(np.abs(s - s_or)) <= 1e-11 * s_or[0]
    U = out["U"].cpu().numpy()
    V = out["V"].cpu().numpy()
    assert np.linalg.norm(T @ V - U * s[None, :]) <= 1e-11 * s_or[0] * 3


def test_lanczos_cap_not_converged(pb, orc):
    """max_rank < rank: NOT_CONVERGED, the rank-max_rank Lanczos approximation: orthonormal bases and
    singular values interlaced below T's (B = U_k^H T V_k is a compression of T)."""
    d, n, m = 2, 10, 8
    prob = _problem(d, n, m, 55)
    out = pb.lanczos_svd(dev(prob.grid), d, n, max_rank=5, seed=1)
    assert out["status"] == pb.PRONY_ERR_NOT_CONVERGED
    assert out["rank"] == 5
    T = orc.T_dense(prob.grid, d, n, 0)
    s_or = np.linalg.svd(T, compute_uv=False)
    s = out["sigma"].cpu().numpy()
    assert np.all(s <= s_or[:5] * (1 + 1e-12))
    assert s[0] >= 0.9 * s_or[0]
    U = out["U"].cpu().numpy()
    np.testing.assert_allclose(U.conj().T @ U, np.eye(5), atol=1e-12)


def test_lanczos_zero_operator(pb):
    d, n = 2, 4
    grid = torch.zeros((2 * n + 2) ** d, dtype=torch.complex128, device="cuda")
    out = pb.lanczos_svd(grid, d, n, max_rank=4, check=False)
    assert out["status"] == pb.PRONY_ERR_RANK
    assert out["rank"] == 0


def test_lanczos_ldo_and_determinism(pb):
    d, n, m = 2, 12, 6
    prob = _problem(d, n, m, 91)
    a = pb.lanczos_svd(dev(prob.grid), d, n, max_rank=12, ldo=4, seed=5)
    b = pb.lanczos_svd(dev(prob.grid), d, n, max_rank=12, ldo=4, seed=5)
    assert a["rank"] == m and a["U"].shape == (prob.cfg.N, 4)
    assert torch.equal(a["U"], b["U"]) and torch.equal(a["sigma"], b["sigma"])


@pytest.mark.parametrize("name", ["cfg5", "cfg4"])
def test_lanczos_full_size_planted(pb, name):
    """Full-size configurations: rank found with no m given, singular values and left subspace vs the
    planted closed-form SVD of the noise-free T (cfg4 carries 1e-6 noise: tolerance at that level)."""
    prob = W.make_problem(name)
    c = prob.cfg
    tol = 1e-6 if c.noise else None
    out = pb.lanczos_svd(dev(prob.grid), c.d, c.n, max_rank=min(2 * c.m + 5, 255), tol=tol, seed=11)
    assert out["status"] == pb.PRONY_OK
    assert out["rank"] == c.m
    s = out["sigma"].cpu().numpy()[:c.m]
    rtol = 1e-10 if not c.noise else 1e-4
    assert np.max(np.abs(s - prob.sigma) / prob.sigma[0]) <= rtol
    U = out["U"][:, :c.m]
    Upl = dev(prob.U)
    # ||P_U - P_planted||_F^2 = 2m - 2 ||Upl^H U||_F^2 (both orthonormal)
    overlap = torch.linalg.norm(Upl.conj().T @ U).item() ** 2
    assert 2 * c.m - 2 * overlap <= (1e-16 if not c.noise else 1e-6)


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_algorithm1_with_lanczos_svd(pb, orc, name):
    """Algorithm 1 with the SVD step done by Lanczos (m not given to the SVD): the rank it finds sizes
    the pencil, then S_l, C_mu eig, W^-1 S_l W and t on the device recover the planted nodes."""
    prob = W.make_problem(name, with_svd=False)
    c = prob.cfg
    grid = dev(prob.grid)
    tol = 1e-6 if c.noise else None
    lz = pb.lanczos_svd(grid, c.d, c.n, max_rank=2 * c.m + 5, tol=tol, seed=2)
    r = lz["rank"]
    assert lz["status"] == pb.PRONY_OK and r == c.m
    S = pb.project(grid, lz["U"][:, :r].contiguous(), lz["V"][:, :r].contiguous(), lz["sigma"][:r].contiguous(),
                   c.d, c.n, r)
    mu = dev(orc.random_mu(c.d, 4))
    z, t, _ = pb.diagonalize(S, mu, c.d, r)
    t = t.cpu().numpy()
    perm = orc.match_nodes(t, prob.t)
    assert W.torus_dist_inf(t[perm], prob.t).max() <= (1e-8 if c.noise else 1e-11)
