"""Seeded random sweep of the CUDA path against the CPU oracle: shapes drawn across d = 1..8, n, m (m up to
128; N up to what the oracle finishes in about a second), noise on or off, random orthonormal U, V and sigma, random unit
and column sub-ranges in every unit order, and the three ways a pencil is launched (prony_project +
prony_vandermonde_ls, the one-call prony_pencil, the host-input prony_pencil_host with its split-K copy
pipeline). Every case is compared element by element within the north_star tolerance (relative Frobenius
<= 1e-10). The draws are fixed (seed 20121143), so a failure names a reproducible case."""
import numpy as np
import pytest
import torch

import workload as W

pytestmark = pytest.mark.gpu

TOL = 1e-10
SEED = 20121143


def _cases(k=64):
    rng = np.random.default_rng(SEED)
    out = []
    while len(out) < k:
        d = int(rng.integers(1, 9))
        nmax = {1: 600, 2: 40, 3: 11, 4: 6, 5: 4, 6: 3, 7: 2, 8: 2}[d]
        n = int(rng.integers(1, nmax + 1))
        N = (n + 1) ** d
        if N < 2:
            continue
        m = int(rng.integers(1, min(N, 128 if d <= 2 else 48) + 1))
        noise = float(rng.choice([0.0, 1e-6]))
        out.append((d, n, m, noise, int(rng.integers(1 << 30))))
    return out


CASES = _cases()


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2012_11430_b200 as pb
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return pb


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def problem(d, n, m, noise, seed):
    cfg = W.custom_config(d, n, m, noise, seed)
    prob = W.make_problem(cfg, with_svd=False)
    rng = np.random.default_rng(seed + 1)
    prob.U = W.random_orthonormal(cfg.N, m, rng)
    prob.V = W.random_orthonormal(cfg.N, m, rng)
    prob.sigma = np.sort(rng.random(m) + 0.5)[::-1].copy()
    return prob


@pytest.mark.parametrize("d,n,m,noise,seed", CASES)
def test_fuzz_pencil_vs_oracle(pb, orc, d, n, m, noise, seed):
    prob = problem(d, n, m, noise, seed)
    c = prob.cfg
    N = c.N
    rng = np.random.default_rng(seed + 2)
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    A_or = orc.vandermonde(prob.z, d, n)
    G_or, b_or = orc.ls_products(A_or, prob.grid, d, n)
    g, U, V, s, z = (dev(x) for x in (prob.grid, prob.U, prob.V, prob.sigma, prob.z))

    # 1. the two entry points over the full ranges
    S = pb.project(g, U, V, s, d, n, m)
    for ell in range(d):
        assert rel(S[ell], S_or[ell]) <= TOL, ("project", ell)
    ls = pb.vandermonde_ls(z, g, d, n, m)
    assert rel(ls["G"], G_or) <= TOL and rel(ls["b"], b_or) <= TOL

    # 2. a random split of the units (every order) and of the columns: the partial sums add up
    for order in (pb.UNITS_L_MAJOR, pb.UNITS_ROW_MAJOR, pb.UNITS_SHARED):
        units = (n + 2) ** d if order == pb.UNITS_SHARED else d * N
        cut = int(rng.integers(0, units + 1))
        S1 = pb.project(g, U, V, s, d, n, m, 0, cut, order)
        S2 = pb.project(g, U, V, s, d, n, m, cut, units, order)
        for ell in range(d):
            assert rel(S1[ell] + S2[ell], S_or[ell]) <= TOL, ("units", order, cut, ell)
    cc = int(rng.integers(0, N + 1))
    l1 = pb.vandermonde_ls(z, g, d, n, m, 0, cc)
    l2 = pb.vandermonde_ls(z, g, d, n, m, cc, N)
    assert rel(l1["G"] + l2["G"], G_or) <= TOL and rel(l1["b"] + l2["b"], b_or) <= TOL

    # 3. the one-call pencil and the host-input pencil
    pencil = pb.sharding.DistributedPencil(d, n, m, torch.device("cuda", 0))
    S3, c3, t3 = pencil(g, U, V, s, z)
    torch.cuda.synchronize()
    for ell in range(d):
        assert rel(S3[ell], S_or[ell]) <= TOL, ("pencil", ell)
    assert rel(pencil.G, G_or) <= TOL
    out = pb.pencil_host(prob.grid, prob.U, prob.V, prob.sigma, prob.z, d, n, m)
    assert out["status"] == 0
    for ell in range(d):
        assert rel(out["S"][ell], S_or[ell]) <= TOL, ("pencil_host", ell)
    assert rel(out["G"], G_or) <= TOL and rel(out["b"], b_or) <= TOL
    assert np.array_equal(out["t"], t3.cpu().numpy())
