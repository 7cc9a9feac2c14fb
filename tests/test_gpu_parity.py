"""CUDA path (libprony.so through the C ABI) vs the CPU oracle, element by element.

Tolerances (north_star / DESIGN.md §4): relative Frobenius <= 1e-10 on S_l, G and b (2-norm
for b); |t - t_planted| <= 1e-8 on noise-free data. Observed errors are ~1e-15.
"""
import numpy as np
import pytest
import torch

import workload as W

pytestmark = pytest.mark.gpu

TOL = 1e-10


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
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def problem(d, n, m, seed, noise=0.0, random_uv=False):
    cfg = W.custom_config(d, n, m, noise, seed)
    prob = W.make_problem(cfg, with_svd=not random_uv)
    if random_uv:
        rng = np.random.default_rng(seed + 1)
        N = cfg.N
        prob.U = W.random_orthonormal(N, m, rng)
        prob.V = W.random_orthonormal(N, m, rng)
        prob.sigma = np.sort(rng.random(m) + 0.5)[::-1].copy()
    return prob


def run_project(pb, prob, **kw):
    c = prob.cfg
    return pb.project(dev(prob.grid), dev(prob.U), dev(prob.V), dev(prob.sigma), c.d, c.n, c.m, **kw)


# ------------------------------------------------------------------ projection parity
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_project_configs_full_oracle(pb, orc, name):
    prob = W.make_problem(name)
    c = prob.cfg
    S = run_project(pb, prob)
    torch.cuda.synchronize()
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n)
    for l in range(c.d):
        assert rel(S[l], S_or[l]) <= TOL


@pytest.mark.parametrize("d,n,m,noise", [
    (1, 40, 7, 1e-6),      # d = 1
    (2, 6, 1, 0.0),        # m = 1
    (2, 7, 9, 1e-3),       # ragged: N = 64, m = 9 (two n-tiles, pad 7)
    (2, 13, 33, 1e-6),     # N = 196 (ragged row block), m = 33
    (3, 4, 17, 0.0),       # d = 3, N = 125
    (4, 3, 12, 1e-6),      # d = 4
    (5, 2, 8, 0.0),        # d = 5, N = 243
    (2, 11, 64, 0.0),      # m = 64 (WN = 1, NT = 8 -> WN = 2 path)
    (2, 12, 100, 1e-6),    # m = 100 (WN = 2, NT = 7), N = 169
    (2, 11, 128, 0.0),     # m = 128 = PRONY_MAX_M (NT = 8, WN = 2)
    (6, 1, 5, 1e-6),       # d = 6: E = 729 > dN = 384
    (8, 1, 3, 0.0),        # d = 8 = PRONY_MAX_D, N = 256, E = 6561
    (1, 3, 4, 0.0),        # d = 1, N = 4 = m (full rank), E = N + 1
])
@pytest.mark.parametrize("order", [2, 0])
def test_project_edge_shapes(pb, orc, d, n, m, noise, order):
    prob = problem(d, n, m, 1000 + d * 100 + n + m, noise, random_uv=True)
    S = run_project(pb, prob, unit_order=order)
    torch.cuda.synchronize()
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    for l in range(d):
        assert rel(S[l], S_or[l]) <= TOL


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 7, 8, 9, 12, 13, 20, 36, 44, 76, 80, 81, 84, 97, 100, 101, 104, 105, 124, 128])
def test_project_packed_last_tile_every_m_class(pb, orc, m):
    """k_project packs the last n-tile (2 real products, 4M form) exactly when m % 8 is 1..4: every residue
    class of m, both consumer layouts (m <= 80: 2 column warps; m > 80: 3), both complex modes of the
    other tiles' engine, against the oracle. N = 169 > m, ragged row blocks."""
    d, n = 2, 12
    prob = problem(d, n, m, 2000 + m, 1e-6, random_uv=True)
    S = run_project(pb, prob)
    torch.cuda.synchronize()
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    for l in range(d):
        assert rel(S[l], S_or[l]) <= TOL


def test_project_shared_random_partitions(pb, orc):
    """Random partitions of the SHARED unit space [0, (n+2)^d) over 2-9 'ranks' sum to the full pencil
    (the multi-GPU decomposition), each partial equal to the oracle's rows of T_l it stands for."""
    rng = np.random.default_rng(2024)
    for d, n, m in [(2, 20, 12), (3, 7, 9)]:
        prob = problem(d, n, m, 300 + d, 1e-6, random_uv=True)
        E = (n + 2) ** d
        full = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
        for parts in (2, 5, 9):
            cuts = np.sort(rng.choice(np.arange(1, E), size=parts - 1, replace=False))
            cuts = [0, *cuts.tolist(), E]
            acc = torch.zeros((d, m, m), dtype=torch.complex128, device="cuda")
            for a, b in zip(cuts, cuts[1:]):
                S = run_project(pb, prob, unit_begin=a, unit_end=b, unit_order=2)
                acc += S
                if parts == 2:
                    S_or = orc.project_units(prob.grid, prob.U, prob.V, prob.sigma, d, n, a, b, 2)
                    for l in range(d):
                        assert rel(S[l], S_or[l]) <= TOL
            for l in range(d):
                assert rel(acc[l], full[l]) <= TOL


@pytest.mark.parametrize("order", [0, 1, 2])
def test_project_unit_ranges_partition(pb, orc, order):
    """Partial pencils over unit sub-ranges match the oracle and sum to the full pencil."""
    prob = problem(3, 6, 10, 77, 1e-6, random_uv=True)
    c = prob.cfg
    N = c.N
    E = (c.n + 2) ** c.d
    cuts = [0, 5, 343, 344, 700, 3 * N - 1, 3 * N] if order < 2 else [0, 5, 63, 64, 300, E - 1, E]
    acc = torch.zeros((c.d, c.m, c.m), dtype=torch.complex128, device="cuda")
    for a, b in zip(cuts, cuts[1:]):
        S = run_project(pb, prob, unit_begin=a, unit_end=b, unit_order=order)
        torch.cuda.synchronize()
        S_or = orc.project_units(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n, a, b, order)
        for l in range(c.d):
            if np.linalg.norm(S_or[l]) == 0:
                assert float(S[l].abs().max()) == 0.0
            else:
                assert rel(S[l], S_or[l]) <= TOL
        acc += S
    full = orc.project(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n)
    for l in range(c.d):
        assert rel(acc[l], full[l]) <= TOL


@pytest.mark.parametrize("mode", ["4m", "3m"])
@pytest.mark.parametrize("d,n,m", [(2, 12, 100), (3, 5, 20)])
def test_project_cmul_modes(pb, orc, mode, d, n, m, monkeypatch):
    """Both complex-product formulations of k_project (3M default, 4M via PRONY_CMUL=4m)."""
    monkeypatch.setenv("PRONY_CMUL", mode)
    prob = problem(d, n, m, 4242, 1e-6, random_uv=True)
    S = run_project(pb, prob)
    torch.cuda.synchronize()
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    for l in range(d):
        assert rel(S[l], S_or[l]) <= 1e-13


@pytest.mark.parametrize("u0,u1,order", [(0, 100, 0), (4096 + 7, 4096 + 300, 0), (11, 913, 1), (0, 8192, 1),
                                          (0, 100, 2), (3999, 4225, 2)])
def test_project_small_ranges_many_chunks(pb, orc, u0, u1, order):
    """Small unit ranges over a long K (N = 4096) make the planner split K into many chunks:
    exercises the split-K arrival counters and the last-arriver fixup of k_project."""
    prob = problem(2, 63, 20, 5151, 1e-6, random_uv=True)
    c = prob.cfg
    S = run_project(pb, prob, unit_begin=u0, unit_end=u1, unit_order=order)
    S2 = run_project(pb, prob, unit_begin=u0, unit_end=u1, unit_order=order)
    torch.cuda.synchronize()
    assert torch.equal(S, S2)                       # deterministic whatever the arrival order
    S_or = orc.project_units(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n, u0, u1, order)
    for l in range(c.d):
        if np.linalg.norm(S_or[l]) == 0:
            assert float(S[l].abs().max()) == 0.0
        else:
            assert rel(S[l], S_or[l]) <= TOL


def test_project_empty_range_is_zero(pb):
    prob = problem(2, 5, 4, 5, random_uv=True)
    S = run_project(pb, prob, unit_begin=7, unit_end=7)
    torch.cuda.synchronize()
    assert float(S.abs().max()) == 0.0


def test_project_deterministic(pb):
    prob = W.make_problem("cfg2")
    S1 = run_project(pb, prob)
    S2 = run_project(pb, prob)
    torch.cuda.synchronize()
    assert torch.equal(S1, S2)


def test_project_spectrum_recovers_nodes(pb):
    """F2 on the GPU result: eig(S_l) = {z_j(l)} with the planted SVD (noise-free cfg3)."""
    prob = W.make_problem("cfg3")
    S = run_project(pb, prob).cpu().numpy()
    for l in range(prob.cfg.d):
        ev = np.linalg.eigvals(S[l])
        for zj in prob.z[:, l]:
            assert np.min(np.abs(ev - zj)) < 1e-10


# ------------------------------------------------------------------ NEXT-4: B_mu / C_mu in one projection
@pytest.mark.parametrize("d,n,m,noise", [(2, 12, 9, 1e-6), (3, 5, 20, 0.0), (1, 30, 4, 1e-6), (4, 3, 7, 0.0)])
def test_project_mu_equals_combination(pb, orc, d, n, m, noise):
    """C_mu = U* (sum mu_l T_l) V Sigma^-1 equals sum_l mu_l S_l of the oracle."""
    prob = problem(d, n, m, 3300 + d + n + m, noise, random_uv=True)
    mu = orc.random_mu(d, 9)
    C = pb.project_mu(dev(prob.grid), dev(prob.U), dev(prob.V), dev(prob.sigma), dev(mu), d, n, m)
    torch.cuda.synchronize()
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    want = np.tensordot(mu, S_or, axes=1)
    assert rel(C, want) <= TOL


# ------------------------------------------------------------------ Toeplitz apply (NEXT-1 operator)
@pytest.mark.parametrize("d,n,r,noise", [(2, 7, 5, 1e-6), (3, 4, 130, 0.0), (1, 30, 3, 1e-3), (4, 3, 17, 1e-6)])
def test_toeplitz_apply_dense_oracle(pb, orc, d, n, r, noise):
    """Y = T_l X, T X and T^H X against the oracle's dense T_l times X."""
    prob = problem(d, n, 3, 600 + d + n + r, noise, random_uv=True)
    N = prob.cfg.N
    rng = np.random.default_rng(r)
    X = rng.standard_normal((N, r)) + 1j * rng.standard_normal((N, r))
    Xd = dev(X)
    for ell in range(0, d + 1):
        Y = pb.toeplitz_apply(dev(prob.grid), Xd, d, n, ell).cpu().numpy()
        T = orc.T_dense(prob.grid, d, n, ell)
        assert rel(Y, T @ X) <= 1e-13
    Yh = pb.toeplitz_apply(dev(prob.grid), Xd, d, n, 0, conj=True).cpu().numpy()
    T = orc.T_dense(prob.grid, d, n, 0)
    assert rel(Yh, T.conj().T @ X) <= 1e-13


def test_toeplitz_apply_strided_columns(pb, orc):
    """X and Y as column slices of wider matrices (row strides ldx, ldy > r)."""
    prob = problem(2, 9, 3, 77, 1e-6, random_uv=True)
    N = prob.cfg.N
    rng = np.random.default_rng(5)
    Xw = rng.standard_normal((N, 40)) + 1j * rng.standard_normal((N, 40))
    Xd = dev(Xw)
    Yw = torch.zeros((N, 50), dtype=torch.complex128, device="cuda")
    pb.toeplitz_apply(dev(prob.grid), Xd[:, 6:29], 2, 9, 1, out=Yw[:, 10:33])
    T1 = orc.T_dense(prob.grid, 2, 9, 1)
    Y = Yw.cpu().numpy()
    assert rel(Y[:, 10:33], T1 @ Xw[:, 6:29]) <= 1e-13
    assert np.all(Y[:, :10] == 0) and np.all(Y[:, 33:] == 0)


# ------------------------------------------------------------------ full-size configs
def _closed_form_S(prob):
    """F1 (noise-free, any U V sigma): S_l = (U* B) diag(c z_l) (B^H V) Sigma^-1."""
    c = prob.cfg
    k = W.index_set(c.d, c.n).astype(np.float64)
    ph = k @ prob.t.T
    B = np.exp(-2j * np.pi * (ph - np.floor(ph)))
    UB = prob.U.conj().T @ B
    BV = B.conj().T @ prob.V
    return np.stack([(UB * (prob.c * prob.z[:, l])) @ BV / prob.sigma[None, :] for l in range(c.d)])


def test_cfg5_full_size_closed_form(pb):
    prob = W.make_problem("cfg5")
    S = run_project(pb, prob)
    torch.cuda.synchronize()
    want = _closed_form_S(prob)
    for l in range(prob.cfg.d):
        assert rel(S[l], want[l]) <= TOL


@pytest.mark.parametrize("name,cols", [("cfg4", [0, 57, 99]), ("cfg5", [3, 29])])
def test_full_size_sampled_columns_oracle(pb, orc, name, cols):
    """Full BASELINE sizes, the launch configuration bench.py times: sampled columns of S_l
    computed one by one by the oracle (T_l v_j in full, then U^*)."""
    prob = W.make_problem(name)
    c = prob.cfg
    S = run_project(pb, prob).cpu().numpy()
    ells = [1, c.d] if c.d > 1 else [1]
    for ell in ells:
        want = orc.project_columns(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n, ell, cols)
        assert rel(S[ell - 1][:, cols], want) <= TOL


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_all_entries_fft_convolution(pb, name):
    """Every entry of S_l at full BASELINE size against F7: U* (T_l V) Sigma^-1 with T_l V by FFT
    convolution of the (noisy, for cfg4) grid (tests/f7_fft.py, pinned to the oracle on CPU)."""
    from f7_fft import fft_apply
    prob = W.make_problem(name)
    c = prob.cfg
    S = run_project(pb, prob).cpu().numpy()
    for ell in range(1, c.d + 1):
        want = prob.U.conj().T @ fft_apply(prob.grid, c.d, c.n, ell, prob.V) / prob.sigma[None, :]
        assert rel(S[ell - 1], want) <= TOL, ell


@pytest.mark.parametrize("m", [128, 97])
def test_full_size_max_m_all_entries(pb, orc, m):
    """The headline grid (d=2, n=200, N=40401, noisy) at m = PRONY_MAX_M = 128 (16 n-tiles: the 4-column-warp
    k_project layout and the 8-n-tile k_reduce_ws warps) and m = 97 (a packed 1-column last n-tile): every
    entry of S_l against F7, two sampled columns against the oracle, and the LS products against the oracle
    on a column sub-range."""
    from f7_fft import fft_apply
    cfg = W.custom_config(2, 200, m, 1e-6, 4242 + m)
    prob = W.make_problem(cfg, with_svd=False)
    rng = np.random.default_rng(m)
    N = cfg.N
    prob.U = W.random_orthonormal(N, m, rng)
    prob.V = W.random_orthonormal(N, m, rng)
    prob.sigma = np.sort(rng.random(m) + 0.5)[::-1].copy()
    S = run_project(pb, prob).cpu().numpy()
    for ell in (1, 2):
        want = prob.U.conj().T @ fft_apply(prob.grid, 2, 200, ell, prob.V) / prob.sigma[None, :]
        assert rel(S[ell - 1], want) <= TOL, ell
    cols = [0, m - 1]
    want = orc.project_columns(prob.grid, prob.U, prob.V, prob.sigma, 2, 200, 2, cols)
    assert rel(S[1][:, cols], want) <= TOL
    a, e = 1000, 9000
    out = pb.vandermonde_ls(dev(prob.z), dev(prob.grid), 2, 200, m, a, e, want_A=True)
    torch.cuda.synchronize()
    A_or = orc.vandermonde(prob.z, 2, 200, a, e)
    G_or, b_or = orc.ls_products(A_or, prob.grid, 2, 200, a, e)
    assert rel(out["A"], A_or) <= TOL and rel(out["G"], G_or) <= TOL and rel(out["b"], b_or) <= TOL


# ------------------------------------------------------------------ Vandermonde / LS parity
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_vandermonde_ls_configs(pb, orc, name):
    prob = W.make_problem(name, with_svd=False)
    c = prob.cfg
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = pb.vandermonde_ls(dev(prob.z), dev(prob.grid), c.d, c.n, c.m, want_A=True, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    A_or = orc.vandermonde(prob.z, c.d, c.n)
    G_or, b_or = orc.ls_products(A_or, prob.grid, c.d, c.n)
    assert rel(out["A"], A_or) <= TOL
    assert rel(out["G"], G_or) <= TOL
    assert rel(out["b"], b_or) <= TOL
    c_or = orc.cholesky_solve(G_or, b_or)
    assert rel(out["c"], c_or) <= 1e-9
    t = out["t"].cpu().numpy()
    assert W.torus_dist_inf(t, prob.t).max() <= 1e-8
    if c.noise == 0.0:
        assert rel(out["c"], prob.c) <= 1e-9


def test_vandermonde_ls_cfg4_full_size(pb, orc):
    prob = W.make_problem("cfg4", with_svd=False)
    c = prob.cfg
    out = pb.vandermonde_ls(dev(prob.z), dev(prob.grid), c.d, c.n, c.m, want_A=True)
    torch.cuda.synchronize()
    A_or = orc.vandermonde(prob.z, c.d, c.n)
    G_or, b_or = orc.ls_products(A_or, prob.grid, c.d, c.n)
    assert rel(out["A"], A_or) <= TOL
    assert rel(out["G"], G_or) <= TOL
    assert rel(out["b"], b_or) <= TOL
    assert W.torus_dist_inf(out["t"].cpu().numpy(), prob.t).max() <= 1e-8
    assert rel(out["c"], prob.c) <= 1e-5          # noisy sigma = 1e-6 data: c error ~ eps


@pytest.mark.parametrize("d,n,m", [(1, 30, 5), (2, 9, 1), (3, 5, 70), (4, 3, 9), (2, 11, 128)])
def test_vandermonde_ls_edges_and_ranges(pb, orc, d, n, m):
    rng = np.random.default_rng(d * 1000 + n * 10 + m)
    z = W.node_vectors(rng.random((m, d))) * (1.0 + 0.01 * (rng.random((m, d)) - 0.5))   # non-unit nodes
    grid = W.sample_grid(rng.random((3, d)), np.array([1.0, 0.5j, -2.0]), n, 1e-6, 3)
    N = (n + 1) ** d
    for a, e in [(0, N), (0, 1), (3, N - 2), (N // 2, N)]:
        out = pb.vandermonde_ls(dev(z), dev(grid), d, n, m, a, e, want_A=True)
        torch.cuda.synchronize()
        A_or = orc.vandermonde(z, d, n, a, e)
        G_or, b_or = orc.ls_products(A_or, grid, d, n, a, e)
        assert rel(out["A"], A_or) <= TOL
        assert rel(out["G"], G_or) <= TOL
        assert rel(out["b"], b_or) <= TOL


def test_ls_solve_singular_status(pb):
    m, d = 3, 2
    G = torch.tensor([[1, 2, 0], [2, 1, 0], [0, 0, 1]], dtype=torch.complex128, device="cuda")
    b = torch.ones(m, dtype=torch.complex128, device="cuda")
    z = torch.ones((m, d), dtype=torch.complex128, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    c, _ = pb.ls_solve(G, b, z, d, m, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == pb.PRONY_ERR_SINGULAR
    assert torch.isnan(c.real).all()


# ------------------------------------------------------------------ end to end from host buffers
def test_pencil_host_matches_device_path(pb, orc):
    prob = W.make_problem("cfg2")
    c = prob.cfg
    out = pb.pencil_host(prob.grid, prob.U, prob.V, prob.sigma, prob.z, c.d, c.n, c.m)
    assert out["status"] == 0
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n)
    for l in range(c.d):
        assert rel(out["S"][l], S_or[l]) <= TOL
    A_or = orc.vandermonde(prob.z, c.d, c.n)
    G_or, b_or = orc.ls_products(A_or, prob.grid, c.d, c.n)
    assert rel(out["G"], G_or) <= TOL and rel(out["b"], b_or) <= TOL
    assert W.torus_dist_inf(out["t"], prob.t).max() <= 1e-8


def test_pencil_host_context_reuse(pb, orc):
    """prony_host_context: one context serves many calls (different shapes included); results are bitwise those
    of the per-call-stream path (the same kernels in the same order) and match the oracle."""
    ctx = pb.HostContext()
    for name in ("cfg2", "cfg1", "cfg2"):
        prob = W.make_problem(name)
        c = prob.cfg
        a = pb.pencil_host(prob.grid, prob.U, prob.V, prob.sigma, prob.z, c.d, c.n, c.m, context=ctx)
        b = pb.pencil_host(prob.grid, prob.U, prob.V, prob.sigma, prob.z, c.d, c.n, c.m)
        assert a["status"] == 0 and b["status"] == 0
        for k in ("S", "G", "b", "c", "t"):
            assert np.array_equal(a[k], b[k]), k
        S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n)
        for l in range(c.d):
            assert rel(a["S"][l], S_or[l]) <= TOL
    ctx.close()


@pytest.mark.parametrize("d,n,m,noise", [(1, 300, 9, 1e-6), (3, 9, 13, 0.0), (2, 40, 37, 1e-6), (2, 5, 3, 0.0)])
def test_pencil_host_shapes(pb, orc, d, n, m, noise):
    """prony_pencil_host over shapes whose plans split K into several chunks (the copy/compute overlap
    path: chunk 0 on the caller's stream, chunks 1.. behind the rest of V) and a single-chunk one."""
    prob = problem(d, n, m, 700 + d + n + m, noise, random_uv=True)
    c = prob.cfg
    out = pb.pencil_host(prob.grid, prob.U, prob.V, prob.sigma, prob.z, d, n, m)
    assert out["status"] == 0
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    for l in range(d):
        assert rel(out["S"][l], S_or[l]) <= TOL
    A_or = orc.vandermonde(prob.z, d, n)
    G_or, b_or = orc.ls_products(A_or, prob.grid, d, n)
    assert rel(out["G"], G_or) <= TOL and rel(out["b"], b_or) <= TOL


@pytest.mark.parametrize("kc,cmul", [("2", "3m"), ("5", "3m"), ("7", "3m"), ("5", "4m")])
def test_pencil_host_chunk_groups(pb, orc, kc, cmul, monkeypatch):
    """The host-input pencil's copy pipeline with the split-K chunk count forced (PRONY_KC, read per call):
    the narrow lead chunk plus 1..3 launch groups of one or several chunks, each released by its own copy
    event (3M and 4M complex products); S, G, b against the oracle."""
    monkeypatch.setenv("PRONY_KC", kc)
    monkeypatch.setenv("PRONY_CMUL", cmul)
    prob = W.make_problem("cfg2")
    c = prob.cfg
    out = pb.pencil_host(prob.grid, prob.U, prob.V, prob.sigma, prob.z, c.d, c.n, c.m)
    assert out["status"] == 0
    S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n)
    for l in range(c.d):
        assert rel(out["S"][l], S_or[l]) <= TOL
    A_or = orc.vandermonde(prob.z, c.d, c.n)
    G_or, b_or = orc.ls_products(A_or, prob.grid, c.d, c.n)
    assert rel(out["G"], G_or) <= TOL and rel(out["b"], b_or) <= TOL


def test_end_to_end_recovery_with_oracle_tail(pb, orc):
    """Algorithm 1 with the GPU pencil: S from the device, then the oracle's eig / diagonalization
    (NEXT-1 runs those on the device); t within 1e-8 of planted (noise-free cfg3)."""
    prob = W.make_problem("cfg3")
    S = run_project(pb, prob).cpu().numpy()
    z, _, off = orc.diagonalize(S, orc.random_mu(prob.cfg.d, 1))
    t = orc.t_from_z(z)
    perm = orc.match_nodes(t, prob.t)
    assert W.torus_dist_inf(t[perm], prob.t).max() <= 1e-8
    out = pb.vandermonde_ls(dev(z), dev(prob.grid), prob.cfg.d, prob.cfg.n, prob.cfg.m)
    assert rel(out["c"].cpu().numpy()[perm], prob.c) <= 1e-8


@pytest.mark.parametrize("bad", ["tiny", "zero", "nan"])
def test_project_sigma_guard(pb, orc, bad):
    """Scale guard (SURVEY §8(b) conventions; SPEC compute_S errors): sigma_min <= N eps sigma_max,
    a zero or a non-finite sigma -> PRONY_ERR_SINGULAR in the device status word; a healthy sigma -> 0."""
    prob = problem(2, 6, 4, 31, random_uv=True)
    c = prob.cfg
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    run_project(pb, prob, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    sigma = prob.sigma.copy()
    sigma[-1] = {"tiny": sigma[0] * c.N * 1e-17, "zero": 0.0, "nan": np.nan}[bad]
    st.zero_()
    pb.project(dev(prob.grid), dev(prob.U), dev(prob.V), dev(sigma), c.d, c.n, c.m, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == pb.PRONY_ERR_SINGULAR


@pytest.mark.parametrize("d,n", [(2, 63), (3, 9), (4, 7)])
def test_toeplitz_matvec_dfma_dense(pb, orc, d, n):
    """The single-vector apply (DFMA Toeplitz matvec: q = 1 inner coordinate for n + 1 >= 64, q = 2 for
    shorter runs at d >= 3; NEXT-3's operator) against the oracle's dense T_l and T^H, with a strided
    input column and output column."""
    prob = problem(d, n, 3, 881 + d + n, 1e-6, random_uv=True)
    N = prob.cfg.N
    rng = np.random.default_rng(9)
    Xw = rng.standard_normal((N, 5)) + 1j * rng.standard_normal((N, 5))
    Xd = dev(Xw)
    grid = dev(prob.grid)
    Yw = torch.zeros((N, 3), dtype=torch.complex128, device="cuda")
    for ell in range(0, d + 1):
        pb.toeplitz_apply(grid, Xd[:, 2:3], d, n, ell, out=Yw[:, 1:2])
        T = orc.T_dense(prob.grid, d, n, ell)
        assert rel(Yw[:, 1].cpu().numpy(), T @ Xw[:, 2]) <= 1e-13
        del T
    pb.toeplitz_apply(grid, Xd[:, 2:3], d, n, 0, conj=True, out=Yw[:, 1:2])
    T = orc.T_dense(prob.grid, d, n, 0)
    assert rel(Yw[:, 1].cpu().numpy(), T.conj().T @ Xw[:, 2]) <= 1e-13
    Y = Yw.cpu().numpy()
    assert np.all(Y[:, 0] == 0) and np.all(Y[:, 2] == 0)


@pytest.mark.parametrize("d,n", [(3, 63), (3, 20), (4, 12)])
def test_toeplitz_matvec_dfma_sampled(pb, orc, monkeypatch, d, n):
    """Large shapes (d = 3, n = 63: N = 262144, q = 1; cfg3 / cfg5 sizes, q = 2): sampled rows of T_l x
    against the oracle (one row of T_l at a time via oracle.project_rows with a one-hot U); T x and
    T^H x against the DMMA apply path."""
    prob = problem(d, n, 2, 882, 0.0, random_uv=True)
    N = prob.cfg.N
    rng = np.random.default_rng(10)
    x = rng.standard_normal((N, 1)) + 1j * rng.standard_normal((N, 1))
    xd, grid = dev(x), dev(prob.grid)
    rows = sorted({0, 1, n, n + 1, (n + 1) ** 2 - 1, (n + 1) ** 2, N // 2 + 17, N - n - 2, N - 1})
    one = np.ones(1)
    for ell in sorted({1, 2, d}):
        y = pb.toeplitz_apply(grid, xd, d, n, ell).cpu().numpy()[:, 0]
        ref = []
        for k in rows:
            e = np.zeros((N, 1), complex)
            e[k, 0] = 1.0
            ref.append(orc.project_rows(prob.grid, e, x, one, d, n, ell, k, k + 1)[0, 0])
        assert rel(y[rows], np.array(ref)) <= 1e-13
    y0 = pb.toeplitz_apply(grid, xd, d, n, 0).cpu().numpy()
    yh = pb.toeplitz_apply(grid, xd, d, n, 0, conj=True).cpu().numpy()
    monkeypatch.setenv("PRONY_APPLY", "dmma")
    assert rel(y0, pb.toeplitz_apply(grid, xd, d, n, 0).cpu().numpy()) <= 1e-13
    assert rel(yh, pb.toeplitz_apply(grid, xd, d, n, 0, conj=True).cpu().numpy()) <= 1e-13


def test_cuda_graph_capture_and_replay(pb, orc):
    """prony.h promises stream-ordered, allocation-free calls that a CUDA graph can capture: one pencil
    (projection + LS products + solve) captured once and replayed on new inputs copied into the same
    buffers gives the oracle's pencil for those inputs."""
    probs = [problem(2, 20, 9, 1500 + i, 1e-6, random_uv=True) for i in range(2)]
    c = probs[0].cfg
    d, n, m = c.d, c.n, c.m
    bufs = {k: dev(getattr(probs[0], k)) for k in ("grid", "U", "V", "sigma", "z")}
    ws_p = pb.alloc_workspace(pb.WS_PROJECT, d, n, m)
    ws_l = pb.alloc_workspace(pb.WS_LS, d, n, m)
    S = torch.empty((d, m, m), dtype=torch.complex128, device="cuda")
    out = {"G": torch.empty((m, m), dtype=torch.complex128, device="cuda"),
           "b": torch.empty(m, dtype=torch.complex128, device="cuda"),
           "c": torch.empty(m, dtype=torch.complex128, device="cuda"),
           "t": torch.empty((m, d), dtype=torch.float64, device="cuda")}
    st = torch.cuda.Stream()

    def pencil():
        pb.project(bufs["grid"], bufs["U"], bufs["V"], bufs["sigma"], d, n, m, out=S, workspace=ws_p,
                   stream=torch.cuda.current_stream())
        pb.vandermonde_ls(bufs["z"], bufs["grid"], d, n, m, out=out, workspace=ws_l,
                          stream=torch.cuda.current_stream())

    with torch.cuda.stream(st):
        pencil()  # warm-up (sets kernel attributes outside the capture)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        pencil()
    for prob in probs[::-1]:
        for k in bufs:
            bufs[k].copy_(torch.from_numpy(np.ascontiguousarray(getattr(prob, k))))
        graph.replay()
        torch.cuda.synchronize()
        S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
        for l in range(d):
            assert rel(S[l], S_or[l]) <= TOL
        A_or = orc.vandermonde(prob.z, d, n)
        G_or, b_or = orc.ls_products(A_or, prob.grid, d, n)
        assert rel(out["G"], G_or) <= TOL and rel(out["b"], b_or) <= TOL


def test_project_random_shapes_and_ranges(pb, orc):
    """Seeded random sweep: d in 1..4, n, m (ragged tiles, m up to 40), random sub-ranges in all three
    unit orders, noise or not — each partial pencil against the oracle's rows of T_l."""
    rng = np.random.default_rng(4242)
    for it in range(24):
        d = int(rng.integers(1, 5))
        n = int(rng.integers(2, {1: 60, 2: 14, 3: 6, 4: 4}[d]))
        N = (n + 1) ** d
        m = int(rng.integers(1, min(40, N) + 1))
        prob = problem(d, n, m, 5000 + it, float(rng.choice([0.0, 1e-6])), random_uv=True)
        order = int(rng.integers(0, 3))
        U_tot = (n + 2) ** d if order == 2 else d * N
        a = int(rng.integers(0, U_tot))
        b = int(rng.integers(a, U_tot + 1))
        S = run_project(pb, prob, unit_begin=a, unit_end=b, unit_order=order)
        torch.cuda.synchronize()
        S_or = orc.project_units(prob.grid, prob.U, prob.V, prob.sigma, d, n, a, b, order)
        for l in range(d):
            if np.linalg.norm(S_or[l]) == 0:
                assert float(S[l].abs().max()) == 0.0, (it, d, n, m, order, a, b)
            else:
                assert rel(S[l], S_or[l]) <= TOL, (it, d, n, m, order, a, b)


def test_workspace_too_small_is_rejected(pb):
    """Every entry point checks workspace_bytes against prony_workspace_size before launching."""
    prob = problem(2, 6, 4, 77, random_uv=True)
    c = prob.cfg
    small = torch.empty(256, dtype=torch.uint8, device="cuda")
    with pytest.raises(pb.PronyError) as e:
        run_project(pb, prob, workspace=small)
    assert e.value.code == pb.PRONY_ERR_WORKSPACE
    with pytest.raises(pb.PronyError) as e:
        pb.vandermonde_ls(dev(prob.z), dev(prob.grid), c.d, c.n, c.m, workspace=small)
    assert e.value.code == pb.PRONY_ERR_WORKSPACE
    with pytest.raises(pb.PronyError) as e:
        pb.toeplitz_apply(dev(prob.grid), dev(prob.U), c.d, c.n, 0, workspace=small)
    assert e.value.code == pb.PRONY_ERR_WORKSPACE


def test_pencil_host_part_empty_and_partial(pb, orc):
    """prony_pencil_host_part: an empty unit / column range gives zero partials; a partial range equals
    the oracle's partial pencil and LS products over the same units / columns."""
    prob = problem(3, 5, 6, 909, 1e-6, random_uv=True)
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    S = torch.empty((d, m, m), dtype=torch.complex128, device="cuda")
    G = torch.empty((m, m), dtype=torch.complex128, device="cuda")
    b = torch.empty(m, dtype=torch.complex128, device="cuda")
    args = [pin(prob.grid), pin(prob.U), pin(prob.V), pin(prob.sigma), pin(prob.z), d, n, m]
    pb.pencil_host_part(*args, 40, 40, 17, 17, S, G, b)
    torch.cuda.synchronize()
    assert float(S.abs().max()) == 0.0 and float(G.abs().max()) == 0.0 and float(b.abs().max()) == 0.0
    E = (n + 2) ** d
    pb.pencil_host_part(*args, 37, E - 50, 11, N - 9, S, G, b)
    torch.cuda.synchronize()
    S_or = orc.project_units(prob.grid, prob.U, prob.V, prob.sigma, d, n, 37, E - 50, 2)
    for l in range(d):
        assert rel(S[l], S_or[l]) <= TOL
    A = orc.vandermonde(prob.z, d, n, 11, N - 9)
    G_or, b_or = orc.ls_products(A, prob.grid, d, n, 11, N - 9)
    assert rel(G, G_or) <= TOL and rel(b, b_or) <= TOL


def test_pencil_resets_and_reports_status(pb):
    """prony_pencil zeroes dev_status itself (first kernel, stream-ordered): a stale nonzero word from an earlier
    failure is cleared by a good pencil, and a bad sigma (below the scale guard) is reported by the next call."""
    prob = problem(2, 12, 5, 1777, 0.0, random_uv=True)
    c0 = prob.cfg
    d, n, m = c0.d, c0.n, c0.m
    pencil = pb.sharding.DistributedPencil(d, n, m, torch.device("cuda", 0))
    args = [dev(getattr(prob, k)) for k in ("grid", "U", "V", "sigma", "z")]
    pencil.status.fill_(pb.PRONY_ERR_SINGULAR)
    pencil(*args)
    torch.cuda.synchronize()
    assert int(pencil.status.item()) == 0
    bad_sigma = args[3].clone()
    bad_sigma[-1] = 0.0
    pencil(args[0], args[1], args[2], bad_sigma, args[4])
    torch.cuda.synchronize()
    assert int(pencil.status.item()) == pb.PRONY_ERR_SINGULAR
    pencil(*args)
    torch.cuda.synchronize()
    assert int(pencil.status.item()) == 0


def test_pencil_one_call_and_graph_replay(pb, orc):
    """prony_pencil (one C call: projection on the stream, LS + solve on the context's side stream) through
    sharding.DistributedPencil at N = 1, eager and captured once in a CUDA graph then replayed on new inputs
    copied into the same buffers: S, G, b, c, t against the oracle each time."""
    probs = [problem(2, 18, 11, 1700 + i, 1e-6, random_uv=True) for i in range(2)]
    c0 = probs[0].cfg
    d, n, m = c0.d, c0.n, c0.m
    bufs = {k: dev(getattr(probs[0], k)) for k in ("grid", "U", "V", "sigma", "z")}
    pencil = pb.sharding.DistributedPencil(d, n, m, torch.device("cuda", 0))
    st = torch.cuda.Stream()

    def check(prob, S, c, t):
        S_or = orc.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
        for l in range(d):
            assert rel(S[l], S_or[l]) <= TOL
        A_or = orc.vandermonde(prob.z, d, n)
        G_or, b_or = orc.ls_products(A_or, prob.grid, d, n)
        assert rel(pencil.G, G_or) <= TOL and rel(pencil.b, b_or) <= TOL
        assert rel(c, orc.cholesky_solve(G_or, b_or)) <= 1e-9
        assert np.max(np.abs(t.cpu().numpy() - orc.t_from_z(prob.z))) <= 1e-12
        assert int(pencil.status.item()) == 0

    with torch.cuda.stream(st):
        S, c, t = pencil(bufs["grid"], bufs["U"], bufs["V"], bufs["sigma"], bufs["z"], stream=st)
    torch.cuda.synchronize()
    check(probs[0], S, c, t)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        S, c, t = pencil(bufs["grid"], bufs["U"], bufs["V"], bufs["sigma"], bufs["z"], stream=st)
    for prob in probs[::-1]:
        for k in bufs:
            bufs[k].copy_(torch.from_numpy(np.ascontiguousarray(getattr(prob, k))))
        graph.replay()
        torch.cuda.synchronize()
        check(prob, S, c, t)
