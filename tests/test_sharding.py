"""Multi-GPU sharding host logic on CPU: world_size-2 gloo processes each compute their share of the
pencil (unit range / column range) with the oracle, and sharding.allreduce_pencil (the same call the
GPU path makes over NCCL) must reproduce the single-process pencil."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2012_11430_b200 import sharding  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, d, n, m, order, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workload as W
    prob = W.make_problem(W.custom_config(d, n, m, 1e-6, 97), with_svd=True)
    u0, u1 = sharding.unit_range(d, n, world, rank, order)
    c0, c1 = sharding.column_range(d, n, world, rank)
    S = oracle.project_units(prob.grid, prob.U, prob.V, prob.sigma, d, n, u0, u1, order)
    A = oracle.vandermonde(prob.z, d, n, c0, c1)
    G, b = oracle.ls_products(A, prob.grid, d, n, c0, c1)
    Sr, Gr, br = sharding.allreduce_pencil(torch.from_numpy(S), torch.from_numpy(G), torch.from_numpy(b))
    if rank == 0:
        np.savez(out_path, S=Sr.numpy(), G=Gr.numpy(), b=br.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,n,m,order,world", [(3, 4, 6, 1, 2), (3, 4, 6, 0, 2), (2, 9, 5, 1, 2), (2, 9, 5, 2, 2),
                                               (3, 4, 6, 2, 2), (2, 9, 5, 2, 3)])
def test_allreduce_pencil_world2_gloo(tmp_path, oracle_mod, d, n, m, order, world):
    """world 2 (the contract's case) and an uneven world 3 split of the units and columns."""
    import workload as W
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), d, n, m, order, out), nprocs=world, join=True)
    res = np.load(out)
    prob = W.make_problem(W.custom_config(d, n, m, 1e-6, 97), with_svd=True)
    S = oracle_mod.project(prob.grid, prob.U, prob.V, prob.sigma, d, n)
    A = oracle_mod.vandermonde(prob.z, d, n)
    G, b = oracle_mod.ls_products(A, prob.grid, d, n)
    assert np.linalg.norm(res["S"] - S) / np.linalg.norm(S) < 1e-13
    assert np.linalg.norm(res["G"] - G) / np.linalg.norm(G) < 1e-13
    assert np.linalg.norm(res["b"] - b) / np.linalg.norm(b) < 1e-13


@pytest.mark.parametrize("total,parts", [(0, 1), (10, 3), (80802, 8), (7, 8)])
def test_split_range_partitions(total, parts):
    ranges = [sharding.split_range(total, parts, i) for i in range(parts)]
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    for (a, b), (c, _) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_default_unit_order():
    for d, world in [(3, 3), (2, 2), (3, 2), (2, 8), (2, 1)]:
        assert sharding.default_unit_order(d, world) == sharding.UNITS_SHARED
    assert sharding.unit_count(2, 200, sharding.UNITS_SHARED) == 202 ** 2
    assert sharding.unit_count(2, 200, sharding.UNITS_L_MAJOR) == 2 * 201 ** 2


@pytest.mark.parametrize("d,n", [(1, 6), (2, 3), (3, 2)])
def test_shared_units_cover_every_row_once(oracle_mod, d, n):
    """Unit order 2: over [0, (n+2)^d) every row k of every T_l is covered exactly once (so a partition
    of the units over ranks sums to the full pencil), and splitting the range splits the runs."""
    N = (n + 1) ** d
    E = (n + 2) ** d
    for ell in range(1, d + 1):
        runs = oracle_mod._shared_runs(d, n, ell, 0, E)
        rows = [k for a, b in runs for k in range(a, b)]
        assert rows == list(range(N))
        cut = E // 3
        left = oracle_mod._shared_runs(d, n, ell, 0, cut)
        right = oracle_mod._shared_runs(d, n, ell, cut, E)
        assert [k for a, b in left + right for k in range(a, b)] == list(range(N))


def test_pack_unpack_roundtrip():
    d, m = 3, 5
    S = torch.randn(d, m, m, dtype=torch.complex128)
    G = torch.randn(m, m, dtype=torch.complex128)
    b = torch.randn(m, dtype=torch.complex128)
    S2, G2, b2 = sharding.unpack(sharding.pack(S, G, b), d, m)
    assert torch.equal(S, S2) and torch.equal(G, G2) and torch.equal(b, b2)


@pytest.mark.parametrize("d,n", [(1, 5), (2, 4), (3, 3), (2, 9)])
def test_shared_u_rows_is_the_exact_range(d, n):
    """The U rows a SHARED unit slab pairs with (what prony_pencil_host_part copies): brute force over the
    slab's units and every l."""
    import random
    rng = random.Random(d * 10 + n)
    E = (n + 2) ** d
    for _ in range(60):
        a = rng.randrange(0, E)
        b = rng.randrange(a, E + 1)
        rows = set()
        for e in range(a, b):
            c, r = [], e
            for _ in range(d):
                c.append(r % (n + 2))
                r //= n + 2
            c = c[::-1]
            for ell in range(d):
                cc = list(c)
                cc[ell] -= 1
                if min(cc) < 0 or max(cc) > n:
                    continue
                k = 0
                for ci in cc:
                    k = k * (n + 1) + ci
                rows.add(k)
        want = (min(rows), max(rows) + 1) if rows else (0, 0)
        assert sharding.shared_u_rows(d, n, a, b) == want


def _gather_worker(rank, world, port, N, m, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V = torch.arange(N * m, dtype=torch.float64).reshape(N, m) * (1 + 1j)
    chunk, (v0, v1), _ = sharding.host_rows(2, int(round(N ** 0.5)) - 1, world, rank, sharding.UNITS_SHARED)
    buf = torch.zeros((chunk * world, m), dtype=torch.complex128)
    buf[v0:v1] = V[v0:v1]                       # only this rank's slice arrives from its host
    sharding.allgather_rows(buf, world, rank)
    ok = bool(torch.equal(buf[:N], V))
    torch.save(ok, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 9), (3, 4)])
def test_scatter_v_allgather_gloo(tmp_path, world, n):
    """The N > 1 end-to-end path copies 1/world of V per rank from the host and all_gathers the rest over
    the device interconnect: every rank must end with all of V (gloo, CPU)."""
    N, m = (n + 1) ** 2, 3
    out = str(tmp_path / "ok")
    mp.spawn(_gather_worker, args=(world, _free_port(), N, m, out), nprocs=world, join=True)
    assert all(torch.load(f"{out}.{r}") for r in range(world))


def test_h2d_bytes_scatter_model():
    """per-rank H2D of the N > 1 end-to-end path at cfg4 (d=2, n=200, m=100): the V scatter
    moves at most half of what the full-V path moved, at every N in {2, 4, 8}; the V slices partition [0, N)."""
    d, n, m = 2, 200, 100
    N = (n + 1) ** d
    for world in (2, 4, 8):
        rows = []
        for r in range(world):
            _, (v0, v1), (ulo, uhi) = sharding.host_rows(d, n, world, r)
            rows.append((v0, v1))
            new = sharding.h2d_bytes(d, n, m, world, r, scatter_v=True)
            old = sharding.h2d_bytes(d, n, m, world, r, scatter_v=False)
            assert new <= 0.5 * old if world >= 4 else new < 0.8 * old
        assert rows[0][0] == 0 and rows[-1][1] == N
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
