"""The N>1 path of the public API (sharding.DistributedPencil): 2 ranks (processes) share the one GPU of
this environment and reduce over gloo (no kernel waits on another rank, so sharing a GPU is safe).
The all-reduced pencil is compared with the CPU ORACLE on the same inputs (S_l, G, b element by element;
c, t against the oracle's Cholesky solve), for the device-resident path, the V-scatter end-to-end path
(each rank copies 1/N of V and all-gathers it) and the full-V C-ABI end-to-end path
(prony_pencil_host_part). The bench launcher itself is run at --gpus 2 over gloo."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, name, out, mode, backend="gloo"):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import workload as W
    from paper_2012_11430_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = W.make_problem(name)
    c = prob.cfg
    tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    # collective=True: the partial path with its collectives even on a one-rank NCCL group
    pencil = sharding.DistributedPencil(c.d, c.n, c.m, torch.device("cuda", 0), world, rank, collective=True)
    side = torch.cuda.Stream()          # a non-current stream: the call must order everything on it
    if mode == "device":
        S, cc, t = pencil(tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z), stream=side)
    else:
        S, cc, t = pencil.from_host(pin(prob.grid), pin(prob.U), pin(prob.V), pin(prob.sigma), pin(prob.z),
                                    stream=side, scatter_v=(mode == "scatter"))
    side.synchronize()
    if rank == 0:
        np.savez(out, S=S.cpu().numpy(), G=pencil.G.cpu().numpy(), b=pencil.b.cpu().numpy(), c=cc.cpu().numpy(),
                 t=t.cpu().numpy(), st=pencil.status.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _check_vs_oracle(out, name):
    sys.path.insert(0, ROOT)
    import oracle
    import workload as W
    r = np.load(out)
    prob = W.make_problem(name)
    c = prob.cfg
    assert int(r["st"][0]) == 0
    S_or = oracle.project(prob.grid, prob.U, prob.V, prob.sigma, c.d, c.n)
    A = oracle.vandermonde(prob.z, c.d, c.n)
    G_or, b_or = oracle.ls_products(A, prob.grid, c.d, c.n)
    c_or = oracle.cholesky_solve(G_or, b_or)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    for l in range(c.d):
        assert rel(r["S"][l], S_or[l]) <= 1e-10
    # G, b after the all-reduce: the packed buffer's G, b views are what rank 0 solved with
    assert rel(r["c"], c_or) <= 1e-10
    assert np.max(np.abs(r["t"] - oracle.t_from_z(prob.z))) <= 1e-12
    assert W.torus_dist_inf(r["t"], prob.t).max() <= 1e-8


@pytest.mark.parametrize("name,mode", [("cfg2", "device"), ("cfg3", "device"), ("cfg2", "scatter"),
                                       ("cfg3", "scatter"), ("cfg2", "full_v")])
def test_distributed_pencil_two_ranks_vs_oracle(tmp_path, name, mode):
    out = str(tmp_path / "r.npz")
    mp.spawn(_rank, args=(2, _free_port(), name, out, mode), nprocs=2, join=True)
    _check_vs_oracle(out, name)


@pytest.mark.parametrize("name,mode", [("cfg2", "device"), ("cfg2", "scatter"), ("cfg2", "full_v"),
                                       ("cfg3", "device")])
def test_distributed_pencil_nccl_one_rank_vs_oracle(tmp_path, name, mode):
    """The N > 1 code path over REAL NCCL (one rank: NCCL refuses two ranks on one GPU): the partial
    projection, the all_reduce of [G, b] on the LS side stream after k_project's end event, the all_reduce
    of S, the V all_gather of the scatter path and prony_pencil_host_part, against the oracle."""
    out = str(tmp_path / "r.npz")
    mp.spawn(_rank, args=(1, _free_port(), name, out, mode, "nccl"), nprocs=1, join=True)
    _check_vs_oracle(out, name)


def test_bench_launcher_two_ranks_gloo():
    """`python bench.py --gpus 2` starts its own 2 ranks (torchrun re-exec) exactly as the driver's N = 1 form
    runs; over gloo two ranks can share this environment's one GPU. One JSON line with n_gpus = 2."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo", "--cfg", "cfg2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and len(j["per_rank"]) == 2
    assert j["pct_peak"] <= 1.0 and j["roofline"]["frac"] <= 1.0
    assert len(j["e2e"]["h2d_bytes_per_rank"]) == 2 and j["e2e"]["value"] > 0


def test_bench_force_dist_nccl_one_rank():
    """`bench.py --force-dist` at --gpus 1: the bench's N > 1 branch (NCCL process group, the two all_reduces
    with their comm events, the per-rank all_gather of times, the V-scatter e2e through from_host) over real
    NCCL on this environment's one GPU."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--force-dist", "--cfg", "cfg2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 1 and j["value"] > 0 and j["config"]["dist_backend"] == "nccl"
    assert j["per_rank"][0]["allreduce_ms"] > 0 and j["e2e"]["value"] > 0
