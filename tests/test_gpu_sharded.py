"""The N>1 path of the public API (sharding.DistributedPencil): 2 ranks (processes) share the one GPU of
this environment and reduce over gloo (no kernel waits on another rank, so sharing a GPU is safe);
the all-reduced pencil and the solved c, t must equal the single-process result."""
import os
import socket
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


def _rank(rank, world, port, name, out, from_host=False):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import workload as W
    from paper_2012_11430_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    prob = W.make_problem(name)
    c = prob.cfg
    tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    pencil = sharding.DistributedPencil(c.d, c.n, c.m, torch.device("cuda", 0), world, rank)
    if from_host:  # end to end from pinned host inputs: prony_pencil_host_part per rank
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        S, cc, t = pencil.from_host(pin(prob.grid), pin(prob.U), pin(prob.V), pin(prob.sigma), pin(prob.z),
                                    tg(prob.z))
    else:
        S, cc, t = pencil(tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z))
    torch.cuda.synchronize()
    if rank == 0:
        np.savez(out, S=S.cpu().numpy(), c=cc.cpu().numpy(), t=t.cpu().numpy(), st=pencil.status.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,from_host", [("cfg2", False), ("cfg3", False), ("cfg2", True), ("cfg3", True)])
def test_distributed_pencil_two_ranks(tmp_path, name, from_host):
    sys.path.insert(0, ROOT)
    import paper_2012_11430_b200 as pb
    import workload as W
    out = str(tmp_path / "r.npz")
    mp.spawn(_rank, args=(2, _free_port(), name, out, from_host), nprocs=2, join=True)
    r = np.load(out)
    prob = W.make_problem(name)
    c = prob.cfg
    tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    S1 = pb.project(tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), c.d, c.n, c.m).cpu().numpy()
    ls = pb.vandermonde_ls(tg(prob.z), tg(prob.grid), c.d, c.n, c.m)
    assert int(r["st"][0]) == 0
    for l in range(c.d):
        assert np.linalg.norm(r["S"][l] - S1[l]) / np.linalg.norm(S1[l]) <= 1e-12
    assert np.linalg.norm(r["c"] - ls["c"].cpu().numpy()) / np.linalg.norm(prob.c) <= 1e-12
    assert np.max(np.abs(r["t"] - ls["t"].cpu().numpy())) <= 1e-12
    assert W.torus_dist_inf(r["t"], prob.t).max() <= 1e-8
