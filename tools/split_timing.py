"""Per-rank device time of the N-way sharded pencil, measured rank by rank on ONE B200 (no collective): for
N in {1, 2, 4, 8}, rank r runs its SHARED unit slab of prony_project and its column range of
prony_vandermonde_ls (+ the solve), with the streams of sharding.DistributedPencil at N > 1: the projection on a
high-priority stream, the LS branch on a normal one released right before k_project (so it runs in k_project's
last wave). The max over ranks plus an all-reduce estimate is the modelled step of an N-GPU run;
the driver's scaling run measures the real one."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
from paper_2012_11430_b200 import sharding  # noqa: E402
import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
prob = W.make_problem(name)
c = prob.cfg
d, n, m, N = c.d, c.n, c.m, c.N
tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
grid, U, V, sigma, z = tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z)
ws_p = pb.alloc_workspace(pb.WS_PROJECT, d, n, m)
ws_l = pb.alloc_workspace(pb.WS_LS, d, n, m)
S = torch.empty((d, m, m), dtype=torch.complex128, device="cuda")
G = torch.empty((m, m), dtype=torch.complex128, device="cuda")
b = torch.empty(m, dtype=torch.complex128, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()
main = torch.cuda.Stream(priority=-1)
out = {"cfg": name}
for world in (1, 2, 4, 8):
    per_rank = []
    for rank in range(world):
        u0, u1 = sharding.unit_range(d, n, world, rank)
        c0, c1 = sharding.column_range(d, n, world, rank)
        ts = []
        for rep in range(6):
            flush.fill_(rep & 0xFF)
            e0, e1, ep, pb0, pb1 = (torch.cuda.Event(enable_timing=True) for _ in range(5))
            for x in (pb0, pb1):
                x.record(main)
            torch.cuda.synchronize()
            e0.record(main)
            pb.project(grid, U, V, sigma, d, n, m, u0, u1, pb.UNITS_SHARED, out=S, workspace=ws_p, stream=main,
                       info=pb.make_exec_info(pb0, pb1))
            side.wait_event(pb0)  # recorded by the library right before k_project
            ls = pb.vandermonde_ls(z, grid, d, n, m, c0, c1, want_solution=False, out={"G": G, "b": b},
                                   workspace=ws_l, stream=side)
            pb.ls_solve(G, b, z, d, m, stream=side)
            ep.record(side)
            main.wait_event(ep)
            e1.record(main)
            torch.cuda.synchronize()
            if rep >= 2:
                ts.append(e0.elapsed_time(e1))
        per_rank.append(statistics.median(ts))
    out[f"N{world}"] = {"max_rank_ms": max(per_rank), "min_rank_ms": min(per_rank),
                        "speedup_vs_N1_model": None}
    print(json.dumps({"N": world, "per_rank_ms": [round(x, 3) for x in per_rank]}), flush=True)
base = out["N1"]["max_rank_ms"]
for world in (1, 2, 4, 8):
    out[f"N{world}"]["speedup_vs_N1_model"] = base / out[f"N{world}"]["max_rank_ms"]
print(json.dumps(out))
