"""The paper's §2 timing table configurations (d=3, n=20, N=9261, m = 5/10/15/20, paper family,
noise-free) run through Algorithm 1 on one B200: block power SVD (Alg. 3) + S_l (build_pencil), the S_l
projection alone, diagonalization, A + LS. CUDA-event / wall timings, median of 5. Context only: the paper
ran on a Tesla K40c + 2 Xeons (full SVD ~80% of its total)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

d, n = 3, 20
N = (n + 1) ** d
for m in (5, 10, 15, 20):
    t_pl, c_pl = W.paper_family(d, m)
    grid = torch.from_numpy(W.sample_grid(t_pl, c_pl, n)).cuda()
    tol = N * 2.220446049250313e-16
    ws = pb.alloc_workspace(pb.WS_BUILD, d, n, m)
    mu = torch.from_numpy(W.random_mu(d, 2)).cuda()
    rec = {"build": [], "project": [], "diag": [], "ls": [], "total": []}
    for rep in range(7):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = pb.build_pencil(grid, d, n, m, seed=1, tol=tol, workspace=ws)
        t1 = time.perf_counter()
        z, t, _ = pb.diagonalize(out["S"], mu, d, m)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ls = pb.vandermonde_ls(z, grid, d, n, m)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pb.project(grid, out["U"], out["V"], out["sigma"], d, n, m)
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            rec["build"].append(t1 - t0)
            rec["diag"].append(t2 - t1)
            rec["ls"].append(t3 - t2)
            rec["total"].append(t3 - t0)
            rec["project"].append(e0.elapsed_time(e1) * 1e-3)
    tt = t.cpu().numpy()
    perm = oracle.match_nodes(tt, t_pl) if out["rank"] == m else None
    res = {"d": d, "n": n, "N": N, "m": m, "rank": out["rank"]}
    res.update({f"{k}_s": statistics.median(v) for k, v in rec.items()})
    if perm is not None:
        res["t_err"] = float(W.torus_dist_inf(tt[perm], t_pl).max())
        res["c_err"] = float(np.linalg.norm(ls["c"].cpu().numpy()[perm] - c_pl) / np.linalg.norm(c_pl))
    print(json.dumps(res), flush=True)
