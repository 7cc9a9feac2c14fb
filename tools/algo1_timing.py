"""Time Algorithm 1 on the device at a config (build_pencil = SVD + projection, diagonalize, LS) and
report recovery errors vs the planted parameters. Run on a GPU box."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
prob = W.make_problem(name, with_svd=False)
c = prob.cfg
grid = torch.from_numpy(prob.grid).cuda()
tol = 1e-6 if c.noise else None
ws = pb.alloc_workspace(pb.WS_BUILD, c.d, c.n, c.m)
mu = torch.from_numpy(W.random_mu(c.d, 2)).cuda()
res = {}
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pb.build_pencil(grid, c.d, c.n, c.m, seed=1, tol=tol, workspace=ws)
    t1 = time.perf_counter()
    z, t, _ = pb.diagonalize(out["S"], mu, c.d, c.m)
    ls = pb.vandermonde_ls(z, grid, c.d, c.n, c.m)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = {"cfg": name, "build_pencil_s": t1 - t0, "diag_ls_s": t2 - t1, "rank": out["rank"], "resid": out["resid"],
           "status": out["status"]}
# NEXT-3: the rank-agnostic Lanczos SVD (no m given; max_rank 2m+5) + projection
wl = pb.alloc_workspace(pb.WS_LANCZOS, c.d, c.n, min(2 * c.m + 5, 255))
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lz = pb.lanczos_svd(grid, c.d, c.n, max_rank=min(2 * c.m + 5, 255), tol=tol, seed=1, ldo=c.m, workspace=wl)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    S_lz = pb.project(grid, lz["U"], lz["V"], lz["sigma"], c.d, c.n, c.m)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
res.update({"lanczos_s": t1 - t0, "lanczos_project_s": t2 - t1, "lanczos_rank": lz["rank"],
            "lanczos_steps": lz["steps"], "lanczos_status": lz["status"]})
z2, t_lz, _ = pb.diagonalize(S_lz, mu, c.d, c.m)
tl = t_lz.cpu().numpy()
res["lanczos_t_err"] = float(W.torus_dist_inf(tl[oracle.match_nodes(tl, prob.t)], prob.t).max())
tt = t.cpu().numpy()
perm = oracle.match_nodes(tt, prob.t)
res["t_err"] = float(W.torus_dist_inf(tt[perm], prob.t).max())
res["c_err"] = float(np.linalg.norm(ls["c"].cpu().numpy()[perm] - prob.c) / np.linalg.norm(prob.c))
print(json.dumps(res))
