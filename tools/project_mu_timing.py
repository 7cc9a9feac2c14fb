"""NEXT-4 vs the shared-row projection at cfg4: C_mu = U* B_mu V Sigma^-1 in one projection on the
combined grid (prony_project_mu) against all S_1..S_d (prony_project, SHARED units). Device-timed, median
of 5. GPU box only."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

prob = W.make_problem("cfg4")
c = prob.cfg
tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
grid, U, V, s = tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma)
mu = tg(W.random_mu(c.d, 3))
ws = pb.alloc_workspace(pb.WS_PROJECT_MU, c.d, c.n, c.m)
wsp = pb.alloc_workspace(pb.WS_PROJECT, c.d, c.n, c.m)


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


print({"project_mu_ms": timed(lambda: pb.project_mu(grid, U, V, s, mu, c.d, c.n, c.m, workspace=ws)),
       "project_all_S_ms": timed(lambda: pb.project(grid, U, V, s, c.d, c.n, c.m, workspace=wsp))})
