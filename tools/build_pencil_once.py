"""One prony_build_pencil call at a config (for ncu launch lists of the NEXT-1 SVD): warm-up call, then one
profiled call bracketed by cudaProfilerStart/Stop."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
prob = W.make_problem(name, with_svd=False)
c = prob.cfg
grid = torch.from_numpy(prob.grid).cuda()
tol = 1e-6 if c.noise else None
ws = pb.alloc_workspace(pb.WS_BUILD, c.d, c.n, c.m)
walls = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pb.build_pencil(grid, c.d, c.n, c.m, seed=1, tol=tol, workspace=ws)
    torch.cuda.synchronize()
    walls.append(round(time.perf_counter() - t0, 5))
torch.cuda.cudart().cudaProfilerStart()
out = pb.build_pencil(grid, c.d, c.n, c.m, seed=1, tol=tol, workspace=ws)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({"cfg": name, "rank": out["rank"], "status": out["status"], "resid": out["resid"], "wall_s": walls})
