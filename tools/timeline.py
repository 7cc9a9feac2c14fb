"""Per-step timeline of one pencil (device-resident inputs, N = 1): CUDA events on the main stream (before
the projection, around k_project, after k_finalize) and on the LS side stream (around k_vls, after k_solve),
all relative to the step's start. Shows what sits on the critical path outside k_project."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prob = W.make_problem(name)
c = prob.cfg
d, n, m, N = c.d, c.n, c.m, c.N
dev = torch.device("cuda", 0)
tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
grid, U, V, sigma, z = tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z)
ws_p = pb.alloc_workspace(pb.WS_PROJECT, d, n, m, dev)
ws_l = pb.alloc_workspace(pb.WS_LS, d, n, m, dev)
S = torch.empty((d, m, m), dtype=torch.complex128, device=dev)
# "hi": the projection on a high-priority stream (as sharding.DistributedPencil does), the LS on a normal one
main = torch.cuda.Stream(priority=-1) if "hi" in sys.argv[3:] else torch.cuda.current_stream()
side = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(main)
    return e


rows = []
for r in range(reps + 3):
    flush.fill_(r & 0xFF)
    e = {k: ev() for k in ("start", "p0", "p1", "main_end", "v0", "v1", "side_end", "all")}
    ip = pb.make_exec_info(e["p0"], e["p1"])
    il = pb.make_exec_info(e["v0"], e["v1"])
    torch.cuda.synchronize()
    torch.cuda.set_stream(main)
    e["start"].record(main)
    pb.project(grid, U, V, sigma, d, n, m, out=S, workspace=ws_p, stream=main, info=ip)
    e["main_end"].record(main)
    side.wait_event(e["start"])
    out = pb.vandermonde_ls(z, grid, d, n, m, workspace=ws_l, stream=side, info=il)
    e["side_end"].record(side)
    main.wait_stream(side)
    e["all"].record(main)
    torch.cuda.synchronize()
    if r >= 3:
        rows.append({k: e["start"].elapsed_time(v) for k, v in e.items() if k != "start"})
med = {k: statistics.median(x[k] for x in rows) for k in rows[0]}
print(json.dumps({"cfg": name, "priority_main": "hi" if "hi" in sys.argv[3:] else "default", "median_ms_from_start": med,
                  "k_project_ms": med["p1"] - med["p0"], "after_k_project_main_ms": med["main_end"] - med["p1"],
                  "before_k_project_ms": med["p0"], "k_vls_ms": med["v1"] - med["v0"],
                  "ls_tail_after_main_ms": med["all"] - med["main_end"], "step_ms": med["all"]}))
