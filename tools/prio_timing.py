"""A/B: prony_pencil with the caller's stream at default vs high priority (cfg4, L2 flushed, CUDA events):
does the LS side stream's k_vls delay k_project's last wave when both have the same priority?"""
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
K = 10
prob = W.make_problem(name)
c = prob.cfg
d, n, m = c.d, c.n, c.m
dev = torch.device("cuda", 0)
tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
grid, U, V, sigma, z = tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z)
outs = {"S": torch.empty((d, m, m), dtype=torch.complex128, device=dev),
        "G": torch.empty((m, m), dtype=torch.complex128, device=dev),
        "b": torch.empty(m, dtype=torch.complex128, device=dev), "c": torch.empty(m, dtype=torch.complex128, device=dev),
        "t": torch.empty((m, d), dtype=torch.float64, device=dev)}
ws = pb.alloc_workspace(pb.WS_PENCIL, d, n, m, dev)
ctx = pb.HostContext()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
ws_p = pb.alloc_workspace(pb.WS_PROJECT, d, n, m, dev)
ws_l = pb.alloc_workspace(pb.WS_LS, d, n, m, dev)
side = torch.cuda.Stream()
ev_in = torch.cuda.Event()


def split_call(st, info_p, info_l=None):
    """the timeline's form: prony_project on st, prony_vandermonde_ls on a torch side stream, joined"""
    ev_in.record(st)
    pb.project(grid, U, V, sigma, d, n, m, out=outs["S"], workspace=ws_p, stream=st, info=info_p)
    side.wait_event(ev_in)
    pb.vandermonde_ls(z, grid, d, n, m, workspace=ws_l, stream=side, info=info_l)
    st.wait_stream(side)


modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["default", "high", "split", "default2", "split2"]
for label in modes:
    prio = -1 if label.startswith("high") else 0
    st = torch.cuda.Stream(priority=prio) if prio else torch.cuda.current_stream()
    evs = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(K)]  # noqa: E731
    es, ee, ps, pe, vs, ve = evs(), evs(), evs(), evs(), evs(), evs()
    for e in es + ee + ps + pe + vs + ve:
        e.record(st)
    call = (lambda st, ip, il: split_call(st, ip, il)) if label.startswith("split") else (
        lambda st, ip, il: pb.pencil(grid, U, V, sigma, z, d, n, m, outs, ws, context=ctx, stream=st, info_p=ip,
                                     info_l=il))
    for _ in range(3):
        call(st, None, None)
    torch.cuda.synchronize()
    for i in range(K):
        if "noflush" not in label:
            with torch.cuda.stream(st):
                flush.fill_(i & 0xFF)
        if "sync" in label:
            torch.cuda.synchronize()
        es[i].record(st)
        call(st, pb.make_exec_info(ps[i], pe[i]), pb.make_exec_info(vs[i], ve[i]))
        ee[i].record(st)
    torch.cuda.synchronize()
    step = [es[i].elapsed_time(ee[i]) for i in range(K)]
    proj = [ps[i].elapsed_time(pe[i]) for i in range(K)]
    res[label] = {"step_ms": statistics.median(step), "k_project_ms": statistics.median(proj),
                  "outside_ms": statistics.median([a - b for a, b in zip(step, proj)]),
                  "before_ms": statistics.median([es[i].elapsed_time(ps[i]) for i in range(K)]),
                  "after_ms": statistics.median([pe[i].elapsed_time(ee[i]) for i in range(K)]),
                  "vls_start_ms": statistics.median([es[i].elapsed_time(vs[i]) for i in range(K)]),
                  "vls_end_ms": statistics.median([es[i].elapsed_time(ve[i]) for i in range(K)])}
print(json.dumps({"cfg": name, **res}))
