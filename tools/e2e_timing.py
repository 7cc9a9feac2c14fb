"""Where does the e2e (host-buffer) pencil lose time against the device-resident one? For prony_pencil_host_ctx:
wall-clock per call, device time e0 -> e1 as the bench measures it, and the same with the GPU kept busy by a
sleep kernel while the host enqueues the call (device-side cost only: the copies and kernels)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

for name in sys.argv[1:] or ["cfg4"]:
    prob = W.make_problem(name)
    c = prob.cfg
    d, n, m = c.d, c.n, c.m
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hg, hU, hV, hs, hz = pin(prob.grid), pin(prob.U), pin(prob.V), pin(prob.sigma), pin(prob.z)
    outs = {k: torch.empty(s, dtype=dt).pin_memory() for k, s, dt in
            [("S", (d, m, m), torch.complex128), ("G", (m, m), torch.complex128), ("b", (m,), torch.complex128),
             ("c", (m,), torch.complex128), ("t", (m, d), torch.float64)]}
    ws = pb.alloc_workspace(pb.WS_PENCIL_HOST, d, n, m)
    ctx = pb.HostContext()
    st = torch.cuda.current_stream()
    for _ in range(3):
        pb.pencil_host(hg, hU, hV, hs, hz, d, n, m, workspace=ws, outputs=outs, stream=st, context=ctx)
    res = {}
    for mode in ("plain", "sleep", "plain2"):
        wall, dev = [], []
        for i in range(8):
            torch.cuda.synchronize()
            if mode == "sleep":
                torch.cuda._sleep(4_000_000)  # ~2 ms of GPU busy-wait: the host enqueues behind it
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            t0 = time.perf_counter()
            pb.pencil_host(hg, hU, hV, hs, hz, d, n, m, workspace=ws, outputs=outs, stream=st, context=ctx)
            t1 = time.perf_counter()
            e1.record(st)
            e1.synchronize()
            wall.append((t1 - t0) * 1e3)
            dev.append(e0.elapsed_time(e1))
        res[mode] = {"wall_ms": statistics.median(wall), "event_ms": statistics.median(dev)}
    # host enqueue cost alone: time of the C call with the GPU held busy, up to its final synchronize
    print(json.dumps({"cfg": name, **res}))
