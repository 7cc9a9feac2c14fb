"""Host cost of one small pencil (cfg1): the public call path (sharding.DistributedPencil), the binding
(binding.pencil), and the bare C entry point with pre-marshalled arguments — where the eager launch time
goes when the GPU work is ~25 us. Wall clock per call, the GPU kept busy ahead (no host waits)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
from paper_2012_11430_b200 import binding as B  # noqa: E402
import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
prob = W.make_problem(name)
c = prob.cfg
d, n, m = c.d, c.n, c.m
dev = torch.device("cuda", 0)
tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
grid, U, V, sigma, z = tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z)
pencil = pb.sharding.DistributedPencil(d, n, m, dev)
st = torch.cuda.current_stream()
R = 2000


def timed(fn):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(50_000_000)  # keep the GPU busy so the host never waits on it
    t0 = time.perf_counter()
    for _ in range(R):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / R * 1e6


res = {"cfg": name}
res["DistributedPencil_us"] = timed(lambda: pencil(grid, U, V, sigma, z, stream=st))
ws = pencil.ws_pencil
ctx = pencil.ctx
outs = pencil.outs
res["binding_pencil_us"] = timed(lambda: pb.pencil(grid, U, V, sigma, z, d, n, m, outs, ws, context=ctx, stream=st))
L = B.lib()
args = (ctx.handle, d, n, m, B._ptr(grid), B._ptr(U), B._ptr(V), B._ptr(sigma), B._ptr(z), B._ptr(outs["S"]),
        B._ptr(outs["G"]), B._ptr(outs["b"]), B._ptr(outs["c"]), B._ptr(outs["t"]), B._ptr(ws), ws.numel(), None,
        B._stream(st), None, None)
res["bare_c_us"] = timed(lambda: L.prony_pencil(*args))
res["status_zero_us"] = timed(lambda: pencil.status.zero_())
print(json.dumps(res))
