"""Pencils/s of one GPU with the pencil (projection + LS products + solve, LS on a side stream as in
sharding.DistributedPencil) replayed from a CUDA graph vs launched eagerly — the serving case of many
small pencils, where launch overhead matters. Device-timed (CUDA events), L2 not flushed (steady-state
serving of resident inputs). GPU box only; one JSON line per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402


def main(names):
    for name in names:
        prob = W.make_problem(name)
        c = prob.cfg
        d, n, m = c.d, c.n, c.m
        tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        grid, U, V, sigma, z = (tg(getattr(prob, k)) for k in ("grid", "U", "V", "sigma", "z"))
        pencil = pb.sharding.DistributedPencil(d, n, m, torch.device("cuda", 0))
        st = torch.cuda.Stream()
        K = max(10, min(2000, int(2.0 / max(1e-5, 8 * m * c.N * (c.n + 2) ** d / 35e12))))
        with torch.cuda.stream(st):
            for _ in range(3):
                pencil(grid, U, V, sigma, z, stream=st)
        torch.cuda.synchronize()

        def timed(fn):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record(st)
                for _ in range(K):
                    fn()
                e1.record(st)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / K

        eager = timed(lambda: pencil(grid, U, V, sigma, z, stream=st))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            pencil(grid, U, V, sigma, z, stream=st)
        graph = timed(g.replay)
        print(json.dumps({"cfg": name, "reps": K, "eager_ms": eager, "graph_ms": graph,
                          "eager_pencils_per_s": 1e3 / eager, "graph_pencils_per_s": 1e3 / graph}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5", "cfg4"])
