"""Roofline of the Toeplitz apply that the NEXT rows run on (block power SVD: r = 2m columns; Lanczos:
r = 1): Y = T X at cfg4 for several r, device-timed with CUDA events (median of 5 after 2 warm-ups,
workspace preallocated), against the cuBLAS ZGEMM rate measured in the same process. Algorithmic flops
8 r N^2 (ZGEMM convention). GPU box only; prints one JSON line."""
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


def ev_time(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main(name="cfg4"):
    prob = W.make_problem(name, with_svd=False)
    c = prob.cfg
    N = c.N
    grid = torch.from_numpy(prob.grid).cuda()
    ws = pb.alloc_workspace(pb.WS_APPLY, c.d, c.n, 1)
    a = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
    zg_ms = ev_time(lambda: a @ a, reps=5)
    zgemm = 8 * 4096 ** 3 / (zg_ms * 1e-3) / 1e12
    res = {"cfg": name, "N": N, "zgemm_tflops": zgemm, "apply": []}
    for r in (1, 8, 32, 100, 200):
        X = torch.randn(N, r, dtype=torch.complex128, device="cuda")
        Y = torch.empty_like(X)
        for conj in (False, True):
            ms = ev_time(lambda: pb.toeplitz_apply(grid, X, c.d, c.n, 0, conj, out=Y, workspace=ws))
            tf = 8.0 * r * N * N / (ms * 1e-3) / 1e12
            res["apply"].append({"r": r, "conj": conj, "ms": ms, "tflops": tf, "frac_vs_zgemm": tf / zgemm})
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:])
