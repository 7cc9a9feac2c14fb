"""Time the non-dominant sub-steps of one cfg4 pencil on the device (CUDA events around the library's
own main-kernel events) and report their rates: the LS step with and without the optional A write
(HBM-bound: 16 m N bytes), and the projection's k_project for context. Run on a GPU box; writes one JSON
line (profiles/r01_substeps.json keeps a copy)."""
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


def timed(fn, reps=10):
    ms = []
    for _ in range(3):
        fn(None)
    torch.cuda.synchronize()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e1.record()  # force creation before handing the handles to the library
        info = pb.make_exec_info(e0, e1)
        fn(info)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def main(name="cfg4"):
    prob = W.make_problem(name)
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    grid, z = tg(prob.grid), tg(prob.z)
    ws = pb.alloc_workspace(pb.WS_LS, d, n, m)
    A = torch.empty((m, N), dtype=torch.complex128, device="cuda")
    out = {"A": A, "G": torch.empty((m, m), dtype=torch.complex128, device="cuda"),
           "b": torch.empty(m, dtype=torch.complex128, device="cuda")}
    res = {"cfg": name, "N": N, "m": m}
    ms_noA = timed(lambda info: pb.vandermonde_ls(z, grid, d, n, m, want_solution=False, out=dict(out, A=None),
                                                  workspace=ws, info=info))
    ms_A = timed(lambda info: pb.vandermonde_ls(z, grid, d, n, m, want_A=True, want_solution=False, out=out,
                                                workspace=ws, info=info))
    a_bytes = 16.0 * m * N
    res["k_vls_ms"] = ms_noA
    res["k_vls_with_A_ms"] = ms_A
    res["A_write_bytes"] = a_bytes
    res["A_write_GBps_incremental"] = a_bytes / ((ms_A - ms_noA) * 1e-3) / 1e9 if ms_A > ms_noA else None
    res["k_vls_with_A_GBps"] = a_bytes / (ms_A * 1e-3) / 1e9
    res["k_vls_TFLOPs"] = (8.0 * m * m * N + 8.0 * m * N) / (ms_noA * 1e-3) / 1e12
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:])
