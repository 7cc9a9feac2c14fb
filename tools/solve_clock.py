"""k_solve phase clocks (build variant with -DPRONY_SOLVE_TIMING, loaded through PRONY_LIB): load / panel
factorizations / trailing updates / substitutions, printed by the kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402

for m in (20, 50, 100, 128):
    rng = np.random.default_rng(m)
    X = rng.standard_normal((m, 3 * m)) + 1j * rng.standard_normal((m, 3 * m))
    G = torch.from_numpy(X @ X.conj().T).cuda()
    b = torch.from_numpy(rng.standard_normal(m) + 1j * rng.standard_normal(m)).cuda()
    z = torch.ones((m, 2), dtype=torch.complex128, device="cuda")
    for _ in range(3):
        c, _ = pb.ls_solve(G, b, z, 2, m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c, _ = pb.ls_solve(G, b, z, 2, m)
    e1.record()
    torch.cuda.synchronize()
    err = np.linalg.norm(G.cpu().numpy() @ c.conj().cpu().numpy() - b.cpu().numpy()) / np.linalg.norm(b.cpu().numpy())
    print(f"m={m} ls_solve {e0.elapsed_time(e1) * 1e3:.1f} us residual {err:.2e}", flush=True)
