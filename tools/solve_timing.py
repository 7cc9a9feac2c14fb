"""Host-side timing of prony_ls_solve at m = 100 (one CTA Cholesky + substitutions); for the kernel's
own duration run it under `ncu --metrics gpu__time_duration.sum -k regex:k_solve`. GPU box only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402

m, d = 100, 2
rng = np.random.default_rng(0)
A = rng.standard_normal((m, 400)) + 1j * rng.standard_normal((m, 400))
G = torch.from_numpy(A @ A.conj().T).cuda()
b = torch.from_numpy(A @ (rng.standard_normal(400) + 0j)).cuda()
z = torch.from_numpy(np.exp(2j * np.pi * rng.random((m, d)))).cuda()
for _ in range(5):
    pb.ls_solve(G, b, z, d, m)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    c, t = pb.ls_solve(G, b, z, d, m)
e1.record()
torch.cuda.synchronize()
print("ls_solve ms per call (incl. host launch gaps):", e0.elapsed_time(e1) / 20)
