"""Time prony_diagonalize (C_mu eig + W^-1 S_l W + t) at several m on the device (CUDA events), on a known
pencil S_l = X diag(z_l) X^-1. GPU box only; one JSON line per m."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_11430_b200 as pb  # noqa: E402
import workload as W  # noqa: E402

for m in [int(x) for x in (sys.argv[1:] or ["20", "50", "100"])]:
    d = 2
    rng = np.random.default_rng(m)
    z = W.node_vectors(rng.random((m, d)))
    X = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    S = np.stack([X @ np.diag(z[:, l]) @ np.linalg.inv(X) for l in range(d)])
    Sd = torch.from_numpy(S).cuda()
    mu = torch.from_numpy(W.random_mu(d, 1)).cuda()
    ws = pb.alloc_workspace(pb.WS_DIAG, d, m, m)
    for _ in range(2):
        pb.diagonalize(Sd, mu, d, m, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    zz, t, Wm = pb.diagonalize(Sd, mu, d, m, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    err = min(np.abs(zz.cpu().numpy()[:, 0][:, None] - z[None, :, 0]).min(axis=0).max(), 1.0)
    print(json.dumps({"m": m, "diagonalize_ms": e0.elapsed_time(e1), "max_node_err": float(err)}), flush=True)
