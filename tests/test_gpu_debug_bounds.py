"""Debug build (-DPRONY_DEBUG) of libprony: the implicit-Toeplitz gather checks every grid index it
forms against [0, box) and counts violations (compute-sanitizer is not available on this pool).
Runs the projection / apply paths of several shapes in a subprocess against that build."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes, os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch
import paper_2012_11430_b200 as pb
import workload as W
cases = [(2, 10, 3, 0.0), (2, 63, 20, 1e-6), (3, 6, 10, 0.0), (4, 3, 12, 1e-6), (1, 40, 7, 0.0), (2, 12, 100, 1e-6)]
for d, n, m, noise in cases:
    prob = W.make_problem(W.custom_config(d, n, m, noise, 3 + d + n + m))
    g = torch.from_numpy(prob.grid).cuda()
    U = torch.from_numpy(prob.U).cuda(); V = torch.from_numpy(prob.V).cuda(); s = torch.from_numpy(prob.sigma).cuda()
    N = prob.cfg.N
    pb.project(g, U, V, s, d, n, m)
    pb.project(g, U, V, s, d, n, m, 3, d * N - 5, 1)
    for ell in range(d + 1):
        pb.toeplitz_apply(g, V, d, n, ell)
    pb.toeplitz_apply(g, V, d, n, 0, conj=True)
L = ctypes.CDLL(os.environ["PRONY_LIB"])
L.prony_debug_violations.restype = ctypes.c_ulonglong
print("VIOLATIONS", L.prony_debug_violations())
"""


def test_gather_indices_in_bounds_debug_build():
    from paper_2012_11430_b200 import _build
    path = os.path.join(ROOT, "build", "libprony_debug.so")
    if _build._stale(path):
        os.makedirs(os.path.dirname(path), exist_ok=True)
        _build.build_variant(path, ["PRONY_DEBUG"])
    env = dict(os.environ, PRONY_LIB=path, ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("VIOLATIONS")][0]
    assert int(line.split()[1]) == 0, line
