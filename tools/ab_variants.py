"""Build k_project variants (-D flags) and print their spill counts; run with --time on a GPU box."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2012_11430_b200 import _build  # noqa: E402

VARIANTS = {
    "debug": ["PRONY_DEBUG"],
    "w8": ["PRONY_CONSUMER_WARPS=8"],
    "w8r224": ["PRONY_CONSUMER_WARPS=8", "PRONY_CONSUMER_REGS=224", "PRONY_PRODUCER_REGS=40"],
    "base": [],
    "kk2": ["PRONY_KK_UNROLL=2"],
    "kk1": ["PRONY_KK_UNROLL=1"],
    "g2": ["PRONY_GATHER_UNROLL=2"],
    "kk2g2": ["PRONY_KK_UNROLL=2", "PRONY_GATHER_UNROLL=2"],
    "r152p40": ["PRONY_CONSUMER_REGS=152", "PRONY_PRODUCER_REGS=40"],
    "bk8s6": ["PRONY_BK=8", "PRONY_STAGES=6"],
    "vt32": ["PRONY_VLS_TILE=32"],
    "vt64": ["PRONY_VLS_TILE=64"],
    "bk8s5": ["PRONY_BK=8", "PRONY_STAGES=5"],
    "solvet": ["PRONY_SOLVE_TIMING"],
    "sreg": ["PRONY_PROJ_SREG=1"],
    "sregkk2": ["PRONY_PROJ_SREG=1", "PRONY_KK_UNROLL=2"],
    "sregkk1": ["PRONY_PROJ_SREG=1", "PRONY_KK_UNROLL=1"],
}

if __name__ == "__main__":
    names = sys.argv[2:] if len(sys.argv) > 2 else list(VARIANTS)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    if sys.argv[1] == "--build":
        for n in names:
            path = os.path.join(ROOT, "build", f"libprony_{n}.so")
            os.makedirs(os.path.dirname(path), exist_ok=True)
            _build.build_variant(path, VARIANTS[n])
            for fn in ("_ZN5prony9k_projectILi5ELi3ELi3EEEvNS_10ProjParamsE",
                       "_ZN5prony9k_projectILi7ELi2ELi3EEEvNS_10ProjParamsE"):
                r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_loops.py"), path, fn],
                                   capture_output=True, text=True)
                if r.returncode == 0:
                    print(n, fn[14:30], r.stdout.splitlines()[0],
                          [l for l in r.stdout.splitlines() if "instrs 1" not in l and "loop" in l][:6])
    elif sys.argv[1] == "--time":
        for n in names:
            path = os.path.join(ROOT, "build", f"libprony_{n}.so")
            env = dict(os.environ, PRONY_LIB=path)
            try:
                out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                                      "--no-cpu-baseline"], capture_output=True, text=True, env=env, timeout=240).stdout
            except subprocess.TimeoutExpired:
                print(n, "TIMEOUT", flush=True)
                continue
            j = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])
            print(n, "k_project_ms=%.3f" % j["kernels_ms"]["k_project"], "TF=%.2f" % j["roofline"]["achieved"],
                  "pencils/s=%.3f" % j["value"], flush=True)
