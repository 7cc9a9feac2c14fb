#!/bin/bash
# row-owner gather (BM = 96 shapes): parity + per-config bench lines
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_bounds.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity.log
for c in cfg2 cfg3 cfg5 cfg4; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cfg $c > gpurun_out/bench_$c.log 2>&1
  python - $c << 'PY'
import json, sys
c = sys.argv[1]
l = [x for x in open(f"gpurun_out/bench_{c}.log") if x.startswith("{")]
if not l: print(c, "FAILED"); print(open(f"gpurun_out/bench_{c}.log").read()[-1500:]); sys.exit()
j = json.loads(l[-1])
print(c, "pencils/s=%.1f" % j["value"], "step_ms=%.4f" % j["ms_per_step"], "k_project_ms=%.4f" % j["kernels_ms"]["k_project"], "frac=%.3f" % j["roofline"]["frac"], "e2e=%.1f" % j["e2e"]["value"])
PY
done
