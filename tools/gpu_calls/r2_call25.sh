#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "project" > gpurun_out/r2_call25_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_call25_tests.log
for c in cfg2 cfg5 cfg3 cfg4; do timeout 300 python bench.py --cfg $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench25_$c.log 2>&1
python - $c << 'PY'
import json, sys; j = json.loads([l for l in open(f"gpurun_out/r2_bench25_{sys.argv[1]}.log") if l.startswith("{")][-1])
print(sys.argv[1], "value", round(j["value"],2), "ms", round(j["ms_per_step"],4), "k_project", round(j["kernels_ms"]["k_project"],4), "frac", round(j["roofline"]["frac"],3), "e2e", round(j["e2e"]["value"],2))
PY
done
