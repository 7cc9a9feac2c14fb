#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2_call34_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r2_call34_parity.log
timeout 300 python bench.py --cfg cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench34_cfg4.log 2>&1
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench34_cfg4.log") if l.startswith("{")][-1])
print("value", round(j["value"],2), "ms", round(j["ms_per_step"],4), "k_project", round(j["kernels_ms"]["k_project"],4), "outside", round(j["kernels_ms"]["outside_k_project"],4), "frac", round(j["roofline"]["frac"],3), "e2e", round(j["e2e"]["value"],2))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches34.csv python bench.py --cfg cfg4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 python tools/timeline.py cfg4 > gpurun_out/r2_timeline34_cfg4.json 2>&1; tail -c 600 gpurun_out/r2_timeline34_cfg4.json
