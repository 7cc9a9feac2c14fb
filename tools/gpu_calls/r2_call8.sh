#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/r2_call8_tests.log 2>&1; echo "pytest sharded rc=$?"; tail -3 gpurun_out/r2_call8_tests.log
timeout 600 python bench.py --gpus 2 --dist-backend gloo --cfg cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench8_g2.log 2>&1; echo "bench g2 rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench8_g2.log") if l.startswith("{")][-1])
print("gloo x2 on 1 GPU: value", j["value"], "ms", j["ms_per_step"], "per_rank", j["per_rank"], "e2e", j["e2e"])
PY
