#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q -k "sharded or two_ranks or launcher or pencil" > gpurun_out/r2_call17_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_call17_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench17.log 2>&1; echo "bench rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench17.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "kernels", j["kernels_ms"], "frac", j["roofline"]["frac"], "exec", j["roofline"]["executed_frac"], "launches", j["gpu_launches"], "grid", j["roofline"]["grid"], "e2e", j["e2e"]["value"])
PY
timeout 600 python bench.py --gpus 2 --dist-backend gloo --cfg cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench17_g2.log 2>&1; echo "bench g2 rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench17_g2.log") if l.startswith("{")][-1])
print("gloo x2 cfg3: value", j["value"], "per_rank", j["per_rank"], "launches", j["gpu_launches"])
PY
