#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
PRONY_LIB=build/libprony_solvet.so timeout 120 python tools/solve_clock.py > gpurun_out/r2_solve_clock3.log 2>&1; grep "m=100 clocks\|m=20 clocks\|m=128 clocks" gpurun_out/r2_solve_clock3.log | tail -3; grep residual gpurun_out/r2_solve_clock3.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_call7_tests.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/r2_call7_tests.log
for c in cfg4 cfg2; do timeout 300 python tools/timeline.py $c 8 hi > gpurun_out/r2_timeline7_$c.json 2>&1; cat gpurun_out/r2_timeline7_$c.json; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench7.log 2>&1; echo "bench rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench7.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "kernels", j["kernels_ms"], "frac", j["roofline"]["frac"], "traffic", j["roofline"]["traffic"], j["roofline"]["traffic_source"], "e2e", j["e2e"]["value"])
PY
timeout 300 python bench.py --cfg cfg2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench7_cfg2.log 2>&1
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench7_cfg2.log") if l.startswith("{")][-1])
print("cfg2 value", j["value"], "ms", j["ms_per_step"], "kernels", j["kernels_ms"], "e2e", j["e2e"]["value"])
PY
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_v4.csv python $SHORT > gpurun_out/ncu_launch7.log 2>&1; echo "ncu launch rc=$?"
