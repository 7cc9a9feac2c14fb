#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_call5_tests.log 2>&1; echo "pytest gpu rc=$?"; tail -5 gpurun_out/r2_call5_tests.log
for c in cfg4 cfg2 cfg3 cfg5; do timeout 300 python tools/timeline.py $c 8 hi > gpurun_out/r2_timeline5_$c.json 2>&1; cat gpurun_out/r2_timeline5_$c.json; done
timeout 300 python tools/timeline.py cfg4 8 > gpurun_out/r2_timeline5_cfg4_default.json 2>&1; cat gpurun_out/r2_timeline5_cfg4_default.json
PRONY_LIB=build/libprony_solvet.so timeout 120 python tools/solve_clock.py > gpurun_out/r2_solve_clock.log 2>&1; cat gpurun_out/r2_solve_clock.log | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench3.log 2>&1; echo "bench rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench3.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "kernels", j["kernels_ms"], "frac", j["roofline"]["frac"], "exec", j["roofline"]["executed_frac"], "e2e", j["e2e"]["value"])
PY
for c in cfg2 cfg3 cfg5; do timeout 300 python bench.py --cfg $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench3_$c.log 2>&1
python - $c << 'PY'
import json, sys; j = json.loads([l for l in open(f"gpurun_out/r2_bench3_{sys.argv[1]}.log") if l.startswith("{")][-1])
print(sys.argv[1], "value", round(j["value"],2), "ms", round(j["ms_per_step"],4), "kernels", j["kernels_ms"], "frac", round(j["roofline"]["frac"],3), "e2e", round(j["e2e"]["value"],2))
PY
done
