#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_call11_tests.log 2>&1; echo "pytest gpu rc=$?"; tail -15 gpurun_out/r2_call11_tests.log
timeout 300 python tools/timeline.py cfg4 8 > gpurun_out/r2_timeline11_cfg4.json 2>&1; cat gpurun_out/r2_timeline11_cfg4.json
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench11.log 2>&1; echo "bench rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench11.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "kernels", j["kernels_ms"], "frac", j["roofline"]["frac"], "e2e", j["e2e"]["value"])
PY
for c in cfg2 cfg3 cfg5; do timeout 300 python bench.py --cfg $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench11_$c.log 2>&1
python - $c << 'PY'
import json, sys; j = json.loads([l for l in open(f"gpurun_out/r2_bench11_{sys.argv[1]}.log") if l.startswith("{")][-1])
print(sys.argv[1], "value", round(j["value"],2), "ms", round(j["ms_per_step"],4), "k_project", round(j["kernels_ms"]["k_project"],4), "frac", round(j["roofline"]["frac"],3), "e2e", round(j["e2e"]["value"],2))
PY
done
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_v6.csv python $SHORT > gpurun_out/ncu_launch11.log 2>&1; echo "ncu launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reduce_ws -s 3 -c 1 -o gpurun_out/r2_prof_k_reduce_ws_v2 python $SHORT > gpurun_out/r2_ncu_krws2.log 2>&1; echo "ncu krws rc=$?"
