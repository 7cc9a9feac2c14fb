#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_call32_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2_call32_parity.log
for c in cfg4 cfg3 cfg5 cfg2; do timeout 300 python bench.py --cfg $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench32_$c.log 2>&1
python - $c << 'PY'
import json, sys; j = json.loads([l for l in open(f"gpurun_out/r2_bench32_{sys.argv[1]}.log") if l.startswith("{")][-1])
print(sys.argv[1], "value", round(j["value"],2), "ms", round(j["ms_per_step"],4), "k_project", round(j["kernels_ms"]["k_project"],4), "outside", round(j["kernels_ms"]["outside_k_project"],4), "frac", round(j["roofline"]["frac"],3), "e2e", round(j["e2e"]["value"],2))
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_reduce --csv --log-file gpurun_out/r2_reduce_launches32.csv python bench.py --cfg cfg4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_reduce_ws -s 2 -c 1 -o gpurun_out/r2_prof_k_reduce_ws_v5 python bench.py --cfg cfg4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
