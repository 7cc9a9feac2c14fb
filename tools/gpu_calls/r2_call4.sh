#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "vandermonde or ls_solve or pencil_host or cuda_graph or end_to_end" > gpurun_out/r2_call4_tests.log 2>&1; echo "pytest parity rc=$?"; tail -3 gpurun_out/r2_call4_tests.log
timeout 900 python -m pytest tests/test_gpu_algorithm1.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2_call4_tests2.log 2>&1; echo "pytest alg1 rc=$?"; tail -3 gpurun_out/r2_call4_tests2.log
for c in cfg4 cfg2; do timeout 300 python tools/timeline.py $c 8 > gpurun_out/r2_timeline_$c.json 2>&1; cat gpurun_out/r2_timeline_$c.json; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench2.log 2>&1; echo "bench rc=$?"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench2.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "kernels", j["kernels_ms"], "frac", j["roofline"]["frac"], "e2e", j["e2e"]["value"])
PY
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for K in k_vls k_solve; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K} -s 3 -c 1 -o gpurun_out/r2_prof_${K}_v1 python $SHORT > gpurun_out/r2_ncu_${K}_v1.log 2>&1; echo "ncu $K rc=$?"
done
