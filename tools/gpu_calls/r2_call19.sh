#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_algorithm1.py -x -q > gpurun_out/r2_call19_tests.log 2>&1; echo "pytest alg1 rc=$?"; tail -25 gpurun_out/r2_call19_tests.log | grep -v "^$" | tail -20
timeout 300 python tools/diag_timing.py 20 50 100 128 > gpurun_out/r2_diag_timing2.jsonl 2>&1; cat gpurun_out/r2_diag_timing2.jsonl
for c in cfg4; do timeout 600 python tools/algo1_timing.py $c > gpurun_out/r2_algo1b_$c.json 2>&1; tail -1 gpurun_out/r2_algo1b_$c.json; done
