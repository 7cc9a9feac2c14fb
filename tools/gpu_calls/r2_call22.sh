#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_call22_tests.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/r2_call22_tests.log
timeout 300 python tools/diag_timing.py 20 50 100 119 128 > gpurun_out/r2_diag_timing3.jsonl 2>&1; cat gpurun_out/r2_diag_timing3.jsonl
for c in cfg2 cfg3 cfg5 cfg4; do timeout 600 python tools/algo1_timing.py $c > gpurun_out/r2_algo1c_$c.json 2>&1; tail -1 gpurun_out/r2_algo1c_$c.json | cut -c1-200; done
