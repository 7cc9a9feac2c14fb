#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_algorithm1.py -x -q > gpurun_out/r2_call27_alg1.log 2>&1; echo "alg1 rc=$?"; tail -15 gpurun_out/r2_call27_alg1.log
timeout 300 python tools/paper_table_timing.py > gpurun_out/r2_paper_table_hqr2.jsonl 2>&1; echo "table rc=$?"; cat gpurun_out/r2_paper_table_hqr2.jsonl | tail -5
for c in cfg2 cfg3 cfg5 cfg4; do timeout 300 python tools/algo1_timing.py $c; done > gpurun_out/r2_algo1_timing_hqr2.jsonl 2>&1; echo "algo1 rc=$?"; cat gpurun_out/r2_algo1_timing_hqr2.jsonl | cut -c1-300
