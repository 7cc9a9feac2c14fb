#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/paper_table_timing.py > gpurun_out/r2_paper_table_final.jsonl 2>&1; echo "table rc=$?"
for c in cfg2 cfg3 cfg5 cfg4; do timeout 300 python tools/algo1_timing.py $c; done > gpurun_out/r2_algo1_timing_final.jsonl 2>&1; echo "algo1 rc=$?"
