#!/bin/bash
# refresh: per-rank split timing (N-way model), Algorithm 1 device timings, the paper's table timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python tools/split_timing.py cfg4 > gpurun_out/split_cfg4.jsonl 2>&1; tail -1 gpurun_out/split_cfg4.jsonl
python tools/split_timing.py cfg5 > gpurun_out/split_cfg5.jsonl 2>&1; tail -1 gpurun_out/split_cfg5.jsonl
for c in cfg2 cfg3 cfg5 cfg4; do timeout 600 python tools/algo1_timing.py $c >> gpurun_out/algo1.jsonl 2>&1; done; cat gpurun_out/algo1.jsonl | tail -4
timeout 600 python tools/paper_table_timing.py > gpurun_out/paper_table.jsonl 2>&1; tail -4 gpurun_out/paper_table.jsonl
