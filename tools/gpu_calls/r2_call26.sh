#!/bin/bash
# (first Householder-QR run: two passes per step; superseded by r2_call27)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_algorithm1.py -x -q > gpurun_out/r2_call26_alg1.log 2>&1
timeout 300 python tools/paper_table_timing.py > gpurun_out/r2_paper_table_hqr.jsonl 2>&1
for c in cfg2 cfg3 cfg5 cfg4; do timeout 300 python tools/algo1_timing.py $c; done > gpurun_out/r2_algo1_timing_hqr.jsonl 2>&1
