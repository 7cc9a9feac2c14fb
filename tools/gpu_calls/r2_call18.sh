#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python tools/diag_timing.py 20 50 100 128 > gpurun_out/r2_diag_timing.jsonl 2>&1; cat gpurun_out/r2_diag_timing.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_diag_launches.csv python tools/diag_timing.py 100 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/r2_diag_launches.csv --prony | head -8
for c in cfg2 cfg3 cfg5 cfg4; do timeout 600 python tools/algo1_timing.py $c > gpurun_out/r2_algo1_$c.json 2>&1; tail -1 gpurun_out/r2_algo1_$c.json; done
