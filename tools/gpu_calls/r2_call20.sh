#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_diag_launches2.csv python tools/diag_timing.py 100 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/r2_diag_launches2.csv | head -10
