#!/bin/bash
# Full GPU suite + smoke + bench + launch list on the current code (round 2, re-entry).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
bash tools/gpu_round.sh
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
