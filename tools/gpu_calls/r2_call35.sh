#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_algorithm1.py tests/test_gpu_lanczos.py -x -q > gpurun_out/r2_call35_alg1.log 2>&1; echo "alg1 rc=$?"; tail -3 gpurun_out/r2_call35_alg1.log
for c in cfg3 cfg5 cfg4; do timeout 300 python tools/build_pencil_once.py $c || exit 1; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bp_launches_cfg4_v3.csv python tools/build_pencil_once.py cfg4 > /dev/null 2>&1; echo "ncu list rc=$?"
