#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for c in cfg3 cfg5 cfg4; do timeout 300 python tools/build_pencil_once.py $c || exit 1; done
timeout 900 python -m pytest tests/test_gpu_algorithm1.py -x -q > gpurun_out/r2_call29_alg1.log 2>&1; echo "alg1 rc=$?"; tail -3 gpurun_out/r2_call29_alg1.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bp_launches_cfg4_v2.csv python tools/build_pencil_once.py cfg4 > gpurun_out/r2_ncu29a.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_house_qr -s 1 -c 1 -o gpurun_out/r2_house_qr_cfg4_v2 python tools/build_pencil_once.py cfg4 > gpurun_out/r2_ncu29b.log 2>&1; echo "ncu full rc=$?"
