#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/build_pencil_once.py cfg4 || exit 1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bp_launches_cfg4.csv python tools/build_pencil_once.py cfg4 > gpurun_out/r2_ncu28a.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_house_qr -s 1 -c 1 -o gpurun_out/r2_house_qr_cfg4 python tools/build_pencil_once.py cfg4 > gpurun_out/r2_ncu28b.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/r2_ncu28b.log
