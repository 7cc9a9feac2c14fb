#!/bin/bash
# Stamped ncu --set full of k_project (cfg4, current sources) + a cfg5 capture with source for analysis.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 python $SHORT > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project -s 3 -c 1 -o gpurun_out/prof_k_project_cfg4 python $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_k_project_cfg4.ncu-rep gpurun_out/ncu_k_project_current.json --stamp > gpurun_out/ncu_k_project_cfg4_summary.txt 2>&1
head -40 gpurun_out/ncu_k_project_cfg4_summary.txt
timeout 300 python $SHORT --cfg cfg5 > gpurun_out/plain5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_project -s 3 -c 1 -o gpurun_out/prof_k_project_cfg5 python $SHORT --cfg cfg5 > gpurun_out/ncu_full5.log 2>&1; echo "ncu full5 rc=$?"
python tools/ncu_summary.py gpurun_out/prof_k_project_cfg5.ncu-rep gpurun_out/ncu_k_project_cfg5_v10.json > gpurun_out/ncu_k_project_cfg5_summary.txt 2>&1
