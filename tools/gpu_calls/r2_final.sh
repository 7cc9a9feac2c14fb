#!/bin/bash
# Round-2 evidence refresh: GPU suite, smoke, bench (+cpu_baseline), reference arm, other configs, launch list,
# stamped ncu --set full of k_project. Output under gpurun_out/.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
for c in cfg1 cfg2 cfg3 cfg5; do timeout 300 python bench.py --cfg $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project -s 3 -c 1 -o gpurun_out/prof_k_project_cfg4 python $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_k_project_cfg4.ncu-rep gpurun_out/ncu_k_project_current.json --stamp > gpurun_out/ncu_k_project_cfg4_summary.txt 2>&1
head -5 gpurun_out/ncu_k_project_cfg4_summary.txt
