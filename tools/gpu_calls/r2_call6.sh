#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
PRONY_LIB=build/libprony_solvet.so timeout 120 python tools/solve_clock.py > gpurun_out/r2_solve_clock2.log 2>&1; grep -v "^k_solve m=1[02]" gpurun_out/r2_solve_clock2.log | tail -8; grep "m=100 clocks" gpurun_out/r2_solve_clock2.log | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_algorithm1.py -x -q -k "ls_solve or vandermonde or pencil_host or algorithm1 or accuracy or end_to_end" > gpurun_out/r2_call6_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_call6_tests.log
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 python $SHORT > gpurun_out/plain6.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_v3.csv python $SHORT > gpurun_out/ncu_launch6.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project -s 3 -c 1 -o gpurun_out/r2_prof_k_project_v3 python $SHORT > gpurun_out/r2_ncu_kp.log 2>&1; echo "ncu kp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 3 -c 1 -o gpurun_out/r2_prof_k_reduce_v3 python $SHORT > gpurun_out/r2_ncu_kr.log 2>&1; echo "ncu kr rc=$?"
