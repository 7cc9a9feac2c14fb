#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench0.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2_bench0.log | cut -c1-600
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for K in k_vls k_reduce k_finalize k_solve; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K} -s 3 -c 1 -o gpurun_out/r2_prof_${K}_v0 python $SHORT > gpurun_out/r2_ncu_${K}.log 2>&1; echo "ncu $K rc=$?"
done
