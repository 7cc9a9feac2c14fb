#!/bin/bash
# bench (default), then a short bench plain + ncu launch list + ncu --set full of k_project.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline ${SHORT_ARGS}"
timeout 300 python $SHORT > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
if [ -n "${FULL_KERNEL}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${FULL_KERNEL} -s ${FULL_SKIP:-3} -c 1 -o gpurun_out/prof_${FULL_KERNEL} python $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
fi
