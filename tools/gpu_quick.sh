#!/bin/bash
# quick kernel timing of both complex modes + one ncu capture of k_project
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
for mode in 3m 4m; do
  PRONY_CMUL=$mode timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${QARGS} > gpurun_out/quick_$mode.log 2>&1
  python - "$mode" << 'PY'
import json, sys
l = [x for x in open(f"gpurun_out/quick_{sys.argv[1]}.log") if x.startswith("{")]
if not l: print(sys.argv[1], "FAILED"); print(open(f"gpurun_out/quick_{sys.argv[1]}.log").read()[-2000:]); sys.exit()
j = json.loads(l[-1])
print(sys.argv[1], j["config"]["workload"], "pencils/s=%.3f" % j["value"], "step_ms=%.3f" % j["ms_per_step"], "k_project_ms=%.3f" % j["kernels_ms"]["k_project"], "k_vls_ms=%.3f" % j["kernels_ms"]["k_vls"], "proj_TF=%.2f" % j["roofline"]["achieved"], "frac=%.3f" % j["roofline"]["frac"], "grid", j["roofline"]["grid"])
PY
done
if [ -n "${FULL_KERNEL}" ]; then
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline ${QARGS}"
timeout 300 python $SHORT > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${FULL_KERNEL} -s ${FULL_SKIP:-3} -c 1 -o gpurun_out/prof_${FULL_KERNEL} python $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
