#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/r2_bench14_full.log 2> gpurun_out/r2_bench14_full.err; echo "bench rc=$?"; grep "Elapsed" gpurun_out/r2_bench14_full.err
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench14_full.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "frac", j["roofline"]["frac"], "traffic", j["roofline"]["traffic"], j["roofline"]["traffic_source"], "e2e", j["e2e"]["value"], "cpu", j["cpu_baseline"]["value"], j["cpu_baseline"]["small_configs_1core"], "clocks", j["clocks"])
PY
/usr/bin/time -v timeout 900 python bench.py --impl reference > gpurun_out/r2_ref14.log 2> gpurun_out/r2_ref14.err; echo "ref rc=$?"; grep "Elapsed" gpurun_out/r2_ref14.err; cut -c1-400 gpurun_out/r2_ref14.log
SHORT="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_v8.csv python $SHORT > gpurun_out/ncu_launch14.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project -s 3 -c 1 -o gpurun_out/r2_prof_k_project_v10 python $SHORT > gpurun_out/r2_ncu_kp10.log 2>&1; echo "ncu kp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reduce_ws -s 3 -c 1 -o gpurun_out/r2_prof_k_reduce_ws_v4 python $SHORT > gpurun_out/r2_ncu_krws4.log 2>&1; echo "ncu krws rc=$?"
