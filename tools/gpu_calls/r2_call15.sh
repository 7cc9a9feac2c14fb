#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
S=$(date +%s.%N); timeout 900 python bench.py > gpurun_out/r2_bench15_full.log 2> gpurun_out/r2_bench15_full.err; echo "bench rc=$? wall $(echo "$(date +%s.%N) - $S" | bc)"
python - << 'PY'
import json; j = json.loads([l for l in open("gpurun_out/r2_bench15_full.log") if l.startswith("{")][-1])
print("value", j["value"], "ms", j["ms_per_step"], "frac", j["roofline"]["frac"], "traffic", j["roofline"]["traffic"], j["roofline"]["traffic_source"], "e2e", j["e2e"]["value"], "cpu", j["cpu_baseline"]["value"], j["cpu_baseline"]["small_configs_1core"], "clocks", j["clocks"])
PY
S=$(date +%s.%N); timeout 900 python bench.py --impl reference > gpurun_out/r2_ref15.log 2> gpurun_out/r2_ref15.err; echo "ref rc=$? wall $(echo "$(date +%s.%N) - $S" | bc)"; cut -c1-600 gpurun_out/r2_ref15.log
