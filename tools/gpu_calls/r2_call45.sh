#!/bin/bash
# A/B: split-K chunk count (default 3 at cfg4) for the device and the e2e pencil
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for kc in 3 6 4 5 3; do
PRONY_KC=$kc timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cfg cfg4 > gpurun_out/bench_kc$kc.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/bench_kc$kc.log') if x.startswith('{')][-1]; j=json.loads(l); print('KC=$kc', round(j['value'],3), round(j['ms_per_step'],3), round(j['kernels_ms']['k_project'],3), 'e2e', round(j['e2e']['value'],3), round(j['e2e']['ms_per_step'],3), j['roofline']['grid'])"; done
