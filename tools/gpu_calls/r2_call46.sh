#!/bin/bash
# narrow lead chunk for the host-input pencil: parity + e2e A/B
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_p.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_p.log
for c in cfg4 cfg4 cfg5 cfg3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cfg $c > gpurun_out/bench_$c.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/bench_$c.log') if x.startswith('{')][-1]; j=json.loads(l); print('$c', round(j['value'],3), round(j['ms_per_step'],3), round(j['kernels_ms']['k_project'],3), 'e2e', round(j['e2e']['value'],3), round(j['e2e']['ms_per_step'],3))"; done
