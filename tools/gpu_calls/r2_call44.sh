#!/bin/bash
# LS side stream released after the prep kernels: timing A/B + the pencil/sharded tests
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
python tools/prio_timing.py cfg4 default,default_sync,split,split_sync
python tools/prio_timing.py cfg2 default,default_sync
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q -k "pencil or sharded or distributed or graph or bench" > gpurun_out/pytest_p.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_p.log
for c in cfg4 cfg2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cfg $c > gpurun_out/bench_$c.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/bench_$c.log') if x.startswith('{')][-1]; j=json.loads(l); print('$c', j['value'], j['ms_per_step'], j['kernels_ms'], j['e2e']['value'])"; done
timeout 300 python bench.py --gpus 1 --force-dist --cfg cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fd.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/bench_fd.log') if x.startswith('{')][-1]; j=json.loads(l); print('force-dist', j['value'], j['ms_per_step'], j['kernels_ms'], j['e2e']['value'])"
