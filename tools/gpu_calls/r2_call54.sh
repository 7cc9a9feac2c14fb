#!/bin/bash
# N > 1 path without the wait on k_project's end: sharded tests (gloo 2 ranks, NCCL 1 rank) + force-dist bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1; echo "sharded rc=$?"; tail -2 gpurun_out/pytest_sharded.log
for c in cfg4 cfg5; do
timeout 300 python bench.py --gpus 1 --force-dist --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fd_$c.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/bench_fd_$c.log') if x.startswith('{')][-1]; j=json.loads(l); print('force-dist $c', round(j['value'],3), round(j['ms_per_step'],4), j['kernels_ms'], j['per_rank'][0]['allreduce_ms'], j['e2e']['value'])"
done
