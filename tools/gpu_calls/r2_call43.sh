#!/bin/bash
# the sharded tests (gloo 2 ranks + NCCL one rank + bench --force-dist)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1; echo "sharded rc=$?"; tail -30 gpurun_out/pytest_sharded.log
timeout 300 python bench.py --gpus 1 --force-dist --cfg cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_force_dist.log 2>&1; echo "bench fd rc=$?"; grep -E "NCCL INFO (comm|Init)" gpurun_out/bench_force_dist.log | head -3; tail -1 gpurun_out/bench_force_dist.log | cut -c1-600
