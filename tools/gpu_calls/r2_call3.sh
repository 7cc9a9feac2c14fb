#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_algorithm1.py tests/test_gpu_sharded.py -v -rA > gpurun_out/r2_call3_tests.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|Error|assert " gpurun_out/r2_call3_tests.log | head -40
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2_bench1.log | cut -c1-3000
