#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_algorithm1.py -v -rA ${PYTEST_ARGS} > gpurun_out/r2_alg1.log 2>&1; echo "pytest rc=$?"
grep -E "PASS|FAIL|Error|assert" gpurun_out/r2_alg1.log | head -40
tail -3 gpurun_out/r2_alg1.log
