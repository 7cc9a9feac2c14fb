#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_call31_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/r2_call31_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
