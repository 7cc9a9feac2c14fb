#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_call16_tests.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/r2_call16_tests.log
timeout 300 python tools/substeps.py > gpurun_out/r2_substeps.json 2>&1; cat gpurun_out/r2_substeps.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vls -s 13 -c 1 -o gpurun_out/r2_prof_k_vls_A python tools/substeps.py > gpurun_out/r2_ncu_vlsA.log 2>&1; echo "ncu vlsA rc=$?"
