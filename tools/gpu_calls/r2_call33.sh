#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python tools/ab_variants.py --time base sreg sregkk2 sregkk1 base 2>&1 | tee gpurun_out/r2_ab_sreg.txt
