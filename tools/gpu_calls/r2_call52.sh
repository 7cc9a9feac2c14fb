#!/bin/bash
# A/B: V/Vsum bulk copies with an L2 evict_last policy (default build) vs the default policy
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "
from paper_2012_11430_b200 import _build; import os
os.makedirs('build', exist_ok=True); _build.build_variant('build/libprony_noevict.so', ['PRONY_V_EVICT_LAST=0'])" || exit 1
SHORT="bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for lib in paper_2012_11430_b200/libprony.so build/libprony_noevict.so paper_2012_11430_b200/libprony.so build/libprony_noevict.so; do
  PRONY_LIB=$lib timeout 300 python $SHORT > /tmp/b.log 2>&1; python -c "
import json; l=[x for x in open('/tmp/b.log') if x.startswith('{')][-1]; j=json.loads(l); print('$lib', round(j['value'],3), round(j['kernels_ms']['k_project'],4), round(j['roofline']['frac'],4))"
done
for lib in paper_2012_11430_b200/libprony.so build/libprony_noevict.so; do
  PRONY_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_project -s 3 -c 1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__|duration|hit_rate" | sed "s|^|$lib |"
done
