#!/bin/bash
# ncu HBM counters of the staging / HBM-side kernels at cfg4: k_prep (P table, gsum, Vsum plane, E tables),
# k_vsum (e2e path), k_vls with and without the A write, k_powers
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_prep|k_vsum|k_powers|k_vls|k_ls_reduce|k_finalize" -s 10 -c 12 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_hbm.csv 2>/dev/null; echo "rc=$?"
python - << 'PY'
import csv, io
rows = list(csv.reader(open("gpurun_out/ncu_hbm.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
from collections import defaultdict
acc = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    key = (r[h.index("ID")], r[ki].split("(")[0].replace("void ", ""))
    acc[key][r[mi]] = (r[vi], r[ui])
for (i, k), d in acc.items():
    print(i, k, {m.split("__")[1].split(".")[0] if "__" in m else m: f"{v} {u}" for m, (v, u) in d.items()})
PY
