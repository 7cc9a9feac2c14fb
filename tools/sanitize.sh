#!/bin/bash
# compute-sanitizer on the small pencil paths (smoke: cfg1 project / LS / one-call pencil; host pencil cfg1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
cat > /tmp/san_case.py << 'PY'
import __graft_entry__ as g
g.smoke()
import numpy as np, paper_2012_11430_b200 as pb, workload as W
p = W.make_problem("cfg1"); c = p.cfg
out = pb.pencil_host(p.grid, p.U, p.V, p.sigma, p.z, c.d, c.n, c.m)
assert out["status"] == 0
print("SAN_CASE_OK")
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_case.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c SAN_CASE_OK gpurun_out/san_$tool.log) $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -1)"
done
