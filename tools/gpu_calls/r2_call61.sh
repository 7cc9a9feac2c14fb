#!/bin/bash
# ncu --set full of one k_toeplitz_mv launch (the Lanczos apply, cfg4)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
cat > /tmp/mv_case.py << 'PY'
import sys, os; sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch, paper_2012_11430_b200 as pb, workload as W
p = W.make_problem("cfg4", with_svd=False); c = p.cfg
g = torch.from_numpy(p.grid).cuda()
x = torch.randn(c.N, 1, dtype=torch.complex128, device="cuda")
for _ in range(4):
    y = pb.toeplitz_apply(g, x, c.d, c.n, 0, False)
torch.cuda.synchronize()
print("ok")
PY
grep -n "def toeplitz_apply" -A3 paper_2012_11430_b200/binding.py | head -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_mv -s 2 -c 1 -o gpurun_out/prof_mv python /tmp/mv_case.py > gpurun_out/ncu_mv.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_mv.log
python tools/ncu_summary.py gpurun_out/prof_mv.ncu-rep gpurun_out/ncu_mv.json > gpurun_out/ncu_mv_summary.txt 2>&1; head -30 gpurun_out/ncu_mv_summary.txt
