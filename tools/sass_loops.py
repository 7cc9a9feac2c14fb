"""List inner loops (backward branches) of a kernel's SASS with DMMA / spill counts."""
import re
import subprocess
import sys

lib, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s+Function : ", out)
body = [b for b in blocks if b.startswith(fn)]
if not body:
    sys.exit(f"function {fn} not found")
addr = []
for ln in body[0].splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        addr.append((int(m.group(1), 16), m.group(2).strip()))
print("instructions", len(addr), "DMMA", sum("DMMA" in i for _, i in addr),
      "LDL/STL", sum(("LDL" in i or "STL" in i) for _, i in addr))
for a, ins in addr:
    m = re.search(r"BRA (0x[0-9a-f]+)", ins)
    if m:
        t = int(m.group(1), 16)
        if t < a:
            b = [(x, i) for x, i in addr if t <= x <= a]
            nd = sum("DMMA" in i for _, i in b)
            nl = sum(("LDL" in i or "STL" in i) for _, i in b)
            if nd or nl:
                print(f"loop {hex(t)}-{hex(a)} instrs {len(b)} DMMA {nd} LDL/STL {nl}")
