"""Instruction mix per kernel from `cuobjdump -sass libvf.so` (run here, no GPU)."""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1009_0959_b200/libvf.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    ops = []
    for line in re.findall(r"/\*[0-9a-f]{4,6}\*/\s+(.*?);", f):
        l = line.strip()
        if l.startswith("@"):
            l = l.split(None, 1)[1]
        ops.append(l.split()[0].split(".")[0])
    c = Counter(ops)
    fp = c["FFMA"] + c["FMUL"] + c["FADD"]
    print(f"{name[:60]:60s} n={len(ops):6d} FP32={fp:6d} MUFU={c['MUFU']:4d} LDL={c['LDL']} STL={c['STL']} "
          + ", ".join(f"{k}:{v}" for k, v in c.most_common(10)))
