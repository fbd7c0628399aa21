"""Summarise `ncu -i rep --page source --csv` (SASS view): per kernel, the
dynamic instruction mix (warp-level instructions executed by opcode) and the
warp-stall samples by opcode.  Usage: python tools/ncu_source_summary.py rep.ncu-rep [kernel-substring]"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    kernels = []
    cur = None
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            kernels.append(cur)
            hdr = None
            continue
        if row[0] == "Address":
            hdr = row
            continue
        if cur is not None and hdr is not None:
            cur["rows"].append(dict(zip(hdr, row)))
    return kernels


FLOP_WEIGHTS = {"FFMA": 2, "FADD": 1, "FMUL": 1, "FFMA2": 4, "FADD2": 2, "FMUL2": 2}


def main():
    rep = sys.argv[1]
    sel = sys.argv[2] if len(sys.argv) > 2 else ""
    seen = set()
    for k in load(rep):
        if sel not in k["name"] or k["name"] in seen:   # the source page lists each kernel twice
            continue
        seen.add(k["name"])
        inst = Counter()
        stall = Counter()
        total_i = 0
        for r in k["rows"]:
            src = r.get("Source", "").strip()
            if src.startswith("@"):
                src = src.split(None, 1)[1]
            op = src.split()[0].split(".")[0] if src else "?"
            n = int(r.get("Instructions Executed", "0") or 0)
            s = int(r.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst[op] += n
            stall[op] += s
            total_i += n
        ts = sum(stall.values())
        print(f"== {k['name'][:90]}  warp-inst {total_i}")
        for op, n in inst.most_common(16):
            print(f"   {op:12s} {n:12d} {100*n/total_i:6.1f}%   stall-samples {100*stall[op]/max(ts,1):5.1f}%")
        # FP32 flops executed, counting the packed sm_100 forms (FFMA2 = 2 FMAs
        # = 4 flops per lane); warp instructions x 32 lanes (an upper bound:
        # partial warps are counted full)
        fl = 32 * sum(inst[o] * w for o, w in FLOP_WEIGHTS.items())
        print(f"   exec-fp32-flops {fl}")


if __name__ == "__main__":
    main()
