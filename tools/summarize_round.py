"""Turn a round's gpurun_out/ artefacts into committed evidence under profiles/:
  profiles/<tag>_launches_summary.md   kernel shares of the bench command's ncu launch list
  profiles/<tag>_launches.csv          the launch list itself (ncu --metrics gpu__time_duration.sum)
  profiles/<tag>_ncu_<cfg>.md          per-kernel ncu --set full metrics (C2, C4)
  profiles/<tag>_bench_<cfg>.json      bench JSON lines
  profiles/ncu_summary.json            per-launch DRAM bytes etc. (read by bench.py for roofline.traffic)
Usage: python tools/summarize_round.py r01
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("VF_PROF_DIR", os.path.join(ROOT, "profiles"))
CRIT = {0: "angular", 1: "exp", 2: "log"}
VAR = {0: "exact", 1: "minimax", 2: "poly4", 3: "reach"}


def kernel_key(name):
    name = name.replace("(int)", "")
    m = re.search(r"vf_angular_role_kernel<(\d), (\d)", name)   # <WIN, VAR, NT, PPT>
    if m:
        return f"angular/{VAR[int(m.group(2))]}", int(m.group(1))
    m = re.search(r"vf_angular_(shared|window)_kernel<(\d), (\d)(?:, \d)?>", name)
    if m:
        return f"angular/{VAR[int(m.group(3))]}", int(m.group(2))
    m = re.search(r"vf_el(?:_tma)?_kernel<(\d), (\d), (\d)(?:, \d)*>", name)
    if m:
        return f"{CRIT[int(m.group(2))]}/{VAR[int(m.group(3))]}", int(m.group(1))
    return None, None


def launches(tag):
    src = os.path.join(OUT, "launches.csv")
    if not os.path.exists(src):
        return
    lines = open(src).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    shutil.copy(src, os.path.join(PROF, f"{tag}_launches.csv"))
    agg = defaultdict(list)
    for r in rows:
        agg[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    ours = sum(sum(v) for k, v in agg.items() if "vf::" in k)
    with open(os.path.join(PROF, f"{tag}_launches_summary.md"), "w") as fh:
        fh.write(f"# {tag}: ncu launch list of `python bench.py` (default C2 workload)\n\n")
        fh.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole bench command "
                 "(cold-cache, serialised launches: compare shares, not absolutes; the bench itself runs the 7 "
                 "filters concurrently in one CUDA graph).\n\n")
        fh.write(f"Total device time {tot/1e6:.3f} ms over {len(rows)} launches; libvf kernels {100*ours/tot:.1f}%.\n\n")
        fh.write("| kernel | launches | mean µs | share of all | share of libvf |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            s = sum(v)
            fh.write(f"| `{k[:90]}` | {len(v)} | {s/len(v)/1e3:.2f} | {100*s/tot:.1f}% | "
                     f"{(100*s/ours if 'vf::' in k else 0):.1f}% |\n")


METRICS = [
    ("gpu__time_duration.sum", "time", 1e-3, "µs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1, ""),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1, ""),
    ("launch__registers_per_thread", "regs", 1, ""),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %", 1, ""),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %", 1, ""),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %", 1, ""),
    ("dram__bytes_read.sum", "DRAM read", 1, "B"),
    ("dram__bytes_write.sum", "DRAM write", 1, "B"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak", 1, ""),
    ("smsp__inst_executed.sum", "warp inst", 1, ""),
]


TIME_TO_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def sass_mix_flops(path):
    """kernel name (normalised, 60 chars) -> executed FP32 flops, from a SASS mix file."""
    if not os.path.exists(path):
        return {}
    res, cur = {}, None
    for line in open(path):
        if line.startswith("== "):
            cur = line[3:].split("  warp-inst")[0].replace("(int)", "").replace("vf::", "")[:60]
        elif "exec-fp32-flops" in line and cur:
            res[cur] = float(line.split()[-1])
    return res


def ncu_full(tag, cfg, npix, summary):
    rep = os.path.join(OUT, f"prof_{cfg}.ncu-rep")
    if not os.path.exists(rep):
        return
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    with open(os.path.join(PROF, f"{tag}_ncu_{cfg}.md"), "w") as fh:
        fh.write(f"# {tag}: ncu --set full, {cfg} ({npix} pixels per launch), all filter kernels\n\n")
        fh.write("`ncu --set full --import-source on --clock-control none -k regex:vf_` on "
                 f"`tools/prof_driver.py --config {cfg}` (second round of launches).\n\n")
        names = [r[col["Kernel Name"]] for r in data]
        fh.write("| metric | " + " | ".join(kernel_key(n)[0] + f" ({kernel_key(n)[1]}x{kernel_key(n)[1]})"
                                             for n in names) + " |\n")
        fh.write("|---|" + "---|" * len(names) + "\n")
        for m, label, scale, _ in METRICS:
            if m not in col:
                continue
            vals = []
            for r in data:
                v = r[col[m]]
                if m.startswith("dram__bytes"):
                    vals.append(f"{to_bytes(v, units[col[m]])/1e6:.2f} MB")
                elif m == "gpu__time_duration.sum":   # in µs
                    vals.append(f"{to_bytes(v, 'x') * TIME_TO_US[units[col[m]]]:.1f}")
                elif m == "smsp__inst_executed.sum":
                    vals.append(f"{float(v.replace(',', ''))*32/npix:.0f} /px")
                else:
                    vals.append(v[:6])
            fh.write(f"| {label} | " + " | ".join(vals) + " |\n")
        # executed FP32 flops per elapsed second over the FP32 peak (2 x 128 x
        # SMs x clock), from the SASS mix (tools/ncu_source_summary.py: FFMA 2,
        # FADD/FMUL 1, packed FFMA2 4, FADD2/FMUL2 2 flops per lane; ncu's
        # op_ffma metrics do not count the packed sm_100 forms)
        mix = sass_mix_flops(os.path.join(PROF, f"{tag}_sass_mix_{cfg}.txt"))
        if mix and "gpu__time_duration.sum" in col:
            vals = []
            for r in data:
                fl = mix.get(r[col["Kernel Name"]].replace("(int)", "").replace("vf::", "")[:60])
                t = to_bytes(r[col["gpu__time_duration.sum"]], "x") * TIME_TO_US[units[col["gpu__time_duration.sum"]]] * 1e-6
                if fl is None:
                    vals.append("-")
                    continue
                frac = fl / t / (2 * 128 * 148 * 1.965e9)
                vals.append(f"{100 * frac:.1f}%")
                summary.setdefault("executed_fp32_frac", {})[f"{cfg}/{kernel_key(r[col['Kernel Name']])[0]}"] = frac
            fh.write("| executed FP32 flops (FFMA/FFMA2/FADD/FADD2/FMUL/FMUL2, SASS mix) % of peak at 1965 MHz | "
                     + " | ".join(vals) + " |\n")
        fh.write("\nKernel names: " + "; ".join(f"`{n[:80]}`" for n in names) + "\n")
    for r in data:
        key, w = kernel_key(r[col["Kernel Name"]])
        rd = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wr = to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        summary["dram_bytes_per_launch"][f"{cfg}/{key}"] = rd + wr
        summary["algorithmic_bytes_per_launch"][f"{cfg}/{key}"] = 6 * npix
        summary["thread_inst_per_pixel"][f"{cfg}/{key}"] = float(r[col["smsp__inst_executed.sum"]].replace(",", "")) * 32 / npix


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    summary = {"round": tag, "dram_bytes_per_launch": {}, "algorithmic_bytes_per_launch": {},
               "thread_inst_per_pixel": {},
               "note": "DRAM bytes = dram__bytes_read.sum + dram__bytes_write.sum of one launch (ncu --set full); "
                       "algorithmic bytes = 3 B in + 3 B out per pixel"}
    ncu_full(tag, "C2", 512 * 512, summary)
    ncu_full(tag, "C4", 16 * 512 * 768, summary)
    ncu_full(tag, "C3", 8 * 2048 * 2048, summary)
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    for cfg, src in (("C2", "bench.json"), ("C3", "bench_C3.json"), ("C4", "bench_C4.json")):
        p = os.path.join(OUT, src)
        if os.path.exists(p) and os.path.getsize(p) > 0:
            shutil.copy(p, os.path.join(PROF, f"{tag}_bench_{cfg}.json"))
    print("ok", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main()
