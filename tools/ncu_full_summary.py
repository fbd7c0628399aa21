"""Summarise an `ncu --set full` report (one row per captured launch) as
markdown: duration, issue / pipe / warp activity, DRAM bytes, executed
instructions, and the largest stall reasons (PC sampling).

    ncu -i report.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_full_summary.py raw.csv > profiles/r02_ncu_full.md
"""
import csv
import io
import sys

# (metric, label, target unit) -- values are converted from the unit row of the CSV
UNITS = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
ROWS = [("gpu__time_duration.sum", "duration", 1e-3, "ms"),
        ("launch__grid_size", "blocks", 1, ""),
        ("launch__registers_per_thread", "registers", 1, ""),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1, ""),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1, ""),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %", 1, ""),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %", 1, ""),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %", 1, ""),
        ("smsp__inst_executed.sum", "warp instructions", 1e-6, "M"),
        ("dram__bytes_read.sum", "DRAM read", 1e6, "MB"),
        ("dram__bytes_write.sum", "DRAM write", 1e6, "MB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %", 1, "")]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main(path):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    names = [d[col["Kernel Name"]][:60] for d in data]
    print("| metric | " + " | ".join(f"`{n}`" for n in names) + " |")
    print("|---|" + "---|" * len(names))
    for key, label, scale, unit in ROWS:
        if key not in col:
            continue
        vals = []
        u = units[col[key]]
        for d in data:
            x = num(d[col[key]])
            if x is not None and u in UNITS:        # to SI, then to the target unit (scale = its size)
                x = x * UNITS[u] / scale
            elif x is not None and scale != 1:
                x = x * scale
            vals.append("—" if x is None else (f"{x:,.2f}{(' ' + unit) if unit else ''}"))
        print(f"| {label} | " + " | ".join(vals) + " |")
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    print("\nPC-sampling stall reasons (share of samples per launch, top 6):\n")
    for j, d in enumerate(data):
        tot = sum(num(d[col[h]]) or 0 for h in stall)
        top = sorted(((num(d[col[h]]) or 0, h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall),
                     reverse=True)[:6]
        print(f"- `{names[j]}`: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top if tot))


if __name__ == "__main__":
    main(sys.argv[1])
