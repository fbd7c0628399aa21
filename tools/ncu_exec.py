"""ncu CSV (tools/prof_kernels.py capture) -> profiles/ncu_exec.json: per kernel
launch (mangled name | grid) the pipe utilisations, issue activity and DRAM
bytes, tagged with the sha256 of the libvf.so that was profiled (bench.py
attaches a record only when it runs that same library).

    python tools/ncu_exec.py --metrics            # the metric list for ncu --metrics
    python tools/ncu_exec.py exec.csv [libvf.so]  # -> profiles/ncu_exec.json
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "launch__registers_per_thread": "registers",
}


def main():
    if sys.argv[1:] == ["--metrics"]:
        print(",".join(METRICS))
        return
    src = sys.argv[1]
    lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "paper_1009_0959_b200", "libvf.so")
    text = open(src).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    recs = {}
    for row in csv.DictReader(io.StringIO(text)):
        name = row.get("Kernel Name", "")
        grid = row.get("Grid Size", "").strip("()").replace(" ", "")
        key = f"{name}|{grid}"
        m = row.get("Metric Name")
        if m not in METRICS:
            continue
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "")
        if unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        elif unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        r = recs.setdefault(key, {})
        r[METRICS[m]] = v
    for r in recs.values():
        if "dram_read_bytes" in r:
            r["dram_bytes"] = r["dram_read_bytes"] + r.get("dram_write_bytes", 0.0)
    sys.path.insert(0, ROOT)
    import bench
    h = bench.lib_sha256(lib)
    out = {"libvf_sha256": h, "src_sha256": bench.src_sha256(), "command": "ncu --metrics <tools/ncu_exec.py --metrics> python tools/prof_kernels.py",
           "note": "ncu replays each kernel (serialised, cold caches); pipe percentages are of the kernel's own "
                   "active cycles", "kernels": recs}
    with open(os.path.join(ROOT, "profiles", "ncu_exec.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"{len(recs)} kernel records -> profiles/ncu_exec.json (libvf sha256 {h[:16]})")


if __name__ == "__main__":
    main()
