"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (the
bench command under ncu): launches, total and mean duration and share per
kernel.  ncu serialises and cold-starts every launch, so the SHARES (not the
absolute times) are what compares with the bench's step.

    python tools/ncu_launches.py profiles/r02_launches.csv > profiles/r02_launches_summary.md
"""
import collections
import csv
import io
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(io.StringIO(text)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(r["Metric Value"].replace(",", "")) * UNIT.get(r.get("Metric Unit", "usecond"), 1.0)
        k = r["Kernel Name"]
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"`{path}`: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.1f} ms in all\n")
    print("| kernel | launches | total ms | mean ms | share |")
    print("|---|---|---|---|---|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:90]}` | {n} | {us / 1e3:.2f} | {us / n / 1e3:.3f} | {100 * us / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
