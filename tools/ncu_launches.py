"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (the
bench command under ncu): launches, total and mean duration and share per
kernel.  ncu serialises and cold-starts every launch, so the SHARES (not the
absolute times) are what compares with the bench's step.

    python tools/ncu_launches.py profiles/r02_launches.csv > profiles/r02_launches_summary.md

With `--step PATTERN:COUNT ...` it also composes one bench step from the mean
launch time of each of the step's kernels (COUNT launches per step of the
kernels whose name contains PATTERN) and prints each kernel's share of that
sum -- the figure to compare with the bench's `roofline.share_of_step`.
"""
import collections
import csv
import io
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(path, step=()):
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
    if step:
        rows = []
        for spec in step:
            pat, cnt = spec.rsplit(":", 1)
            hits = [(k, v) for k, v in agg.items() if pat in k]
            n = sum(v[0] for _, v in hits)
            us = sum(v[1] for _, v in hits)
            if n:
                rows.append((pat, int(cnt), us / n))
        tot_step = sum(c * m for _, c, m in rows)
        print(f"\nOne step composed from the mean launch times (serialised, cold cache): {tot_step / 1e3:.2f} ms\n")
        print("| step kernel (name contains) | launches per step | mean ms | share of the step |")
        print("|---|---|---|---|")
        for pat, c, m in rows:
            print(f"| `{pat}` | {c} | {m / 1e3:.3f} | {100 * c * m / tot_step:.1f}% |")


if __name__ == "__main__":
    args = sys.argv[1:]
    step = args[args.index("--step") + 1:] if "--step" in args else []
    main(args[0], step)
