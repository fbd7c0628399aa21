"""Table 5 / Table 6 of the paper on a synthetic corpus stand-in
(SURVEY.md 8(f4)): for the paper's three filters -- BVDF (the angular order
statistic, Eq. 5), AMNFE (Eq. 8) and EVMF (Eq. 9) -- the per-image percentage
change of MAE / MSE / NCD against the noise-free image when the exact
elementary functions are replaced by the minimax approximants,
    delta% = 100 (Q_exact - Q_approx) / Q_exact     (negative: approximant worse),
its mean and standard deviation over the corpus, and the execution-time
ratio Time% = 100 t_exact / t_approx (the paper's definition, R20)
measured on the B200 with CUDA events over the whole corpus batch.

Corpus: N synthetic 384x512 images (smooth gradients + 32 rectangles/edges,
vfsynth), the same clean images under every noise model (Eq. 10):
  Table 5: uncorrelated phi_k = 0.10; correlated phi = 0.10, phi_k = 0.25;
           mixed (Gaussian sigma = 10, then correlated phi = 0.10, phi_k = 0.25);
  Table 6: correlated phi = 0.20, 0.30, 0.40 (phi_k = 0.25).
The paper's corpus (100 internet images) is not available; these are
stand-in numbers, not a reproduction.

Usage (GPU): python tools/paper_tables.py [--n 24] [--out profiles/r01_paper_tables]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402

FILTERS = {"BVDF": "angular", "AMNFE": "amnfe", "EVMF": "evmf"}
PAPER_T5 = {   # Table 5: Mean(%) for MAE, MSE, NCD, Time; uncorrelated / correlated / mixed
    "BVDF": {"uncorrelated": (-1.000, -0.571, -0.783, 1381.783), "correlated": (-0.926, 0.171, -0.759, 1371.314),
             "mixed": (-0.022, -0.131, 0.007, 1408.964)},
    "AMNFE": {"uncorrelated": (-0.025, -0.070, -0.020, 142.700), "correlated": (-0.016, -0.064, -0.031, 143.496),
              "mixed": (-0.001, -0.006, -0.004, 140.814)},
    "EVMF": {"uncorrelated": (-0.141, -0.376, -0.147, 236.582), "correlated": (-0.108, -0.203, -0.149, 236.105),
             "mixed": (0.000, 0.013, -0.004, 215.000)},
}


def spec_for(model, p, n, H=384, W=512):
    base = dict(H=H, W=W, batch=n, window=(3,), n_objects=32, rects_only=False, p=p, seed=10090959 + 77)
    if model == "uncorrelated":
        return vfsynth.ImageSpec("corpus", noise="uncorrelated", **base)
    if model == "correlated":
        return vfsynth.ImageSpec("corpus", noise="correlated_phik", **base)
    return vfsynth.ImageSpec("corpus", noise="mixed", sigma=10.0, **base)


def per_image_quality(clean, out):
    s = vfb.vf_image_stats(clean, out).cpu().numpy()          # [B, 8]
    B, H, W, _ = clean.shape
    n3 = 3.0 * H * W
    return {"mae": s[:, 1] / n3, "mse": s[:, 2] / n3, "ncd": s[:, 3] / s[:, 4]}


def timed(x, crit, var, reps=5):
    o = torch.empty_like(x)
    vfb.vf_filter_batch(x, 3, crit, var, out=o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        vfb.vf_filter_batch(x, 3, crit, var, out=o)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return o, statistics.median(ts)


def run_model(model, p, n):
    spec = spec_for(model, p, n)
    imgs = [vfsynth.make_image(spec, i) for i in range(n)]
    clean = torch.from_numpy(np.stack([c for c, _ in imgs])).cuda()
    noisy = torch.from_numpy(np.stack([x for _, x in imgs])).cuda()
    res = {"noisy_mae": float(per_image_quality(clean, noisy)["mae"].mean())}
    for name, crit in FILTERS.items():
        oe, te = timed(noisy, crit, "exact")
        om, tm = timed(noisy, crit, "minimax")
        qe, qm = per_image_quality(clean, oe), per_image_quality(clean, om)
        row = {}
        for m in ("mae", "mse", "ncd"):
            d = 100.0 * (qe[m] - qm[m]) / qe[m]
            row[m] = {"mean": float(d.mean()), "stdev": float(d.std(ddof=1)), "exact": float(qe[m].mean()),
                      "approx": float(qm[m].mean())}
        row["time_pct"] = 100.0 * te / tm
        row["ms_exact"], row["ms_approx"] = te, tm
        res[name] = row
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_paper_tables"))
    a = ap.parse_args()
    vfb.load_library()
    t5 = {m: run_model(m, 0.10, a.n) for m in ("uncorrelated", "correlated", "mixed")}
    t6 = {f"correlated {int(100 * p)}%": run_model("correlated", p, a.n) for p in (0.20, 0.30, 0.40)}
    with open(a.out + ".json", "w") as fh:
        json.dump({"table5": t5, "table6": t6, "n_images": a.n, "size": "384x512"}, fh, indent=1)
    lines = [f"# Table 5 / 6 on a synthetic stand-in corpus ({a.n} images, 384x512, B200)", "",
             "`python tools/paper_tables.py` -- delta% = 100 (Q_exact - Q_approx) / Q_exact per image "
             "(negative: the minimax version is worse), mean and stdev over the corpus; Time% = 100 t_exact / "
             "t_approx on the GPU (the paper's: Pentium D, C, x87 libm).  Paper values (P:311-326) in brackets.", ""]

    def table(title, cols, data, paper=None):
        out = [f"## {title}", "", "| Filter | Measure | " + " | ".join(f"{c} Mean(%) | {c} Stdev(%)" for c in cols)
               + " |", "|---|---|" + "---|---|" * len(cols)]
        for f in FILTERS:
            for mi, m in enumerate(("mae", "mse", "ncd")):
                cells = []
                for c in cols:
                    r = data[c][f][m]
                    pv = f" [{paper[f][c][mi]:+.3f}]" if paper else ""
                    cells.append(f"{r['mean']:+.3f}{pv} | {r['stdev']:.3f}")
                out.append(f"| {f} | {m.upper()} | " + " | ".join(cells) + " |")
            cells = []
            for c in cols:
                pv = f" [{paper[f][c][3]:.1f}]" if paper else ""
                cells.append(f"{data[c][f]['time_pct']:.1f}{pv} | -")
            out.append(f"| {f} | Time | " + " | ".join(cells) + " |")
        return out + [""]

    lines += table("Table 5 analogue: 10% noise", ["uncorrelated", "correlated", "mixed"], t5, PAPER_T5)
    lines += table("Table 6 analogue: correlated impulsive noise", list(t6), t6)
    with open(a.out + ".md", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
