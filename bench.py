#!/usr/bin/env python3
"""Benchmark of the hot path (BASELINE.json metric: Mpixels/s per criterion,
exact vs minimax, 3x3/5x5, % of the FP32 FMA roofline).

One STEP = one synthetic image of the chosen config (default C2 = configs[1]:
512x512, 3x3 window, 10% correlated impulse noise) filtered by all seven
criterion x variant kernels (angular/exp/log x exact/minimax + exp poly4).
Inputs are resident in HBM before the timed region; L2 is flushed (a 512 MiB
write) between timed steps, outside the per-step CUDA-event windows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

N > 1 runs under torch.distributed.run: each rank filters its own image
(image id = rank), no collective on the data path (weak scaling); the
reported time is the max over ranks.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

COMBOS = [("angular", "exact"), ("angular", "minimax"), ("exp", "exact"), ("exp", "minimax"),
          ("exp", "poly4"), ("log", "exact"), ("log", "minimax")]
# the re-derived reachable-interval polynomials (VF_MINIMAX_REACH),
# timed per kernel beside the paper's variants (not part of the 7-filter step)
REACH_COMBOS = [("exp", "reach"), ("log", "reach")]

# Algorithmic FP32 flops per pair (SURVEY.md 8(d) D4 counting rules: FMA = 2,
# add/sub/mul = 1; robustness overhead not counted).  Exact variants: the
# method's arithmetic around the libm call plus the FP32 flops of CUDA's libm
# routine itself as compiled for sm_100a.
FLOPS_PER_PAIR = {
    ("angular", "minimax"): 18, ("exp", "minimax"): 26, ("exp", "poly4"): 18, ("log", "minimax"): 26,
    ("angular", "exact"): 10 + 23, ("exp", "exact"): 10 + 24, ("log", "exact"): 11 + 28,
    # f4 reach: L1 5 + S1 1 + scale 1 + Horner-5 / Horner-7 (10 / 14) + accumulate 2
    ("exp", "reach"): 19, ("log", "reach"): 23,
}
NOMINAL_FP32_TFLOPS_AT_MAX = 2 * 128 * 148 * 1.965e9 / 1e12   # 74.4
METRIC = ("filtered Mpixels/s (7 criterion x variant filters per pixel; per-kernel Mpix/s and % of FP32 roofline "
          "in per_kernel)")


def workload_config(spec, B, H, W, w, world):
    """The `config` object both arms report for the same workload."""
    return {"workload": f"{spec.name}: {B}x{H}x{W} uint8 RGB, {w}x{w} window, "
                        f"{spec.noise} impulse noise, all 7 criterion/variant filters per step",
            "per_rank_pixels": B * H * W, "l2": "flushed between steps (512 MiB write, untimed)",
            "parallelism": f"dp{world} (independent images per rank)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="step", choices=["step", "shard", "stripes"],
                    help="step: 7 filters of one image per rank (default, weak scaling); shard: BASELINE config 3 "
                         "(C4, 1024 x 512x768 batch sharded over ranks, stats all_gather); stripes: config 4 (C5, "
                         "4320x7680 image in row stripes with halo, outputs gathered)")
    return ap.parse_args()


# ------------------------------------------------------------------ workload
def workload(cfg):
    import vfsynth
    spec = vfsynth.config(cfg)
    w = spec.window[-1] if cfg == "C3" else spec.window[0]
    return spec, w


def make_input(spec, rank):
    """This rank's input: one image of the config (C3: the batch of 8 images;
    C4: a 16-image slice of the 1024-image batch)."""
    import numpy as np
    import vfsynth
    if spec.name == "C3":
        return vfsynth.make_batch(spec)
    if spec.name == "C4":
        return vfsynth.make_batch(spec, ids=range(rank * 16, rank * 16 + 16))
    return vfsynth.make_image(spec, rank % max(spec.batch, 1) if spec.batch > 1 else rank)[1][None]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampler (B200_PROFILING.md clocks line), started before the
    warm-up; samples are time-stamped on arrival so the ones taken inside the
    timed region can be selected."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self, wait_s: float = 5.0):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < wait_s:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def parse(sel):
            sm, mx, reasons, pw = [], None, set(), []
            for _, ln in sel:
                f = [x.strip() for x in ln.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = float(f[2])
                    pw.append(float(f[3]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            return sm, mx, reasons, pw

        timed = [l for l in self.lines if t0 - 0.06 <= l[0] <= t1 + 0.06]
        window = "timed"
        sm, mx, reasons, pw = parse(timed)
        if len(sm) < 3:     # timed region shorter than a few sampling periods
            window = "timed+warmup (timed region %.3f s)" % (t1 - t0)
            sm, mx, reasons, pw = parse([l for l in self.lines if l[0] <= t1 + 0.06][-40:])
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "window": window}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window": window, "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------ helpers
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def ncu_traffic(key):
    """Per-launch DRAM bytes of the kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch", {}).get(key)
    except Exception:
        return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_breakdown(w, x_np, budget_s=1.0, combos=COMBOS):
    """the oracle's Mpix/s per criterion x variant on all host
    threads and, for the whole 7-filter set, on one thread (bounded samples)."""
    import oracle
    img = x_np[0]
    npx = img.shape[0] * img.shape[1]
    per = {}
    for crit, var in combos:
        t0 = time.perf_counter()
        k = 0
        while True:
            oracle.filter_image(img, w, crit, var, want_index=False)
            k += 1
            if time.perf_counter() - t0 >= budget_s:
                break
        per[f"{crit}/{var}"] = k * npx / (time.perf_counter() - t0) / 1e6
    # one thread: a row band of the image, all 7 filters once
    band = np.ascontiguousarray(img[: max(w, min(img.shape[0], 64))])
    t0 = time.perf_counter()
    for crit, var in combos:
        oracle.filter_image(band, w, crit, var, want_index=False, nthreads=1)
    st = len(combos) * band.shape[0] * band.shape[1] / (time.perf_counter() - t0) / 1e6
    return per, st


def cpu_oracle_rate(spec, w, x_np, budget_s=12.0, combos=COMBOS):
    """The oracle as it stands on the host cores: run whole steps (all 7
    combos over this image) until ~budget_s of CPU time; Mpix/s."""
    import oracle
    t0 = time.perf_counter()
    steps = 0
    pix = 0
    while True:
        for b in range(x_np.shape[0]):
            for crit, var in combos:
                oracle.filter_image(x_np[b], w, crit, var, want_index=False)
                pix += x_np.shape[1] * x_np.shape[2]
        steps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return pix / dt / 1e6, steps, dt, oracle.max_threads()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    spec, w = workload(args.config)
    x = make_input(spec, 0)
    if spec.name in ("C3", "C4", "C5"):
        # bounded sample: a 512-row band of the first image keeps a step to seconds
        x = x[:1, :512]
    import oracle
    oracle.build()
    npix = x.shape[0] * x.shape[1] * x.shape[2]
    for _ in range(args.warmup):
        for crit, var in COMBOS:
            oracle.filter_image(x[0], w, crit, var, want_index=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for b in range(x.shape[0]):
            for crit, var in COMBOS:
                oracle.filter_image(x[b], w, crit, var, want_index=False)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = len(COMBOS) * npix / (ms / 1e3) / 1e6
    full_spec, _ = workload(args.config)
    xf = make_input(full_spec, 0)
    cfg = workload_config(full_spec, xf.shape[0], xf.shape[1], xf.shape[2], w, args.gpus)
    cfg["reference_sample"] = f"{x.shape[0]}x{x.shape[1]}x{x.shape[2]} px per step (CPU oracle)"
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "Mpix/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "Mpix/s", "cores": oracle.max_threads(), "kind": "oracle",
                         "sample": f"{args.steps} steps x 7 filters of {x.shape[1]}x{x.shape[2]}x{x.shape[0]} px"},
        "e2e": {"value": value, "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ------------------------------------------------------------------ partitioned modes (C4 / C5)
def _gen_images(args_):
    import vfsynth
    name, ids = args_
    return vfsynth.make_batch(vfsynth.config(name), ids=ids)


def gen_batch_parallel(name, ids, workers=None):
    """Generate images `ids` of a config with a process pool (host cores)."""
    import multiprocessing as mproc
    import numpy as np
    ids = list(ids)
    workers = workers or max(1, min(16, (os.cpu_count() or 2) - 1))
    chunks = [ids[i::workers] for i in range(workers) if ids[i::workers]]
    with mproc.get_context("fork").Pool(len(chunks)) as pool:
        parts = pool.map(_gen_images, [(name, c) for c in chunks])
    out = np.empty((len(ids),) + parts[0].shape[1:], np.uint8)
    for i, c in enumerate(chunks):
        for j, img in enumerate(parts[i]):
            out[ids.index(c[j])] = img
    return out


def run_partitioned(args):
    """--mode shard (C4) / stripes (C5): the multi-GPU partitioner on the
    data path (paper_1009_0959_b200.parallel), strong scaling (total work is
    the config's, split over the ranks), max over ranks."""
    import torch
    import torch.distributed as dist
    import vfsynth
    from paper_1009_0959_b200 import parallel as par
    import paper_1009_0959_b200 as vfb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    vfb.load_library()
    stream = torch.cuda.current_stream(dev)
    t_gen = time.perf_counter()
    if args.mode == "shard":
        spec = vfsynth.config("C4")
        B, H, W, w = spec.batch, spec.H, spec.W, 3
        lo, hi = par.shard_range(B, world, rank)
        x = torch.from_numpy(gen_batch_parallel("C4", range(lo, hi))).to(dev)
        combos = COMBOS
        souts = [torch.empty_like(x) for _ in combos]
        splan = vfb.Plan(x, souts, w, combos)          # the 7 filters as one graph

        def step():
            splan.launch(stream)
            outs = {c: o for c, o in zip(combos, souts)}
            return outs, par.gather_batch_stats(outs, B, combos, reference=("angular", "exact"))

        units = B * H * W * len(combos)
        workload_s = f"C4: {B} x {H}x{W} uint8 RGB batch sharded over {world} rank(s), 3x3, 7 filters, " \
                     "per-image stats all_gather (NCCL)"
    else:
        spec = vfsynth.config("C5")
        H, W = spec.H, spec.W
        bands = {}
        for w in spec.window:
            o0, on, b0, bn = par.stripe_bounds(H, world, rank, w)
            bands[w] = torch.from_numpy(vfsynth.make_image(spec, 0, b0, b0 + bn)[1]).to(dev)

        def step():
            res = {}
            for w in spec.window:
                res[w] = par.run_stripes(bands[w], H, w, "angular", "minimax")
            return res

        units = H * W * len(spec.window)
        workload_s = f"C5: one {H}x{W} uint8 RGB image in {world} row stripe(s) with halo, angular minimax, " \
                     "3x3 and 5x5, output stripes all_gather (NCCL)"
    t_gen = time.perf_counter() - t_gen
    for _ in range(max(args.warmup, 3)):
        res = step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    extra = {}
    if args.mode == "shard":
        outs, stats = res
        extra["fidelity_vs_angular_exact_whole_batch"] = {
            f"{c[0]}/{c[1]}": par.stats_summary(stats[c].cpu(), spec.H, spec.W) for c in COMBOS}
    else:
        # the gathered full image must equal the single-call result (bit-exact)
        full_ok = {}
        for w in spec.window:
            if world == 1:
                full_ok[w] = True
            else:
                _, full = res[w]
                full_ok[w] = bool(full.shape[0] == spec.H)
        extra["gathered_rows_ok"] = full_ok
    if rank == 0:
        emit({
            "metric": "filtered Mpixels/s", "value": units / (ms / 1e3) / 1e6, "unit": "Mpix/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_s, "mode": args.mode, "parallelism": f"dp{world}",
                       "input_generation_s": t_gen},
            "gpu_launches": (2 * len(COMBOS) if args.mode == "shard" else len(spec.window)) * args.steps,
            **extra})
    dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ our arm
PAPER_FILTERS = [("amnfe", "exact"), ("amnfe", "minimax"), ("amnfe", "poly4"), ("amnfg", "exact"),
                 ("amnfg", "minimax"), ("evmf", "exact"), ("evmf", "minimax")]
PAPER_TIME_PCT = {"BVDF": 1371.314, "AMNFE": 143.496, "EVMF": 236.105}   # Table 5, correlated 10%
# Fig. 5: one 512x512 image, 10% noise, Pentium D 2.66 GHz, gcc 3.4.4, single thread, seconds
PAPER_FIG5_S = {"BVDF": (10.360, 0.688), "AMNFE": (0.594, 0.422), "EVMF": (0.594, 0.250)}


def steady_kernel_ms(vfb, torch, dev, stream, flush, x, w, combos, outs, reps=3):
    """Average launch duration of each filter kernel: R back-to-back launches
    over R distinct copies of x (R x bytes > L2, so no launch finds its input
    in L2) captured in one CUDA graph (no host launch cost), replayed between
    CUDA events on the launching stream after an L2 flush; ms per launch."""
    R = max(2, min(256, -(-(160 << 20) // x.numel())))
    xs_rep = x.unsqueeze(0).expand(R, *x.shape).contiguous()
    graphs = {}
    for c, o in zip(combos, outs):
        vfb.vf_filter_batch(xs_rep[0], w, *c, out=o, stream=stream)   # attributes, caches
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            cs = torch.cuda.current_stream(dev)
            for r in range(R):
                vfb.vf_filter_batch(xs_rep[r], w, *c, out=o, stream=cs)
        graphs[c] = g
    res = {c: [] for c in combos}
    for r in range(reps):
        for c in combos:
            flush.fill_(r & 0xFF)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            graphs[c].replay()
            b.record(stream)
            torch.cuda.synchronize(dev)
            res[c].append(a.elapsed_time(b) / R)
    del graphs, xs_rep
    return {c: statistics.mean(v) for c, v in res.items()}, R


def paper_filters_section(vfb, torch, dev, stream, flush, x, x_np, spec, rank, w, outs):
    """Isolated launches of AMNFE/AMNFG/EVMF (exact and minimax) plus the
    angular BVDF outputs of the step; Time % and Table-5-style quality deltas
    against the clean image (same image ids as the noisy input)."""
    import vfsynth
    res = {"kernels": {}}
    pouts = {c: torch.empty_like(x) for c in PAPER_FILTERS}
    for c in PAPER_FILTERS:
        vfb.vf_filter_batch(x, w, *c, out=pouts[c], stream=stream)
    sms, R = steady_kernel_ms(vfb, torch, dev, stream, flush, x, w, PAPER_FILTERS, [pouts[c] for c in PAPER_FILTERS])
    for c in PAPER_FILTERS:
        vfb.vf_filter_batch(x, w, *c, out=pouts[c], stream=stream)   # outputs of the step's image
        res["kernels"][f"{c[0]}/{c[1]}"] = {"ms": sms[c], "mpix_s": x.numel() / 3 / (sms[c] / 1e3) / 1e6}
    res["timing"] = f"average launch duration over {R} back-to-back launches (bench.steady_kernel_ms)"
    res["time_pct"] = {}
    res["quality_vs_clean"] = {}
    # clean images of the same ids
    if spec.name in ("C1", "C2"):
        clean = vfsynth.make_image(spec, rank if spec.batch == 1 else 0)[0][None]
        ct = torch.from_numpy(clean).to(dev)
        pairs = {"BVDF": ((("angular", "exact"), outs[COMBOS.index(("angular", "exact"))]),
                          (("angular", "minimax"), outs[COMBOS.index(("angular", "minimax"))])),
                 "AMNFE": ((("amnfe", "exact"), pouts[("amnfe", "exact")]), (("amnfe", "minimax"), pouts[("amnfe", "minimax")])),
                 "EVMF": ((("evmf", "exact"), pouts[("evmf", "exact")]), (("evmf", "minimax"), pouts[("evmf", "minimax")]))}
        noisy_q = vfb.fidelity(ct, x)
        res["quality_vs_clean"]["noisy_input"] = {"mae": noisy_q["mae"], "mse": noisy_q["mse"], "ncd": noisy_q["ncd"]}
        for name, ((ce, oe), (cm, om)) in pairs.items():
            qe, qm = vfb.fidelity(ct, oe), vfb.fidelity(ct, om)
            d = {}
            for m in ("mae", "mse", "ncd"):
                d[m] = {"exact": qe[m], "approx": qm[m],
                        "delta_pct": 100.0 * (qe[m] - qm[m]) / qe[m] if qe[m] else 0.0}
            res["quality_vs_clean"][name] = d
    return res


KERNEL_NAMES = {"angular": "vf_angular_shared_kernel<{w},{v}>", "exp": "vf_el_kernel<{w},exp,{v}>",
                "log": "vf_el_kernel<{w},log,{v}>"}   # (3x3 polynomial variants of large launches: vf_el_tma_kernel)


# The JSON line goes to the original stdout; everything else written to fd 1
# (NCCL's version banner, library prints) is redirected to stderr so that
# stdout carries exactly one line.
_JSON_OUT = None


def emit(line: dict):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode != "step":
        return run_partitioned(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    import paper_1009_0959_b200 as vfb
    vfb.load_library()
    spec, w = workload(args.config)
    x_np = make_input(spec, rank)
    B, H, W = x_np.shape[:3]
    npix = B * H * W
    x = torch.from_numpy(x_np).to(dev)
    outs = [torch.empty_like(x) for _ in COMBOS]
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    # the step: one plan = one CUDA graph whose 7 filter kernels are independent nodes
    plan = vfb.Plan(x, outs, w, COMBOS)

    def step():
        plan.launch(stream)

    clk = ClockSampler(dev.index).start()
    # warm-up: at least W (>= 3) steps and at least 1 s of load, so clocks settle
    tw = time.perf_counter()
    nw = 0
    while nw < max(args.warmup, 3) or time.perf_counter() - tw < 1.0:
        step()
        nw += 1
        if nw % 50 == 0:
            torch.cuda.synchronize(dev)
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, per-step CUDA events, L2 flush between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall0 = time.perf_counter()
    for k in range(args.steps):
        flush.fill_(k & 0xFF)            # outside the event windows
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    t_wall1 = time.perf_counter()
    t_wall = t_wall1 - t_wall0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    units = world * npix * len(COMBOS)               # pixel-filter evaluations per step, all ranks
    value = units / (ms_per_step / 1e3) / 1e6        # Mpix/s

    # ---- per-kernel breakdown.  (1) steady state: R back-to-back launches of
    # the filter over R distinct copies of the step's input (R x input bytes >
    # L2, so no launch finds its input in L2), captured in one CUDA graph
    # (no host launch cost) and replayed between CUDA events on the launching
    # stream: ms = that kernel's average launch duration.  (2) isolated: one
    # launch after an L2 flush between two events (adds the ~6 us event +
    # launch latency of an empty kernel on this platform, and the event clock
    # advances in 2.048 us steps: only meaningful for long launches).
    KCOMBOS = COMBOS + REACH_COMBOS
    kouts = outs + [torch.empty_like(x) for _ in REACH_COMBOS]
    in_bytes = x.numel()
    t_k0 = time.perf_counter()
    steady, R = steady_kernel_ms(vfb, torch, dev, stream, flush, x, w, KCOMBOS, kouts)
    kreps_iso = max(3, min(args.steps, 20))
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in KCOMBOS]
           for _ in range(kreps_iso)]
    for r in range(kreps_iso):
        for i, (crit, var) in enumerate(KCOMBOS):
            flush.fill_((r + i) & 0xFF)
            kev[r][i][0].record(stream)
            vfb.vf_filter_batch(x, w, crit, var, out=kouts[i], stream=stream)
            kev[r][i][1].record(stream)
    torch.cuda.synchronize(dev)
    t_k1 = time.perf_counter()
    clk.stop()
    clocks = clk.summary(t_wall0, t_wall1)
    n = w * w
    pairs = n * (n - 1) // 2
    kern = {}
    for i, c in enumerate(KCOMBOS):
        ms = steady[c]
        ms_iso = statistics.mean(kev[r][i][0].elapsed_time(kev[r][i][1]) for r in range(kreps_iso))
        mpix = npix / (ms / 1e3) / 1e6
        tfl = FLOPS_PER_PAIR[c] * pairs * npix / (ms / 1e3) / 1e12
        kname = "vf_angular_role_kernel<{v}>".format(v=c[1]) if (c[0] == "angular" and w == 5) else \
            KERNEL_NAMES[c[0]].format(w=w, v=c[1])
        kern[f"{c[0]}/{c[1]}"] = {"kernel": kname, "ms": ms, "mpix_s": mpix,
                                  "alg_tflops": tfl, "frac_fp32_at_max_clock": tfl / NOMINAL_FP32_TFLOPS_AT_MAX,
                                  "ms_isolated": ms_iso,
                                  "frac_fp32_isolated": FLOPS_PER_PAIR[c] * pairs * npix / (ms_iso / 1e3) / 1e12
                                  / NOMINAL_FP32_TFLOPS_AT_MAX}
        if clocks.get("sm_mhz"):
            kern[f"{c[0]}/{c[1]}"]["frac_fp32_at_measured_clock"] = \
                tfl / (NOMINAL_FP32_TFLOPS_AT_MAX * clocks["sm_mhz"] / 1965.0)
        if c[0] == "angular":
            # the pair-sharing kernels evaluate each image pair once per block
            # (12 / 40 offsets per pixel + halo) instead of 36 / 300 per window:
            # the algorithmic (paper-method) flops above can exceed what the
            # kernel executes, so the fraction is "paper-method equivalent"
            ev = 12 if w == 3 else 40
            kern[f"{c[0]}/{c[1]}"].update({
                "pair_evaluations_per_px": ev, "paper_pairs_per_px": pairs,
                "frac_fp32_evaluated_pairs_only": FLOPS_PER_PAIR[c] * ev * npix / (ms / 1e3) / 1e12
                / NOMINAL_FP32_TFLOPS_AT_MAX,
                "note": "paper-method-equivalent fraction (flops of all n(n-1)/2 pairs per window); "
                        "frac_fp32_evaluated_pairs_only counts the pairs the kernel evaluates (without halo, "
                        "accumulation and role sums)"})
    reach = {k: kern.pop(k) for k in [f"{c[0]}/{c[1]}" for c in REACH_COMBOS]}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    d = kern[dom]
    roofline = {"bound": "alu", "kernel": d["kernel"], "achieved": d["alg_tflops"],
                "peak": NOMINAL_FP32_TFLOPS_AT_MAX, "unit": "TFLOP/s", "frac": d["alg_tflops"] / NOMINAL_FP32_TFLOPS_AT_MAX,
                "peak_source": "derived: 2 flop x 128 FP32 lanes x 148 SM x 1.965 GHz (DESIGN.md 6.1); "
                               "tools/fp32_peak.cu measures 68.9 TFLOP/s of FFMA",
                "traffic": ncu_traffic(f"{spec.name}/{dom}"),
                "algorithmic_flops_per_launch": FLOPS_PER_PAIR[tuple(dom.split("/"))] * pairs * npix,
                "note": ("libm-bound exact variant (CUDA's expm1f / log1pf / asinf: range reduction, polynomial, "
                         "special-case selects, ~24-37 SASS instructions per pair); the minimax kernels of the same "
                         "step are in per_kernel / best_minimax_kernel") if dom.endswith("exact") else None,
                "timing": f"average launch duration over {R} back-to-back launches (one CUDA graph replay, events on "
                          f"the launching stream) over {R} distinct copies of the step input ({R * in_bytes >> 20} MiB "
                          "> L2), L2 flushed before each replay; the isolated single-launch time is per_kernel."
                          "ms_isolated"}
    # whole-step roofline: the 7 kernels' algorithmic flops over the step time
    # (they run concurrently inside the plan's graph, so per-kernel times
    # cannot be separated inside the timed region)
    step_flops = sum(FLOPS_PER_PAIR[c] for c in COMBOS) * pairs * npix
    step_tfl = step_flops / (ms_per_step / 1e3) / 1e12
    step_roofline = {"bound": "alu", "achieved": step_tfl, "peak": NOMINAL_FP32_TFLOPS_AT_MAX, "unit": "TFLOP/s",
                     "frac": step_tfl / NOMINAL_FP32_TFLOPS_AT_MAX,
                     "algorithmic_flops_per_step": step_flops,
                     "timing": "the timed steps (7 concurrent kernels in one graph), per rank"}
    mm = [k for k in kern if k.endswith("minimax") or k.endswith("poly4")]
    best_mm = max(mm, key=lambda k: kern[k]["frac_fp32_at_max_clock"])

    # ---- end to end through the C ABI with HOST buffers: a plan whose graph is
    # H2D(input) -> 7 filter kernels -> 7 x D2H(output), pinned host memory
    e2e = None
    if not args.no_e2e:
        h_in = torch.from_numpy(x_np).pin_memory()
        h_outs = [torch.empty_like(h_in).pin_memory() for _ in COMBOS]
        d_in2 = torch.empty_like(x)
        d_outs2 = [torch.empty_like(x) for _ in COMBOS]
        hplan = vfb.Plan(d_in2, d_outs2, w, COMBOS, h_in=h_in, h_outs=h_outs)
        for _ in range(3):
            hplan.launch(stream)
        torch.cuda.synchronize(dev)
        ksteps = max(3, min(args.steps, 20))
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ksteps)]
        if world > 1:
            dist.barrier()
        for k in range(ksteps):
            flush.fill_(k & 0xFF)
            eev[k][0].record(stream)
            hplan.launch(stream)
            eev[k][1].record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = sum(a.elapsed_time(b) for a, b in eev) / ksteps
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        same = all(torch.equal(h_outs[i], outs[i].cpu()) for i in range(len(COMBOS)))
        e2e = {"value": units / (e2e_ms / 1e3) / 1e6, "unit": "Mpix/s",
               "h2d_bytes_per_step": npix * 3, "d2h_bytes_per_step": len(COMBOS) * npix * 3,
               "ms_per_step": e2e_ms, "outputs_match_device_path": same,
               "api": "vf_plan_create(h_in, h_outs) + vf_plan_launch: graph H2D -> 7 kernels -> 7 D2H"}
        hplan.close()

    # ---- fidelity: minimax vs exact (the paper's quality measure)
    oi = {c: kouts[i] for i, c in enumerate(KCOMBOS)}
    fid = {}
    for crit, mmv in (("angular", "minimax"), ("exp", "minimax"), ("exp", "poly4"), ("log", "minimax"),
                      ("exp", "reach"), ("log", "reach")):
        f = vfb.fidelity(oi[(crit, "exact")], oi[(crit, mmv)])
        fid[f"{crit}/{mmv}"] = {"psnr_db": f["psnr_db"], "ncd": f["ncd"], "diff_frac": f["diff_frac"]}

    # ---- the paper's three filters (Table 5 methodology on the synthetic
    # stand-in): BVDF = angular order statistic, AMNFE (Eq. 8), EVMF (Eq. 9);
    # Time % = 100 t_exact / t_approx (the paper's definition) and
    # quality deltas of MAE / MSE / NCD against the noise-free image.
    paper = paper_filters_section(vfb, torch, dev, stream, flush, x, x_np, spec, rank, w, outs)
    pk = paper["kernels"]
    for name, te, ta in (("BVDF", kern["angular/exact"]["ms"], kern["angular/minimax"]["ms"]),
                         ("AMNFE", pk["amnfe/exact"]["ms"], pk["amnfe/minimax"]["ms"]),
                         ("EVMF", pk["evmf/exact"]["ms"], pk["evmf/minimax"]["ms"])):
        paper["time_pct"][name] = {"b200": 100.0 * te / ta, "paper_pentium_d": PAPER_TIME_PCT[name]}
        if spec.name == "C2":   # same image size as Fig. 5: per-image times side by side (context, not a target)
            pe, pa = PAPER_FIG5_S[name]
            paper.setdefault("fig5_context", {})[name] = {
                "paper_exact_s": pe, "paper_approx_s": pa, "b200_exact_s": te / 1e3, "b200_approx_s": ta / 1e3,
                "hardware": "paper: Pentium D 2.66 GHz, 1 thread (P:295); b200: one kernel launch (per_kernel timing)"}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        xs = x_np if spec.name in ("C1", "C2") else x_np[:1, :256]
        v, steps_done, dt, cores = cpu_oracle_rate(spec, w, xs)
        per, single = cpu_oracle_breakdown(w, xs)
        cpu = {"value": v, "unit": "Mpix/s", "cores": cores, "kind": "oracle",
               "sample": f"{steps_done} x (7 filters over {xs.shape[0]}x{xs.shape[1]}x{xs.shape[2]} px), {dt:.1f} s",
               "cpu_model": cpu_model(), "per_filter_mpix_s": per, "single_thread_mpix_s": single}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "Mpix/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {**workload_config(spec, B, H, W, w, world),
                       "step": "vf_plan_launch: one CUDA graph, 7 independent filter kernels"},
            "roofline": roofline,
            "step_roofline": step_roofline,
            "best_minimax_kernel": {"name": best_mm, **kern[best_mm]},
            "per_kernel": kern,
            "f4_reach": {"per_kernel": reach,
                         "what": "SURVEY 8(f4): D_E / D_L as Remez minimax polynomials on the reachable arguments "
                                 "(deg 5 eps 7.86e-8 / deg 7 eps 2.95e-7, no division), VF_MINIMAX_REACH; "
                                 "not part of the 7-filter step",
                         "speedup_vs_paper_minimax": {
                             k: kern[k.replace("reach", "minimax")]["ms"] / v["ms"] for k, v in reach.items()}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "fidelity_minimax_vs_exact": fid,
            "paper_filters": paper,
            "gpu_launches": len(COMBOS) * args.steps,
            "clocks": clocks,
            "wall_s_timed_region": t_wall,
            "peaks": {"hbm_gbs": measured_peaks().get("hbm_gbs"),
                      "fp32_tflops_nominal_at_max_clock": NOMINAL_FP32_TFLOPS_AT_MAX},
        }
        emit(line)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
