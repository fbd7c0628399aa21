"""Quick per-kernel timing (CUDA events, median of N launches, L2 flushed) for
tuning iterations: python tools/kbench.py [C2 C3 C4 ...] [--algo window|shared]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

args = sys.argv[1:]
skip = {i + 1 for i, a in enumerate(args) if a in ("--algo", "--only")}
cfgs = [a for i, a in enumerate(args) if not a.startswith("--") and i not in skip] or ["C2", "C4", "C3"]
algo = "auto"
if "--algo" in sys.argv:
    algo = sys.argv[sys.argv.index("--algo") + 1]
only = None
if "--only" in sys.argv:
    only = sys.argv[sys.argv.index("--only") + 1]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for cfg in cfgs:
    spec, w = bench.workload(cfg)
    x = torch.from_numpy(bench.make_input(spec, 0)).cuda()
    npix = x.numel() // 3
    out = torch.empty_like(x)
    n = w * w
    pairs = n * (n - 1) // 2
    line = [f"{cfg}({w}x{w},{npix/1e6:.1f}Mpx)"]
    combos = [c for c in bench.COMBOS + bench.REACH_COMBOS if not only or only in f"{c[0]}/{c[1]}"]
    outs = [torch.empty_like(x) for _ in combos]
    if algo == "auto":
        # average launch duration over back-to-back launches (bench.steady_kernel_ms)
        sms, R = bench.steady_kernel_ms(vfb, torch, torch.device("cuda"), torch.cuda.current_stream(), flush, x, w,
                                        combos, outs)
    for c in combos:
        if algo == "auto":
            ms = sms[c]
        else:
            for _ in range(3):
                vfb.vf_filter_batch_algo(x, w, *c, algo, out=out)
            ts = []
            for _ in range(9):
                flush.fill_(1)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                vfb.vf_filter_batch_algo(x, w, *c, algo, out=out)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
        frac = bench.FLOPS_PER_PAIR[c] * pairs * npix / (ms / 1e3) / 1e12 / bench.NOMINAL_FP32_TFLOPS_AT_MAX
        line.append(f"{c[0][:3]}/{c[1][:3]} {ms*1e3:8.1f}us {frac*100:4.1f}%")
    print(" | ".join(line), flush=True)
