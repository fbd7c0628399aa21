"""Launch every criterion x variant kernel once on the bench's workloads (C4
full batch 3x3, C3 5x5) and the step's statistics passes, for an ncu capture
whose per-kernel records bench.py can attach (tools/ncu_exec.py):

    ncu --metrics $(python tools/ncu_exec.py --metrics) --csv --log-file gpurun_out/exec.csv \\
        python tools/prof_kernels.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

dev = torch.device("cuda")
stream = torch.cuda.current_stream()
images = int(os.environ.get("PROF_IMAGES", "1024"))
for cfg, w, ids in (("C4", 3, range(images)), ("C3", 5, range(8))):
    x = torch.from_numpy(bench.gen_batch(cfg, ids)).to(dev)
    outs = {}
    for c in bench.COMBOS + bench.REACH_COMBOS:
        outs[c] = torch.empty_like(x)
        vfb.vf_filter_batch(x, w, *c, out=outs[c], stream=stream)
    if cfg == "C4":
        # the step's fused plan nodes (exp/log; angular exact + minimax)
        for gcs in ([c for c in bench.COMBOS if c[0] in ("exp", "log")], [c for c in bench.COMBOS if c[0] == "angular"]):
            gp = vfb.Plan(x, [outs[c] for c in gcs], w, gcs)
            gp.launch(stream)
            torch.cuda.synchronize()
            gp.close()
        n = sum(len(cs) for _, cs in bench.FIDELITY_GROUPS)
        st = torch.empty((n, x.shape[0], 8), dtype=torch.float64, device=dev)
        k = 0
        for ref, cs in bench.FIDELITY_GROUPS:
            vfb.vf_image_stats_multi(outs[ref], [outs[c] for c in cs], st[k:k + len(cs)], stream)
            k += len(cs)
    torch.cuda.synchronize()
    del x, outs
print("prof_kernels done")
