import os, sys, itertools, statistics
sys.path.insert(0, "/root/repo")
import torch, bench, paper_1009_0959_b200 as vfb
spec, w = bench.workload("C2")
x = torch.from_numpy(bench.make_input(spec, 0)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
orders = {
 "default": bench.COMBOS,
 "long_first": [("exp","exact"),("log","exact"),("angular","exact"),("angular","minimax"),("exp","minimax"),("log","minimax"),("exp","poly4")],
 "short_first": [("exp","poly4"),("log","minimax"),("exp","minimax"),("angular","minimax"),("angular","exact"),("log","exact"),("exp","exact")],
}
for name, combos in orders.items():
    outs = [torch.empty_like(x) for _ in combos]
    plan = vfb.Plan(x, outs, w, combos)
    for _ in range(20): plan.launch()
    ts = []
    for r in range(50):
        flush.fill_(r & 255)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.launch(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(name, "median %.4f ms  min %.4f" % (statistics.median(ts), min(ts)))
    plan.close()
# sequential for reference
ts=[]
outs = [torch.empty_like(x) for _ in bench.COMBOS]
for r in range(30):
    flush.fill_(r & 255)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for c, o in zip(bench.COMBOS, outs): vfb.vf_filter_batch(x, w, *c, out=o)
    b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("sequential median %.4f" % statistics.median(ts))
