import sys, torch
sys.path.insert(0, '.')
import paper_1009_0959_b200 as vfb, vfsynth
x = torch.from_numpy(vfsynth.random_image(1, 64, 64)).cuda()
for a in ["auto:1", "auto:2", "auto:3"]:
    for c in [("exp","minimax"), ("exp","exact")]:
        try:
            vfb.filter(x, 3, *c, algo=a); torch.cuda.synchronize(); print(a, c, "ok")
        except Exception as e:
            print(a, c, "ERR", str(e)[:200]); sys.exit(1)
