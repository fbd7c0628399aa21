"""The partitioner on the GPU with the NCCL backend (world size 1 on the one
GPU available: the same code path the 8-GPU runs take, minus the peers)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402
from paper_1009_0959_b200 import parallel as par  # noqa: E402


@pytest.fixture(scope="module")
def nccl1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_batch_sharded_nccl(nccl1):
    import dataclasses
    spec = dataclasses.replace(vfsynth.config("C4"), H=64, W=96, batch=5)
    xb = torch.from_numpy(vfsynth.make_batch(spec)).cuda()
    combos = [("angular", "exact"), ("angular", "minimax"), ("exp", "poly4")]
    outs, stats = par.run_batch_sharded(xb, 5, 3, combos)
    torch.cuda.synchronize()
    for c in combos:
        ref, _, _ = vfb.filter(xb, 3, *c)
        assert torch.equal(outs[c], ref)
        assert stats[c].shape == (5, 8)
    assert torch.all(stats[combos[0]][:, 0] == 0)           # reference vs itself
    s = par.stats_summary(stats[("angular", "minimax")].cpu(), 64, 96)
    assert s["psnr_db"] > 40


@pytest.mark.parametrize("w", [3, 5])
def test_stripes_nccl(nccl1, w):
    x = vfsynth.random_image(3, 45, 70)
    xt = torch.from_numpy(x).cuda()
    ref, _, _ = vfb.filter(xt, w, "angular", "minimax")
    o0, on, b0, bn = par.stripe_bounds(45, 1, 0, w)
    stripe, full = par.run_stripes(xt[b0:b0 + bn].contiguous(), 45, w, "angular", "minimax")
    torch.cuda.synchronize()
    assert torch.equal(full, ref) and torch.equal(stripe, ref)
