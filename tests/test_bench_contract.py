"""bench.py output contract on the host (the reference arm runs the CPU
oracle, so it needs no GPU): stdout carries exactly one JSON line with the
keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "Mpix/s" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C2")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == "", (r.stdout, r.stderr[-1000:])


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """Our arm on the GPU (short run): one JSON line with roofline, clocks,
    gpu_launches and an end-to-end figure that moved host bytes."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["dtype"] == "f32" and d["scaling"] == "weak" and d["gpu_launches"] == 7 * 3
    rf = d["roofline"]
    assert rf["bound"] == "alu" and 0 < rf["frac"] < 1.5 and rf["unit"] == "TFLOP/s" and rf["peak"] > 70
    assert d["e2e"]["h2d_bytes_per_step"] == 512 * 512 * 3 and d["e2e"]["d2h_bytes_per_step"] == 7 * 512 * 512 * 3
    assert d["e2e"]["outputs_match_device_path"] is True
    assert d["clocks"]["sm_mhz"] is None or d["clocks"]["sm_mhz"] > 0
    for k, v in d["per_kernel"].items():
        assert v["ms"] > 0 and v["ms_isolated"] > 0, k
