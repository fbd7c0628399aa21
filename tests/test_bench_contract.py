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
    assert d["config"]["workload"].startswith("C4: 1024 x 512x768")      # the headline workload (BASELINE config 3)
    assert d["scaling"] == "strong"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == "", (r.stdout, r.stderr[-1000:])


def test_ncu_exec_attach_rule(tmp_path, monkeypatch):
    """profiles/ncu_exec.json is attached only if it was captured from this
    library's device code, or from a library built from these same kernel
    sources and flags (src_sha256); anything else is reported as stale."""
    sys.path.insert(0, ROOT)
    import bench
    src = bench.src_sha256()
    assert src == bench.src_sha256() and len(src) == 64
    os.makedirs(tmp_path / "profiles")
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))

    def put(d):
        with open(tmp_path / "profiles" / "ncu_exec.json", "w") as fh:
            json.dump(d, fh)
    assert bench.load_ncu_exec("a" * 64)[0] is None                      # absent
    put({"libvf_sha256": "a" * 64, "kernels": {}})
    assert bench.load_ncu_exec("a" * 64)[0] is not None                  # same device code
    d, why = bench.load_ncu_exec("b" * 64)
    assert d is None and "stale" in why                                  # other device code, no source hash
    put({"libvf_sha256": "a" * 64, "src_sha256": src, "kernels": {}})
    d, why = bench.load_ncu_exec("b" * 64)
    assert d is not None and "src_sha256" in why                         # rebuilt from the same sources
    put({"libvf_sha256": "a" * 64, "src_sha256": "c" * 64, "kernels": {}})
    assert bench.load_ncu_exec("b" * 64)[0] is None                      # other sources


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """Our arm on the GPU (short run on the first 64 C4 images): one JSON line
    with roofline, roofline_minimax, per-kernel SURVEY 8(d) fractions, clocks,
    gpu_launches and an end-to-end figure that moved host bytes."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--images", "64", "--no-cpu-baseline", "--no-c3", "--no-paper"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    # fused plan with statistics: exp/log node, angular node + remainder strips, 3 statistics nodes, finalize
    assert d["dtype"] == "f32" and d["scaling"] == "strong" and d["gpu_launches"] == 7 * 3
    assert d["config"]["images"] == 64
    rf = d["roofline"]
    assert rf["bound"] == "alu" and 0 < rf["frac"] < 1.5 and rf["unit"] == "TFLOP/s" and rf["peak"] > 70
    rm = d["roofline_minimax"]
    assert 0 < rm["frac"] < 1.5 and rm["target"] == 0.6 and len(rm["minimax_fracs"]) == 4
    px = 64 * 512 * 768
    assert d["e2e"]["h2d_bytes_per_step"] == px * 3 and d["e2e"]["d2h_bytes_per_step"] == 7 * px * 3
    assert d["e2e"]["outputs_match_device_path"] is True
    assert d["clocks"]["sm_mhz"] is None or d["clocks"]["sm_mhz"] > 0
    assert len(d["per_kernel"]) == 7
    for k, v in d["per_kernel"].items():
        assert v["ms"] > 0 and 0 < v["frac_fp32_alg"] < 1.5 and v["frac_sfu_alg"] >= 0, k
        assert v["kernel"].startswith("_Z"), k                      # vf_kernel_info: mangled kernel name
    a = d["per_kernel"]["angular/minimax"]
    assert a["frac_fp32_evaluated_pairs_only"] < a["frac_fp32_alg"]
    # the step's gathered fidelity statistics (each approximant vs its exact filter, all images)
    fid = d["fidelity_minimax_vs_exact"]
    for k in ("angular/minimax", "exp/minimax", "exp/poly4", "log/minimax"):
        assert fid[k]["images"] == 64 and 0 <= fid[k]["diff_frac"] < 0.5, (k, fid[k])
