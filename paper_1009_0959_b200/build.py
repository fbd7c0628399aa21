"""Build libvf.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvf.so")
LIB_DEBUG = os.path.join(HERE, "libvf_debug.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "vf.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


# Per-translation-unit extra flags (ptxas's register-usage
# level 2 helps the 3x3 exp/log non-libm kernels, hurts the libm ones).
SOURCE_FLAGS = {"vf_el_ty4.cu": ["-Xptxas", "--register-usage-level=2"],
                "vf_ang_mm.cu": ["-Xptxas", "--register-usage-level=2"]}


def build(force: bool = False, verbose: bool = False, debug: bool = False, variant: str = "",
          defines=(), variant_tus=None) -> str:
    """debug=True builds libvf_debug.so with the VF_CHECK device bounds checks;
    variant="x" with defines=["-DKNOB=1", ...] builds libvf_x.so (tuning A/B,
    selected at run time with VF_LIB; variant_tus: the .cu files the defines
    apply to, default all).  Each .cu is compiled to an object with its own
    flags (concurrently), then linked into the shared library."""
    import tempfile
    target = LIB_DEBUG if debug else (os.path.join(HERE, f"libvf_{variant}.so") if variant else LIB)
    if not force and not debug and not variant and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc" if nvcc == "nvcc" and subprocess.call(
            ["which", "nvcc"], stdout=subprocess.DEVNULL) != 0 else nvcc
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-Xptxas", "-v"] if verbose else []) + \
        (["-DVF_DEBUG"] if debug else [])
    # object cache (build/objcache, git- and gpurun-ignored): a translation unit
    # is recompiled only when its flags or any source / header changed
    import hashlib
    import shutil
    cache = os.path.join(ROOT, "build", "objcache")
    os.makedirs(cache, exist_ok=True)
    h_all = hashlib.sha256()
    for d in deps():
        with open(d, "rb") as fh:
            h_all.update(d.encode() + fh.read())
    with tempfile.TemporaryDirectory(prefix="vfbuild") as tmpd:
        procs, objs = [], []
        for src in sources():
            flags = compile_flags + SOURCE_FLAGS.get(os.path.basename(src), []) + \
                (list(defines) if variant_tus is None or os.path.basename(src) in variant_tus else [])
            key = hashlib.sha256(h_all.digest() + " ".join(flags + [os.path.basename(src)]).encode()).hexdigest()[:24]
            cached = os.path.join(cache, key + ".o")
            obj = os.path.join(tmpd, os.path.basename(src) + ".o")
            if os.path.exists(cached) and not verbose:
                shutil.copyfile(cached, obj)
            else:
                cmd = [nvcc] + flags + ["-c", "-o", obj, src]
                procs.append((subprocess.Popen(cmd), cmd, obj, cached))
            objs.append(obj)
        rcs = [(p.wait(), cmd, obj, cached) for p, cmd, obj, cached in procs]   # all finished before cleanup
        for rc, cmd, obj, cached in rcs:
            if rc != 0:
                raise subprocess.CalledProcessError(rc, cmd)
            shutil.copyfile(obj, cached + ".tmp%d" % os.getpid())
            os.replace(cached + ".tmp%d" % os.getpid(), cached)
        tmp = target + ".tmp%d" % os.getpid()
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs, check=True)
    os.replace(tmp, target)
    return target


# The paper's exp / log functions as the exact variants (DESIGN.md reading
# R26; the default library follows the survey's expm1f / log1pf): a variant
# build measured beside the default and parity-tested
# (tests/test_gpu_exact_libm.py); selected at run time with VF_LIB.
PAPER_LIBM = ("paperlibm", ["-DVF_EXACT_LIBM=1"], ["vf_api.cu", "vf_fused.cu"])


def build_all(verbose: bool = False) -> None:
    """libvf.so, libvf_debug.so and libvf_paperlibm.so, compiled concurrently."""
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(3) as ex:
        futs = [ex.submit(build, True, verbose, False), ex.submit(build, True, False, True),
                ex.submit(build, True, False, False, PAPER_LIBM[0], PAPER_LIBM[1], PAPER_LIBM[2])]
        for f in futs:
            f.result()


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a for a in sys.argv if a.startswith("-D")]
    tus = next((a.split("=", 1)[1].split(",") for a in sys.argv if a.startswith("--tus=")), None)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv, variant=var,
                defines=defs, variant_tus=tus))
