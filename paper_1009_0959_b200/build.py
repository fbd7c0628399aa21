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


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """debug=True builds libvf_debug.so with the VF_CHECK device bounds checks.
    Each .cu is compiled to an object with its own flags (concurrently), then
    linked into the shared library."""
    import tempfile
    target = LIB_DEBUG if debug else LIB
    if not force and not debug and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc" if nvcc == "nvcc" and subprocess.call(
            ["which", "nvcc"], stdout=subprocess.DEVNULL) != 0 else nvcc
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-Xptxas", "-v"] if verbose else []) + \
        (["-DVF_DEBUG"] if debug else [])
    with tempfile.TemporaryDirectory(prefix="vfbuild") as tmpd:
        procs, objs = [], []
        for src in sources():
            obj = os.path.join(tmpd, os.path.basename(src) + ".o")
            cmd = [nvcc] + compile_flags + SOURCE_FLAGS.get(os.path.basename(src), []) + ["-c", "-o", obj, src]
            procs.append((subprocess.Popen(cmd), cmd))
            objs.append(obj)
        rcs = [(p.wait(), cmd) for p, cmd in procs]   # all finished before the directory goes away
        for rc, cmd in rcs:
            if rc != 0:
                raise subprocess.CalledProcessError(rc, cmd)
        tmp = target + ".tmp%d" % os.getpid()
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs, check=True)
    os.replace(tmp, target)
    return target


def build_all(verbose: bool = False) -> None:
    """libvf.so and libvf_debug.so, compiled concurrently (one nvcc each)."""
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(2) as ex:
        futs = [ex.submit(build, True, verbose, False), ex.submit(build, True, False, True)]
        for f in futs:
            f.result()


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
