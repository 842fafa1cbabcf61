"""Build the CUDA library libpm.so in-tree with nvcc for sm_100a.

The library is the whole CUDA path behind include/pm.h; the Python binding
(pm.py) only loads it.  Called by __graft_entry__.build() and the tests.
"""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpm.so")
LIB_CHECKS = os.path.join(HERE, "libpm_checks.so")  # -DPM_CHECKS: device bounds checks

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-v",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "pm.h")]


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel, then link libpm.so
    (checks=True: libpm_checks.so with the device bounds checks PM_CHECK;
    load it with PM_LIB=<path>)."""
    target = LIB_CHECKS if checks else LIB
    if not force and not stale(target):
        return target
    from concurrent.futures import ThreadPoolExecutor
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DPM_CHECKS"] if checks else [])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + f".{os.getpid()}{'.chk' if checks else ''}.o")
        cmd = [nvcc, *flags, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, res

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    log = []
    for src, obj, res in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n" + res.stdout + res.stderr)
        log.append(res.stderr)
    tmp = target + f".tmp{os.getpid()}"
    objs = [obj for _, obj, _ in results]
    res = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                          tmp, *objs, "-ldl"], capture_output=True, text=True)
    for o in objs:
        os.remove(o)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    if verbose:
        print("".join(log))
    os.replace(tmp, target)
    if not checks:
        with open(os.path.join(HERE, "libpm.ptxas.txt"), "w") as f:
            # (without ptxas' compile times, so that the log only changes with the code)
            f.write("".join(l for l in "".join(log).splitlines(True)
                            if "Compile time" not in l))
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
