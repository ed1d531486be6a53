"""Build libspo_b200.so in-tree with nvcc for sm_100a (no torch involvement).

    python -m paper_1611_02665_b200.build          # or __graft_entry__.build()

The library links the CUDA runtime statically, so it does not depend on the
runtime version torch ships; device pointers and streams come from the caller.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libspo_b200.so")
SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [
    os.path.join(ROOT, "include", "spo_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu to an object in parallel (one nvcc per file), then
    link the shared library."""
    from concurrent.futures import ThreadPoolExecutor

    if not force and not needs_build():
        return LIB
    tag = f"{os.getpid()}.tmp"  # concurrent builders never share a temp file
    tmp = f"{LIB}.{tag}"
    objs = [os.path.join(PKG, "csrc", os.path.basename(s)[:-3] + f".{tag}.o") for s in SOURCES]
    cmds = [[nvcc(), *NVCC_FLAGS, "-c", "-o", o, s] for s, o in zip(SOURCES, objs)]
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    if all(r.returncode == 0 for r in results):
        results.append(subprocess.run(link, capture_output=True, text=True))
        cmds.append(link)
    log = os.path.join(PKG, "csrc", "build.log")
    with open(log, "w") as f:
        for c, r in zip(cmds, results):
            f.write(" ".join(c) + "\n" + r.stdout + r.stderr)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    bad = [r for r in results if r.returncode != 0]
    if bad or len(results) != len(cmds):
        sys.stderr.write("".join(r.stderr for r in bad))
        raise RuntimeError(f"nvcc failed; see {log}")
    os.replace(tmp, LIB)
    if verbose:
        print("".join(r.stderr for r in results))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
