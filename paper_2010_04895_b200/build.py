"""Build libmhw.so in-tree with nvcc for sm_100a (no JIT cache, no torch).

python -m paper_2010_04895_b200.build  [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmhw.so")
OBJ = os.path.join(PKG, "_obj")
SOURCES = ["graph.cu", "walk.cu", "exact.cu", "corpus.cu", "loader.cu", "api.cu"]
HEADERS = ["mhw_device.cuh", "internal.h", "walk.h", "loader.h", "jsonfmt.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden", "-Xptxas", "-O3",
    "-I", os.path.join(ROOT, "include"),
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "mhw.h")]
    objs, cmds = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s, *hdrs]):
            cmds.append([NVCC, *ARCH, *FLAGS, "-c", s, "-o", o])
    # translation units compile in parallel
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(run, cmds))
    if force or _stale(LIB, objs):
        # export only the C ABI: the visibility flag hides everything else,
        # the mhw_* symbols are re-exported by the version script.
        vs = os.path.join(OBJ, "exports.map")
        with open(vs, "w") as f:
            f.write("{ global: mhw_*; local: *; };\n")
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xlinker", f"--version-script={vs}", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
