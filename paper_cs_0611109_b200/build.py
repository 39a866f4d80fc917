#!/usr/bin/env python3
"""Build libraid6c.so in-tree for sm_100a (nvcc, parallel per translation unit).

    python -m paper_cs_0611109_b200.build [--force] [--verbose]

Each csrc/*.cu is compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo, then
linked into paper_cs_0611109_b200/libraid6c.so (shipped to the GPU box with the tree).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libraid6c.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --compress-mode=size: the 28 x 13 fast-path instantiations are ~170 MB of SASS + line tables
# uncompressed; the size mode brings libraid6c.so to about an eighth (driver >= 570 decompresses
# a translation unit's image on first use)
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "--compress-mode=size", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I", INC, "-I", CSRC]


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(INC, "raid6c.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src, force, verbose, objdir=OBJ, defines=()):
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    if not force and not _stale(obj, [src] + _deps()):
        return obj, None
    cmd = [NVCC] + ARCH + FLAGS + [f"-D{d}" for d in defines] + (["-Xptxas", "-v"] if verbose else []) + \
        ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, (r.stderr if verbose else None)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Build the library (``out``); ``defines`` builds an experiment variant in its own object dir."""
    objdir = OBJ if not defines else os.path.join(ROOT, "build", "obj_" + "_".join(defines))
    os.makedirs(objdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        res = list(ex.map(lambda s: _compile(s, force or bool(defines), verbose, objdir, defines), srcs))
    objs = [o for o, _ in res]
    if verbose:
        for o, log in res:
            if log:
                print(f"== {os.path.basename(o)}\n{log}", file=sys.stderr)
    LIBO = out
    if force or defines or _stale(LIBO, objs):
        tmp = LIBO + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIBO)
    return LIBO


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=LIB)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.out, tuple(a.defines)))
