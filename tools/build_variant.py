#!/usr/bin/env python3
"""A/B library variant that differs in a few translation units only: recompile the named
csrc/*.cu files with extra -D defines, link them with the main build's other objects.
usage: python tools/build_variant.py OUT.so "zp_fast_p13.cu zp_fast_p61.cu" DEF1 [DEF2 ...]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_cs_0611109_b200 import build as B  # noqa: E402

out, units, defines = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
B.build()  # main objects up to date
tmp = os.path.join(ROOT, "build", "obj_variant")
os.makedirs(tmp, exist_ok=True)
for f in glob.glob(os.path.join(tmp, "*.o")):
    os.remove(f)
objs = {os.path.basename(o): o for o in glob.glob(os.path.join(B.OBJ, "*.o"))}
for u in units:
    o, _ = B._compile(os.path.join(B.CSRC, u), True, False, tmp, tuple(defines))
    objs[os.path.basename(o)] = o
cmd = [B.NVCC] + B.ARCH + ["-shared", "-o", out] + sorted(objs.values()) + ["-lcudart"]
subprocess.run(cmd, check=True)
print(out)
