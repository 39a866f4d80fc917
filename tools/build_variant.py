#!/usr/bin/env python3
"""A/B library variant that differs in a few translation units only: recompile the named
csrc/*.cu files with extra -D defines, link them with the main build's other objects.
--slim: a small library with the fast kernels of the five configs' primes only (5, 13, 59, 61,
257; every other prime takes the generic kernel) -- A/B builds of the config kernels that fit
the gpurun snapshot.
usage: python tools/build_variant.py [--slim] OUT.so "zp_fast_p13.cu zp_fast_p61.cu" DEF1 [DEF2 ...]"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_cs_0611109_b200 import build as B  # noqa: E402

args = sys.argv[1:]
slim = args and args[0] == "--slim"
if slim:
    args = args[1:]
out, units, defines = args[0], args[1].split(), args[2:]
if not os.environ.get("ZP_VARIANT_NO_MAIN"):  # (set: link against the main objects as they are)
    B.build()  # main objects up to date
tmp = os.path.join(ROOT, "build", "obj_variant")
os.makedirs(tmp, exist_ok=True)
for f in glob.glob(os.path.join(tmp, "*.o")):
    os.remove(f)
objs = {os.path.basename(o): o for o in glob.glob(os.path.join(B.OBJ, "*.o"))}
keep = {"zp_fast_p5.o", "zp_fast_p13.o", "zp_fast_p59.o", "zp_fast_p61.o", "zp_fast_p257.o"}
if slim:
    objs = {k: v for k, v in objs.items() if not k.startswith("zp_fast_p") or k in keep}
    units = sorted(set(units) | {"raid6c_host.cu"})
with cf.ThreadPoolExecutor(max_workers=8) as ex:
    res = list(ex.map(lambda u: B._compile(os.path.join(B.CSRC, u), True, False, tmp,
                                           tuple(defines) + (("ZP_SLIM",) if slim else ())), units))
for o, _ in res:
    objs[os.path.basename(o)] = o
cmd = [B.NVCC] + B.ARCH + ["-shared", "-o", out] + sorted(objs.values()) + ["-lcudart"]
subprocess.run(cmd, check=True)
print(out)
