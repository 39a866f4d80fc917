"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/raid6c.h declares, and its host-only helpers agree with the oracle's size rules.
(No compute call is made here; parity tests are in test_gpu_parity.py.)"""
import os
import re
import subprocess

import pytest

import oracle
from paper_cs_0611109_b200 import raid6c as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "raid6c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(raid6c_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = _declared()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", R.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(raid6c_[a-z0-9_]+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(R.EXPORTED) == set(names)


def test_sizes_agree_with_oracle():
    for p in [3, 5, 7, 13, 17, 59, 61, 97, 257]:
        for nb in [1, 2, 3, 7, 100, 4097, 65536, 4 << 20]:
            assert R.word_count(p, nb) == oracle.word_count(p, nb)
            assert R.parity_bytes(p, nb) == oracle.parity_bytes(p, nb)
    assert R.parity_bytes(9, 100) == 0 and R.word_count(4, 10) == 0


def test_valid_p_and_fast_set():
    primes = [q for q in range(3, 258) if all(q % d for d in range(2, int(q ** 0.5) + 1))]
    for q in range(0, 300):
        assert R.valid_p(q) == (q in primes and q >= 3 and q <= 257)
    for q in [5, 13, 59, 61, 257]:
        assert R.has_fast_path(q)
    # the fast (compile-time-p) kernel exists for exactly the primes whose period lcm(p-1, 32)
    # fits 32 lanes; the others run the generic kernel
    from math import gcd
    fits = [q for q in primes if (q - 1) // gcd(q - 1, 32) <= 32]
    assert len(fits) == 28 and len(primes) - len(fits) == 26
    for q in primes:
        assert R.has_fast_path(q) == (q in fits), q


def test_ext_supported_matches_oracle():
    """Theorem 25.3 check in the library (host code) vs the oracle's, for all p <= 257."""
    for q in range(3, 258):
        if R.valid_p(q):
            assert R.ext_supported(q) == oracle.ext_condition(q), q
    assert not R.ext_supported(9)


def test_status_strings():
    for st in range(9):
        assert R._lib.raid6c_status_string(st)


def test_no_device_is_reported_not_faked():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(R.Raid6Error, match="NO_DEVICE"):
        R.Plan(13, 12, 4096)
    with pytest.raises(R.Raid6Error):
        R.encode(13, 1, [0], 0, 0, 16)  # NULL pointers are rejected before any device call


def test_single_erasure_argument_checks_need_no_device():
    """lost_j = RAID6C_NONE is completed on the host before any device call: a bad lost_i is still
    an index error, and a well-formed single erasure gets past the index check (to the NULL-strip
    check here), with or without a GPU."""
    assert R.NONE == -1
    null4 = [0, 0, 0, 0]
    for bad_i in (-1, 4, 7):
        with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
            R.recover(5, 2, bad_i, R.NONE, null4, 16)
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        R.recover(5, 2, 0, -2, null4, 16)
    for i in range(4):
        with pytest.raises(R.Raid6Error, match="E_NULL"):
            R.recover(5, 2, i, R.NONE, null4, 16)


def test_build_and_shard_import_without_library():
    """A fresh checkout has no libraid6c.so: the build module (which makes it) and the host
    sharding logic must import, while the binding itself must fail loudly (no fallback)."""
    import sys
    env = dict(os.environ, RAID6C_LIB="/nonexistent/libraid6c.so")
    code = ("import paper_cs_0611109_b200.build, paper_cs_0611109_b200.shard\n"
            "try:\n"
            "    from paper_cs_0611109_b200 import raid6c\n"
            "except ImportError as e:\n"
            "    assert 'no CPU fallback' in str(e); print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr


def _build_c_example(out):
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_api_roundtrip.c"), "-L", os.path.dirname(R.LIB_PATH), "-lraid6c",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{os.path.dirname(R.LIB_PATH)}", "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_example_compiles_and_links(tmp_path):
    """The boundary is a plain C ABI: a C program includes raid6c.h and links libraid6c.so."""
    if os.path.basename(R.LIB_PATH) != "libraid6c.so":
        pytest.skip("variant library")
    r = _build_c_example(str(tmp_path / "c_api_roundtrip"))
    assert r.returncode == 0, r.stderr
