"""Thin Python binding of libraid6c.so (include/raid6c.h) -- argument marshalling only.

Every step of the method runs in the library's sm_100a kernels.  PyTorch is used here only
to hand over device/host memory and streams.  If the shared library is missing the import
fails loudly: there is no fallback implementation.

Names follow the C ABI: ``encode`` / ``recover`` are the north-star single-stripe calls
(raid6c_encode / raid6c_recover), ``Plan`` wraps raid6c_plan_* and the batched calls.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAID6C_LIB") or os.path.join(_HERE, "libraid6c.so")  # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libraid6c.so not found at {LIB_PATH}: build it with `python -m paper_cs_0611109_b200.build` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

_u8p = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int
_vp = ctypes.c_void_p


class Erasure(ctypes.Structure):
    _fields_ = [("lost_i", ctypes.c_int32), ("lost_j", ctypes.c_int32)]


# (name, restype, argtypes) -- must match include/raid6c.h
_SIGS = [
    ("raid6c_word_count", _sz, [_i, _sz]),
    ("raid6c_parity_bytes", _sz, [_i, _sz]),
    ("raid6c_valid_p", _i, [_i]),
    ("raid6c_has_fast_path", _i, [_i]),
    ("raid6c_ext_supported", _i, [_i]),
    ("raid6c_status_string", ctypes.c_char_p, [_i]),
    ("raid6c_last_cuda_error", ctypes.c_char_p, []),
    ("raid6c_launch_count", ctypes.c_uint64, []),
    ("raid6c_plan_create", _i, [ctypes.POINTER(_vp), _i, _i, _sz, _i, _vp]),
    ("raid6c_plan_destroy", _i, [_vp]),
    ("raid6c_plan_set_stream", _i, [_vp, _vp]),
    ("raid6c_sync", _i, [_vp]),
    ("raid6c_encode", _i, [_i, _i, ctypes.POINTER(_vp), _vp, _vp, _sz]),
    ("raid6c_recover", _i, [_i, _i, _i, _i, ctypes.POINTER(_vp), _sz]),
    ("raid6c_encode_strided", _i, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _i]),
    ("raid6c_recover_strided", _i, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _i, _vp, _i, _i]),
    ("raid6c_scrub_strided", _i, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _i, _vp]),
    ("raid6c_update_strided", _i, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _i, _vp, _sz, _vp, _i, _i]),
    ("raid6c_rs_encode_strided", _i, [_i, _sz, _vp, _sz, _sz, _vp, _vp, _sz, _i, _vp]),
    ("raid6c_rs_recover_strided", _i, [_i, _sz, _vp, _sz, _sz, _vp, _vp, _sz, _i, _vp, _i, _i, _vp]),
    ("raid6c_xgpu_range_bytes", _sz, [_i, _sz, _i]),
    ("raid6c_partial_strided", _i, [_vp, ctypes.POINTER(_vp), _sz, _sz, _i, _vp, _i, _i, _i, _i, _i,
                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _sz]),
    ("raid6c_combine_strided", _i, [_vp, ctypes.POINTER(_vp), _sz, _sz, _i, _vp, _i, _i, _i,
                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _sz, _sz]),
    ("raid6c_dev_alloc", _i, [_sz, _i, ctypes.POINTER(_vp)]),
    ("raid6c_dev_free", _i, [_vp]),
    ("raid6c_ipc_export", _i, [_vp, ctypes.c_char_p]),
    ("raid6c_ipc_open", _i, [ctypes.c_char_p, _i, ctypes.POINTER(_vp)]),
    ("raid6c_ipc_close", _i, [_vp]),
    ("raid6c_encode_host", _i, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _i]),
    ("raid6c_recover_host", _i, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _i, _vp, _i]),
    ("raid6c_host_traffic", _i, [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
    ("raid6c_fill", _i, [_vp, _sz, _sz, _sz, _i, _i, ctypes.c_uint64, _i, _i, _i, _i, _vp]),
    ("raid6c_count_mismatch", _i, [_vp, _vp, _sz, _vp, _vp]),
    ("raid6c_digest", _i, [_vp, _sz, _sz, _sz, _i, _i, _vp, _vp]),
]
for _name, _res, _args in _SIGS:
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = [s[0] for s in _SIGS]
STATUS = {0: "RAID6C_OK", 1: "RAID6C_E_INVALID_P", 2: "RAID6C_E_INVALID_N", 3: "RAID6C_E_INVALID_INDEX",
          4: "RAID6C_E_NULL", 5: "RAID6C_E_SIZE", 6: "RAID6C_E_CUDA", 7: "RAID6C_E_NO_DEVICE", 8: "RAID6C_E_PLAN"}


NONE = -1  # RAID6C_NONE: lost_j of a single erasure (host arguments only)


class Raid6Error(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.raid6c_status_string(status).decode()
        cuda = _lib.raid6c_last_cuda_error().decode() if status == 6 else ""
        super().__init__(f"{where}: {STATUS.get(status, status)} ({msg}){' ' + cuda if cuda else ''}")


def _check(st: int, where: str):
    if st != 0:
        raise Raid6Error(st, where)


def _ptr(x) -> int:
    """Device/host address of a tensor (or an int address)."""
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream_handle(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


# ------------------------------------------------------------------ host-side helpers
def word_count(p: int, nbytes: int) -> int:
    return int(_lib.raid6c_word_count(p, nbytes))


def parity_bytes(p: int, nbytes: int) -> int:
    return int(_lib.raid6c_parity_bytes(p, nbytes))


def valid_p(p: int) -> bool:
    return bool(_lib.raid6c_valid_p(p))


def has_fast_path(p: int) -> bool:
    return bool(_lib.raid6c_has_fast_path(p))


def ext_supported(p: int) -> bool:
    """Theorem 25.3: p admits the extended code (up to 2p-1 data strips)."""
    return bool(_lib.raid6c_ext_supported(p))


def launch_count() -> int:
    return int(_lib.raid6c_launch_count())


# ------------------------------------------------------------------ north-star calls
def encode(p: int, N: int, strips, P, Q, nbytes: int) -> None:
    """raid6c_encode: strips = N device tensors/addresses; P, Q device (parity_bytes)."""
    arr = (_vp * N)(*[_ptr(s) for s in strips])
    _check(_lib.raid6c_encode(p, N, arr, _ptr(P), _ptr(Q), nbytes), "raid6c_encode")


def recover(p: int, N: int, lost_i: int, lost_j: int, strips, nbytes: int) -> None:
    """raid6c_recover: strips = N+2 device tensors/addresses (0..N-1 data, N = P, N+1 = Q).
    lost_j = NONE: strip lost_i alone (runs as the pair (lost_i, Q), or (P, Q) for lost_i = Q)."""
    arr = (_vp * (N + 2))(*[_ptr(s) for s in strips])
    _check(_lib.raid6c_recover(p, N, lost_i, lost_j, arr, nbytes), "raid6c_recover")


def _erasure_array(pairs):
    """Host erasure pairs as a ctypes array of raid6c_erasure (a prebuilt one passes through)."""
    if isinstance(pairs, ctypes.Array) and getattr(pairs, "_type_", None) is Erasure:
        return pairs
    arr = (Erasure * len(pairs))()
    for s, (i, j) in enumerate(pairs):
        arr[s].lost_i, arr[s].lost_j = int(i), int(j)
    return arr


erasure_array = _erasure_array  # marshal a host pair list once, reuse it across calls


def fill(dst, strip_stride: int, stripe_stride: int, nbytes: int, nstrips: int, nstripes: int, seed: int,
         cfg: int, stripe0: int, strip0: int, sparse_mode: int = 0, stream=None) -> None:
    _check(_lib.raid6c_fill(_ptr(dst), strip_stride, stripe_stride, nbytes, nstrips, nstripes, seed, cfg, stripe0,
                            strip0, sparse_mode, _stream_handle(stream)), "raid6c_fill")


def count_mismatch(a, b, nbytes: int, count_dev, stream=None) -> None:
    _check(_lib.raid6c_count_mismatch(_ptr(a), _ptr(b), nbytes, _ptr(count_dev), _stream_handle(stream)),
           "raid6c_count_mismatch")


def digest(src, strip_stride: int, stripe_stride: int, nbytes: int, nstrips: int, nstripes: int, out_dev,
           stream=None) -> None:
    """raid6c_digest: out_dev[s*nstrips + t] = 64-bit digest of strip t of stripe s (device int64/uint64
    tensor of nstrips*nstripes entries; the host definition is synthetic/digest.py)."""
    _check(_lib.raid6c_digest(_ptr(src), strip_stride, stripe_stride, nbytes, nstrips, nstripes, _ptr(out_dev),
                              _stream_handle(stream)), "raid6c_digest")


# ------------------------------------------------------------------ NEXT-3: RS baseline
def rs_encode_strided(N, nbytes, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, stream=None):
    _check(_lib.raid6c_rs_encode_strided(N, nbytes, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                         parity_stride, num_stripes, _stream_handle(stream)), "raid6c_rs_encode_strided")


def rs_recover_strided(N, nbytes, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, erasures,
                       stream=None):
    if hasattr(erasures, "is_cuda") and erasures.is_cuda:
        _check(_lib.raid6c_rs_recover_strided(N, nbytes, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                              parity_stride, num_stripes, _ptr(erasures), erasures.shape[0], 1,
                                              _stream_handle(stream)), "raid6c_rs_recover_strided")
    else:
        arr = _erasure_array(erasures)
        _check(_lib.raid6c_rs_recover_strided(N, nbytes, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                              parity_stride, num_stripes, ctypes.cast(arr, _vp), len(arr), 0,
                                              _stream_handle(stream)), "raid6c_rs_recover_strided")


# ------------------------------------------------------------------ plans
class Plan:
    """raid6c_plan for (p, N, nbytes) on `device`, ordered on `stream` (torch stream or handle)."""

    def __init__(self, p: int, N: int, nbytes: int, device: int = 0, stream=None):
        h = _vp()
        _check(_lib.raid6c_plan_create(ctypes.byref(h), p, N, nbytes, device, _stream_handle(stream)),
               "raid6c_plan_create")
        self._h = h
        self.p, self.N, self.nbytes, self.device = p, N, nbytes, device
        self.pbytes = parity_bytes(p, nbytes)

    def close(self):
        if getattr(self, "_h", None):
            _lib.raid6c_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream):
        _check(_lib.raid6c_plan_set_stream(self._h, _stream_handle(stream)), "raid6c_plan_set_stream")

    def sync(self):
        _check(_lib.raid6c_sync(self._h), "raid6c_sync")

    # raw-address forms (the C signatures)
    def encode_strided(self, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes):
        _check(_lib.raid6c_encode_strided(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                          parity_stride, num_stripes), "raid6c_encode_strided")

    def recover_strided(self, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, erasures):
        """erasures: list of (i, j) host pairs (1 or num_stripes), or an int32 CUDA tensor [S, 2]."""
        if hasattr(erasures, "is_cuda") and erasures.is_cuda:
            n = erasures.shape[0]
            _check(_lib.raid6c_recover_strided(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                               parity_stride, num_stripes, _ptr(erasures), n, 1),
                   "raid6c_recover_strided")
        else:
            arr = _erasure_array(erasures)
            _check(_lib.raid6c_recover_strided(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                               parity_stride, num_stripes, ctypes.cast(arr, _vp), len(arr), 0),
                   "raid6c_recover_strided")

    def scrub_strided(self, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, bad_words):
        """bad_words: uint32 (or int32) CUDA tensor [num_stripes], overwritten with per-stripe counts."""
        _check(_lib.raid6c_scrub_strided(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                         parity_stride, num_stripes, _ptr(bad_words)), "raid6c_scrub_strided")

    def update_strided(self, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, new_data,
                       new_stride, disks):
        """disks: list of strip indices (1 or num_stripes) or an int32 CUDA tensor [S]."""
        if hasattr(disks, "is_cuda") and disks.is_cuda:
            _check(_lib.raid6c_update_strided(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                              parity_stride, num_stripes, _ptr(new_data), new_stride, _ptr(disks),
                                              disks.shape[0], 1), "raid6c_update_strided")
        else:
            arr = (ctypes.c_int32 * len(disks))(*[int(k) for k in disks])
            _check(_lib.raid6c_update_strided(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                              parity_stride, num_stripes, _ptr(new_data), new_stride,
                                              ctypes.cast(arr, _vp), len(arr), 0), "raid6c_update_strided")

    def encode_host(self, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes):
        _check(_lib.raid6c_encode_host(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                       parity_stride, num_stripes), "raid6c_encode_host")

    def recover_host(self, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, erasures):
        arr = _erasure_array(erasures)
        _check(_lib.raid6c_recover_host(self._h, _ptr(data), strip_stride, stripe_stride, _ptr(P), _ptr(Q),
                                        parity_stride, num_stripes, ctypes.cast(arr, _vp), len(arr)),
               "raid6c_recover_host")

    def host_traffic(self):
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.raid6c_host_traffic(self._h, ctypes.byref(a), ctypes.byref(b)), "raid6c_host_traffic")
        return int(a.value), int(b.value)

    # tensor-layout forms: data [S, N, strip_stride] uint8, parity [S, 2, parity_stride] uint8
    def encode_batch(self, data, parity):
        S, N, ss = data.shape
        assert N == self.N and parity.shape[0] == S and parity.shape[1] == 2
        ps = parity.shape[2]
        f = self.encode_host if not data.is_cuda else self.encode_strided
        f(data, ss, N * ss, parity, _ptr(parity) + ps, 2 * ps, S)

    def recover_batch(self, data, parity, erasures):
        S, N, ss = data.shape
        assert N == self.N and parity.shape[0] == S and parity.shape[1] == 2
        ps = parity.shape[2]
        if data.is_cuda:
            self.recover_strided(data, ss, N * ss, parity, _ptr(parity) + ps, 2 * ps, S, erasures)
        else:
            self.recover_host(data, ss, N * ss, parity, _ptr(parity) + ps, 2 * ps, S, erasures)


    # ------------------------------------------------ NEXT-4: cross-GPU stripe layout
    def xgpu_range_bytes(self, num_ranks: int) -> int:
        return xgpu_range_bytes(self.p, self.nbytes, num_ranks)

    def _erasure_args(self, erasures):
        """(pointer, count, on_device) for None (encode), host pairs, or an int32 CUDA tensor [S, 2]."""
        if erasures is None:
            return None, 0, 0, None
        if hasattr(erasures, "is_cuda") and erasures.is_cuda:
            return _ptr(erasures), int(erasures.shape[0]), 1, None
        arr = _erasure_array(erasures)
        return ctypes.cast(arr, _vp), len(arr), 0, arr

    def partial_strided(self, strips, data_stride, parity_stride, num_stripes, erasures, k_lo, k_hi,
                        part_p, part_q, part_stride, range_bytes):
        """raid6c_partial_strided.  strips: N+2 device addresses by global index (None = not held);
        part_p / part_q: one device address per word range (owner slots)."""
        st = (_vp * (self.N + 2))(*[None if x is None else _ptr(x) for x in strips])
        pp = (_vp * len(part_p))(*[_ptr(x) for x in part_p])
        pq = (_vp * len(part_q))(*[_ptr(x) for x in part_q])
        ep, en, eo, _keep = self._erasure_args(erasures)
        _check(_lib.raid6c_partial_strided(self._h, st, data_stride, parity_stride, num_stripes, ep, en, eo, k_lo, k_hi,
                                           len(part_p), pp, pq, part_stride, range_bytes), "raid6c_partial_strided")

    def combine_strided(self, strips, data_stride, parity_stride, num_stripes, erasures, src_p, src_q, part_stride,
                        range_lo, range_hi):
        """raid6c_combine_strided.  strips: N+2 device addresses by global index (outputs written);
        src_p / src_q: one device address per partial source."""
        st = (_vp * (self.N + 2))(*[None if x is None else _ptr(x) for x in strips])
        sp = (_vp * len(src_p))(*[_ptr(x) for x in src_p])
        sq = (_vp * len(src_q))(*[_ptr(x) for x in src_q])
        ep, en, eo, _keep = self._erasure_args(erasures)
        _check(_lib.raid6c_combine_strided(self._h, st, data_stride, parity_stride, num_stripes, ep, en, eo, len(src_p),
                                           sp, sq, part_stride, range_lo, range_hi), "raid6c_combine_strided")


# ------------------------------------------------------------------ NEXT-4: cross-GPU layout helpers
def xgpu_range_bytes(p: int, nbytes: int, num_ranks: int) -> int:
    """raid6c_xgpu_range_bytes: word-range size for num_ranks owners (host only)."""
    r = int(_lib.raid6c_xgpu_range_bytes(p, nbytes, num_ranks))
    if r == 0:
        raise Raid6Error(5, "raid6c_xgpu_range_bytes")
    return r


# ------------------------------------------------------------------ inter-process device memory (NEXT-4)
def dev_alloc(nbytes: int, device: int) -> int:
    h = _vp()
    _check(_lib.raid6c_dev_alloc(nbytes, device, ctypes.byref(h)), "raid6c_dev_alloc")
    return int(h.value)


def dev_free(ptr: int) -> None:
    _check(_lib.raid6c_dev_free(ptr), "raid6c_dev_free")


def ipc_export(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(_lib.raid6c_ipc_export(ptr, buf), "raid6c_ipc_export")
    return buf.raw


def ipc_open(handle: bytes, device: int) -> int:
    assert len(handle) == 64
    h = _vp()
    _check(_lib.raid6c_ipc_open(handle, device, ctypes.byref(h)), "raid6c_ipc_open")
    return int(h.value)


def ipc_close(ptr: int) -> None:
    _check(_lib.raid6c_ipc_close(ptr), "raid6c_ipc_close")


def aligned_stride(nbytes: int, align: int = 256) -> int:
    return (nbytes + align - 1) // align * align
