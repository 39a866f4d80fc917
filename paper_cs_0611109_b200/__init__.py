"""B200-native Z_p-RAID (arxiv cs/0611109): C-ABI library libraid6c.so over hand-written
sm_100a kernels, plus this thin ctypes binding.  See include/raid6c.h and DESIGN.md.

The binding (``raid6c``) is imported on first attribute access, so that ``build`` (which
produces libraid6c.so) and ``shard`` (host-side sharding logic) import in a tree where the
library has not been built yet.  Any use of the method itself goes through ``raid6c``, which
raises ImportError when libraid6c.so is missing -- there is no CPU fallback.
"""
_BINDING = ("Erasure", "Plan", "Raid6Error", "aligned_stride", "count_mismatch", "encode", "fill",
            "has_fast_path", "ext_supported", "launch_count", "parity_bytes", "recover", "valid_p",
            "word_count", "LIB_PATH", "EXPORTED")


def __getattr__(name):
    if name in _BINDING:
        from . import raid6c
        return getattr(raid6c, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
