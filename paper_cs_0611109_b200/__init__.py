"""B200-native Z_p-RAID (arxiv cs/0611109): C-ABI library libraid6c.so over hand-written
sm_100a kernels, plus this thin ctypes binding.  See include/raid6c.h and DESIGN.md."""
from .raid6c import (Erasure, Plan, Raid6Error, aligned_stride, count_mismatch, encode, fill,  # noqa: F401
                     has_fast_path, ext_supported, launch_count, parity_bytes, recover, valid_p, word_count, LIB_PATH, EXPORTED)
