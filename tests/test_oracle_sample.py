"""The segmented full-size oracle harness (tests/oracle_sample.py) equals the oracle run on whole
strips: same P/Q and rebuilt strips (as digests), for ragged lengths, several segments, every
erasure class.  This pins the harness that bench.py's oracle sample and the full-size GPU tests
rely on."""
import numpy as np
import pytest

import oracle
import synthetic
from tests import oracle_sample as OS


@pytest.mark.parametrize("p,N,nbytes,seg", [(5, 4, 1001, 8), (13, 6, 3001, 48), (59, 5, 2051, 232),
                                            (61, 7, 1503, 120), (257, 3, 700, 256)])
def test_segmented_oracle_equals_whole_strips(p, N, nbytes, seg):
    assert OS.segment_bytes(p, seg) % 8 == 0 and OS.segment_bytes(p, seg) % (p - 1) == 0
    assert len(OS.segments(p, nbytes, seg)) >= 2
    pairs = [(0, 1), (1, N), (2, N + 1), (N, N + 1)]
    items = [(3, pairs), (8, pairs[:1])]
    dig, info = OS.stripe_digests(p, N, nbytes, cfg=2, items=items, sparse_of=lambda s: s == 8, threads=3,
                                  seg_target=seg, keep=True)
    assert info["user_bytes"] == (5 + 2) * N * nbytes
    for s, prs in items:
        data = synthetic.stripe_strips(0, 2, s, N, nbytes, sparse=(s == 8))
        P, Q = oracle.encode(p, data, nbytes)
        assert dig[s]["P"] == synthetic.digest(P) and dig[s]["Q"] == synthetic.digest(Q)
        assert np.array_equal(info["strips"][s]["P"], P) and np.array_equal(info["strips"][s]["Q"], Q)
        for (x, y) in prs:
            st = [d.copy() for d in data] + [P.copy(), Q.copy()]
            st[x][:] = 0
            st[y][:] = 0
            oracle.recover(p, N, x, y, st, nbytes)
            orig = data + [P, Q]
            for k in (x, y):
                assert np.array_equal(st[k], orig[k])  # the oracle's own round trip
                assert dig[s][(x, y, k)] == synthetic.digest(st[k])
                assert np.array_equal(info["strips"][s][(x, y, k)], st[k])


def test_data_digests_and_sampling():
    d = OS.data_digests(3, 777, 4, [0, 1], sparse_of=lambda s: s % 2 == 1, threads=2)
    assert d[1][2] == synthetic.digest(synthetic.strip_bytes(0, 4, 1, 2, 777, True))
    assert OS.sample_stripes(4096, 64) == sorted(set(OS.sample_stripes(4096, 64)))
    ss = OS.sample_stripes(4096, 64)
    assert len(ss) == 64 and all(0 <= s < 4096 for s in ss)
    for G in (1, 2, 4, 8):  # every block shard holds sampled stripes
        for r in range(G):
            lo, hi = r * 4096 // G, (r + 1) * 4096 // G
            assert any(lo <= s < hi for s in ss)
    assert OS.sample_stripes(3, 64) == [0, 1, 2]
