"""CPU model of the fused peer-memory step's routing (partition.py,
spmvk_dist_set_rows): after any number of steps every rank's window holds the
exact iterate on the rows it reads, for the all-gather and halo plans."""
import numpy as np
import pytest

import oracle as orc
from paper_1012_2270_b200 import partition as pt


def slab_matvec_factory(m, slabs):
    rp, col, val = m.rp, m.col, m.val

    def mv(rank, x):
        s = slabs[rank]
        out = np.zeros(s.rows)
        for r in range(s.row_begin, s.row_end):
            acc = 0.0
            for k in range(rp[r], rp[r + 1]):
                acc += val[k] * x[col[k]]
            out[r - s.row_begin] = acc * 0.0625
        return out
    return mv


def col_range(m, s):
    if s.rows == 0 or m.rp[s.row_end] == m.rp[s.row_begin]:
        return (1, 0)
    c = m.col[m.rp[s.row_begin]: m.rp[s.row_end]]
    return (int(c.min()), int(c.max()))


@pytest.mark.parametrize("mode", ["allgather", "halo"])
@pytest.mark.parametrize("P,G", [(1, 4), (2, 4), (3, 8), (5, 2), (8, 4)])
def test_windows_hold_the_iterate(mode, P, G):
    m = orc.stencil(7, 6)  # 216 rows, banded: halo = neighbouring planes
    slabs = pt.slab_bounds(m.rows, G, P)
    ranges = [col_range(m, s) for s in slabs]
    recv = pt.fused_receive_ranges(slabs, ranges, mode)
    x0 = orc.random_vector(m.cols, 1)
    mv = slab_matvec_factory(m, slabs)
    want = x0.copy()
    for k in range(4):
        want = np.concatenate([mv(s.rank, want) for s in slabs])
        got = pt.simulate_fused_routing(slabs, recv, mv, x0, k + 1)
        for s, w in zip(slabs, got):
            lo, hi = recv[s.rank]
            assert np.array_equal(w[lo:hi], want[lo:hi]), (mode, P, s.rank, k)
            cmin, cmax = ranges[s.rank]
            if cmin <= cmax:
                assert lo <= cmin and cmax < hi
    if mode == "halo" and P > 1:  # only neighbouring planes travel
        assert all(hi - lo < m.rows for lo, hi in recv)


def test_receive_ranges_edge_cases():
    slabs = pt.slab_bounds(10, 4, 4)  # last slab empty
    assert slabs[-1].rows == 0
    recv = pt.fused_receive_ranges(slabs, [(0, 5), (2, 9), (8, 9), (1, 0)], "halo")
    assert recv == [(0, 6), (2, 10), (8, 10), (0, 0)]
    assert pt.fused_receive_ranges(slabs, None, "allgather") == [(0, 10)] * 4
