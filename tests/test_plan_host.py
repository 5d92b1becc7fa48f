"""The row-slab planner behind the C-ABI (spmvk_plan_*, csrc/nccl_dist.cu) --
pure host code, no GPU -- against a direct Python statement of SURVEY §8e:
group-aligned slabs, slot-balanced cuts, the fused path's receive ranges and
the halo's send / receive lists (every send on one side is the matching
receive on the other)."""
import ctypes as C

import numpy as np
import pytest

from paper_1012_2270_b200 import partition as pt
from paper_1012_2270_b200._lib import lib


def model_slabs(n, G, P):
    groups = (n + G - 1) // G
    S = (groups + P - 1) // P * G
    return [(min(n, p * S), min(n, (p + 1) * S)) for p in range(P)], S


def model_weighted(lens, G, P):
    n = len(lens)
    groups = (n + G - 1) // G
    cum, acc = [], 0
    for g in range(groups):
        s = min(G, n - g * G)
        acc += s * max(lens[g * G: g * G + s])
        cum.append(acc)
    cuts = [0]
    for p in range(1, P):
        g = next((i for i, c in enumerate(cum) if c * P >= acc * p), groups) + 1 if acc else 0
        cuts.append(min(n, max(cuts[-1], g * G)))
    cuts.append(n)
    return list(zip(cuts, cuts[1:]))


@pytest.mark.parametrize("n,G,P", [(0, 32, 1), (1, 32, 4), (1000, 32, 3), (4096, 32, 8),
                                   (4097, 256, 8), (100, 1, 7), (134217728, 32, 8)])
def test_slab_bounds(n, G, P):
    want, S = model_slabs(n, G, P)
    got = pt.slab_bounds(n, G, P)
    assert [(s.row_begin, s.row_end) for s in got] == want
    assert all(s.pad_rows == S for s in got)
    assert all(s.row_begin % G == 0 or s.row_begin == n for s in got)


def test_plan_errors():
    b = (C.c_uint64 * 4)()
    assert lib().spmvk_plan_slabs(10, 0, 3, b, None) == 1
    assert lib().spmvk_plan_slabs(10, 4, 0, b, None) == 1
    assert lib().spmvk_plan_receive(2, b, b, 7, b) == 1
    nr, ns = C.c_int(), C.c_int()
    assert lib().spmvk_plan_halo(2, 2, b, b, b, C.byref(nr), b, C.byref(ns)) == 1


@pytest.mark.parametrize("seed", range(12))
def test_weighted_slab_bounds(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    lens = np.minimum(rng.pareto(1.5, n) * 4, 4096).astype(np.uint32)
    if seed % 4 == 0:
        lens[:] = 0
    G = int(rng.choice([1, 4, 32, 64]))
    P = int(rng.integers(1, 9))
    assert pt.weighted_slab_bounds(lens, G, P) == model_weighted(lens.tolist(), G, P)


@pytest.mark.parametrize("seed", range(20))
def test_receive_and_halo_lists(seed):
    rng = np.random.default_rng(100 + seed)
    P = int(rng.integers(1, 9))
    n = int(rng.integers(P, 5000))
    slabs = pt.slab_bounds(n, int(rng.choice([1, 8, 32])), P)
    ranges = []
    for s in slabs:
        if s.rows == 0 or rng.random() < 0.15:
            ranges.append((1, 0))  # no entries
            continue
        a = int(rng.integers(0, n))
        b = int(rng.integers(a, n))
        ranges.append((a, b))
    rec = pt.fused_receive_ranges(slabs, ranges, "halo")
    for s, (lo, hi), (cmin, cmax) in zip(slabs, rec, ranges):
        want_lo, want_hi = s.row_begin, s.row_end
        if cmin <= cmax:
            want_lo, want_hi = min(want_lo, cmin), max(want_hi, cmax + 1)
        assert (lo, hi) == ((want_lo, want_hi) if want_lo < want_hi else (0, 0))
    assert pt.fused_receive_ranges(slabs, ranges, "allgather") == [(0, slabs[-1].row_end)] * P
    # halo lists: receive = columns read that a peer owns; sends mirror them
    bounds = (C.c_uint64 * (P + 1))(*([s.row_begin for s in slabs] + [slabs[-1].row_end]))
    cr = (C.c_uint64 * (2 * P))(*[v for r in ranges for v in r])
    sends, recvs = {}, {}
    for s in slabs:
        rv, sv = (C.c_uint64 * (3 * P))(), (C.c_uint64 * (3 * P))()
        nr, ns = C.c_int(), C.c_int()
        assert lib().spmvk_plan_halo(s.rank, P, bounds, cr, rv, C.byref(nr), sv,
                                     C.byref(ns)) == 0
        recvs[s.rank] = [tuple(rv[3 * k: 3 * k + 3]) for k in range(nr.value)]
        sends[s.rank] = [tuple(sv[3 * k: 3 * k + 3]) for k in range(ns.value)]
        cmin, cmax = ranges[s.rank]
        want = [(q.rank, max(cmin, q.row_begin), min(cmax + 1, q.row_end)) for q in slabs
                if q.rank != s.rank and cmin <= cmax and max(cmin, q.row_begin) <
                min(cmax + 1, q.row_end)]
        assert recvs[s.rank] == want
        assert pt.halo_plan(s, cmin, cmax, slabs) == want
    for r, lst in recvs.items():
        for q, c0, c1 in lst:
            assert (r, c0, c1) in sends[q]
    assert sum(map(len, recvs.values())) == sum(map(len, sends.values()))
