"""Descending row reordering on the device against the
reference: descending_row_permutation (src/reorder.cpp:35-42) and
apply_permutation RowsOnly (:44-61); the reference's tests pin the M8 map
[6,0,5,7,1,2,3,4] (tests/test_reorder.cpp:62-65), padding 7 -> 3 on M8 with
groups of 4 (:88-96) and optimality under exhaustive enumeration when the
groups divide the rows (tests/acceptance.cpp:190-218)."""
import itertools

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import bitwise, golden_csr, triplets
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu


def permute_rows(m: orc.Csr, p) -> orc.Csr:
    """Host restatement of apply_permutation(m, p, RowsOnly)."""
    lens = m.lens().astype(np.int64)
    rp = np.concatenate([[0], np.cumsum(lens[p])]).astype(np.uint32)
    idx = np.concatenate([np.arange(m.rp[o], m.rp[o + 1]) for o in p]) if m.nnz else np.array([], int)
    return orc.Csr(m.rows, m.cols, rp, m.col[idx], m.val[idx])


def padding_of(lens, g):
    slots = nnz = 0
    for s0 in range(0, len(lens), g):
        blk = lens[s0:s0 + g]
        slots += len(blk) * max(blk)
        nnz += sum(blk)
    return slots - nnz


def test_example8_map_and_padding(cuda, golden):
    g = golden["example8"]
    m = triplets(golden_csr(g, "m"))
    p = sk.descending_row_permutation(m)
    assert p.tolist() == [6, 0, 5, 7, 1, 2, 3, 4] and bitwise(p, g["descending_map"])
    before = sk.fill_report(sk.build_rgcsr(m, 4)).artificial_zeros
    csr2, p2 = sk.apply_descending_permutation(m)
    assert bitwise(p2, p)
    after = sk.fill_report(sk.build_rgcsr(csr2, 4)).artificial_zeros
    assert (before, after) == (7, 3)


def test_random_maps_and_permuted_arrays(cuda):
    for seed in range(700, 760):
        om = orc.random_small(seed)
        want = orc.descending_map(om)
        if orc.ref_available():
            assert bitwise(want, orc.RefMatrix.from_csr(om).descending_map())
        csr2, p = sk.apply_descending_permutation(triplets(om))
        assert bitwise(p, want), seed
        pm = permute_rows(om, want)
        rp, col, val = csr2.to_host()
        assert bitwise(rp, pm.rp) and bitwise(col, pm.col) and bitwise(val, pm.val), seed
        x = orc.random_vector(om.cols, seed)
        y = sk.spmv_rgcsr(sk.build_rgcsr(triplets(om), 4), x)
        y2 = sk.spmv_rgcsr(sk.build_rgcsr(csr2, 4), x)
        assert bitwise(y2, y[want])  # spmv(P m, x)[i] == spmv(m, x)[map[i]]


def test_descending_is_optimal_by_enumeration(cuda):
    """tests/acceptance.cpp:190-218: 60 cases with rows in {4, 8}, G in {2, 4}."""
    for seed in range(60):
        st = orc._MT(seed)
        rows = 8 if seed % 2 == 0 else 4
        cols = 1 + st.next() % 8
        density = 0.1 + 0.5 * st.unit_real()
        om = orc.random_matrix(rows, cols, density, -8, 8, True, True, st.next())
        csr2, _ = sk.apply_descending_permutation(triplets(om))
        lens = sorted(om.lens().tolist())
        for G in (2, 4):
            got = sk.fill_report(sk.build_rgcsr(csr2, G)).artificial_zeros
            best = min(padding_of(list(q), G) for q in set(itertools.permutations(lens)))
            assert got == best, (seed, G)


def test_powerlaw_padding_collapses(cuda):
    """Config 3 at 1M rows: RgCSR G=32 fill before / after descending order."""
    om = orc.powerlaw(1_000_000, 7)
    csr = sk.build_csr(triplets(om))
    before = sk.fill_report(sk.build_rgcsr(csr, 32)).fill_percent
    csr2, p = sk.apply_descending_permutation(csr)
    after = sk.fill_report(sk.build_rgcsr(csr2, 32)).fill_percent
    assert before > 300 and after < 5, (before, after)
    x = torch.from_numpy(orc.random_vector(om.cols, 1)).cuda()
    y = sk.spmv_rgcsr(sk.build_rgcsr(csr, 32), x)
    y2 = sk.spmv_rgcsr(sk.build_rgcsr(csr2, 32), x)
    assert torch.equal(y2, y[torch.from_numpy(p.astype(np.int64)).cuda()])
