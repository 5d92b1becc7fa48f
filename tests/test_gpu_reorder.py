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


# ------------------------------------------- general permutations (both modes)
def permute_sym(m: orc.Csr, p) -> orc.Csr:
    """Host restatement of apply_permutation(m, p, Symmetric): entries
    (inv[r], inv[c], v), canonical order."""
    p = np.asarray(p, np.int64)
    inv = np.empty_like(p)
    inv[p] = np.arange(p.size)
    rows = np.repeat(np.arange(m.rows), np.diff(m.rp.astype(np.int64)))
    r2, c2 = inv[rows], inv[m.col.astype(np.int64)]
    o = np.lexsort((c2, r2))
    rp = np.concatenate([[0], np.cumsum(np.bincount(r2, minlength=m.rows))]).astype(np.uint32)
    return orc.Csr(m.rows, m.cols, rp, c2[o].astype(np.uint32), m.val[o])


def same_csr(a: sk.CsrMatrix, w: orc.Csr) -> bool:
    rp, col, val = a.to_host()
    return bitwise(rp, w.rp) and bitwise(col, w.col) and bitwise(val, w.val.astype(val.dtype))


def test_apply_permutation_reference_cases(cuda, golden):
    """tests/test_reorder.cpp:55-60, 75-86, 98-106."""
    om = golden_csr(golden["example8"], "m")
    m = triplets(om)
    assert same_csr(sk.apply_permutation(m, sk.Permutation.identity(8)), om)
    tiny = sk.canonicalize([(0, 0, 1.0)], 2, 2)
    rp, col, val = sk.apply_permutation(tiny, sk.Permutation([1, 0])).to_host()
    assert rp.tolist() == [0, 0, 1] and col.tolist() == [0] and val.tolist() == [1.0]
    with pytest.raises(sk.InvalidArgument, match="permutation length 1 does not match 2 rows"):
        sk.apply_permutation(tiny, sk.Permutation([0]))
    sym = sk.canonicalize([(0, 1, 5.0)], 2, 2)
    rp, col, val = sk.apply_permutation(sym, sk.Permutation([1, 0]), "symmetric").to_host()
    assert rp.tolist() == [0, 0, 1] and col.tolist() == [0] and val.tolist() == [5.0]
    rect = sk.canonicalize([(0, 1, 5.0)], 2, 3)
    with pytest.raises(sk.InvalidArgument, match="symmetric mode needs a square matrix"):
        sk.apply_permutation(rect, sk.Permutation([1, 0]), "symmetric")
    with pytest.raises(sk.InvalidArgument, match="not a bijection on 0..1"):
        sk.Permutation([0, 0])
    with pytest.raises(sk.InvalidArgument, match="not a bijection"):
        sk.Permutation([2, 0])


@pytest.mark.parametrize("prec", [8, 4])
def test_random_permutations_both_modes(cuda, prec):
    """Random bijections (tests/test_reorder.cpp:108-133): rows-only and
    symmetric results equal the host restatement bitwise; rows-only commutes
    with the SpMV (y_perm[i] == y[p[i]], permute_vector back = y)."""
    rng = np.random.default_rng(11)
    for seed in range(40):
        om = orc.random_small(seed)
        m = triplets(om)
        p = sk.Permutation(rng.permutation(om.rows))
        a = sk.build_csr(m, prec)
        want = permute_rows(om, p.map())
        assert same_csr(sk.apply_permutation(a, p), want), seed
        if om.rows == om.cols:
            assert same_csr(sk.apply_permutation(a, p, "symmetric"),
                            permute_sym(om, p.map())), seed
        dt = torch.float64 if prec == 8 else torch.float32
        x = torch.from_numpy(orc.random_vector(om.cols, seed)).cuda().to(dt)
        y = sk.spmv_csr(a, x)
        yp = sk.spmv_csr(sk.apply_permutation(a, p), x)
        assert torch.equal(yp, y[torch.from_numpy(p.map().astype(np.int64)).cuda()]), seed
        assert torch.equal(sk.permute_vector(p, yp, inverse=True), y), seed
        assert torch.equal(sk.permute_vector(p, y), yp), seed


def test_symmetric_permutation_at_scale(cuda):
    """Symmetric mode on a 7-point 48^3 stencil with a random bijection:
    segmented re-sort of 770k entries; A' x' = (A x)' (x' = x permuted)."""
    csr = sk.CsrMatrix.stencil(7, 48)
    n = csr.num_rows
    p = sk.Permutation(np.random.default_rng(3).permutation(n))
    b = sk.apply_permutation(csr, p, "symmetric")
    rp, col, val = b.to_host()
    assert all(np.all(np.diff(col[rp[i]:rp[i + 1]].astype(np.int64)) > 0) for i in range(0, n, 997))
    x = torch.from_numpy(orc.random_vector(n, 1)).cuda()
    y = sk.spmv_csr(csr, x)
    yp = sk.spmv_csr(b, sk.permute_vector(p, x))
    # same entries per row, but a different summation order: compare to 1e-12
    assert torch.allclose(sk.permute_vector(p, y), yp, rtol=1e-12, atol=1e-12)
