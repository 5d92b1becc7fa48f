"""The product's host generators (libspmvk.so) against the oracle's
independent restatement of SURVEY Appendix B and the reference's
banded_matrix / random_vector; config-scale counts pinned by the survey's
probes."""
import numpy as np
import pytest

import oracle as orc
from helpers import bitwise
from paper_1012_2270_b200 import generators as gen


@pytest.mark.parametrize("kind,n", [(5, 1), (5, 2), (5, 37), (7, 1), (7, 9), (27, 2), (27, 11)])
def test_stencils_match_oracle(kind, n):
    a, b = gen.stencil(kind, n), orc.stencil(kind, n)
    assert bitwise(a.row_ptr, b.rp) and bitwise(a.col, b.col) and bitwise(a.val, b.val)


def test_stencil_nnz_formulas():
    assert gen.stencil(5, 1024).nnz == 5 * 1024 ** 2 - 4 * 1024 == 5_238_784
    assert orc.O().orc_stencil(27, 128, None, None, None) == (3 * 128 - 2) ** 3 == 55_742_968
    assert orc.O().orc_stencil(7, 64, None, None, None) == 7 * 64 ** 3 - 6 * 64 ** 2


def test_powerlaw_matches_oracle_and_shape():
    a, b = gen.powerlaw(100_000, 7), orc.powerlaw(100_000, 7)
    assert bitwise(a.row_ptr, b.rp) and bitwise(a.col, b.col) and bitwise(a.val, b.val)
    lens = np.diff(a.row_ptr.astype(np.int64))
    assert lens.min() >= 1 and lens.max() <= 4096 and 14 < lens.mean() < 18


def test_random_vector_matches_reference_convention():
    assert bitwise(gen.random_vector(1000, 1), orc.random_vector(1000, 1))
    if orc.ref_available():
        v = np.empty(1000)
        orc.R().ref_random_vector(1000, 1, v.ctypes.data)
        assert bitwise(gen.random_vector(1000, 1), v)


def test_banded_matches_reference():
    for n, hbw, seed in ((1, 0, 1), (17, 4, 42), (1024, 4, 42), (300, 40, 3)):
        a, b = gen.banded(n, hbw, seed), orc.banded(n, hbw, seed)
        assert bitwise(a.row_ptr, b.rp) and bitwise(a.col, b.col) and bitwise(a.val, b.val)
        if orc.ref_available():
            r = orc.RefMatrix.banded(n, hbw, seed).to_csr()
            assert bitwise(a.val, r.val) and bitwise(a.col, r.col)


def test_sweep_cases_are_canonical():
    for seed in range(9):
        name, m = gen.sweep_case(seed, max_rows=20_000, min_rows=1_000)
        m._validate()
        assert m.nnz > 0 and name
