"""GPU parity of the Hybrid ELL+COO path (K3 width/build, K4/K5 fused SpMV).

Mirrors tests/test_formats.cpp:125-202 (cost table, exhaustive width scan,
K1=1 golden COO, degenerate splits, partition, spmv_hybrid) and the Hybrid
leg of tests/acceptance.cpp:138-173 / :262-295.  Bar: arrays and y bitwise.
"""
import numpy as np
import pytest
import torch

import oracle as orc
from helpers import assert_hybrid_equal, bitwise, golden_csr, triplets
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_example8_golden(cuda, golden):
    g = golden["example8"]
    m = triplets(golden_csr(g, "m"))
    for k1, name in ((None, "hyd"), (0, "hy0"), (1, "hy1"), (3, "hy3")):
        h = sk.build_hybrid(m, k1)
        assert h.slots_per_row == int(g[f"{name}_k1"][0])
        assert_hybrid_equal(h.to_host(), g, f"{name}_")
        assert bitwise(sk.spmv_hybrid(h, np.ones(8)), g[f"{name}_y_ones"])
        az, bs, bd = (int(v) for v in g[f"{name}_fill"])
        f = sk.fill_report(h)
        assert (f.artificial_zeros, f.bytes_single, f.bytes_double) == (az, bs, bd)
    # test_formats.cpp:160-169 verbatim
    h = sk.build_hybrid(m, 1).to_host()
    assert h["coo_rows"].tolist() == [0, 5, 6, 6, 7]
    assert h["coo_columns"].tolist() == [3, 5, 4, 6, 7]
    assert h["coo_values"].tolist() == [2, 8, 10, 11, 13]
    with pytest.raises(sk.InvalidArgument, match="exceeds the maximum row length"):
        sk.build_hybrid(m, 4)


@pytest.mark.parametrize("kind", ["i", "r"])
def test_small_golden_seeds(cuda, golden, kind):
    g = golden["small"]
    for seed in range(600, 650):
        t = f"s{seed}_{kind}"
        m = triplets(golden_csr(g, t))
        h = sk.build_hybrid(m)
        assert h.slots_per_row == int(g[f"{t}_hy_k1"][0])
        assert_hybrid_equal(h.to_host(), g, f"{t}_hy_")
        x = g[f"{t}_x"]
        f = sk.fill_report(h)  # includes the reference's ell_nnz recount of stored zeros
        assert [f.artificial_zeros, f.bytes_single, f.bytes_double] == \
            [int(v) for v in g[f"{t}_hy_fill"]], t
        assert bitwise(sk.spmv_hybrid(h, x), g[f"{t}_hy_y"]), t
        assert bitwise(sk.spmv_hybrid(h, dev(x)).cpu().numpy(), g[f"{t}_hy_y"]), t


def test_acceptance_200_seeds(cuda, golden):
    g = golden["acceptance"]
    for seed in range(200):
        m = triplets(golden_csr(g, f"a{seed}"))
        y = sk.spmv_hybrid(sk.build_hybrid(m), dev(g[f"a{seed}_xi"])).cpu().numpy()
        assert bitwise(y, g[f"a{seed}_hy_yi"]), seed


def test_device_width_matches_exhaustive_scan(cuda):
    """acceptance.cpp:270-292 / test_formats.cpp:138-158 on device histograms."""
    for seed in range(1000, 1050):
        om = orc.random_case(seed, 48)
        if om.rows == 0:
            continue
        h = sk.build_hybrid(triplets(om))
        assert h.slots_per_row == orc.choose_ell_width(om.lens())
        ml = int(om.lens().max())
        assert sk.build_hybrid(triplets(om), ml).coo_nnz() == 0


@pytest.mark.parametrize("prec", [8, 4])
def test_powerlaw_small_bitwise(cuda, prec):
    """Config 3's generator at 200k rows: long COO tails through the fused kernel."""
    om = orc.powerlaw(200_000, 7)
    h = sk.build_hybrid(triplets(om), None, prec)
    want = orc.build_hybrid(om, None, prec)
    assert h.slots_per_row == want["k1"]
    assert_hybrid_equal(h.to_host(), want)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    assert bitwise(sk.spmv_hybrid(h, dev(x)).cpu().numpy(), orc.spmv_hybrid(want, x))


@pytest.mark.parametrize("prec", [8, 4])
def test_config2_27pt_128_bitwise(cuda, prec):
    om = orc.stencil(27, 128)
    h = sk.build_hybrid(sk.CsrMatrix.stencil(27, 128), None, prec)
    want = orc.build_hybrid(om, None, prec)
    assert h.slots_per_row == 27 and h.coo_nnz() == 0
    assert_hybrid_equal(h.to_host(), want)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    y = sk.spmv_hybrid(h, dev(x)).cpu().numpy()
    assert bitwise(y, orc.spmv_hybrid(want, x))
    if prec == 8:
        assert float(np.cumsum(y)[-1]) == 1674.3573800651031


def test_csr_spmv_bitwise(cuda, golden):
    g = golden["small"]
    for seed in range(600, 650):
        t = f"s{seed}_r"
        a = sk.build_csr(triplets(golden_csr(g, t)))
        y = sk.spmv_csr(a, dev(g[f"{t}_x"])).cpu().numpy()
        assert bitwise(y, g[f"{t}_csr_y"]), t
