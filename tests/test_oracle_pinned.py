"""Pins the oracle (oracle/oracle.c, the plain-C restatement) before it is
trusted: against the golden vectors the reference produced
(tests/golden/*.npz, shapes.json) and, when oracle/_ref is built, against the
unmodified reference library live.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle as orc
from helpers import RG_KEYS, HY_KEYS, bitwise, golden_csr

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_example8_golden(golden):
    g = golden["example8"]
    m = golden_csr(g, "m")
    assert m.rp.tolist() == [0, 2, 3, 4, 5, 6, 8, 11, 13]  # test_formats.cpp:37-41
    for G in (4, 8):
        for prec in (8, 4):
            a = orc.build_rgcsr(m, G, prec)
            for k in RG_KEYS:
                assert bitwise(a[k], g[f"rg{G}_p{prec}_{k}"])
            ones = np.ones(8, a["values"].dtype)
            y, madds = orc.spmv_rgcsr(a, ones)
            assert bitwise(y, g[f"rg{G}_p{prec}_y_ones"]) and madds == 13
            slots, nnz, az, bs, bd = orc.rgcsr_fill(a)
            assert [az, bs, bd, nnz] == [int(v) for v in g[f"rg{G}_p{prec}_fill"]]
    for k1, name in ((None, "hyd"), (0, "hy0"), (1, "hy1"), (3, "hy3")):
        h = orc.build_hybrid(m, k1)
        for k in HY_KEYS:
            assert bitwise(h[k], g[f"{name}_{k}"])
        assert bitwise(orc.spmv_hybrid(h, np.ones(8)), g[f"{name}_y_ones"])
    assert g["y_ref_ones"].tolist() == [3, 3, 4, 5, 6, 15, 30, 25]
    assert bitwise(orc.spmv_reference(m, np.ones(8)), g["y_ref_ones"])
    assert bitwise(orc.descending_map(m), g["descending_map"])
    assert g["descending_map"].tolist() == [6, 0, 5, 7, 1, 2, 3, 4]  # test_reorder.cpp:62-65


def test_small_golden(golden):
    g = golden["small"]
    for seed in range(600, 650):
        for kind in "ir":
            t = f"s{seed}_{kind}"
            m = golden_csr(g, t)
            om = orc.random_small(seed, True, kind == "i")  # generator restatement
            assert bitwise(om.rp, m.rp) and bitwise(om.col, m.col) and bitwise(om.val, m.val)
            x = g[f"{t}_x"]
            if kind == "r":
                assert bitwise(orc.random_vector(m.cols, seed), x)
            else:
                assert bitwise(orc.random_integer_x(m.cols, seed * 77 + 1), x)
            G = 1 + seed % 9
            a = orc.build_rgcsr(m, G)
            for k in RG_KEYS:
                assert bitwise(a[k], g[f"{t}_rg_{k}"])
            assert bitwise(orc.spmv_rgcsr(a, x)[0], g[f"{t}_rg_y"])
            a32 = orc.build_rgcsr(m, G, 4)
            for k in RG_KEYS:
                assert bitwise(a32[k], g[f"{t}_rg32_{k}"])
            assert bitwise(orc.spmv_rgcsr(a32, x.astype(np.float32))[0], g[f"{t}_rg32_y"])
            h = orc.build_hybrid(m)
            for k in HY_KEYS:
                assert bitwise(h[k], g[f"{t}_hy_{k}"])
            assert bitwise(orc.spmv_hybrid(h, x), g[f"{t}_hy_y"])
            assert bitwise(orc.spmv_csr(m, x), g[f"{t}_csr_y"])
            assert bitwise(orc.spmv_reference(m, x), g[f"{t}_ref_y"])


def test_acceptance_golden(golden):
    g = golden["acceptance"]
    for seed in range(200):
        m = golden_csr(g, f"a{seed}")
        om = orc.random_case(seed, 64)
        assert bitwise(om.col, m.col) and bitwise(om.val, m.val)
        xi = g[f"a{seed}_xi"]
        assert bitwise(orc.random_integer_x(m.cols, seed + 11), xi)
        a = orc.build_rgcsr(m, 1 + seed % 9)
        for k in RG_KEYS:
            assert bitwise(a[k], g[f"a{seed}_rg_{k}"])
        y = orc.spmv_rgcsr(a, xi)[0]
        assert bitwise(y, g[f"a{seed}_rg_yi"]) and bitwise(y, g[f"a{seed}_ref_yi"])
        assert bitwise(orc.spmv_hybrid(orc.build_hybrid(m), xi), g[f"a{seed}_hy_yi"])


def test_config_shapes_golden():
    """Config-scale scalars the reference computed (configs 1 and 2)."""
    with open(os.path.join(GOLD, "shapes.json")) as f:
        s = json.load(f)
    x_seed = 1
    for name, gen in (("5pt_1024", lambda: orc.stencil(5, 1024)),
                      ("27pt_128", lambda: orc.stencil(27, 128))):
        e = s[name]
        m = gen()
        assert m.nnz == e["nnz"] and int(m.lens().max()) == e["max_len"]
        x = orc.random_vector(m.cols, x_seed)
        for G in (32, 64, 128, 256):
            a = orc.build_rgcsr(m, G)
            slots, nnz, az, bs, bd = orc.rgcsr_fill(a)
            assert (slots, az, bd, bs) == (e[f"rg{G}"]["slots"], e[f"rg{G}"]["artificial_zeros"],
                                          e[f"rg{G}"]["bytes_double"], e[f"rg{G}"]["bytes_single"])
            if G == 32:
                y = orc.spmv_rgcsr(a, x)[0]
                assert float(np.cumsum(y)[-1]) == e["rg32"]["checksum_f64"]
                y32 = orc.spmv_rgcsr(orc.build_rgcsr(m, G, 4), x.astype(np.float32))[0]
                assert float(np.cumsum(y32.astype(np.float64))[-1]) == e["rg32"]["checksum_f32"]
            del a
        assert orc.choose_ell_width(m.lens()) == e["hybrid"]["k1"]
        h = orc.build_hybrid(m)
        assert h["coo_rows"].size == e["hybrid"]["coo"]
        assert float(np.cumsum(orc.spmv_hybrid(h, x))[-1]) == e["hybrid"]["checksum_f64"]
        assert float(np.cumsum(orc.spmv_reference(m, x))[-1]) == e["checksum_reference"]


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_live_reference_random_corpora():
    """Restatement vs the live reference over fresh seeds and group sizes."""
    rng = np.random.default_rng(0)
    for seed in range(2000, 2060):
        r = orc.RefMatrix.random_small(seed, seed % 2 == 0, seed % 3 == 0)
        m = r.to_csr()
        x = orc.random_vector(m.cols, seed)
        for G in (1, 2, 3, 7, 32, 65):
            want = r.rgcsr(G)
            got = orc.build_rgcsr(m, G)
            for k in RG_KEYS:
                assert bitwise(got[k], want[k])
            assert bitwise(orc.spmv_rgcsr(got, x)[0], r.rgcsr_spmv(want, x)[0])
            orc.R().ref_rgcsr_free(want["_h"])
        k1 = int(rng.integers(0, int(m.lens().max()) + 1)) if m.nnz else 0
        for kk in (None, k1):
            want = r.hybrid(kk)
            got = orc.build_hybrid(m, kk)
            for k in HY_KEYS:
                assert bitwise(got[k], want[k])
            assert bitwise(orc.spmv_hybrid(got, x), r.hybrid_spmv(want, x))
            orc.R().ref_hybrid_free(want["_h"])
        assert bitwise(orc.descending_map(m), r.descending_map())
