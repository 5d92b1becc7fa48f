"""GPU parity of the RgCSR path (K1 conversion, K2 SpMV) through the C-ABI.

Mirrors the reference's own tests: tests/test_formats.cpp:247-350 (golden M8
arrays, degeneracies, madds, monotone padding, fill bytes, oracle
equivalence, float exactness) and tests/acceptance.cpp:138-173 (200-seed
oracle equivalence).  Bar: converted arrays and y BITWISE equal to the
reference's (stronger than the 1e-12 / 1e-5 tolerance north_star allows).
"""
import numpy as np
import pytest
import torch

import oracle as orc
from helpers import RG_KEYS, assert_rgcsr_equal, bitwise, golden_csr, triplets
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu


VARIANTS = ["auto", "grp6", "grp7_mpf", "grp8", "grp8_r64", "lite", "lite8", "lite8_full",
            "vec2", "pipe", "grpv4"]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.fixture(params=VARIANTS)
def k2(request, cuda):
    """Runs the test once per K2 kernel variant (all must be bitwise equal)."""
    from paper_1012_2270_b200._lib import lib
    assert lib().spmvk_set_rgcsr_kernel(request.param.encode()) == 0
    yield request.param
    lib().spmvk_set_rgcsr_kernel(b"auto")


def test_example8_golden_arrays(cuda, golden):
    g = golden["example8"]
    m = triplets(golden_csr(g, "m"))
    for G in (4, 8):
        for prec in (8, 4):
            a = sk.build_rgcsr(m, G, prec)
            assert_rgcsr_equal(a.to_host(), g, f"rg{G}_p{prec}_")
            dt = np.float64 if prec == 8 else np.float32
            y, madds = sk.spmv_rgcsr(a, np.ones(8, dt), multiply_add_count=True)
            assert bitwise(y, g[f"rg{G}_p{prec}_y_ones"])
            assert madds == 13  # one per stored nonzero (test_formats.cpp:267-275)
            az, bs, bd, nnz = (int(v) for v in g[f"rg{G}_p{prec}_fill"])
            f = sk.fill_report(a)
            assert (f.artificial_zeros, f.bytes_single, f.bytes_double, f.nnz) == (az, bs, bd, nnz)
    # tests/test_formats.cpp:247-256 verbatim
    a = sk.build_rgcsr(m, 4).to_host()
    assert a["group_pointers"].tolist() == [0, 8, 20]
    assert a["row_lengths"].tolist() == [2, 1, 1, 1, 1, 2, 3, 2]
    assert a["values"].tolist() == [1, 3, 4, 5, 2, 0, 0, 0, 6, 7, 9, 12, 0, 8, 10, 13, 0, 0, 11, 0]
    assert a["columns"].tolist() == [0, 1, 2, 0, 3, 0, 0, 0, 4, 0, 1, 2, 0, 5, 4, 7, 0, 0, 6, 0]


def test_errors_match_reference(cuda, golden):
    m = triplets(golden_csr(golden["example8"], "m"))
    with pytest.raises(sk.InvalidArgument, match="group size must be nonzero"):
        sk.build_rgcsr(m, 0)
    a = sk.build_rgcsr(m, 4)
    with pytest.raises(sk.InvalidArgument, match="spmv_rgcsr: dimension mismatch"):
        sk.spmv_rgcsr(a, np.ones(9))
    with pytest.raises(sk.InvalidArgument, match="dimension mismatch"):
        sk.spmv_rgcsr(a, dev(np.ones(8)), y=torch.empty(7, dtype=torch.float64, device="cuda"))
    with pytest.raises(sk.InvalidArgument):
        sk.spmv_rgcsr(a, np.ones(8, np.float32))  # precision mismatch
    # TripletMatrix ctor validation (src/triplet.cpp:22-32), on the device
    bad = orc.Csr(2, 2, [0, 2, 2], [1, 0], [1.0, 2.0])  # decreasing columns
    with pytest.raises(sk.InvalidArgument, match="strictly increasing"):
        sk.build_csr(sk.TripletMatrix(2, 2, bad.rp, bad.col, bad.val, validate=False))
    oob = orc.Csr(2, 2, [0, 1, 1], [5], [1.0])
    with pytest.raises(sk.InvalidArgument, match="outside"):
        sk.build_csr(sk.TripletMatrix(2, 2, oob.rp, oob.col, oob.val, validate=False))


@pytest.mark.parametrize("kind", ["i", "r"])
def test_small_golden_seeds(cuda, golden, kind, k2):
    """random_small seeds 600-649, G = 1 + seed % 9 (test_formats.cpp:325-342)."""
    g = golden["small"]
    for seed in range(600, 650):
        t = f"s{seed}_{kind}"
        m = triplets(golden_csr(g, t))
        G = 1 + seed % 9
        x = g[f"{t}_x"]
        a = sk.build_rgcsr(m, G)
        assert_rgcsr_equal(a.to_host(), g, f"{t}_rg_")
        f = sk.fill_report(a)
        assert [f.artificial_zeros, f.bytes_single, f.bytes_double, f.nnz] == \
            [int(v) for v in g[f"{t}_rg_fill"]], t
        assert bitwise(sk.spmv_rgcsr(a, x), g[f"{t}_rg_y"]), t
        assert bitwise(sk.spmv_rgcsr(a, dev(x)).cpu().numpy(), g[f"{t}_rg_y"]), t
        a32 = sk.build_rgcsr(m, G, 4)
        assert_rgcsr_equal(a32.to_host(), g, f"{t}_rg32_")
        assert bitwise(sk.spmv_rgcsr(a32, x.astype(np.float32)), g[f"{t}_rg32_y"]), t
        if kind == "i":  # integer data: every format bitwise equal to spmv_reference
            assert bitwise(g[f"{t}_rg_y"], g[f"{t}_ref_y"])


def test_acceptance_200_seeds(cuda, golden, k2):
    """tests/acceptance.cpp:138-173: 200 random_case matrices, G = 1 + seed % 9."""
    g = golden["acceptance"]
    for seed in range(200):
        m = triplets(golden_csr(g, f"a{seed}"))
        a = sk.build_rgcsr(m, 1 + seed % 9)
        assert_rgcsr_equal(a.to_host(), g, f"a{seed}_rg_")
        y = sk.spmv_rgcsr(a, dev(g[f"a{seed}_xi"])).cpu().numpy()
        assert bitwise(y, g[f"a{seed}_rg_yi"]) and bitwise(y, g[f"a{seed}_ref_yi"]), seed


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("x0", [np.inf, -np.inf, np.nan, -0.0, -2.5])
def test_padded_walk_exact_for_any_x0(cuda, k2, x0, prec):
    """The group-uniform kernels load pads (value 0, column 0); with a
    non-finite x[0] a pad's 0 * x[0] would be NaN, so they must fall back to
    length predication: y stays bitwise spmv_rgcsr's (rows that never touch
    column 0 stay finite).  Ragged rows in every group, several G."""
    om = orc.random_small(4242, allow_zero=True)
    dt = np.float64 if prec == 8 else np.float32
    for G in (3, 4, 32):
        m = triplets(om)
        want = orc.build_rgcsr(om, G, prec)
        x = orc.random_vector(om.cols, 5).astype(dt)
        x[0] = x0
        y = sk.spmv_rgcsr(sk.build_rgcsr(m, G, prec), dev(x)).cpu().numpy()
        ref = orc.spmv_rgcsr(want, x)[0]
        # NaN rows must coincide; their payload may not: the GPU's fp32 multiply
        # returns the canonical NaN (IEEE leaves the payload open), fp64 keeps it
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(y), nan), (G, x0)
        assert bitwise(y[~nan], ref[~nan]), (G, x0)
        if prec == 8:
            assert bitwise(y, ref), (G, x0)


def test_padding_monotone_and_single_group_is_ell(cuda):
    """test_formats.cpp:277-297 and acceptance.cpp:262-269."""
    for seed in range(300, 320):
        om = orc.random_small(seed)
        m = triplets(om)
        prev, first, last = 0, True, 0
        G = 1
        while G < 2 * om.rows:
            a = sk.build_rgcsr(m, G)
            z = sk.fill_report(a).artificial_zeros
            assert (z == 0) if first else (z >= prev)
            first, prev, last = False, z, a.slot_count()
            G *= 2
        ell_slots = om.rows * int(om.lens().max()) if om.nnz else 0
        assert last == ell_slots
        assert sk.build_rgcsr(m, om.rows + seed % 5).slot_count() == ell_slots


@pytest.mark.parametrize("shape", ["empty_rows", "no_entries", "single_row", "identity", "dense_row"])
def test_edge_shapes(cuda, shape, k2):
    if shape == "empty_rows":
        om = orc.Csr(5, 4, [0, 0, 2, 2, 2, 3], [1, 3, 0], [2.0, -1.0, 5.0])
    elif shape == "no_entries":
        om = orc.Csr(3, 3, [0, 0, 0, 0], [], [])
    elif shape == "single_row":
        om = orc.Csr(1, 3, [0, 1], [2], [7.0])
    elif shape == "identity":
        om = orc.Csr(7, 7, np.arange(8), np.arange(7), np.ones(7))
    else:  # one long row among short ones
        n = 200
        rp = np.concatenate([[0], n + np.arange(n)])  # row 0 dense, then one entry each
        col = np.concatenate([np.arange(n), np.arange(1, n)])
        om = orc.Csr(n, n, rp, col, np.arange(col.size, dtype=np.float64) - 50.5)
    x = orc.random_vector(om.cols, 3)
    for G in (1, 2, 3, 4, 32, 33, 256):
        want = orc.build_rgcsr(om, G)
        a = sk.build_rgcsr(triplets(om), G)
        assert_rgcsr_equal(a.to_host(), want)
        assert bitwise(sk.spmv_rgcsr(a, x), orc.spmv_rgcsr(want, x)[0])


@pytest.mark.parametrize("prec", [8, 4])
def test_powerlaw_long_rows_bitwise(cuda, prec, k2):
    """Config 3's generator at 200k rows: ~600 rows past the long-row cut (up
    to 4096 slots) next to short ones -- the long-row paths of every variant."""
    om = orc.powerlaw(200_000, 7)
    assert int(om.lens().max()) > 1000
    for G in (32, 7):
        want = orc.build_rgcsr(om, G, prec)
        a = sk.build_rgcsr(triplets(om), G, prec)
        dt = np.float64 if prec == 8 else np.float32
        x = orc.random_vector(om.cols, 1).astype(dt)
        assert bitwise(sk.spmv_rgcsr(a, dev(x)).cpu().numpy(), orc.spmv_rgcsr(want, x)[0]), G


@pytest.mark.parametrize("prec", [8, 4])
def test_powerlaw_reordered_long_quads_bitwise(cuda, prec, k2):
    """Descending-reordered power-law rows: the long rows sit together, so most
    go to the four-rows-per-warp (quad) path of rgcsr_spmv_long_mixed, the
    longest (>= 1024 slots) stay single.  y bitwise the oracle's on the
    reordered matrix."""
    csr = sk.build_csr(triplets(orc.powerlaw(200_000, 7)))  # fp64; fp32 RgCSR casts
    c2, _ = sk.apply_descending_permutation(csr)
    rp, col, val = c2.to_host()
    om = orc.Csr(c2.num_rows, c2.num_cols, rp, col, val)
    assert int(om.lens()[:8].min()) > 1024 and int((om.lens() > 128).sum()) > 400
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    for G in (32, 64):
        a = sk.build_rgcsr(c2, G, prec)
        want = orc.build_rgcsr(om, G, prec)
        assert bitwise(sk.spmv_rgcsr(a, dev(x)).cpu().numpy(), orc.spmv_rgcsr(want, x)[0]), G


@pytest.mark.parametrize("G", [32, 64, 128, 256])
@pytest.mark.parametrize("prec", [8, 4])
def test_config1_5pt_1024_bitwise(cuda, G, prec, k2):
    """Config 1 (2D 5-point 1024^2) at full size: arrays and y vs the oracle."""
    om = orc.stencil(5, 1024)
    a = sk.build_rgcsr(sk.CsrMatrix.stencil(5, 1024), G, prec)
    want = orc.build_rgcsr(om, G, prec)
    assert_rgcsr_equal(a.to_host(), want)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    assert bitwise(sk.spmv_rgcsr(a, dev(x)).cpu().numpy(), orc.spmv_rgcsr(want, x)[0])


@pytest.mark.parametrize("prec", [8, 4])
def test_config2_27pt_128_bitwise(cuda, prec, k2):
    """Config 2 (3D 27-point 128^3, 55.7 M nnz) at full size, G = 32."""
    om = orc.stencil(27, 128)
    csr = sk.CsrMatrix.stencil(27, 128)
    rp, col, val = csr.to_host()
    assert bitwise(rp, om.rp) and bitwise(col, om.col) and bitwise(val, om.val)
    a = sk.build_rgcsr(csr, 32, prec)
    want = orc.build_rgcsr(om, 32, prec)
    assert_rgcsr_equal(a.to_host(), want)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    y = sk.spmv_rgcsr(a, dev(x)).cpu().numpy()
    assert bitwise(y, orc.spmv_rgcsr(want, x)[0])
    if prec == 8:  # the reference's checksum on this input
        assert float(np.cumsum(y)[-1]) == 1674.3573800651031


def test_row_slabs_equal_global_slices(cuda, k2):
    """Group-aligned slabs are exactly the global arrays' slices."""
    om = orc.stencil(27, 24)
    csr = sk.CsrMatrix.stencil(27, 24)
    G = 32
    full = sk.build_rgcsr(csr, G).to_host()
    x = orc.random_vector(om.cols, 1)
    y_full = sk.spmv_rgcsr(sk.build_rgcsr(csr, G), x)
    n = om.rows
    groups = (n + G - 1) // G
    for P in (2, 3, 4, 8):
        cuts = [min(n, (groups * p // P) * G) for p in range(P + 1)]
        for r0, r1 in zip(cuts, cuts[1:]):
            s = sk.build_rgcsr(csr, G, row_range=(r0, r1))
            h = s.to_host()
            g0, g1 = r0 // G, (r1 + G - 1) // G
            gp = full["group_pointers"]
            assert bitwise(h["group_pointers"], (gp[g0:g1 + 1] - gp[g0]).astype(np.uint32))
            assert bitwise(h["values"], full["values"][gp[g0]:gp[g1]])
            assert bitwise(h["columns"], full["columns"][gp[g0]:gp[g1]])
            assert bitwise(h["row_lengths"], full["row_lengths"][r0:r1])
            assert bitwise(sk.spmv_rgcsr(s, x), y_full[r0:r1])


def test_scaled_iteration_fused(cuda, k2):
    from paper_1012_2270_b200._lib import lib
    om = orc.stencil(7, 20)
    a = sk.build_rgcsr(sk.CsrMatrix.stencil(7, 20), 32)
    x = dev(orc.random_vector(om.cols, 1))
    y = torch.empty_like(x)
    xn = torch.empty_like(x)
    assert lib().spmvk_rgcsr_spmv_scaled_f64(a._h, x.data_ptr(), x.numel(), y.data_ptr(),
                                             y.numel(), xn.data_ptr(), 0.0625, None) == 0
    torch.cuda.synchronize()
    want = orc.spmv_rgcsr(orc.build_rgcsr(om, 32), x.cpu().numpy())[0]
    assert bitwise(y.cpu().numpy(), want)
    assert bitwise(xn.cpu().numpy(), want * 0.0625)


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("kind,n", [(27, 64), (7, 96), (5, 512)])
def test_pipelined_host_span_equals_device(cuda, prec, kind, n):
    """Pinned host x/y take the pipelined path (chunked H2D / SpMV / D2H on
    three streams); pageable memory takes the single-launch path.  Both must be
    bitwise the device-resident y."""
    dt = np.float64 if prec == 8 else np.float32
    a = sk.build_rgcsr(sk.CsrMatrix.stencil(kind, n), 32, prec)
    xh = orc.random_vector(a.num_cols, 2).astype(dt)
    want = sk.spmv_rgcsr(a, dev(xh)).cpu().numpy()
    xp = torch.from_numpy(xh).pin_memory()
    yp = torch.empty(a.num_rows, dtype=xp.dtype).pin_memory()
    for _ in range(2):
        sk.spmv_rgcsr(a, xp.numpy(), yp.numpy())
        assert bitwise(yp.numpy(), want)
    assert bitwise(sk.spmv_rgcsr(a, xh), want)
    # the pipeline is a captured CUDA graph keyed on (matrix, x, y): switching
    # buffers, inputs or matrices must re-capture, never replay a stale graph
    xh2 = orc.random_vector(a.num_cols, 3).astype(dt)
    want2 = sk.spmv_rgcsr(a, dev(xh2)).cpu().numpy()
    xp2 = torch.from_numpy(xh2).pin_memory()
    yp2 = torch.empty_like(yp).pin_memory()
    for _ in range(2):
        sk.spmv_rgcsr(a, xp2.numpy(), yp2.numpy())
        assert bitwise(yp2.numpy(), want2)
        sk.spmv_rgcsr(a, xp.numpy(), yp.numpy())
        assert bitwise(yp.numpy(), want)
    xp.copy_(xp2)  # same buffers, new contents: the replay reads them afresh
    sk.spmv_rgcsr(a, xp.numpy(), yp.numpy())
    assert bitwise(yp.numpy(), want2)
    del a
    b = sk.build_rgcsr(sk.CsrMatrix.stencil(kind, n), 64, prec)
    sk.spmv_rgcsr(b, xp.numpy(), yp.numpy())
    assert bitwise(yp.numpy(), sk.spmv_rgcsr(b, dev(xh2)).cpu().numpy())


@pytest.mark.parametrize("env", [{"SPMVK_PIPE_MAPPED_Y": "0"},
                                 {"SPMVK_PIPE_CHUNKS": "7"},
                                 {"SPMVK_PIPE_CHUNKS": "1", "SPMVK_PIPE_MAPPED_Y": "0"}])
def test_pipelined_host_span_configurations(env):
    """The pipeline's other shapes (y through D2H copies instead of mapped
    stores, forced equal chunk counts) -- read once per process, so each runs
    in a child -- stay bitwise the device-resident y."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch
import oracle as orc
from paper_1012_2270_b200 import generators as gen, spmvkit as sk
mats = [sk.CsrMatrix.stencil(27, 48), sk.CsrMatrix.stencil(5, 400),
        sk.build_csr(gen.random_rows(90000, 70000, 6, 3)),  # x chunk 0 = all of x
        sk.build_csr(gen.banded(200000, 40, 4))]
for prec, dt in ((8, np.float64), (4, np.float32)):
    for kind, m in enumerate(mats):
        if prec == 4:
            m = sk.build_csr(sk.TripletMatrix(m.num_rows, m.num_cols, *m.to_host()), 4)
        a = sk.build_rgcsr(m, 32, prec)
        xh = orc.random_vector(a.num_cols, 5).astype(dt)
        want = sk.spmv_rgcsr(a, torch.from_numpy(xh).cuda()).cpu().numpy()
        xp = torch.from_numpy(xh).pin_memory()
        yp = torch.empty(a.num_rows, dtype=xp.dtype).pin_memory()
        for _ in range(2):
            sk.spmv_rgcsr(a, xp.numpy(), yp.numpy())
            assert yp.numpy().tobytes() == want.tobytes(), (prec, kind)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, PYTHONPATH=root, **env), timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_l2_persistence_window_keeps_results(cuda):
    """spmvk_stream_persist_x: carve-out + access-policy window over x on a
    stream; y is unchanged (bitwise) with and after the window, bad ratios are
    EINVAL, and x == NULL resets."""
    import ctypes as C

    from paper_1012_2270_b200._lib import SPMVK_EINVAL, lib
    L = lib()
    csr = sk.CsrMatrix.stencil(27, 32)
    a = sk.build_rgcsr(csr, 32)
    x = dev(orc.random_vector(a.num_cols, 4))
    want = sk.spmv_rgcsr(a, x).cpu().numpy()
    s = torch.cuda.Stream()
    g = C.c_uint64()
    assert L.spmvk_stream_persist_x(C.c_void_p(s.cuda_stream), C.c_void_p(x.data_ptr()),
                                    x.numel() * 8, 1.0, C.byref(g)) == 0
    assert 0 < g.value <= x.numel() * 8
    y = torch.empty(a.num_rows, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(3):
            sk.spmv_rgcsr(a, x, y)
    s.synchronize()
    assert bitwise(y.cpu().numpy(), want)
    assert L.spmvk_stream_persist_x(C.c_void_p(s.cuda_stream), C.c_void_p(x.data_ptr()),
                                    8, 1.5, None) == SPMVK_EINVAL
    assert L.spmvk_stream_persist_x(C.c_void_p(s.cuda_stream), None, 0, 1.0, None) == 0
    with torch.cuda.stream(s):  # the Python wrapper (current stream)
        assert sk.persist_x(x) > 0
        sk.spmv_rgcsr(a, x, y)
        assert sk.persist_x(None) == 0
        sk.spmv_rgcsr(a, x, y)
    s.synchronize()
    assert bitwise(y.cpu().numpy(), want)


@pytest.fixture(scope="module")
def powerlaw_pair():
    """A 300k-row power-law matrix in original and descending order (singles,
    quads and short rows all present), as device CSR + oracle CSR."""
    csr = sk.build_csr(triplets(orc.powerlaw(300_000, 7)))
    out = {}
    for name, c in (("orig", csr), ("desc", sk.apply_descending_permutation(csr)[0])):
        rp, col, val = c.to_host()
        out[name] = (c, orc.Csr(c.num_rows, c.num_cols, rp, col, val))
    return out


@pytest.mark.parametrize("variant", ["lite", "lite8", "liteh", "lite8h", "pipe"])
@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("prec", [8, 4])
def test_long_rows_fused_into_tile_kernel(cuda, powerlaw_pair, variant, fused, prec):
    """Long rows taken by the tile kernel's warps (dynamic items, one launch)
    or by the separate long-row launch: y and the scaled iterate bitwise the
    oracle's, over repeated back-to-back launches (the per-stream item counter
    must reset itself) and on two streams at once."""
    from paper_1012_2270_b200._lib import lib
    L = lib()
    assert L.spmvk_set_rgcsr_kernel(variant.encode()) == 0
    assert L.spmvk_set_long_fused(fused) == 0
    dt = np.float64 if prec == 8 else np.float32
    try:
        for order in ("orig", "desc"):
            c, om = powerlaw_pair[order]
            a = sk.build_rgcsr(c, 32, prec)
            want = orc.spmv_rgcsr(orc.build_rgcsr(om, 32, prec), orc.random_vector(om.cols, 1)
                                  .astype(dt))[0]
            x = dev(orc.random_vector(om.cols, 1).astype(dt))
            streams = [torch.cuda.Stream(), torch.cuda.Stream()]
            ys = [torch.empty_like(x) for _ in range(4)]
            for k in range(4):
                with torch.cuda.stream(streams[k % 2]):
                    sk.spmv_rgcsr(a, x, ys[k])
            torch.cuda.synchronize()
            for y in ys:
                assert bitwise(y.cpu().numpy(), want), (order, variant)
            if prec == 8:
                y, xn = torch.empty_like(x), torch.empty_like(x)
                assert L.spmvk_rgcsr_spmv_scaled_f64(a._h, x.data_ptr(), x.numel(), y.data_ptr(),
                                                     y.numel(), xn.data_ptr(), 0.0625, None) == 0
                torch.cuda.synchronize()
                assert bitwise(y.cpu().numpy(), want) and bitwise(xn.cpu().numpy(), want * 0.0625)
    finally:
        L.spmvk_set_rgcsr_kernel(b"auto")
        L.spmvk_set_long_fused(1)


@pytest.mark.parametrize("bulk", ["1", "0"])
def test_k1_scatter_variants_bitwise(cuda, bulk):
    """Both K1 scatters (SPMVK_K1_BULK, read once per process, so each runs in
    a child): the TMA bulk-copy kernel (default) and the shared-memory staged
    one, on full and partial groups, G = 32 and 64, row slabs, fp64 and fp32
    (double -> float cast), stencils and power-law rows past the stage size --
    arrays bitwise the oracle's build_rgcsr."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np
import oracle as orc
from helpers import triplets
from paper_1012_2270_b200 import spmvkit as sk
mats = [orc.stencil(27, 21), orc.stencil(5, 301), orc.powerlaw(40000, 7), orc.banded(7777, 9, 3)]
for om in mats:
    m = sk.build_csr(triplets(om))
    for G in (32, 64, 7):
        for prec in (8, 4):
            got = sk.build_rgcsr(m, G, prec).to_host()
            want = orc.build_rgcsr(om, G, prec)
            for k in ("values", "columns", "group_pointers", "row_lengths"):
                assert np.array_equal(got[k], want[k]), (om.rows, G, prec, k)
    r0 = 32 * (om.rows // 96)
    part = sk.build_rgcsr(m, 32, 8, row_range=(r0, om.rows)).to_host()
    full = orc.build_rgcsr(om, 32, 8)
    gp = full["group_pointers"]
    g0 = r0 // 32
    assert np.array_equal(part["values"], full["values"][gp[g0]:])
    assert np.array_equal(part["columns"], full["columns"][gp[g0]:])
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]),
               SPMVK_K1_BULK=bulk)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("fused", ["1", "0"])
def test_k1_layout_fused_and_unfused_bitwise(cuda, fused):
    """Both K1 layout paths (SPMVK_K1_LAYOUT, read once per process, so each
    runs in a child): the fused two-kernel layout (default; tiles of <= 8,192
    rows, the last CTA scanning the tile sums) and the unfused kernels +
    scans.  Group sizes that stage in shared memory with several groups per
    thread (G = 1, 3), one (G = 32), partial tiles (G = 33, 256), one group
    per tile (G = 8192) and groups past the staging size (G = 10000); more
    than 256 tiles (the last CTA's scan crosses chunks); row slabs; long rows
    (their offsets feed the long-row list: y must be the oracle's)."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np
import oracle as orc
from helpers import triplets
from paper_1012_2270_b200 import spmvkit as sk
cases = [(orc.stencil(5, 1600), (1, 32, 33)), (orc.powerlaw(60000, 7), (1, 3, 32, 256, 8192, 10000)),
         (orc.banded(20001, 5, 3), (3, 8192, 10000))]
for om, Gs in cases:
    m = sk.build_csr(triplets(om))
    x = orc.random_vector(om.cols, 1)
    for G in Gs:
        a = sk.build_rgcsr(m, G, 8)
        got = a.to_host()
        want = orc.build_rgcsr(om, G, 8)
        for k in ("values", "columns", "group_pointers", "row_lengths"):
            assert np.array_equal(got[k], want[k]), (om.rows, G, k)
        y = sk.spmv_rgcsr(a, x)
        assert np.array_equal(y.view(np.uint64), orc.spmv_rgcsr(want, x)[0].view(np.uint64)), (om.rows, G)
        r0 = G * ((om.rows // G) // 3)
        if 0 < r0 < om.rows:
            part = sk.build_rgcsr(m, G, 8, row_range=(r0, om.rows)).to_host()
            gp = want["group_pointers"]
            assert np.array_equal(part["values"], want["values"][gp[r0 // G]:]), (om.rows, G)
            assert np.array_equal(part["row_lengths"], want["row_lengths"][r0:]), (om.rows, G)
            assert np.array_equal(part["group_pointers"].astype(np.int64),
                                  gp[r0 // G:].astype(np.int64) - int(gp[r0 // G])), (om.rows, G)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]),
               SPMVK_K1_LAYOUT=fused)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=env, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_host_array_buffers_through_the_span_overload(cuda):
    """spmvk_host_alloc buffers (sk.host_array: page-locked, 2 MB pages) as x
    and y of the pipelined host-span SpMV: y bitwise the device-resident
    result; zero-length and odd sizes allocate; a foreign pointer is refused
    on free."""
    import ctypes as C
    from paper_1012_2270_b200._lib import lib
    csr = sk.CsrMatrix.stencil(27, 64)
    a = sk.build_rgcsr(csr, 32)
    xh = orc.random_vector(a.num_cols, 1)
    x, y = sk.host_array(a.num_cols), sk.host_array(a.num_rows)
    assert x.ctypes.data % (2 << 20) == 0 and not y.any()
    x[:] = xh
    assert lib().spmvk_rgcsr_spmv_host_f64(a._h, x.ctypes.data, a.num_cols, y.ctypes.data,
                                           a.num_rows, None) == 0
    assert bitwise(y, sk.spmv_rgcsr(a, dev(xh)).cpu().numpy())
    for n in (0, 1, 3, (1 << 18) + 1):
        z = sk.host_array(n, np.float32)
        assert z.shape == (n,) and z.dtype == np.float32
        del z
    assert lib().spmvk_host_free(C.c_void_p(x.ctypes.data + 8)) != 0
    del x, y
