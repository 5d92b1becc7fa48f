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


HYBRID_VARIANTS = ["auto", "v4", "lite", "lite8", "lite8_full", "litef", "lite8f", "dyn", "vec"]


@pytest.fixture(params=HYBRID_VARIANTS)
def hk(request, cuda):
    """Runs the test once per Hybrid SpMV kernel variant (all bitwise equal)."""
    from paper_1012_2270_b200._lib import lib
    assert lib().spmvk_set_hybrid_kernel(request.param.encode()) == 0
    yield request.param
    lib().spmvk_set_hybrid_kernel(b"auto")


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
def test_small_golden_seeds(cuda, hk, golden, kind):
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


def test_acceptance_200_seeds(cuda, hk, golden):
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
def test_powerlaw_small_bitwise(cuda, hk, prec):
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
def test_config2_27pt_128_bitwise(cuda, hk, prec):
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


def _same(a: sk.TripletMatrix, m: orc.Csr) -> bool:
    return (a.num_rows, a.num_cols) == (m.rows, m.cols) and bitwise(a.row_ptr, m.rp) and \
        bitwise(a.col, m.col) and bitwise(a.val, m.val)


def test_round_trip_through_every_format(cuda):
    """tests/test_formats.cpp:314-323 (seeds 500-529, nonzero values) and the
    Hybrid partition check :184-192 (seeds 200-229): to_triplets(build_*(m)) == m."""
    for seed in list(range(500, 530)) + list(range(200, 230)):
        om = orc.random_small(seed, allow_zero=False)
        m = triplets(om)
        assert _same(sk.to_triplets(sk.build_csr(m)), om)
        assert _same(sk.to_triplets(sk.build_rgcsr(m, 1 + seed % 16)), om), seed
        assert _same(sk.to_triplets(sk.build_rgcsr(m, 1 + seed % 16, 4)), om), seed
        h = sk.build_hybrid(m)
        assert h.info.fill_nnz == om.nnz  # ell_nnz + coo == nnz without stored zeros
        assert _same(sk.to_triplets(h), om), seed
        assert _same(sk.to_triplets(sk.build_ellpack(m)), om), seed


def test_hybrid_to_triplets_drops_lone_stored_zero_like_reference(cuda):
    """ellpack.hpp:50-54: a row whose only entry is a stored zero at column 0
    is indistinguishable from an empty row — the reference loses it too."""
    om = orc.Csr(3, 3, [0, 1, 2, 3], [0, 0, 2], [0.0, 5.0, 1.0])
    t = sk.to_triplets(sk.build_hybrid(triplets(om)))
    assert t.entries() == [(1, 0, 5.0), (2, 2, 1.0)]
    if orc.ref_available():
        r = orc.RefMatrix.from_csr(om)
        h = r.hybrid()
        assert h["artificial_zeros"] == sk.fill_report(sk.build_hybrid(triplets(om))).artificial_zeros


# ------------------------------------------------ ELLPACK and the separate parts
ONES_Y = [3, 3, 4, 5, 6, 15, 30, 25]  # kExampleOnesResult (test_matrix_core.cpp:88-91)


def test_ellpack_example_and_shapes(cuda, golden):
    """tests/test_formats.cpp:60-94 (build_ellpack, fill, budget, spmv_ellpack)."""
    m = triplets(golden_csr(golden["example8"], "m"))
    a = sk.build_ellpack(m)
    assert a.slots_per_row == 3 and a.info.ell_slots == 24 and a.coo_nnz() == 0
    f = sk.fill_report(a)
    assert (f.format_name, f.artificial_zeros, f.stored_slots, f.nnz) == ("ellpack", 11, 24, 13)
    assert (f.bytes_single, f.bytes_double) == (24 * 8, 24 * 12)  # index words = slots
    assert a.to_host()["ell_values"].tolist() == [1, 3, 4, 5, 6, 7, 9, 12,
                                                  2, 0, 0, 0, 0, 8, 10, 13,
                                                  0, 0, 0, 0, 0, 0, 11, 0]
    ident = sk.canonicalize([(i, i, 1.0) for i in range(5)], 5, 5)
    assert sk.fill_report(sk.build_ellpack(ident)).artificial_zeros == 0
    skew = sk.canonicalize([(0, 0, 1.0), (0, 1, 1.0), (0, 2, 1.0), (0, 3, 1.0), (1, 1, 2.0),
                            (2, 2, 3.0), (3, 0, 4.0)], 4, 4)
    b = sk.build_ellpack(skew)
    assert (b.slots_per_row, b.info.ell_slots, sk.fill_report(b).artificial_zeros) == (4, 16, 9)
    with pytest.raises(sk.SpmvkRuntimeError, match="exceeds the slot budget of 16"):
        sk.build_ellpack(m, 16)
    sk.build_ellpack(m, 24)
    assert sk.spmv_ellpack(a, np.ones(8)).tolist() == ONES_Y
    assert sk.spmv_ellpack(a, np.zeros(8)).tolist() == [0.0] * 8
    one = sk.canonicalize([(0, 2, 7.0)], 1, 3)
    assert sk.spmv_ellpack(sk.build_ellpack(one), np.array([0, 0, 5.0])).tolist() == [35.0]
    t = sk.to_triplets(a)  # test_formats.cpp:318
    assert t.row_ptr.tolist() == m.row_ptr.tolist() and t.col.tolist() == m.col.tolist()
    assert t.val.tolist() == m.val.tolist()
    with pytest.raises(sk.InvalidArgument, match="spmv_ellpack: dimension mismatch"):
        sk.spmv_ellpack(a, np.ones(9))


def test_spmv_coo_accumulates(cuda, hk, golden):
    """tests/test_formats.cpp:96-122: the COO part adds into y in array order."""
    single = sk.build_hybrid(sk.canonicalize([(0, 0, 2.0)], 1, 1), 0)  # all entries in COO
    y = np.array([1.0])
    sk.spmv_coo(single, np.array([3.0]), y)
    assert y.tolist() == [7.0]
    empty = sk.build_hybrid(sk.canonicalize([(0, 0, 2.0)], 1, 1), 1)  # COO part empty
    sk.spmv_coo(empty, np.array([3.0]), y)
    assert y.tolist() == [7.0]
    m = triplets(golden_csr(golden["example8"], "m"))
    h = sk.build_hybrid(m, 0)
    y = np.zeros(8)
    sk.spmv_coo(h, np.ones(8), y)
    assert y.tolist() == ONES_Y
    yd = torch.zeros(8, dtype=torch.float64, device="cuda")
    sk.spmv_coo(h, dev(np.ones(8)), yd)
    assert yd.cpu().numpy().tolist() == ONES_Y
    with pytest.raises(sk.InvalidArgument, match="spmv_coo: entry outside x/y dimensions"):
        sk.spmv_coo(h, np.ones(8), np.zeros(7))
    with pytest.raises(sk.InvalidArgument, match="spmv_coo: entry outside x/y dimensions"):
        sk.spmv_coo(h, np.ones(7), np.zeros(8))
    longer = np.full(10, 5.0)  # rows past the matrix are left alone
    sk.spmv_coo(h, np.ones(8), longer)
    assert longer.tolist() == [v + 5.0 for v in ONES_Y] + [5.0, 5.0]


@pytest.mark.parametrize("prec", [8, 4])
def test_parts_compose_to_spmv_hybrid(cuda, hk, golden, prec):
    """spmv_ellpack(h.ell) then spmv_coo(h.coo) is spmv_hybrid (ellpack.hpp:
    205-210), bitwise, host and device, on the 200 acceptance matrices."""
    g = golden["acceptance"]
    dt = np.float64 if prec == 8 else np.float32
    for seed in range(0, 200, 3):
        m = triplets(golden_csr(g, f"a{seed}"))
        if len(m.col) == 0:
            continue
        x = g[f"a{seed}_xi"].astype(dt)
        for k1 in (None, 1):
            h = sk.build_hybrid(m, k1, prec)
            want = sk.spmv_hybrid(h, x)
            y = sk.spmv_ellpack(h, x)
            sk.spmv_coo(h, x, y)
            assert bitwise(y, want), (seed, k1)
            yd = sk.spmv_ellpack(h, dev(x))
            sk.spmv_coo(h, dev(x), yd)
            assert bitwise(yd.cpu().numpy(), want), (seed, k1)


@pytest.mark.parametrize("kernel", ["", "dyn", "staged", "warp", "row"])
def test_csr_kernels_bitwise_with_long_rows(kernel):
    """spmv_csr's three kernels (SPMVK_CSR_KERNEL, read once per process, so
    each runs in a child): stencils, a banded matrix and power-law rows up to
    ~3,700 entries -- rows that span several staged chunks of 1,024 entries --
    all bitwise the oracle's spmv_csr, fp64 and fp32."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch
import oracle as orc
from helpers import triplets
from paper_1012_2270_b200 import spmvkit as sk
mats = [orc.stencil(27, 24), orc.stencil(5, 300), orc.powerlaw(60000, 7),
        orc.Csr(3, 3, [0, 0, 2, 2], [0, 2], [1.5, -2.0])]
for prec, dt in ((8, np.float64), (4, np.float32)):
    for kind, om in enumerate(mats):
        a = sk.build_csr(triplets(om), prec)
        x = orc.random_vector(om.cols, 5).astype(dt)
        y = sk.spmv_csr(a, torch.from_numpy(x).cuda()).cpu().numpy()
        assert y.tobytes() == orc.spmv_csr(om, x, prec).tobytes(), (prec, kind)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]),
               SPMVK_CSR_KERNEL=kernel)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("prec", [8, 4])
def test_hybrid_reordered_powerlaw_walks_heavy_tiles(cuda, hk, prec):
    """Descending-reordered power-law rows put the long COO tails together: the
    first tiles hold > 16k COO entries and switch from chunk staging to one
    thread per row walking its own COO run.  y bitwise the oracle's; the
    spmv_coo-only part too."""
    csr = sk.build_csr(triplets(orc.powerlaw(200_000, 7)))
    c2, _ = sk.apply_descending_permutation(csr)
    rp, col, val = c2.to_host()
    om = orc.Csr(c2.num_rows, c2.num_cols, rp, col, val)
    h = sk.build_hybrid(c2, None, prec)
    want = orc.build_hybrid(om, None, prec)
    assert h.coo_nnz() > 16 * 1024 * 2
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    assert bitwise(sk.spmv_hybrid(h, dev(x)).cpu().numpy(), orc.spmv_hybrid(want, x))


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("x0", [np.inf, np.nan, -0.0])
def test_nonfinite_x_matches_reference(cuda, hk, prec, x0):
    """Non-finite x[0]: the reference's spmv_ellpack adds every pad's 0 * x[0]
    (NaN for an infinite x[0]) -- the device Hybrid must do the same, and
    spmv_csr must not.  NaN positions must match (fp32 NaN payloads are the
    GPU's canonical NaN); everything else bitwise."""
    om = orc.powerlaw(3000, 7)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 4).astype(dt)
    x[0] = x0
    m = triplets(om)
    h = sk.build_hybrid(m, None, prec)
    c = sk.build_csr(m, prec)
    for got, ref in ((sk.spmv_hybrid(h, dev(x)).cpu().numpy(),
                      orc.spmv_hybrid(orc.build_hybrid(om, None, prec), x)),
                     (sk.spmv_csr(c, dev(x)).cpu().numpy(), orc.spmv_csr(om, x, prec))):
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(got), nan)
        assert bitwise(got[~nan], ref[~nan])
        if prec == 8:
            assert bitwise(got, ref)


def test_hybrid_all_coo_walk_and_heavy(cuda, hk):
    """K1 = 0 (everything in COO) on the reordered power-law matrix: most tiles
    exceed the walk threshold and many rows are heavy -- the COO-only kernel,
    the per-row walk and the heavy-row kernel carry the whole product, and
    spmv_coo's accumulate form composes with them."""
    csr = sk.build_csr(triplets(orc.powerlaw(100_000, 7)))
    c2, _ = sk.apply_descending_permutation(csr)
    rp, col, val = c2.to_host()
    om = orc.Csr(c2.num_rows, c2.num_cols, rp, col, val)
    h = sk.build_hybrid(c2, 0)
    want = orc.build_hybrid(om, 0, 8)
    x = orc.random_vector(om.cols, 2)
    assert h.coo_nnz() == om.nnz
    assert bitwise(sk.spmv_hybrid(h, dev(x)).cpu().numpy(), orc.spmv_hybrid(want, x))


def test_parts_compose_on_heavy_tiles(cuda, hk):
    """spmv_ellpack then spmv_coo (accumulating in place) equals spmv_hybrid
    bitwise on the reordered power-law matrix, whose COO part goes through the
    per-row walk and the heavy-row kernel -- the accumulate form of both."""
    csr = sk.build_csr(triplets(orc.powerlaw(100_000, 7)))
    c2, _ = sk.apply_descending_permutation(csr)
    h = sk.build_hybrid(c2)
    x = dev(orc.random_vector(c2.num_cols, 6))
    y = sk.spmv_ellpack(h, x)
    sk.spmv_coo(h, x, y)
    assert bitwise(y.cpu().numpy(), sk.spmv_hybrid(h, x).cpu().numpy())


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("order", ["orig", "desc"])
def test_dyn_repeated_launches_two_streams(cuda, prec, order):
    """hybrid_spmv_dyn takes rows and heavy rows from per-stream counters that
    the last warp resets: back-to-back launches alternating over two streams
    must all give the oracle's y bitwise (heavy rows present in both
    orders)."""
    from paper_1012_2270_b200._lib import lib
    csr = sk.build_csr(triplets(orc.powerlaw(300_000, 7)))
    c = csr if order == "orig" else sk.apply_descending_permutation(csr)[0]
    rp, col, val = c.to_host()
    om = orc.Csr(c.num_rows, c.num_cols, rp, col, val)
    h = sk.build_hybrid(c, None, prec)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(om.cols, 1).astype(dt)
    want = orc.spmv_hybrid(orc.build_hybrid(om, None, prec), x)
    assert lib().spmvk_set_hybrid_kernel(b"dyn") == 0
    try:
        xd = dev(x)
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        ys = [torch.empty_like(xd) for _ in range(4)]
        for k in range(4):
            with torch.cuda.stream(streams[k % 2]):
                sk.spmv_hybrid(h, xd, ys[k])
        torch.cuda.synchronize()
        for y in ys:
            assert bitwise(y.cpu().numpy(), want)
    finally:
        lib().spmvk_set_hybrid_kernel(b"auto")


@pytest.mark.parametrize("prec", [8, 4])
def test_dyn_walk_threshold_edges(cuda, prec):
    """Rows of exactly 127-130 entries sit on the work-item cut of the dyn walk
    (COO runs > 128 become warp items; CSR rows > 128 likewise), next to empty
    rows, runs that straddle 128-entry chunks and 32-row sub-slice borders:
    spmv_hybrid (K1 = 0 and chosen K1) and spmv_csr bitwise the oracle's."""
    rng = np.random.default_rng(11)
    n = 4099
    lens = rng.integers(0, 9, n)
    for i, l in zip(range(0, n, 37), [0, 1, 127, 128, 129, 130, 255, 256, 257, 31, 32, 33] * 20):
        lens[i] = l
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(
        np.uint32)
    val = rng.uniform(-1, 1, int(rp[-1]))
    om = orc.Csr(n, n, rp, col, val)
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(n, 3).astype(dt)
    m = triplets(om)
    for k1 in (0, None):
        h = sk.build_hybrid(m, k1, prec)
        assert bitwise(sk.spmv_hybrid(h, dev(x)).cpu().numpy(),
                       orc.spmv_hybrid(orc.build_hybrid(om, k1, prec), x)), k1
    c = sk.build_csr(m, prec)
    assert bitwise(sk.spmv_csr(c, dev(x)).cpu().numpy(), orc.spmv_csr(om, x, prec))
    a = sk.build_rgcsr(m, 32, prec)
    assert bitwise(sk.spmv_rgcsr(a, dev(x)).cpu().numpy(),
                   orc.spmv_rgcsr(orc.build_rgcsr(om, 32, prec), x)[0])


def _ell_row_length_ref(ev, ec, rows, k1):
    """ellpack.hpp:55-72 (ell_row_length) over slot-major arrays, per row."""
    out = np.zeros(rows, np.int64)
    for r in range(rows):
        n, prev = 0, 0
        for slot in range(k1):
            c, v = int(ec[slot * rows + r]), ev[slot * rows + r]
            if slot > 0 and c <= prev:
                break
            if slot == 0 and c == 0 and v == 0:
                if not (k1 > 1 and int(ec[rows + r]) > 0):
                    break
            n += 1
            prev = c
        out[r] = n
    return out


@pytest.mark.parametrize("prec", [8, 4])
def test_ell_nnz_with_stored_zeros_at_column_0(cuda, prec):
    """fill_report's ELL nnz is counted from the CSR (not by re-reading the
    ELL arrays): rows whose only ELL entry is a stored zero at column 0 (also
    -0.0, and 1e-50 which is zero only after the cast to fp32) count as empty,
    exactly as the reference's ell_row_length recount of the layout; K1 = 1
    truncates a stored zero at column 0 with a real successor to empty."""
    rows_ = [[(0, 0.0)], [(0, 1.0)], [(0, 0.0), (5, 1.0)], [], [(3, 0.0)], [(0, -0.0)],
             [(0, 1e-50)], [(c, 0.0 if c == 0 else 1.0) for c in range(0, 20, 2)],
             [(1, 2.0), (2, 0.0)], [(0, 0.0), (1, 0.0), (2, 0.0)]]
    rp = np.zeros(len(rows_) + 1, np.uint32)
    col, val = [], []
    for i, r in enumerate(rows_):
        rp[i + 1] = rp[i] + len(r)
        col += [c for c, _ in r]
        val += [v for _, v in r]
    om = orc.Csr(len(rows_), 24, rp, np.array(col, np.uint32), np.array(val, np.float64))
    m = sk.build_csr(triplets(om))
    for k1 in (1, 2, 3, 10):
        h = sk.build_hybrid(m, k1, prec)
        ref = orc.build_hybrid(om, k1, prec)
        want = int(_ell_row_length_ref(ref["ell_values"], ref["ell_columns"], om.rows, k1).sum())
        want += ref["coo_rows"].size
        assert sk.fill_report(h).nnz == want, (k1, prec)
