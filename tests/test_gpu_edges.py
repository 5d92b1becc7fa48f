"""Edge and error paths the round-1 review found untested.

* rows > 0, cols = 0 (a legal reference shape, triplet.hpp:26-45): every row
  is empty, the reference returns y = +0 -- the device path must not touch x
  (a zero-length CUDA tensor has no storage).
* x as an offset view (only 8- / 4-byte aligned): the group walk's x L2 bulk
  prefetch needs 16-byte alignment, so it must be skipped, not fault.
* uint32 slot overflow: the reference truncates group_pointers silently
  (rgcsr.hpp:56); the device converter reports ERANGE with a message.
* the fused multi-GPU step's flag barrier with a peer that never arrives:
  it must time out into SPMVK_ENCCL, not hang the GPU.
"""
import ctypes as C
import time

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import bitwise
from paper_1012_2270_b200 import generators as gen
from paper_1012_2270_b200 import partition as pt
from paper_1012_2270_b200 import spmvkit as sk
from paper_1012_2270_b200._lib import lib

pytestmark = pytest.mark.gpu

KERNELS = ["auto", "grp6", "grp7_mpf", "grp8", "grp8_r64", "lite", "lite8", "lite8_full",
           "vec2", "pipe"]


@pytest.mark.parametrize("rows", [1, 37, 5000])
def test_zero_columns_gives_positive_zero(cuda, rows):
    m = sk.TripletMatrix(rows, 0, np.zeros(rows + 1, np.uint32), np.zeros(0, np.uint32),
                         np.zeros(0, np.float64))
    for prec, dt in ((8, torch.float64), (4, torch.float32)):
        x = torch.empty(0, dtype=dt, device="cuda")
        for G in (1, 32, 256):
            a = sk.build_rgcsr(m, G, prec)
            for k in KERNELS:
                assert lib().spmvk_set_rgcsr_kernel(k.encode()) == 0
                try:
                    y = torch.full((rows,), -7.0, dtype=dt, device="cuda")
                    sk.spmv_rgcsr(a, x, y)
                    torch.cuda.synchronize()
                finally:
                    lib().spmvk_set_rgcsr_kernel(b"auto")
                got = y.cpu().numpy()
                assert bitwise(got, np.zeros(rows, got.dtype)), (prec, G, k)  # +0, not -0
            # host-span overload and the multiply-add count
            yh, madds = sk.spmv_rgcsr(a, np.zeros(0, got.dtype), multiply_add_count=True)
            assert madds == 0 and bitwise(yh, np.zeros(rows, got.dtype))
        h = sk.build_hybrid(m, precision=prec)
        yh = sk.spmv_hybrid(h, x)
        assert bitwise(yh.cpu().numpy(), np.zeros(rows, yh.cpu().numpy().dtype))
        c = sk.build_csr(m, prec)
        yc = sk.spmv_csr(c, x)
        assert bitwise(yc.cpu().numpy(), np.zeros(rows, yc.cpu().numpy().dtype))
    # the iterated (scaled) form writes x_next = +0 * scale too
    a = sk.build_rgcsr(m, 32, 8)
    y = torch.full((rows,), 3.0, dtype=torch.float64, device="cuda")
    xn = torch.full((rows,), 3.0, dtype=torch.float64, device="cuda")
    sk._check(lib().spmvk_rgcsr_spmv_scaled_f64(a._h, None, 0, y.data_ptr(), rows,
                                                xn.data_ptr(), 0.0625, None))
    assert bitwise(xn.cpu().numpy(), np.zeros(rows))


@pytest.mark.parametrize("kind,n", [(5, 64), (5, 300), (7, 20)])
def test_offset_x_view_bitwise(cuda, kind, n):
    """x = buf[1:] starts 8 (fp64) / 4 (fp32) bytes past a 256-byte boundary."""
    csr = sk.CsrMatrix.stencil(kind, n)
    rp, col, val = csr.to_host()
    om = orc.Csr(csr.num_rows, csr.num_cols, rp, col, val)
    x = gen.random_vector(csr.num_cols, 1)
    for prec, dt in ((8, np.float64), (4, np.float32)):
        xs = x.astype(dt)
        want = orc.spmv_rgcsr(orc.build_rgcsr(om, 32, prec), xs)[0]
        a = sk.build_rgcsr(csr, 32, prec)
        buf = torch.zeros(csr.num_cols + 1, dtype=torch.from_numpy(xs).dtype, device="cuda")
        buf[1:] = torch.from_numpy(xs).cuda()
        xv = buf[1:]
        assert xv.data_ptr() % 16 != 0
        for k in ("auto", "grp6"):
            assert lib().spmvk_set_rgcsr_kernel(k.encode()) == 0
            try:
                y = sk.spmv_rgcsr(a, xv)
                torch.cuda.synchronize()
            finally:
                lib().spmvk_set_rgcsr_kernel(b"auto")
            assert bitwise(y.cpu().numpy(), want), (kind, n, prec, k)


def test_uint32_slot_overflow_is_erange(cuda):
    """2^24 rows, G = 256, one 256-entry row per group: 65,536 groups of
    256 x 256 slots = 2^32 slots -- one past what uint32 group pointers hold.
    The reference would wrap gp to 0 (rgcsr.hpp:56); the device converter
    raises ERANGE (SpmvkRuntimeError) with the slot count."""
    rows, G = 1 << 24, 256
    lens = np.zeros(rows, np.uint32)
    lens[::G] = G
    rp = np.zeros(rows + 1, np.uint32)
    np.cumsum(lens, out=rp[1:])
    nnz = int(rp[-1])
    col = np.tile(np.arange(G, dtype=np.uint32), rows // G)
    val = np.ones(nnz, np.float64)
    m = sk.TripletMatrix(rows, rows, rp, col, val, validate=False)
    csr = sk.build_csr(m)
    with pytest.raises(sk.SpmvkRuntimeError, match=r"4294967296 slots overflow the 32-bit"):
        sk.build_rgcsr(csr, G)
    assert lib().spmvk_rgcsr_build(csr._h, G, 8, None, C.byref(C.c_void_p())) == 2  # ERANGE
    # one row shorter in the last group: 2^32 - 256 slots fit
    lens[-G] = G - 1
    rp2 = np.zeros(rows + 1, np.uint32)
    np.cumsum(lens, out=rp2[1:])
    m2 = sk.TripletMatrix(rows, rows, rp2, col[: int(rp2[-1])], val[: int(rp2[-1])],
                          validate=False)
    a = sk.build_rgcsr(sk.build_csr(m2), G, 4)
    assert a.slot_count() == (1 << 32) - G
    gp = np.empty(a.num_groups() + 1, np.uint32)  # 32 GB of slots stay on the device
    sk._check(lib().spmvk_rgcsr_download(a._h, None, None, gp.ctypes.data, None))
    assert int(gp[-1]) == (1 << 32) - G and int(gp[-2]) == (1 << 32) - G * G


def test_barrier_times_out_on_a_missing_peer(cuda):
    """Two ranks on one GPU (spmvk_dist_open_local); only rank 0 steps with
    the device barrier on.  Its barrier must give up after the timeout, mark
    the window, and spmvk_dist_status must report ENCCL naming rank 1; later
    barriers of the window return at once."""
    L = lib()
    csr = sk.CsrMatrix.stencil(7, 16)
    G, P = 32, 2
    slabs = pt.slab_bounds(csr.num_rows, G, P)
    n = max(csr.num_cols, slabs[-1].row_end)
    wins = [pt.ExchangeWindow(n, 8) for _ in slabs]
    arr = (C.c_void_p * P)(*[w._h.value for w in wins])
    d = C.c_void_p()
    assert L.spmvk_dist_open_local(arr, 0, P, C.byref(d)) == 0
    rr = (C.c_uint64 * 4)(0, n, 0, n)
    sl = slabs[0]
    assert L.spmvk_dist_set_rows(d, sl.row_begin, sl.row_end, rr) == 0
    assert L.spmvk_dist_set_timeout_ms(d, 0) != 0
    assert L.spmvk_dist_set_timeout_ms(d, 200) == 0
    a = sk.build_rgcsr(csr, G, 8, row_range=(sl.row_begin, sl.row_end))
    y = torch.empty(sl.rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    assert L.spmvk_dist_status(d, C.c_void_p(s.cuda_stream)) == 0
    t0 = time.time()
    assert L.spmvk_dist_step_f64(d, a._h, 0.0625, y.data_ptr(), 1, C.c_void_p(s.cuda_stream)) == 0
    for _ in range(20):  # later barriers: status already set, no further waits
        assert L.spmvk_dist_step_f64(d, a._h, 0.0625, y.data_ptr(), 1,
                                     C.c_void_p(s.cuda_stream)) == 0
    rc = L.spmvk_dist_status(d, C.c_void_p(s.cuda_stream))
    dt = time.time() - t0
    assert rc == 4, rc  # SPMVK_ENCCL
    assert "timed out waiting for rank 1" in sk._lib.last_error()
    assert dt < 5.0, dt  # one 200 ms timeout, not 21
    L.spmvk_dist_destroy(d)
    for w in wins:
        w.close()


def test_block_cache_reuse_keeps_inflight_spmv_and_arrays(cuda):
    """Handle arrays released by destroy are reused by the next build of a
    similar size (spmvk.h spmvk_empty_cache): a SpMV still queued on the
    destroyed handle must finish before its block is rewritten, and a rebuilt
    (smaller, reusing the larger block) format is bitwise the oracle's."""
    big = sk.CsrMatrix.stencil(27, 40)
    small = sk.CsrMatrix.stencil(27, 38)
    x_big = torch.from_numpy(gen.random_vector(big.num_cols, 1)).cuda()
    want_big = sk.spmv_rgcsr(sk.build_rgcsr(big, 32), x_big).cpu().numpy()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        a = sk.build_rgcsr(big, 32)
        y = torch.empty_like(x_big)
        with torch.cuda.stream(s1):
            for _ in range(20):  # queue work on the handle, then release it at once
                sk.spmv_rgcsr(a, x_big, y)
        del a
        b = sk.build_rgcsr(small, 32, stream=s2.cuda_stream)
        torch.cuda.synchronize()
        assert bitwise(y.cpu().numpy(), want_big)
        rp, col, val = small.to_host()
        want = orc.build_rgcsr(orc.Csr(small.num_rows, small.num_cols, rp, col, val), 32)
        got = b.to_host()
        for k in ("values", "columns", "group_pointers", "row_lengths"):
            assert np.array_equal(got[k], want[k]), k
        del b
    assert lib().spmvk_empty_cache(-1) == 0
    c = sk.build_rgcsr(big, 32)
    assert bitwise(sk.spmv_rgcsr(c, x_big).cpu().numpy(), want_big)
