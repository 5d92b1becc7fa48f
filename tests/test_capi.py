"""CPU checks of the drop-in boundary: libspmvk.so loads, exports every symbol
include/spmvk.h declares, the host-only entry points agree with the oracle /
reference, and compute entry points refuse to run without a GPU (no CPU
fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as orc
from paper_1012_2270_b200 import _lib
from paper_1012_2270_b200 import spmvkit as sk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spmvk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spmvk_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    decl = declared_symbols()
    assert len(decl) >= 35
    assert set(decl) == set(_lib.SIGNATURES), set(decl) ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert _lib.lib().spmvk_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rp = np.array([0, 1], np.uint32)
    col = np.array([0], np.uint32)
    val = np.array([1.0])
    rc = _lib.lib().spmvk_csr_upload(1, 1, 1, rp.ctypes.data, col.ctypes.data, val.ctypes.data,
                                     8, None, C.byref(h))
    assert rc == _lib.SPMVK_ECUDA
    assert "no CPU fallback" in _lib.last_error() or "CUDA" in _lib.last_error()
    with pytest.raises(sk.CudaError):
        sk.build_rgcsr(sk.TripletMatrix(1, 1, rp, col, val), 4)


def test_choose_ell_width_cost_table():
    """tests/test_formats.cpp:125-136 verbatim."""
    lens = [2, 1, 1, 1, 1, 2, 3, 2]
    assert [sk.hybrid_split_cost(lens, k) for k in range(4)] == [39, 31, 35, 48]
    assert sk.choose_ell_width(lens) == 1
    assert sk.choose_ell_width([3, 3, 3, 3]) == 3
    assert sk.hybrid_split_cost([3, 3, 3, 3], 3) == 24
    assert sk.choose_ell_width([0, 0]) == 0
    assert sk.choose_ell_width([]) == 0


def test_choose_ell_width_matches_exhaustive_scan():
    """The histogram + suffix-sum width equals the reference's O(N*max) scan
    (test_formats.cpp:138-158 with rng 99; acceptance.cpp:270-292 with 4711)."""
    for seed, nmax, lmax in ((99, 32, 12), (4711, 40, 14), (5, 2000, 300)):
        rng = orc._MT(seed)
        for _ in range(100 if nmax < 100 else 10):
            lens = [rng.next() % lmax for _ in range(1 + rng.next() % nmax)]
            assert sk.choose_ell_width(lens) == orc.choose_ell_width(lens)
            if orc.ref_available():
                L = np.array(lens, np.uint64)
                assert sk.choose_ell_width(lens) == orc.R().ref_choose_ell_width(L.ctypes.data,
                                                                                 L.size)


def test_triplet_matrix_validation():
    """TripletMatrix ctor / canonicalize semantics (src/triplet.cpp:22-49)."""
    with pytest.raises(sk.InvalidArgument):
        sk.TripletMatrix.from_entries(2, 2, [(0, 1, 1.0), (0, 0, 1.0)])
    with pytest.raises(sk.InvalidArgument):
        sk.TripletMatrix.from_entries(2, 2, [(0, 2, 1.0)])
    m = sk.canonicalize([(1, 0, 1.0), (0, 1, 2.0), (1, 0, 3.0)], 2, 2)
    assert m.entries() == [(0, 1, 2.0), (1, 0, 4.0)]
    assert sk.row_lengths(m).tolist() == [1, 1]
    assert sk.measured_gflops(1000000, 1e-3) == 2.0  # acceptance.cpp:299
    with pytest.raises(sk.InvalidArgument):
        sk.measured_gflops(1, 0.0)


def test_peak_performance_table():
    """tests/test_memsim.cpp:182-202 at the reference model's 141 GB/s, and the
    B200 default (measured copy bandwidth)."""
    for prec, cached, gf, bpn in ((4, False, 23.5, 12), (8, False, 14.1, 20),
                                  (4, True, 35.25, 8), (8, True, 23.5, 12)):
        p = sk.peak_performance(prec, cached, bandwidth_gb_s=141.0)
        assert (p.gflops, p.bytes_per_nnz) == (gf, bpn)
    assert sk.peak_performance(8, False, 282.0).gflops == 2 * sk.peak_performance(8, False, 141.0).gflops
    assert sk.peak_performance(8, True).gflops == 2 * 6545.3 / 12


def test_kernel_variant_knobs_validate_names():
    """The tuning knobs accept their documented names and reject others
    (EINVAL with the list) -- host-only, no device needed."""
    L = _lib.lib()
    for v in (b"auto", b"v4", b"lite", b"lite8", b"lite8_full", b"litef", b"lite8f", b"g6",
              b"g7", b"g8", b"g8r", b"litefh", b"dyn", b"vec"):
        assert L.spmvk_set_hybrid_kernel(v) == 0, v
    assert L.spmvk_set_hybrid_kernel(b"nope") == _lib.SPMVK_EINVAL
    assert "lite8_full" in _lib.last_error() and "dyn" in _lib.last_error()
    for v in (b"auto", b"grp6", b"grp7_mpf", b"grp8", b"grp8_r64", b"grpv4", b"lite", b"lite8",
              b"lite8_full", b"liteh", b"lite8h", b"vec2", b"pipe"):
        assert L.spmvk_set_rgcsr_kernel(v) == 0, v
    assert L.spmvk_set_rgcsr_kernel(b"nope") == _lib.SPMVK_EINVAL
    assert L.spmvk_set_long_fused(0) == 0 and L.spmvk_set_long_fused(1) == 0
    assert L.spmvk_set_hybrid_kernel(b"auto") == 0 and L.spmvk_set_rgcsr_kernel(b"auto") == 0
