"""spmvkit.run_spmv_bench on the B200 vs the reference's own harness
(src/bench.cpp:47-138, called through oracle/_ref): same BenchRecord
accounting (format, group size, nnz, fill, artificial zeros, bytes) and the
same checksum (y bitwise equal, summed in row order), plus the checksum gate
and the format errors."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
from helpers import golden_csr, triplets
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu

REF_KIND = {"csr": 0, "rgcsr": 1, "hybrid": 2}


def ref_record(om, kind, group, prec):
    r = orc.RefMatrix.from_csr(om)
    out = (C.c_double * 4)()
    orc._rcheck(orc.R().ref_run_spmv_bench(r.h, REF_KIND[kind], -1 if group is None else group,
                                           prec, 3, out))
    return {"median_seconds": out[0], "gflops": out[1], "checksum": out[2], "bytes": int(out[3])}


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("prec", [8, 4])
def test_records_match_reference_harness(cuda, golden, prec):
    g = golden["acceptance"]
    opts = sk.BenchOptions(repetitions=3)
    for seed in (3, 17, 42, 99, 150):
        om = golden_csr(g, f"a{seed}")
        m = triplets(om)
        for kind, group in (("csr", None), ("rgcsr", 1 + seed % 9), ("rgcsr", None),
                            ("hybrid", None)):
            rec = sk.run_spmv_bench(m, f"a{seed}", kind, group, prec, opts)
            ref = ref_record(om, kind, group, prec)
            assert rec.format_name == kind and rec.nnz == om.nnz
            assert rec.precision == ("double" if prec == 8 else "single")
            assert rec.group_size == ((group or 32) if kind == "rgcsr" else None)
            assert rec.bytes == ref["bytes"], (seed, kind)
            assert rec.checksum == ref["checksum"], (seed, kind)  # bitwise y, same sum order
            assert rec.median_seconds > 0 and rec.gflops == pytest.approx(
                2 * om.nnz / rec.median_seconds / 1e9)


def test_ellpack_record_and_errors(cuda, golden):
    m = triplets(golden_csr(golden["example8"], "m"))
    rec = sk.run_spmv_bench(m, "example8", "ellpack", options=sk.BenchOptions(repetitions=3,
                                                                                x_ones=True))
    assert (rec.artificial_zeros, rec.bytes, rec.checksum) == (11, 24 * 12, 91.0)
    with pytest.raises(sk.InvalidArgument, match="coo is benchmarked as part of hybrid"):
        sk.run_spmv_bench(m, "example8", "coo")
    with pytest.raises(sk.InvalidArgument):
        sk.run_spmv_bench(m, "example8", "nope")


def test_checksum_gate_fires(cuda, golden, monkeypatch):
    """A wrong kernel result must raise ChecksumError before any timing."""
    m = triplets(golden_csr(golden["example8"], "m"))
    real = sk.spmv_rgcsr

    def broken(a, x, y=None, **kw):
        out = real(a, x, y, **kw)
        out[0] += 1.0
        return out
    monkeypatch.setattr(sk, "spmv_rgcsr", broken)
    with pytest.raises(sk.ChecksumError, match="rgcsr checksum .* disagrees with oracle"):
        sk.run_spmv_bench(m, "example8", "rgcsr", 4, options=sk.BenchOptions(x_ones=True))
