"""The package's `simulate` report (paper_1012_2270_b200.simulate, SURVEY
§8f-3; reference tools/main.cpp:304-317) from a real ncu pass on the GPU:
the reference's JSON schema, and sector counts that must follow from the
format's layout (every RgCSR slot is one coalesced 8-byte value and 4-byte
column load; y is one coalesced 8-byte store per row)."""
import shutil

import pytest

from paper_1012_2270_b200 import simulate as simm
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu
needs_ncu = pytest.mark.skipif(shutil.which("ncu") is None, reason="ncu not on PATH")

SCHEMA = {"matrix", "format", "precision", "nnz", "artificial_zeros", "transactions",
          "min_possible", "efficiency", "cache", "peak"}


@needs_ncu
def test_rgcsr_report_matches_the_layout(cuda):
    n = 48
    doc = simm.simulate(case=f"7:{n}", format="rgcsr", group_size=32, precision="double")
    assert SCHEMA <= set(doc) and doc["group_size"] == 32
    a = sk.build_rgcsr(sk.CsrMatrix.stencil(7, n), 32)
    f = sk.fill_report(a)
    assert doc["nnz"] == a.nnz() and doc["artificial_zeros"] == f.artificial_zeros
    tx = doc["transactions"]
    slots, rows = a.slot_count(), a.num_rows
    assert tx["values"] == slots * 8 // 32  # fully coalesced, pads included (group walk)
    assert tx["columns"] == slots * 4 // 32
    assert tx["output"] == rows * 8 // 32
    assert tx["x"] > 0 and 0 < doc["efficiency"] <= 1.0
    assert doc["min_possible"] <= sum(tx.values()) + doc["metadata_sectors"]
    assert doc["cache"]["hits"] + doc["cache"]["misses"] >= tx["x"] * 0.5
    assert doc["peak"]["bytes_per_nnz"] == 12 and doc["peak"]["gflops"] > 0


@needs_ncu
@pytest.mark.parametrize("fmt", ["csr", "ellpack"])
def test_other_formats_and_ordering(cuda, fmt):
    doc = simm.simulate(case="0:20000", format=fmt, precision="single",
                        ordering="descending")
    assert SCHEMA <= set(doc) and doc["ordering"] == "descending"
    assert doc["nnz"] > 0 and all(v >= 0 for v in doc["transactions"].values())
    assert doc["peak"]["bytes_per_nnz"] == 8


def test_argument_errors():
    with pytest.raises(ValueError, match="simulate supports"):
        simm.simulate(format="bcsr")
    with pytest.raises(ValueError):
        simm.simulate(precision="half")
