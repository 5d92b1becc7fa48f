"""Shared test helpers: golden-fixture access and oracle <-> product adapters."""
import numpy as np

import oracle as orc
from paper_1012_2270_b200 import spmvkit as sk

RG_KEYS = ("values", "columns", "group_pointers", "row_lengths")
HY_KEYS = ("ell_values", "ell_columns", "coo_rows", "coo_columns", "coo_values")


def golden_csr(npz, prefix) -> orc.Csr:
    rows, cols = (int(v) for v in npz[f"{prefix}_shape"])
    return orc.Csr(rows, cols, npz[f"{prefix}_rp"], npz[f"{prefix}_col"], npz[f"{prefix}_val"])


def triplets(m: orc.Csr) -> sk.TripletMatrix:
    return sk.TripletMatrix(m.rows, m.cols, m.rp, m.col, m.val)


def bitwise(a, b) -> bool:
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def assert_rgcsr_equal(got: dict, want, prefix=""):
    for k in RG_KEYS:
        w = want[f"{prefix}{k}"] if prefix else want[k]
        assert bitwise(got[k], w), f"rgcsr {k} differs"


def assert_hybrid_equal(got: dict, want, prefix=""):
    for k in HY_KEYS:
        w = want[f"{prefix}{k}"] if prefix else want[k]
        assert bitwise(got[k], w), f"hybrid {k} differs"
