"""Generates tests/golden/* from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE ONLY.  Run here (needs /root/reference to build _ref):
    python oracle/make_golden.py
Fixtures (committed; the GPU box never reads /root/reference):
  golden/example8.npz   M8 (tests/fixtures.hpp:17-32): CSR, RgCSR g=4 and g=8
                        arrays, Hybrid K1=1 and default, spmv of ones.
  golden/small.npz      random_small seeds 600-649 (tests/test_formats.cpp:325-342),
                        integer and real values, RgCSR g = 1 + seed % 9, Hybrid
                        default width, x and the reference y of every format.
  golden/acceptance.npz random_case seeds 0-199 (tests/acceptance.cpp:138-173):
                        matrix, integer x, real-valued variant, y per format.
  golden/shapes.json    config-scale scalars computed by the reference: nnz,
                        slot counts per group size, Hybrid K1 / COO count,
                        sequential checksums of y for x = random_vector(N, 1).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as o  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def csr_arrays(prefix, m: o.Csr, d: dict):
    d[f"{prefix}_shape"] = np.array([m.rows, m.cols], np.uint64)
    d[f"{prefix}_rp"] = m.rp
    d[f"{prefix}_col"] = m.col
    d[f"{prefix}_val"] = m.val


def rg_arrays(prefix, a, d):
    for k in ("values", "columns", "group_pointers", "row_lengths"):
        d[f"{prefix}_{k}"] = a[k]


def hy_arrays(prefix, h, d):
    for k in ("ell_values", "ell_columns", "coo_rows", "coo_columns", "coo_values"):
        d[f"{prefix}_{k}"] = h[k]
    d[f"{prefix}_k1"] = np.array([h["k1"]], np.uint64)


def example8():
    d = {}
    r = o.RefMatrix.example8()
    m = r.to_csr()
    csr_arrays("m", m, d)
    ones = np.ones(8)
    for G in (4, 8):
        for prec in (8, 4):
            a = r.rgcsr(G, prec)
            rg_arrays(f"rg{G}_p{prec}", a, d)
            d[f"rg{G}_p{prec}_y_ones"] = r.rgcsr_spmv(a, ones.astype(a["values"].dtype))[0]
            d[f"rg{G}_p{prec}_fill"] = np.array(
                [a["artificial_zeros"], a["bytes_single"], a["bytes_double"], a["nnz"]], np.uint64)
    for k1 in (None, 0, 1, 3):
        h = r.hybrid(k1)
        name = "hyd" if k1 is None else f"hy{k1}"
        hy_arrays(name, h, d)
        d[f"{name}_y_ones"] = r.hybrid_spmv(h, ones)
        d[f"{name}_fill"] = np.array([h["artificial_zeros"], h["bytes_single"], h["bytes_double"]],
                                     np.uint64)
    d["y_ref_ones"] = r.spmv_reference(ones)
    d["descending_map"] = r.descending_map()
    np.savez_compressed(os.path.join(OUT, "example8.npz"), **d)


def small():
    d = {}
    for seed in range(600, 650):
        for integers in (True, False):
            tag = f"s{seed}_{'i' if integers else 'r'}"
            r = o.RefMatrix.random_small(seed, True, integers)
            m = r.to_csr()
            csr_arrays(tag, m, d)
            if integers:
                x = o.random_integer_x(m.cols, seed * 77 + 1)
            else:
                x = np.empty(m.cols)
                o.R().ref_random_vector(m.cols, seed, x.ctypes.data if m.cols else None)
            d[f"{tag}_x"] = x
            G = 1 + seed % 9
            a = r.rgcsr(G)
            rg_arrays(f"{tag}_rg", a, d)
            d[f"{tag}_rg_y"] = r.rgcsr_spmv(a, x)[0]
            a32 = r.rgcsr(G, 4)
            rg_arrays(f"{tag}_rg32", a32, d)
            d[f"{tag}_rg32_y"] = r.rgcsr_spmv(a32, x.astype(np.float32))[0]
            h = r.hybrid()
            hy_arrays(f"{tag}_hy", h, d)
            d[f"{tag}_hy_y"] = r.hybrid_spmv(h, x)
            d[f"{tag}_hy_fill"] = np.array([h["artificial_zeros"], h["bytes_single"],
                                            h["bytes_double"]], np.uint64)
            d[f"{tag}_rg_fill"] = np.array([a["artificial_zeros"], a["bytes_single"],
                                            a["bytes_double"], a["nnz"]], np.uint64)
            d[f"{tag}_csr_y"] = r.csr_spmv(x)
            d[f"{tag}_ref_y"] = r.spmv_reference(x)
    np.savez_compressed(os.path.join(OUT, "small.npz"), **d)


def acceptance():
    d = {}
    for seed in range(200):
        r = o.RefMatrix.random_case(seed, 64)
        m = r.to_csr()
        csr_arrays(f"a{seed}", m, d)
        xi = o.random_integer_x(m.cols, seed + 11)
        d[f"a{seed}_xi"] = xi
        G = 1 + seed % 9
        a = r.rgcsr(G)
        rg_arrays(f"a{seed}_rg", a, d)
        d[f"a{seed}_rg_yi"] = r.rgcsr_spmv(a, xi)[0]
        d[f"a{seed}_hy_yi"] = r.hybrid_spmv(r.hybrid(), xi)
        d[f"a{seed}_ref_yi"] = r.spmv_reference(xi)
    np.savez_compressed(os.path.join(OUT, "acceptance.npz"), **d)


def seq_sum(y):
    return float(np.cumsum(y.astype(np.float64))[-1])


def shapes():
    """Config-scale scalars from the reference (configs 1, 2, 3 of BASELINE.json)."""
    res = {}
    cases = [("5pt_1024", lambda: o.stencil(5, 1024)), ("27pt_128", lambda: o.stencil(27, 128)),
             ("powerlaw_8M", lambda: o.powerlaw(8_000_000, 7))]
    for name, gen in cases:
        m = gen()
        r = o.RefMatrix.from_csr(m)
        x = np.empty(m.cols)
        o.R().ref_random_vector(m.cols, 1, x.ctypes.data)
        e = {"rows": m.rows, "nnz": m.nnz, "max_len": int(m.lens().max())}
        for G in (32, 64, 128, 256):
            a = r.rgcsr(G)
            e[f"rg{G}"] = {"slots": int(a["values"].size), "artificial_zeros": a["artificial_zeros"],
                           "bytes_double": a["bytes_double"], "bytes_single": a["bytes_single"]}
            if G == 32:
                e["rg32"]["checksum_f64"] = seq_sum(r.rgcsr_spmv(a, x)[0])
                o.R().ref_rgcsr_free(a.pop("_h"))
                a4 = r.rgcsr(G, 4)
                e["rg32"]["checksum_f32"] = seq_sum(r.rgcsr_spmv(a4, x.astype(np.float32))[0])
                o.R().ref_rgcsr_free(a4.pop("_h"))
            else:
                o.R().ref_rgcsr_free(a.pop("_h"))
            del a
        h = r.hybrid()
        e["hybrid"] = {"k1": h["k1"], "coo": int(h["coo_rows"].size),
                       "artificial_zeros": h["artificial_zeros"], "bytes_double": h["bytes_double"],
                       "bytes_single": h["bytes_single"],
                       "checksum_f64": seq_sum(r.hybrid_spmv(h, x))}
        o.R().ref_hybrid_free(h.pop("_h"))
        e["checksum_reference"] = seq_sum(r.spmv_reference(x))
        res[name] = e
        print(name, json.dumps(e), flush=True)
        del r
    with open(os.path.join(OUT, "shapes.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    o.build()
    which = sys.argv[1:] or ["example8", "small", "acceptance", "shapes"]
    for w in which:
        globals()[w]()
        print("wrote", w, flush=True)
