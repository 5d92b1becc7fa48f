"""B200-native Row-grouped CSR (RgCSR) / Hybrid ELL+COO SpMV (arxiv/paper_1012_2270).

The product is ``libspmvk.so`` (hand-written sm_100a kernels behind the C-ABI
in ``include/spmvk.h``); ``spmvkit`` mirrors the reference's hot-path API on
top of it, ``generators`` builds the synthetic workloads, ``partition`` is the
row-slab multi-GPU layer.
"""
from . import spmvkit  # noqa: F401
from .spmvkit import (  # noqa: F401
    CsrMatrix, FillReport, HybridMatrix, InvalidArgument, RgcsrMatrix, SpmvkRuntimeError,
    TripletMatrix, build_csr, build_hybrid, build_rgcsr, canonicalize, choose_ell_width,
    fill_report, hybrid_split_cost, measured_gflops, row_lengths, spmv_csr, spmv_hybrid,
    spmv_rgcsr)
