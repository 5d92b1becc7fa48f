"""Interleaved A/B of SpMV kernels on one matrix (same process, same buffers):
RgCSR K2 variants vs Hybrid, back-to-back launches (total events over K
launches) and with a read-only L2 flush before each launch.  Repeats R rounds
so run-to-run drift shows up."""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="27:128")
    ap.add_argument("--prec", type=int, default=8)
    ap.add_argument("--variants", default="lite8,lite,hybrid")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--group", type=int, default=32)
    ap.add_argument("--reorder", action="store_true", help="descending row reordering first")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    if a.case.startswith("b:"):  # b:<rows>:<half bandwidth> -- banded_matrix (synthetic.cpp)
        _, n, hbw = a.case.split(":")
        csr = sk.build_csr(gen.banded(int(n), int(hbw), 3))
    else:
        kind, n = (int(v) for v in a.case.split(":"))
        csr = sk.CsrMatrix.stencil(kind, n) if kind else sk.build_csr(gen.powerlaw(n, 7))
    if a.prec == 4:
        csr = sk.build_csr(sk.TripletMatrix(csr.num_rows, csr.num_cols, *csr.to_host()), 4)
    dt = torch.float64 if a.prec == 8 else torch.float32
    if a.reorder:
        csr = sk.apply_descending_permutation(csr)[0]
    rg = sk.build_rgcsr(csr, a.group, a.prec)
    hy = sk.build_hybrid(csr, None, a.prec)
    x = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda().to(dt)
    y = torch.empty(csr.num_rows, dtype=dt, device="cuda")
    s = torch.cuda.current_stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    f_rg = L.spmvk_rgcsr_spmv_f64 if a.prec == 8 else L.spmvk_rgcsr_spmv_f32
    f_hy = L.spmvk_hybrid_spmv_f64 if a.prec == 8 else L.spmvk_hybrid_spmv_f32

    f_csr = L.spmvk_csr_spmv_f64 if a.prec == 8 else L.spmvk_csr_spmv_f32
    csr_p = csr  # already in the run's precision

    def launcher(v):
        if v == "csr":  # spmv_csr (SPMVK_CSR_KERNEL=row: the thread-per-row kernel)
            return lambda: f_csr(csr_p._h, x.data_ptr(), csr.num_cols, y.data_ptr(),
                                 csr.num_rows, s.cuda_stream)
        if v.startswith("hybrid"):  # hybrid or hybrid:<variant> (spmvk_set_hybrid_kernel)
            hv = (v.split(":", 1)[1] if ":" in v else "auto").encode()
            return lambda: (L.spmvk_set_hybrid_kernel(hv),
                            f_hy(hy._h, x.data_ptr(), csr.num_cols, y.data_ptr(), csr.num_rows,
                                 s.cuda_stream))
        return lambda: (L.spmvk_set_rgcsr_kernel(v.encode()),
                        f_rg(rg._h, x.data_ptr(), csr.num_cols, y.data_ptr(), csr.num_rows,
                             s.cuda_stream))

    res = {v: {"b2b": [], "flushed": []} for v in a.variants.split(",")}
    y0 = None
    for v in res:  # every variant's y must be bitwise the first's
        launcher(v)()
        torch.cuda.synchronize()
        if y0 is None:
            y0 = y.clone()
        elif not torch.equal(y.view(torch.int64 if a.prec == 8 else torch.int32),
                             y0.view(torch.int64 if a.prec == 8 else torch.int32)):
            print(f"{a.case} p{a.prec} {v}: y NOT bitwise equal to {next(iter(res))}", flush=True)
    for _ in range(a.rounds):
        for v in res:
            fn = launcher(v)
            for _ in range(5):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.k):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[v]["b2b"].append(e0.elapsed_time(e1) / a.k * 1e3)
            per = []
            for _ in range(a.k // 2):
                flush.sum()
                s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_.record()
                fn()
                e_.record()
                per.append((s_, e_))
            torch.cuda.synchronize()
            res[v]["flushed"].append(statistics.median(p.elapsed_time(q) for p, q in per) * 1e3)
    L.spmvk_set_rgcsr_kernel(b"auto")
    L.spmvk_set_hybrid_kernel(b"auto")
    for v, d in res.items():
        print(f"{a.case}{'r' if a.reorder else ''} p{a.prec} g{a.group} {v:12s} b2b us " + " ".join(f"{t:7.2f}" for t in d["b2b"]) +
              " | flushed us " + " ".join(f"{t:7.2f}" for t in d["flushed"]), flush=True)


if __name__ == "__main__":
    main()
