"""L2 persistence window for x (spmvk_stream_persist_x): SpMV time with and
without the window on the irregular (power-law, descending-reordered RgCSR
and Hybrid) and regular (27-pt) workloads.  Back-to-back launches (x stays
warm as in an iterated solver) and with a 1 GB read-only flush before each
launch.  y must be bitwise equal with and without the window."""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def b2b(fn, stream, k=30):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


def flushed(fn, stream, scratch, k=15):
    per = []
    for i in range(k + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            scratch.sum()
            a.record(stream)
            fn()
            b.record(stream)
        if i >= 2:
            per.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in per) * 1e3


def main():
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    scratch = torch.zeros(128 << 20, dtype=torch.float64, device="cuda")
    pl = gen.powerlaw(8_000_000, 7)
    cases = []
    for prec in (8, 4):
        c = sk.build_csr(pl, prec, stream=sp)
        c2, _ = sk.apply_descending_permutation(c)
        cases.append(("powerlaw-8M desc rgcsr32", prec, "rg", sk.build_rgcsr(c2, 32, prec, stream=sp)))
        cases.append(("powerlaw-8M hybrid", prec, "hy", sk.build_hybrid(c, None, prec)))
        del c, c2
    st = sk.CsrMatrix.stencil(27, 128)
    cases.append(("27pt-128 rgcsr32", 8, "rg", sk.build_rgcsr(st, 32, 8, stream=sp)))
    for name, prec, kind, a in cases:
        dt = torch.float64 if prec == 8 else torch.float32
        x = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda().to(dt)
        y = torch.empty(a.num_rows, dtype=dt, device="cuda")
        if kind == "rg":
            f = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
        else:
            f = L.spmvk_hybrid_spmv_f64 if prec == 8 else L.spmvk_hybrid_spmv_f32

        def fn():
            assert f(a._h, x.data_ptr(), a.num_cols, y.data_ptr(), a.num_rows, sp) == 0

        res = {"case": name, "prec": prec, "x_MB": x.numel() * prec / 2**20}
        fn()
        torch.cuda.synchronize()
        y0 = y.clone()
        res["b2b_us"], res["flushed_us"] = b2b(fn, stream), flushed(fn, stream, scratch)
        for hr in (1.0, 0.75):
            g = C.c_uint64()
            assert L.spmvk_stream_persist_x(C.c_void_p(sp), C.c_void_p(x.data_ptr()),
                                            x.numel() * prec, hr, C.byref(g)) == 0
            res[f"persist{hr}_b2b_us"] = b2b(fn, stream)
            res[f"persist{hr}_flushed_us"] = flushed(fn, stream, scratch)
            res["granted_MB"] = g.value / 2**20
            res["bitwise"] = bool(torch.equal(y.view(torch.int64 if prec == 8 else torch.int32),
                                              y0.view(torch.int64 if prec == 8 else torch.int32)))
            assert L.spmvk_stream_persist_x(C.c_void_p(sp), None, 0, 1.0, None) == 0
        print(json.dumps({k: round(v, 1) if isinstance(v, float) else v for k, v in res.items()}),
              flush=True)


if __name__ == "__main__":
    main()
