"""BASELINE config 3 (power-law rows, 8M, mean 16, max 4096): RgCSR long-row
cut x K2 variant, descending reordering, vs Hybrid.  L2 flushed (read-only)
before each timed launch; every y checked bitwise against the CSR kernel
(reordered results through the permutation).  One JSON line per case."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def timed(fn, stream, scratch, reps=20):
    per = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            scratch.sum()
            a.record(stream)
            fn()
            b.record(stream)
        stream.synchronize()
        if i >= 3:
            per.append(a.elapsed_time(b))
    return statistics.median(per) * 1e3


def main():
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    scratch = torch.zeros(64 << 20, dtype=torch.float64, device="cuda")
    m = gen.powerlaw(8_000_000, 7)
    nnz = m.nnz
    csr64 = sk.build_csr(m, 8, stream=sp)
    csr2, perm = sk.apply_descending_permutation(csr64)
    permt = torch.from_numpy(perm.astype(np.int64)).cuda()
    for prec in (8, 4):
        dt = torch.float64 if prec == 8 else torch.float32
        iv = torch.int64 if prec == 8 else torch.int32
        x = torch.from_numpy(gen.random_vector(m.num_cols, 1)).cuda().to(dt)
        c = csr64 if prec == 8 else sk.build_csr(m, 4, stream=sp)
        c2 = csr2 if prec == 8 else sk.apply_descending_permutation(c)[0]
        yref = sk.spmv_csr(c, x)
        fn = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
        y = torch.empty_like(yref)

        def run(tag, h, reordered=False, **kw):
            us = timed(lambda: fn(h._h, x.data_ptr(), m.num_cols, y.data_ptr(), m.num_rows, sp),
                       stream, scratch)
            want = yref[permt] if reordered else yref
            print(json.dumps({"prec": prec, "case": tag, "us": round(us, 1),
                              "gflops": round(2 * nnz / us / 1e3, 1),
                              "fill_percent": round(sk.fill_report(h).fill_percent, 2),
                              "bitwise": bool(torch.equal(y.view(iv), want.view(iv))), **kw}),
                  flush=True)

        for cut in (32, 64, 128, 256, 1 << 30):
            L.spmvk_set_long_row_cut(cut)
            h = sk.build_rgcsr(c, 32, prec, stream=sp)
            for v in ("lite8", "lite", "pipe", "ldg_pf"):
                L.spmvk_set_rgcsr_kernel(v.encode())
                run(f"rgcsr32 cut={cut} {v}", h, cut=cut, variant=v)
            del h
        L.spmvk_set_long_row_cut(128)
        L.spmvk_set_rgcsr_kernel(b"auto")
        for G in (32, 128):
            h = sk.build_rgcsr(c2, G, prec, stream=sp)
            run(f"rgcsr{G} descending", h, reordered=True, group_size=G)
            del h
        hy = sk.build_hybrid(c, None, prec, stream=sp)
        fh = L.spmvk_hybrid_spmv_f64 if prec == 8 else L.spmvk_hybrid_spmv_f32
        us = timed(lambda: fh(hy._h, x.data_ptr(), m.num_cols, y.data_ptr(), m.num_rows, sp),
                   stream, scratch)
        print(json.dumps({"prec": prec, "case": "hybrid", "us": round(us, 1),
                          "gflops": round(2 * nnz / us / 1e3, 1),
                          "bitwise": bool(torch.equal(y.view(iv), yref.view(iv)))}), flush=True)
        del hy


if __name__ == "__main__":
    main()
