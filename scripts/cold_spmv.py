"""Cold-cache SpMV time with sub-microsecond resolution: K x (L2 flush; SpMV)
timed as one region minus K x (L2 flush) alone (per-launch events tick in
~2 us steps).  For matrices that fit in L2 (config 1), where the bench rules
require a flush between launches.
    python scripts/cold_spmv.py [--case 5:1024] [--variants auto,grp6,...]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def region(fn, k, stream):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="5:1024")
    ap.add_argument("--variants", default="auto")
    ap.add_argument("--precs", default="8,4")
    ap.add_argument("--k", type=int, default=200)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    kind, n = (int(v) for v in a.case.split(":"))
    csr = sk.CsrMatrix.stencil(kind, n)
    peak, _ = bench.peaks()
    for prec in (int(p) for p in a.precs.split(",")):
        h = sk.build_rgcsr(csr, 32, prec, stream=sp)
        dt = torch.float64 if prec == 8 else torch.float32
        x = torch.from_numpy(gen.random_vector(h.num_cols, 1)).cuda().to(dt)
        y = torch.empty(h.num_rows, dtype=dt, device="cuda")
        f = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
        B = bench.rg_bytes(h.info, prec)

        def fl():
            with torch.cuda.stream(stream):
                flush.sum()
        t_flush = region(fl, a.k, stream)
        for v in a.variants.split(","):
            assert L.spmvk_set_rgcsr_kernel(v.encode()) == 0

            def both():
                fl()
                f(h._h, x.data_ptr(), h.num_cols, y.data_ptr(), h.num_rows, sp)
            t = region(both, a.k, stream) - t_flush
            print(f"{a.case} p{prec} {v:10s} xpf={os.environ.get('SPMVK_X_PREFETCH', 'auto')} "
                  f"cold us {t:7.2f}  frac {B / (t * 1e-6) / 1e9 / peak:.3f}", flush=True)
        L.spmvk_set_rgcsr_kernel(b"auto")


if __name__ == "__main__":
    main()
