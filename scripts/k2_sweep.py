"""Times every K2 (RgCSR SpMV) kernel variant on the stencil workloads and
prints one JSON line per (workload, precision, group size, variant).
Usage (GPU box): python scripts/k2_sweep.py [--steps 200]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--variants", default="auto,lite,lite8,lite8_mpf,vec2,grp6,grp7_mpf,grp8,grp8_r64")
    ap.add_argument("--cases", default="27:128:32,27:128:128,5:1024:32,5:2048:32,7:256:32,7:512:32")
    ap.add_argument("--flush", action="store_true",
                    help="read 512 MB before every timed launch (median of per-launch events)")
    ap.add_argument("--precs", default="8,4")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    assert lib().spmvk_init(0) == 0
    peak, _ = bench.peaks()
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sp = stream.cuda_stream
    L = lib()
    for case in args.cases.split(","):
        kind, n, G = (int(v) for v in case.split(":"))
        csr = sk.CsrMatrix.stencil(kind, n)
        for prec in (int(p) for p in args.precs.split(",")):
            a = sk.build_rgcsr(csr, G, prec, stream=sp)
            dt = torch.float64 if prec == 8 else torch.float32
            x = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda().to(dt)
            y = torch.empty(a.num_rows, dtype=dt, device="cuda")
            fn = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
            B = bench.rg_bytes(a.info, prec)
            ref = None
            for v in args.variants.split(","):
                assert L.spmvk_set_rgcsr_kernel(v.encode()) == 0
                launch = lambda: fn(a._h, x.data_ptr(), a.num_cols, y.data_ptr(),  # noqa: E731
                                    a.num_rows, sp)
                if args.flush:
                    per = []
                    for i in range(args.steps + 3):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        with torch.cuda.stream(stream):
                            flush.sum()
                            e0.record(stream)
                            launch()
                            e1.record(stream)
                        if i >= 3:
                            per.append((e0, e1))
                    torch.cuda.synchronize()
                    us = statistics.median(a_.elapsed_time(b_) for a_, b_ in per) * 1e3
                else:
                    _, per = bench.time_launches(launch, stream, args.steps, 5)
                    us = per * 1e3
                ysum = float(y.double().sum().item())
                ref = ysum if ref is None else ref
                print(json.dumps({"case": f"{kind}pt-{n}", "G": G, "prec": prec, "variant": v,
                                  "us": round(us, 2), "gflops": round(2 * a.nnz() / us / 1e3, 1),
                                  "GBs": round(B / us / 1e3, 1), "frac": round(B / us / 1e3 / peak, 4),
                                  "same_y": ysum == ref}), flush=True)
            del a
        del csr
    L.spmvk_set_rgcsr_kernel(b"auto")


if __name__ == "__main__":
    main()
