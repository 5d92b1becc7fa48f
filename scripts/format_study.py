"""RgCSR-vs-Hybrid study on one B200 (BASELINE configs 1-3): for each workload
and precision, the device conversion time and the SpMV time of RgCSR at
G in {32, 64, 128, 256} (default K2 variant) and of Hybrid ELL+COO, as GFLOP/s
(2 nnz / t), GB/s of the format's algorithmic bytes (B_fmt) and of the
format-independent minimum (B_min = nnz (S + 4) + S (rows + cols)).  Every
result is checked bitwise against the RgCSR G=32 y (all formats accumulate in
the reference's order).  One JSON line per (workload, precision, format).

    python scripts/format_study.py [--workloads 5pt-1024,27pt-128,powerlaw-8M]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def flush_l2(buf):
    """Evicts L2 by READING 512 MB (a write-based flush would leave dirty lines
    whose write-back lands inside the next timed kernel)."""
    return buf.sum()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="5pt-1024,27pt-128,powerlaw-8M")
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    peak, _ = bench.peaks()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    scratch = torch.zeros(64 << 20, dtype=torch.float64, device="cuda")  # 512 MB > L2
    for wl in args.workloads.split(","):
        csr = bench.make_csr(wl)
        rows, cols, nnz = csr.num_rows, csr.num_cols, csr.nnz()
        xh = gen.random_vector(cols, 1)
        for prec in (8, 4):
            dt = torch.float64 if prec == 8 else torch.float32
            x = torch.from_numpy(xh).cuda().to(dt)
            ref = None
            B_min = nnz * (prec + 4) + prec * (rows + cols)
            for fmt in ("rgcsr32", "rgcsr64", "rgcsr128", "rgcsr256", "hybrid"):
                y = torch.empty(rows, dtype=dt, device="cuda")
                torch.cuda.synchronize()
                t = time.perf_counter()
                if fmt == "hybrid":
                    h = sk.build_hybrid(csr, None, prec, stream=sp)
                    B = bench.hy_bytes(h.info, prec)
                    fn = L.spmvk_hybrid_spmv_f64 if prec == 8 else L.spmvk_hybrid_spmv_f32
                    extra = {"ell_width": h.slots_per_row, "coo_nnz": h.coo_nnz()}
                else:
                    G = int(fmt[5:])
                    h = sk.build_rgcsr(csr, G, prec, stream=sp)
                    B = bench.rg_bytes(h.info, prec)
                    fn = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
                    extra = {"group_size": G, "slots": h.slot_count(),
                             "fill_percent": sk.fill_report(h).fill_percent}
                torch.cuda.synchronize()
                conv_ms = (time.perf_counter() - t) * 1e3
                # L2 flushed before every timed launch (small configs fit in L2)
                per = []
                for i in range(args.steps + 3):
                    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(stream):
                        flush_l2(scratch)  # same stream: finishes before the timed launch
                        a_.record(stream)
                        fn(h._h, x.data_ptr(), cols, y.data_ptr(), rows, sp)
                        b_.record(stream)
                    stream.synchronize()
                    if i >= 3:
                        per.append(a_.elapsed_time(b_))
                us = statistics.median(per) * 1e3
                ysum = y.double().cpu().numpy().tobytes()
                ref = ysum if ref is None else ref
                print(json.dumps({"workload": wl, "prec": prec, "format": fmt, "nnz": nnz,
                                  "convert_ms": round(conv_ms, 2), "spmv_us": round(us, 2),
                                  "gflops": round(2 * nnz / us / 1e3, 1),
                                  "fmt_GBs": round(B / us / 1e3, 1),
                                  "min_GBs": round(B_min / us / 1e3, 1),
                                  "frac_fmt": round(B / us / 1e3 / peak, 4),
                                  "frac_min": round(B_min / us / 1e3 / peak, 4),
                                  "bitwise_equal_to_rgcsr32": ysum == ref, **extra}), flush=True)
                del h
        del csr


if __name__ == "__main__":
    main()
