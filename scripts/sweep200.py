"""BASELINE config 4: the synthetic 200-matrix sweep (10^4 - 10^7 rows, random /
banded / block classes; paper_1012_2270_b200.generators.sweep_case), fp32
and fp64, RgCSR G in {32, 64, 128, 256} vs Hybrid ELL+COO — the B200 analogue
of the paper's 1,596-matrix study.

For each matrix and precision: conversion + SpMV time (L2 flushed before
every timed launch), GFLOP/s, and a parity gate against the ORACLE
(oracle/oracle.c, pinned to the unmodified reference by
tests/test_oracle_pinned.py): every format's y must be bitwise the oracle's
spmv_csr y (all formats accumulate each row in the reference's order), and
for matrices up to --array-nnz entries the converted RgCSR (G = 32) and
Hybrid arrays must be bitwise the oracle's build_rgcsr / build_hybrid.  One
JSON line per (matrix, precision); `--summary` renders the statistics table.

    python scripts/sweep200.py [--first 0 --count 200 --max-rows 10000000]
    python scripts/sweep200.py --summary gpurun_out/sweep200.jsonl
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FORMATS = ("rgcsr32", "rgcsr64", "rgcsr128", "rgcsr256", "hybrid")


def timed(fn, stream, scratch, reps):
    import torch
    per = []
    for i in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            scratch.sum()  # read-only L2 flush (no dirty write-back in the timed kernel)
            a.record(stream)
            fn()
            b.record(stream)
        stream.synchronize()
        if i >= 2:
            per.append(a.elapsed_time(b))
    return statistics.median(per) * 1e3


def run(args):
    import torch

    import oracle as orc
    from paper_1012_2270_b200 import generators as gen
    from paper_1012_2270_b200 import spmvkit as sk
    from paper_1012_2270_b200._lib import lib
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    scratch = torch.zeros(64 << 20, dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(1234)
    for seed in range(args.first, args.first + args.count):
        t0 = time.perf_counter()
        name, m = gen.sweep_case(seed, max_rows=args.max_rows)
        t_gen = time.perf_counter() - t0
        csr = sk.build_csr(m, 8, stream=sp)
        xh = gen.random_vector(m.num_cols, seed + 1)
        om = orc.Csr(m.num_rows, m.num_cols, m.row_ptr, m.col, m.val)
        for prec in (8, 4):
            dt = torch.float64 if prec == 8 else torch.float32
            npdt = np.float64 if prec == 8 else np.float32
            x = torch.from_numpy(xh.astype(npdt)).cuda()
            c = csr if prec == 8 else sk.build_csr(m, 4, stream=sp)
            yo = orc.spmv_csr(om, xh.astype(npdt), prec)  # the oracle's y
            yref = torch.from_numpy(yo).cuda()
            ycsr = sk.spmv_csr(c, x)
            torch.cuda.synchronize()
            rec = {"seed": seed, "matrix": name, "rows": m.num_rows, "nnz": m.nnz, "prec": prec,
                   "gen_s": round(t_gen, 2), "parity": "oracle",
                   "csr_bitwise": bool(torch.equal(ycsr.view(torch.int64 if prec == 8 else
                                                             torch.int32),
                                                   yref.view(torch.int64 if prec == 8 else
                                                             torch.int32)))}
            arrays = m.nnz <= args.array_nnz
            iv = torch.int64 if prec == 8 else torch.int32
            for fmt in FORMATS:
                y = torch.empty(m.num_rows, dtype=dt, device="cuda")
                torch.cuda.synchronize()
                t = time.perf_counter()
                if fmt == "hybrid":
                    h = sk.build_hybrid(c, None, prec, stream=sp)
                    fn = L.spmvk_hybrid_spmv_f64 if prec == 8 else L.spmvk_hybrid_spmv_f32
                    fill = sk.fill_report(h).fill_percent
                else:
                    h = sk.build_rgcsr(c, int(fmt[5:]), prec, stream=sp)
                    fn = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
                    fill = sk.fill_report(h).fill_percent
                torch.cuda.synchronize()
                conv = (time.perf_counter() - t) * 1e3
                same_arrays = None
                if arrays and fmt in ("rgcsr32", "hybrid"):
                    got = h.to_host()
                    want = (orc.build_hybrid(om, h.slots_per_row, prec) if fmt == "hybrid"
                            else orc.build_rgcsr(om, 32, prec))
                    same_arrays = all(got[k].tobytes() == want[k].tobytes() for k in got
                                      if k in want)
                us = timed(lambda: fn(h._h, x.data_ptr(), m.num_cols, y.data_ptr(), m.num_rows, sp),
                           stream, scratch, args.reps)
                rec[fmt] = {"gflops": round(2 * m.nnz / us / 1e3, 2), "us": round(us, 2),
                            "fill": round(fill, 2), "convert_ms": round(conv, 2),
                            "bitwise": bool(torch.equal(y.view(iv), yref.view(iv))),
                            "arrays_bitwise": same_arrays}
                del h
            print(json.dumps(rec), flush=True)
            if prec == 4:
                del c
        del csr, m


def summary(path):
    recs = [json.loads(l) for l in open(path) if l.startswith("{")]
    out = ["# Synthetic sweep (BASELINE config 4): RgCSR vs Hybrid on one B200", ""]
    for prec in (4, 8):
        rs = [r for r in recs if r["prec"] == prec]
        if not rs:
            continue
        out += [f"## {'fp32' if prec == 4 else 'fp64'} — {len(rs)} matrices", "",
                "| format | mean GFLOP/s | max GFLOP/s | mean fill % | faster than Hybrid | "
                "mean speed ratio vs Hybrid | all y bitwise |", "|---|---|---|---|---|---|---|"]
        for fmt in FORMATS:
            g = [r[fmt]["gflops"] for r in rs]
            fill = [r[fmt]["fill"] for r in rs]
            bit = all(r[fmt]["bitwise"] for r in rs) and all(
                r.get("sampled_rows_bitwise", r.get("csr_bitwise", False)) for r in rs) and all(
                r[fmt].get("arrays_bitwise") is not False for r in rs)
            if fmt == "hybrid":
                out.append(f"| {fmt} | {statistics.mean(g):.1f} | {max(g):.1f} | "
                           f"{statistics.mean(fill):.1f} | — | — | {bit} |")
            else:
                faster = sum(r[fmt]["gflops"] > r["hybrid"]["gflops"] for r in rs)
                ratio = statistics.mean(r[fmt]["gflops"] / r["hybrid"]["gflops"] for r in rs)
                out.append(f"| {fmt} | {statistics.mean(g):.1f} | {max(g):.1f} | "
                           f"{statistics.mean(fill):.1f} | {100 * faster / len(rs):.1f}% | "
                           f"{ratio:.2f} | {bit} |")
        out.append("")
    print("\n".join(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--count", type=int, default=200)
    ap.add_argument("--max-rows", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--array-nnz", type=int, default=60_000_000,
                    help="compare converted arrays with the oracle up to this many entries")
    ap.add_argument("--summary")
    a = ap.parse_args()
    if a.summary:
        summary(a.summary)
    else:
        run(a)


if __name__ == "__main__":
    main()
