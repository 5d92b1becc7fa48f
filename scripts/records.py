"""SURVEY §8d output: one JSON record per (config, format, G, precision, P=1).

Fields: the reference's BenchRecord (spmvkit/bench.hpp:16-29: matrix_name,
format_name, group_size, precision, repetitions, nnz, median_seconds, gflops,
fill_percent, artificial_zeros, bytes, checksum) plus device, n_gpus, B_fmt,
B_min, achieved_GBps, roofline_frac_nominal (8.0 TB/s), roofline_frac_measured
(MEASURED_PEAKS copy), parity (bitwise | max rel err vs the reference CPU
y), cpu_gflops_1t, cpu_gflops_nt, cpu_cores, conversion times.

GPU: the repo's C-ABI (RgCSR G in {32,64,128,256}, Hybrid), L2 flushed with a
read before each timed launch when the matrix fits in 2x L2, else back-to-back
launches.  CPU: the UNMODIFIED reference spmv_rgcsr / spmv_hybrid
(oracle/_ref) as group-aligned row slabs on all host threads (nt) and the same
slabs run serially on one core (1t).  Test/measurement infrastructure only.

    python scripts/records.py [--workloads 5pt-1024,27pt-128,powerlaw-8M] [--out f.jsonl]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle as orc  # noqa: E402
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

NOMINAL_GBS = 8000.0
L2_BYTES = 126 << 20


def gpu_time_us(fn, stream, flush_buf, fits_l2, steps):
    if not fits_l2:
        total, per = bench.time_launches(fn, stream, steps, 5)
        return per * 1e3

    # cold launches: K x (read-only L2 flush; SpMV) minus K x flush, each timed
    # as one event region (per-launch events tick in ~2 us steps)
    def region(body):
        for _ in range(3):
            body()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            body()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / steps

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.sum()

    def both():
        flush()
        fn()
    return region(both) - region(flush)


def summary(path):
    """Markdown table of a records .jsonl (profiles/r01_records.md)."""
    rs = [json.loads(ln) for ln in open(path) if ln.startswith("{")]
    print("| matrix | prec | format | G | GPU us | GFLOP/s | B_fmt GB/s (frac of measured peak) "
          "| B_min GB/s | ncu DRAM MB / B_fmt MB | ncu L2 hit % | ncu sector eff. % | parity "
          "| CPU 1t GF/s | CPU nt GF/s | GPU / CPU-nt |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rs:
        us = r["median_seconds"] * 1e6
        bmin = r["B_min"] / r["median_seconds"] / 1e9
        prec = "f64" if r["precision"] == "double" else "f32"
        print(f"| {r['matrix_name']} | {prec} | {r['format_name']} | {r['group_size'] or ''} | "
              f"{us:.1f} | {r['gflops']:.0f} | {r['achieved_GBps']:.0f} "
              f"({r['roofline_frac_measured']:.3f}) | {bmin:.0f} | "
              f"{r.get('ncu_dram_bytes', 0) / 1e6:.0f} / {r['B_fmt'] / 1e6:.0f} | "
              f"{r.get('ncu_l2_hit_pct', 0):.1f} | {r.get('ncu_sector_efficiency_pct', 0):.1f} | "
              f"{r['parity']} | "
              f"{r['cpu_gflops_1t']:.2f} | {r['cpu_gflops_nt']:.2f} | "
              f"{r['gflops'] / r['cpu_gflops_nt']:.0f}x |")


def main():
    if len(sys.argv) == 3 and sys.argv[1] == "--summary":
        return summary(sys.argv[2])
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="5pt-1024,27pt-128,powerlaw-8M")
    ap.add_argument("--formats", default="csr,rgcsr32,rgcsr64,rgcsr128,rgcsr256,hybrid")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--out")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    peak, _ = bench.peaks()
    dev_name = torch.cuda.get_device_name(0)
    threads = os.cpu_count() or 1
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = open(args.out, "w") if args.out else None
    R = orc.R() if orc.ref_available() else None
    for wl in args.workloads.split(","):
        m = bench.host_csr(wl)  # the oracle's generators (oracle.Csr)
        rows, cols, rp, col, val = m.rows, m.cols, m.rp, m.col, m.val
        ref_m = orc.RefMatrix.from_csr(m) if R else None
        csr = bench.make_csr(wl)
        nnz = csr.nnz()
        xh = gen.random_vector(cols, 1)
        for prec in (8, 4):
            dt_np = np.float64 if prec == 8 else np.float32
            dt = torch.float64 if prec == 8 else torch.float32
            x_np = xh.astype(dt_np)
            x = torch.from_numpy(x_np).cuda()
            c_prec = csr if prec == 8 else sk.build_csr(
                sk.TripletMatrix(rows, cols, rp, col, val), 4)
            B_min = nnz * (prec + 4) + prec * (rows + cols)
            for fmt in args.formats.split(","):
                y = torch.empty(rows, dtype=dt, device="cuda")
                torch.cuda.synchronize()
                t = time.perf_counter()
                if fmt == "csr":  # the ingest format itself (spmv_csr, csr.hpp:41-53)
                    h = c_prec
                    B = nnz * (prec + 4) + 4 * (rows + 1) + prec * (rows + cols)
                    fn_c = L.spmvk_csr_spmv_f64 if prec == 8 else L.spmvk_csr_spmv_f32
                    G, ref_fmt, k1 = None, 0, -1
                    fr = None
                elif fmt == "hybrid":
                    h = sk.build_hybrid(c_prec, None, prec, stream=sp)
                    B = bench.hy_bytes(h.info, prec)
                    fn_c = L.spmvk_hybrid_spmv_f64 if prec == 8 else L.spmvk_hybrid_spmv_f32
                    G, ref_fmt, k1 = None, 2, h.slots_per_row
                    fr = sk.fill_report(h)
                else:
                    G = int(fmt[5:])
                    h = sk.build_rgcsr(c_prec, G, prec, stream=sp)
                    B = bench.rg_bytes(h.info, prec)
                    fn_c = L.spmvk_rgcsr_spmv_f64 if prec == 8 else L.spmvk_rgcsr_spmv_f32
                    ref_fmt, k1 = 1, -1
                    fr = sk.fill_report(h)
                torch.cuda.synchronize()
                conv_ms = (time.perf_counter() - t) * 1e3
                fn = lambda: fn_c(h._h, x.data_ptr(), cols, y.data_ptr(), rows, sp)  # noqa: E731
                us = gpu_time_us(fn, stream, flush_buf, B < 2 * L2_BYTES, args.steps)
                yg = y.cpu().numpy()
                rec = {"matrix_name": wl, "format_name": fmt if fmt == "csr" else
                       ("rgcsr" if G else "hybrid"),
                       "group_size": G, "precision": "double" if prec == 8 else "single",
                       "repetitions": args.steps, "nnz": nnz, "median_seconds": us * 1e-6,
                       "gflops": 2 * nnz / us / 1e3,
                       "fill_percent": fr.fill_percent if fr else 0.0,
                       "artificial_zeros": fr.artificial_zeros if fr else 0,
                       "bytes": (fr.bytes_double if prec == 8 else fr.bytes_single) if fr else
                       B - prec * (rows + cols),
                       "checksum": float(np.sum(yg, dtype=np.float64)),
                       "device": dev_name, "n_gpus": 1, "B_fmt": B, "B_min": B_min,
                       "achieved_GBps": B / us / 1e3,
                       "roofline_frac_nominal": B / us / 1e3 / NOMINAL_GBS,
                       "roofline_frac_measured": B / us / 1e3 / peak,
                       "convert_ms": conv_ms, "ell_width": k1 if not G else None,
                       "timing": "L2 flushed per launch (region of K flush+SpMV minus K flushes)" if B < 2 * L2_BYTES else "back-to-back"}
                if fmt != "csr":
                    del h
                if R:
                    hs = C.c_void_p()
                    t = time.perf_counter()
                    orc._rcheck(R.ref_slabs_build(ref_m.h, ref_fmt, G or 1, k1, prec, threads,
                                                  C.byref(hs)))
                    cpu_conv = time.perf_counter() - t
                    yc = np.empty(rows, dt_np)
                    runs = {"nt": R.ref_slabs_spmv, "1t": R.ref_slabs_spmv_serial}
                    cpu = {}
                    for k, f in runs.items():
                        f(hs, x_np.ctypes.data, yc.ctypes.data)
                        ts = []
                        for _ in range(args.cpu_reps if k == "nt" else 1):
                            t = time.perf_counter()
                            orc._rcheck(f(hs, x_np.ctypes.data, yc.ctypes.data))
                            ts.append(time.perf_counter() - t)
                        cpu[k] = 2 * nnz / statistics.median(ts) / 1e9
                    R.ref_slabs_free(hs)
                    same = yc.tobytes() == yg.tobytes()
                    rel = float(np.max(np.abs(yc.astype(np.float64) - yg) /
                                       np.maximum(np.abs(yc.astype(np.float64)), 1e-300)))
                    rec.update({"parity": "bitwise" if same else f"max_rel_err={rel:.3e}",
                                "cpu_gflops_1t": cpu["1t"], "cpu_gflops_nt": cpu["nt"],
                                "cpu_cores": threads, "cpu_build_s": cpu_conv,
                                "cpu_kind": "reference (oracle/_ref, unmodified spmv)"})
                else:
                    rec.update({"parity": None, "cpu_gflops_1t": None, "cpu_gflops_nt": None,
                                "cpu_cores": threads, "cpu_kind": "unavailable"})
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
            del c_prec
        del csr, ref_m


if __name__ == "__main__":
    main()
