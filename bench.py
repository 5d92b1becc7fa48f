#!/usr/bin/env python
"""bench.py — RgCSR SpMV GFLOP/s and achieved HBM GB/s (% of roofline) on B200.

Headline workload (BASELINE.json configs[1]): 3D 27-point stencil 128^3
(2,097,152 rows, 55,742,968 nnz), fp64, RgCSR group size 32.  One step = one
y = A x over the whole matrix (K2, one kernel launch) with A and x resident in
HBM; the 681 MB matrix exceeds the 126 MB L2, so no flush is needed between
steps (x, 16.8 MB, stays L2-resident as it would in an iterated solver).
fp32, Hybrid ELL+COO (the paper's comparison format) and the conversion time
ride along in ``variants``.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload 27pt-128|5pt-1024|powerlaw-8M|7pt-512]

N > 1 (torchrun, one rank per GPU): the workload defaults to BASELINE
configs[4] (7-point 512^3, the iterated product the north star asks to scale
near-linearly; strong scaling: the matrix is fixed), cut into group-aligned row
slabs (paper_1012_2270_b200.partition), each step is one slab SpMV with the
next x = y_k * 2^-4 computed in its epilogue, plus the exchange of x —
`--exchange fused` (default: the epilogue itself stores each x row into the
exchange window of every peer whose slab reads it, over NVLink, then a device
flag barrier; csrc/dist.cu), `halo` (NCCL point-to-point of only the column
ranges each slab reads) or `allgather` (NCCL, the whole vector) — timed as the
max over ranks; scaling "strong" (fixed matrix).

``--impl reference`` times the reference's own CPU spmv_rgcsr (oracle/_ref:
the unmodified reference compiled in place; the plain-C port when _ref is not
present) on the same workload with all host threads, as row slabs.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# x up and y down at once over PCIe Gen5 x16: 2 x 16 MiB in 344 us, measured with two
# concurrent copy-engine transfers (scripts/probes/pcie_sm.cu)
PCIE_BIDIR_GBS = 2 * 16 * 1048576 / 344e-6 / 1e9

METRIC = "SpMV GFLOP/s and achieved HBM GB/s (% of roofline) fp32/fp64 at 1/2/4/8 B200"

WORKLOADS = {
    # name: (kind, n or rows, group size, description)
    "27pt-128": ("stencil", 27, 128, "3D 27-point stencil 128^3 (BASELINE configs[1])"),
    "5pt-1024": ("stencil", 5, 1024, "2D 5-point Poisson 1024^2 (BASELINE configs[0])"),
    "7pt-512": ("stencil", 7, 512, "3D 7-point Poisson 512^3 (BASELINE configs[4])"),
    "powerlaw-8M": ("powerlaw", None, 8_000_000, "power-law rows, 8M (BASELINE configs[2])"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def committed_traffic(key):
    """ncu dram bytes per launch of the dominant kernel (profiles/traffic.json,
    written by scripts/ncu_summary.py from one `ncu --set full` capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def traffic_source():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get("_source")
    except Exception:
        return None


def measured_traffic(workload, timeout_s=120):
    """DRAM bytes (read + write) of ONE launch of the headline kernel, measured
    in this run by ncu in a child process (scripts/prof_k2.py: the same
    matrix, the auto K2 kernel, third launch), after -- and apart from -- the
    timed region; None when ncu is unavailable or fails (the committed capture
    is then reported)."""
    import csv
    import io
    import shutil
    import subprocess
    kind, a, b, _ = WORKLOADS[workload]
    if kind != "stencil" or shutil.which("ncu") is None or os.environ.get("CUDA_INJECTION64_PATH"):
        return None  # no ncu, or this process already runs under a profiler
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--csv",
           "--print-units", "base",
           "--clock-control", "none", "-k", "regex:rgcsr_spmv", "-s", "2", "-c", "1",
           sys.executable, os.path.join(ROOT, "scripts", "prof_k2.py"), "--case",
           f"{a}:{b}:32", "--prec", "8", "--variant", "auto", "--format", "rgcsr",
           "--launches", "3"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
        rows = [x for x in csv.reader(io.StringIO(r.stdout)) if len(x) > 10]
        hdr = rows[0]
        im, iv, ik = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Kernel Name")
        tot, kern = 0.0, None
        for x in rows[1:]:
            if x[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(x[iv].replace(",", ""))
                kern = x[ik]
        unit_scale = 1.0
        for x in rows[1:]:  # ncu reports bytes in the unit column (byte / Kbyte / Mbyte / Gbyte)
            if x[im] == "dram__bytes_read.sum":
                u = x[hdr.index("Metric Unit")]
                unit_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        if not tot:
            return None
        return {"bytes": tot * unit_scale, "kernel": (kern or "")[:120]}
    except Exception:  # noqa: BLE001 -- the committed capture is reported instead
        return None


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b and b != 0x1]}


# ---------------------------------------------------------------- inputs
def make_csr(workload):
    """Device CSR of the workload (stencils generated directly in HBM)."""
    from paper_1012_2270_b200 import generators as gen
    from paper_1012_2270_b200 import spmvkit as sk
    kind, a, b, _ = WORKLOADS[workload]
    if kind == "stencil":
        return sk.CsrMatrix.stencil(a, b)
    return sk.build_csr(gen.powerlaw(b, 7))


def host_csr(workload):
    """Host CSR of the same workload for the CPU reference, made by the ORACLE's
    generators (oracle/oracle.c, test infrastructure), so the reference arm
    never loads the product library."""
    import oracle as orc
    kind, a, b, _ = WORKLOADS[workload]
    return orc.stencil(a, b) if kind == "stencil" else orc.powerlaw(b, 7)


GOLDEN_KEY = {"27pt-128": "27pt_128", "5pt-1024": "5pt_1024", "powerlaw-8M": "powerlaw_8M"}


def golden_checksum(workload):
    """Sequential sum of the reference's fp64 y (tests/golden/shapes.json,
    generated from the unmodified reference by oracle/make_golden.py), or None."""
    key = GOLDEN_KEY.get(workload)
    if key is None:
        return None
    with open(os.path.join(ROOT, "tests", "golden", "shapes.json")) as f:
        return json.load(f)[key]["checksum_reference"]


L2_NOTE = {
    "27pt-128": "inputs larger than L2: 681 MB matrix vs 126 MB L2 (no flush); x stays L2-resident",
    "5pt-1024": "matrix (84 MB) fits in the 126 MB L2: back-to-back launches re-read it from L2",
    "7pt-512": "inputs larger than L2: 13.4 GB matrix (no flush)",
    "powerlaw-8M": "inputs larger than L2: 6.9 GB matrix (no flush)",
}


def bench_config(workload, n_gpus, exchange="fused"):
    """The `config` dict both arms print (identical for the same workload / N)."""
    cfg = {"workload": workload, "description": WORKLOADS[workload][3], "format": "rgcsr",
           "group_size": 32, "precision": "fp64", "l2": L2_NOTE[workload]}
    if n_gpus == 1:
        cfg["parallelism"] = "single GPU"
    else:
        cfg["parallelism"] = f"row-slab x{n_gpus}, iterated x <- (A x) * 2^-4, {exchange} x exchange"
    return cfg


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- timing helpers
# Read-only streaming bandwidth measured on B200 (float4 lanes, full occupancy;
# scripts/probes/ld_width.cu, profiles/r01_ld_width.md).
READ_STREAM_GBS = 7164.4


def time_launches(fn, stream, steps, warmup):
    """Warm up, then time `steps` back-to-back launches with CUDA events on
    `stream` around the whole region (synchronize on both sides).  Events
    between launches would add their own gaps (~3 us per launch on the 27-pt
    headline), so the per-launch duration is the region time / steps.
    Returns (total_ms, per-launch ms)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
        for _ in range(steps):
            fn()
        t1.record(stream)
    torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    return total, total / steps


def rg_bytes(info, sv):
    """Algorithmic bytes per SpMV: FillReport bytes + x read + y write."""
    fr = info.bytes_double if sv == 8 else info.bytes_single
    return fr + sv * (info.num_cols + info.num_rows)


def hy_bytes(info, sv):
    fr = info.bytes_double if sv == 8 else info.bytes_single
    return fr + sv * (info.num_cols + info.num_rows)


# ---------------------------------------------------------------- CPU reference
def cpu_reference(workload, sample_reps, threads=None, G=32, prec=8, budget_s=12.0):
    """Times the reference CPU spmv_rgcsr on the host cores, twice: on all
    host threads (group-aligned row slabs, one std::thread each, running the
    unchanged reference template; bitwise equal to one thread) and on ONE core
    (the same slabs in sequence: the reference's own single-threaded SpMV).
    kind 'reference' = the unmodified reference compiled in place
    (oracle/_ref), else the plain-C port (oracle/oracle.c, one core).  Each
    leg is a bounded sample of about `budget_s` seconds."""
    import ctypes as C
    import oracle as orc
    m = host_csr(workload)
    rows, cols, nnz = m.rows, m.cols, m.nnz
    threads = threads or len(os.sched_getaffinity(0)) or 1
    dt = np.float64 if prec == 8 else np.float32
    x = orc.random_vector(cols, 1).astype(dt)
    y = np.empty(rows, dt)

    def timed(run):
        t = time.perf_counter()
        run()
        first = time.perf_counter() - t
        reps = max(3, min(sample_reps, int(budget_s / max(first, 1e-6))))
        times = []
        for _ in range(reps):
            t = time.perf_counter()
            run()
            times.append(time.perf_counter() - t)
        return statistics.median(times), reps

    if orc.ref_available():
        r = orc.RefMatrix.from_csr(m)
        del m
        h = C.c_void_p()
        orc._rcheck(orc.R().ref_slabs_build(r.h, 1, G, -1, prec, threads, C.byref(h)))
        del r
        med_nt, reps_nt = timed(lambda: orc._rcheck(
            orc.R().ref_slabs_spmv(h, x.ctypes.data, y.ctypes.data)))
        med_1t, reps_1t = timed(lambda: orc._rcheck(
            orc.R().ref_slabs_spmv_serial(h, x.ctypes.data, y.ctypes.data)))
        orc.R().ref_slabs_free(h)
        kind, used = "reference", threads
    else:
        a = orc.build_rgcsr(m, G, prec)
        del m

        def run():
            y[:] = orc.spmv_rgcsr(a, x)[0]
        med_1t, reps_1t = timed(run)
        med_nt, reps_nt, kind, used = med_1t, reps_1t, "port", 1
    gf = lambda t: 2.0 * nnz / t / 1e9  # noqa: E731
    what = "unmodified reference spmv_rgcsr" if kind == "reference" else "plain-C port"
    return {"value": gf(med_nt), "unit": "GFLOP/s", "cores": used, "kind": kind,
            "sample": (f"median of {reps_nt} full SpMVs of {workload} "
                       f"({WORKLOADS[workload][3]}), RgCSR G={G}, "
                       f"{'fp64' if prec == 8 else 'fp32'}, {used} row-slab threads of the {what}; "
                       f"1-core leg: median of {reps_1t}"),
            "value_1core": gf(med_1t), "seconds_per_spmv": med_nt,
            "seconds_per_spmv_1core": med_1t, "cpu_model": cpu_model(),
            "host_threads": os.cpu_count(), "checksum": float(np.cumsum(y.astype(np.float64))[-1])}


def cpu_baseline_block(c):
    return {k: c[k] for k in ("value", "unit", "cores", "kind", "sample", "value_1core",
                              "cpu_model", "host_threads")}


# ---------------------------------------------------------------- K1 rate
def convert_rate(csr, stream, peak, G=32, reps=5):
    """Wall time of the device CSR -> RgCSR converter (spmvk_rgcsr_build: the
    layout kernels, one 24-byte readback, the scatter), median of `reps`
    builds after a warm one, against its algorithmic bytes: the CSR read
    (row pointers, columns, values) and the RgCSR arrays written."""
    import torch
    from paper_1012_2270_b200 import spmvkit as sk
    sk.build_rgcsr(csr, G, 8, stream=stream.cuda_stream)
    times, a = [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        a = sk.build_rgcsr(csr, G, 8, stream=stream.cuda_stream)
        times.append(time.perf_counter() - t)
        del a
    a = sk.build_rgcsr(csr, G, 8, stream=stream.cuda_stream)
    nnz, rows = a.nnz(), a.num_rows
    bytes_ = 4 * (rows + 1) + 12 * nnz + a.info.bytes_double
    med = statistics.median(times)
    return {"ms": med * 1e3, "bytes": bytes_, "gbs": bytes_ / med / 1e9,
            "frac_of_peak": bytes_ / med / 1e9 / peak,
            "what": "spmvk_rgcsr_build G=32 fp64, host wall time incl. its readback and "
                    "allocation, median of %d; bytes = CSR read + RgCSR written" % reps}


# ---------------------------------------------------------------- config 3
def powerlaw_block(args, peak):
    """BASELINE configs[2] at full size (8M rows, power-law lengths, 128 M nnz),
    fp64: RgCSR G = 32 in the original and the descending row order, and the
    paper's Hybrid ELL+COO in both, each timed like the headline (back-to-back
    launches, CUDA events on the launching stream).  Roofline on B_min
    (format-independent: every nonzero's value + column once, x and y) and on
    the format's own bytes.  Parity gate: the sequential sum of every y (the
    descending ones mapped back to the original rows) must equal the unmodified
    reference's checksum (tests/golden/shapes.json)."""
    import torch
    from paper_1012_2270_b200 import generators as gen
    from paper_1012_2270_b200 import spmvkit as sk
    from paper_1012_2270_b200._lib import lib
    L = lib()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    t0 = time.perf_counter()
    csr = make_csr("powerlaw-8M")
    desc, pmap = sk.apply_descending_permutation(csr)
    reorder = []  # f1: the device descending row reordering (sort + row gather)
    for _ in range(3):
        torch.cuda.synchronize()
        tr = time.perf_counter()
        d2, _ = sk.apply_descending_permutation(csr)
        torch.cuda.synchronize()
        reorder.append((time.perf_counter() - tr) * 1e3)
        del d2
    perm = sk.Permutation(pmap)
    rows, nnz = csr.num_rows, csr.nnz()
    x = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda()
    y = torch.empty(rows, dtype=torch.float64, device="cuda")
    golden = golden_checksum("powerlaw-8M")
    b_min = nnz * 12 + 8 * (rows + csr.num_cols)
    out = {"workload": "powerlaw-8M", "description": WORKLOADS["powerlaw-8M"][3],
           "precision": "fp64", "nnz": nnz, "b_min": b_min,
           "reference_checksum": golden,
           "reorder_ms": statistics.median(reorder),
           "reorder_what": "apply_descending_permutation (stable device sort of the row "
                           "lengths + row gather of the CSR arrays), host wall time, median of 3"}
    steps = max(5, min(args.steps, 50))
    for label, mat, fmt, reordered in (("rgcsr_g32_original", csr, "rg", False),
                                       ("rgcsr_g32_descending", desc, "rg", True),
                                       ("hybrid_original", csr, "hy", False),
                                       ("hybrid_descending", desc, "hy", True)):
        if fmt == "rg":
            h = sk.build_rgcsr(mat, 32, 8, stream=sp)
            fn, bf = L.spmvk_rgcsr_spmv_f64, rg_bytes(h.info, 8)
        else:
            h = sk.build_hybrid(mat, None, 8, stream=sp)
            fn, bf = L.spmvk_hybrid_spmv_f64, hy_bytes(h.info, 8)
        _, km = time_launches(lambda: fn(h._h, x.data_ptr(), h.num_cols, y.data_ptr(), rows, sp),
                              stream, steps, max(3, args.warmup))
        yy = sk.permute_vector(perm, y, inverse=True) if reordered else y
        ysum = float(np.cumsum(yy.cpu().numpy())[-1])
        if golden is not None and ysum != golden:
            raise SystemExit(f"parity gate failed: powerlaw {label} checksum {ysum!r} != "
                             f"reference {golden!r}")
        out[label] = {"kernel_us": km * 1e3, "gflops": 2.0 * nnz / (km * 1e-3) / 1e9,
                      "frac_b_min": b_min / (km * 1e-3) / 1e9 / peak,
                      "format_bytes": bf, "frac_format_bytes": bf / (km * 1e-3) / 1e9 / peak,
                      "checksum": ysum}
        del h
    out["parity"] = "every checksum == the unmodified reference's (descending y mapped back)"
    out["setup_s"] = time.perf_counter() - t0
    return out


# ---------------------------------------------------------------- scaling anchor
def scale_anchor(args, peak):
    """BASELINE configs[4] at N = 1: 7-point 512^3 fp64 (938 M nnz, 13.4 GB of
    RgCSR), the matrix the N > 1 scaling runs shard.  One step is the
    iterated product's x <- (A x) * 2^-4 (the scaled K2 epilogue), 100 steps
    as the config names, timed like the headline; the iterate's bit checksum
    must equal the unmodified reference's (tests/golden/iterate_7pt512.json,
    oracle/make_iterate_golden.py) and the device CSR kernel's iterate."""
    import torch
    from paper_1012_2270_b200 import generators as gen
    from paper_1012_2270_b200 import spmvkit as sk
    from paper_1012_2270_b200._lib import lib
    L = lib()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    t = time.perf_counter()
    csr = sk.CsrMatrix.stencil(7, 512, stream=sp)
    a = sk.build_rgcsr(csr, 32, 8, stream=sp)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t
    n = a.num_rows
    x0 = torch.from_numpy(gen.random_vector(n, 1)).cuda()
    xs = [x0.clone(), torch.empty_like(x0)]
    y = torch.empty_like(x0)
    cur = [0]

    def step():
        xa, xb = xs[cur[0]], xs[1 - cur[0]]
        L.spmvk_rgcsr_spmv_scaled_f64(a._h, xa.data_ptr(), n, y.data_ptr(), n, xb.data_ptr(),
                                      0.0625, sp)
        cur[0] = 1 - cur[0]
    iters = 100
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    xs[0].copy_(x0)
    cur[0] = 0
    clk = ClockSampler(0)
    with clk:
        total, per = time_launches(step, stream, iters, 0)
    bits = int(xs[cur[0]].view(torch.int64).sum().item())
    # the same 100 iterations through the device CSR kernel (spmv_csr) + scale
    xc = x0.clone()
    yc = torch.empty_like(x0)
    for _ in range(iters):
        sk._check(L.spmvk_csr_spmv_f64(csr._h, xc.data_ptr(), n, yc.data_ptr(), n, sp))
        with torch.cuda.stream(stream):
            torch.mul(yc, 0.0625, out=xc)
    torch.cuda.synchronize()
    bits_csr = int(xc.view(torch.int64).sum().item())
    with open(os.path.join(ROOT, "tests", "golden", "iterate_7pt512.json")) as f:
        bits_ref = int(json.load(f)["bits_sum_int64_after"][str(iters)])
    B = rg_bytes(a.info, 8)
    nnz = a.nnz()
    out = {"workload": "7pt-512", "description": WORKLOADS["7pt-512"][3], "n_gpus": 1,
           "iterations": iters, "ms_per_step": per,
           "gflops": 2.0 * nnz / (per * 1e-3) / 1e9,
           "roofline": {"achieved": B / (per * 1e-3) / 1e9, "peak": peak,
                        "frac": B / (per * 1e-3) / 1e9 / peak, "bytes_per_launch": B},
           "build_s": t_build, "x_bits_checksum": bits, "reference_bits": bits_ref,
           "parity": ("bitwise == the unmodified reference's iterate and the device spmv_csr "
                      "iterate" if bits == bits_csr == bits_ref else "MISMATCH"),
           "sm_mhz": clk.summary().get("sm_mhz")}
    del a, csr, xs, y, xc, yc
    torch.cuda.empty_cache()
    if not bits == bits_csr == bits_ref:
        raise SystemExit(f"parity gate failed: 7pt-512 iterate bits {bits} (CSR kernel "
                         f"{bits_csr}, reference {bits_ref})")
    return out


# ---------------------------------------------------------------- arms
def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = args.steps
    n = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    base = cpu_reference(args.workload, max(steps, 1))
    golden = golden_checksum(args.workload)
    if golden is not None and base["checksum"] != golden:
        raise SystemExit(f"reference checksum {base['checksum']!r} != golden {golden!r}")
    line = {"metric": METRIC, "value": base["value"], "unit": "GFLOP/s", "n_gpus": n,
            "steps": steps, "warmup": args.warmup,
            "ms_per_step": base["seconds_per_spmv"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.workload, n, args.exchange),
            "impl": "reference", "cpu_baseline": cpu_baseline_block(base),
            "e2e": {"value": base["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "checksum": base["checksum"]}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    from paper_1012_2270_b200 import spmvkit as sk
    from paper_1012_2270_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.distributed:
        from paper_1012_2270_b200 import partition
        return partition.bench_distributed(
            args, METRIC, WORKLOADS, ClockSampler, peaks(), rg_bytes,
            config_fn=lambda n, ex: bench_config(args.workload, n, ex),
            cpu_fn=lambda: cpu_baseline_block(cpu_reference(args.workload, args.cpu_reps)),
            traffic=committed_traffic(f"{args.workload}/rgcsr_f64_g32"))

    torch.cuda.set_device(0)
    assert lib().spmvk_init(0) == 0, sk._lib.last_error()
    peak, peak_kind = peaks()
    stream = torch.cuda.Stream()
    G = 32

    t = time.perf_counter()
    csr = make_csr(args.workload)
    torch.cuda.synchronize()
    t_csr = time.perf_counter() - t
    t = time.perf_counter()
    a = sk.build_rgcsr(csr, G, 8, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    t_conv = time.perf_counter() - t
    nnz = a.nnz()
    from paper_1012_2270_b200 import generators as gen
    xh = gen.random_vector(a.num_cols, 1)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty(a.num_rows, dtype=torch.float64, device="cuda")
    sp = stream.cuda_stream
    L = lib()

    def step():
        L.spmvk_rgcsr_spmv_f64(a._h, x.data_ptr(), a.num_cols, y.data_ptr(), a.num_rows, sp)

    clocks = ClockSampler(0)
    torch.cuda.synchronize()
    with clocks:
        total_ms, kern_ms = time_launches(step, stream, args.steps, args.warmup)
    ms = total_ms / args.steps
    B = rg_bytes(a.info, 8)
    achieved = B / (kern_ms * 1e-3) / 1e9
    value = 2.0 * nnz / (ms * 1e-3) / 1e9

    # parity gate on the measured output: the sequential sum of y must equal
    # the unmodified reference's (tests/golden/shapes.json) bit for bit
    ysum = float(np.cumsum(y.cpu().numpy())[-1])
    golden = golden_checksum(args.workload)
    if golden is not None and ysum != golden:
        raise SystemExit(f"parity gate failed: GPU checksum {ysum!r} != reference {golden!r}")

    # ---- e2e: reference-facing C-ABI span overload with pinned HOST buffers
    if args.e2e_host == "torch":  # A/B: torch's pinned host allocator
        xpin = torch.from_numpy(xh).pin_memory()
        ypin = torch.empty(a.num_rows, dtype=torch.float64).pin_memory()
    else:  # the library's page-locked 2 MB-page host buffers (spmvk_host_alloc)
        xpin, ypin = sk.host_array(a.num_cols), sk.host_array(a.num_rows)
        xpin[:] = xh
        xpin, ypin = torch.from_numpy(xpin), torch.from_numpy(ypin)
    e2e_steps = max(3, min(args.steps, 50))
    for _ in range(max(args.warmup, 10)):  # untimed: graph capture, first PCIe traffic
        L.spmvk_rgcsr_spmv_host_f64(a._h, xpin.data_ptr(), a.num_cols, ypin.data_ptr(),
                                    a.num_rows, None)
    torch.cuda.synchronize()
    # five rounds of back-to-back calls, the median round reported: a PCIe /
    # host-memory hiccup from another tenant of the host moves one round,
    # not the number (every round is in the line)
    e2e_rounds = []
    per_round = max(3, e2e_steps // 5)
    for _ in range(5):
        t = time.perf_counter()
        for _ in range(per_round):
            rc = L.spmvk_rgcsr_spmv_host_f64(a._h, xpin.data_ptr(), a.num_cols,
                                             ypin.data_ptr(), a.num_rows, None)
        torch.cuda.synchronize()
        e2e_rounds.append((time.perf_counter() - t) / per_round)
    e2e_s = statistics.median(e2e_rounds)
    assert rc == 0, sk._lib.last_error()
    assert float(np.cumsum(ypin.numpy())[-1]) == ysum

    # ---- variants: fp32 RgCSR, Hybrid fp64/fp32 (same timing method)
    variants = {}
    for label, builder, prec in (("rgcsr_f32_g32", "rg", 4), ("hybrid_f64", "hy", 8),
                                 ("hybrid_f32", "hy", 4), ("csr_f64", "csr", 8)):
        dt = torch.float64 if prec == 8 else torch.float32
        xv = x.to(dt)
        yv = torch.empty(a.num_rows, dtype=dt, device="cuda")
        tt = time.perf_counter()
        if builder == "rg":
            h = sk.build_rgcsr(csr, G, prec, stream=sp)
            fn = L.spmvk_rgcsr_spmv_f32
            Bv = rg_bytes(h.info, prec)
        elif builder == "csr":  # the ingest format's own SpMV (spmv_csr)
            h = csr
            fn = L.spmvk_csr_spmv_f64
            Bv = nnz * 12 + 4 * (a.num_rows + 1) + 8 * (a.num_rows + a.num_cols)
        else:
            h = sk.build_hybrid(csr, None, prec, stream=sp)
            fn = L.spmvk_hybrid_spmv_f64 if prec == 8 else L.spmvk_hybrid_spmv_f32
            Bv = hy_bytes(h.info, prec)
        torch.cuda.synchronize()
        tconv = time.perf_counter() - tt
        vclk = ClockSampler(0)
        with vclk:
            _, pv = time_launches(lambda: fn(h._h, xv.data_ptr(), h.num_cols, yv.data_ptr(),
                                             h.num_rows, sp), stream, args.steps, args.warmup)
        km = pv
        variants[label] = {"gflops": 2.0 * nnz / (km * 1e-3) / 1e9, "kernel_us": km * 1e3,
                           "bytes": Bv, "achieved_gbs": Bv / (km * 1e-3) / 1e9,
                           "frac_of_peak": Bv / (km * 1e-3) / 1e9 / peak,
                           "first_build_ms": tconv * 1e3,
                           "sm_mhz": vclk.summary().get("sm_mhz")}
        if builder == "hy":
            variants[label]["ell_width"] = h.slots_per_row
            variants[label]["coo_nnz"] = h.coo_nnz()
        if builder != "csr":
            del h

    anchor = scale_anchor(args, peak) if args.workload != "7pt-512" else None
    plaw = powerlaw_block(args, peak) if args.powerlaw else None
    cpu = cpu_reference(args.workload, args.cpu_reps)
    if cpu["checksum"] != ysum:
        raise SystemExit(f"parity gate failed: GPU checksum {ysum!r} != CPU reference "
                         f"{cpu['checksum']!r}")
    traffic = committed_traffic(f"{args.workload}/rgcsr_f64_g32")
    t_src = traffic_source()
    live = measured_traffic(args.workload) if args.traffic_live else None
    if live:
        traffic = live["bytes"]
        t_src = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum in a child process "
                 "of this run, one launch of " + live["kernel"])
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.workload, 1, args.exchange),
        "shape": {"nnz": nnz, "rows": a.num_rows, "slots": a.slot_count()},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "bytes_per_launch": B, "kernel_us": kern_ms * 1e3,
                     "traffic": traffic,
                     "traffic_source": t_src,
                     # the peak above is a copy (half writes); SpMV traffic is ~98 % reads
                     "read_stream_peak": READ_STREAM_GBS,
                     "frac_read_stream": achieved / READ_STREAM_GBS,
                     "kernel": "rgcsr_spmv_grp (K2 auto): with x[0] finite it does not read "
                               "row_lengths (4 B/row of B_fmt), so DRAM traffic (ncu) is "
                               "~2 % below bytes_per_launch"},
        "cpu_baseline": cpu_baseline_block(cpu),
        "e2e": {"value": 2.0 * nnz / e2e_s / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": 8 * a.num_cols, "d2h_bytes_per_step": 8 * a.num_rows,
                "ms_per_step": e2e_s * 1e3,
                "rounds_ms_per_step": [round(v * 1e3, 4) for v in e2e_rounds],
                "timing": f"median of 5 rounds x {per_round} back-to-back calls",
                "pcie_gbs": 8 * (a.num_cols + a.num_rows) / e2e_s / 1e9,
                "pcie_peak_gbs": PCIE_BIDIR_GBS,
                "frac_pcie": 8 * (a.num_cols + a.num_rows) / e2e_s / 1e9 / PCIE_BIDIR_GBS,
                "pcie_peak_source": "16 MB up + 16 MB down as two concurrent copy-engine "
                                    "transfers, 344 us (scripts/probes/pcie_sm.cu, "
                                    "profiles/r01_e2e_pipeline.md)",
                "path": "spmvk_rgcsr_spmv_host_f64 (pinned host x,y; H2D + SpMV + D2H)",
                "host_buffers": ("spmvk_host_alloc (page-locked, 2 MB pages)"
                                 if args.e2e_host == "spmvk" else "torch pin_memory")},
        "gpu_launches": args.steps,
        "clocks": clocks.summary(),
        "checksum": ysum,
        "parity": ("checksum == the unmodified reference's (CPU run above and the golden)"
                   if golden is not None else "checksum == the CPU reference run above"),
        "first_call_ms": {"csr_ingest": t_csr * 1e3, "rgcsr_g32_f64": t_conv * 1e3,
                          "note": "the first build of each array in this process: includes "
                                  "cudaMalloc + first-touch page mapping of the handle arrays; "
                                  "the steady-state converter rate is `convert`"},
        "convert": convert_rate(csr, stream, peak),
        "variants": variants,
        "scale_anchor": anchor,
        "config3_powerlaw": plaw,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: 27pt-128 (configs[1]) on one GPU; 7pt-512 (configs[4], the "
                         "iterated, row-slab sharded config) under torchrun with N > 1")
    ap.add_argument("--cpu-reps", type=int, default=10)
    ap.add_argument("--e2e-host", choices=["spmvk", "torch"], default="spmvk",
                    help="host x / y buffers of the e2e leg: spmvk_host_alloc (default) or "
                         "torch pin_memory")
    ap.add_argument("--no-traffic-live", dest="traffic_live", action="store_false",
                    help="report the committed ncu capture instead of measuring the headline "
                         "kernel's DRAM bytes with ncu in a child process")
    ap.add_argument("--no-powerlaw", dest="powerlaw", action="store_false",
                    help="skip the BASELINE configs[2] (power-law 8M) block of the N = 1 line")
    ap.add_argument("--distributed", action="store_true",
                    help="use the row-slab + NCCL path even at world size 1 (under torchrun)")
    ap.add_argument("--exchange", default="fused", choices=["allgather", "halo", "fused"],
                    help="x exchange of the distributed iterated SpMV: NCCL all-gather, NCCL "
                         "halo send/recv, or fused (SpMV epilogue stores into peer windows "
                         "over NVLink + device barrier)")
    args = ap.parse_args()
    if args.workload is None:
        multi = int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.gpus > 1
        args.workload = "7pt-512" if multi else "27pt-128"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
