"""ncu-backed replacement of the reference's `spmvkit simulate` (
reference: tools/main.cpp:262-328 run_simulate, schema at :304-317, models
in src/memsim.cpp:141-199).

The reference models a GTX 280: it replays the RgCSR/CSR/ELL address streams
per half-warp, counts 128-byte segment transactions per array and runs an LRU
texture-cache simulation (src/memsim.cpp:92-199, tools/main.cpp:274-317).
Here the same report is filled from REAL counters of the B200 kernel: one
`ncu --section SourceCounters` pass over one SpMV launch gives, per SASS
memory instruction, the L2 sectors it touched ("L2 Theoretical Sectors
Global") and the ideal count for its bytes; instructions are attributed to
arrays by their cache operator and width:

  values   LDG.NA (no-allocate) of the scalar width     (RgCSR / ELL slots)
  columns  LDG.NA 32-bit                                 (fp32: values and columns
           have identical index patterns, so the NA.32 sectors split evenly)
  x        LDG (L1-allocating, read-only) of the scalar width
  output   STG
  (row lengths / group pointers: the remaining LDG.32, and every warp-uniform
   load -- one sector per executed warp instruction -- reported as "metadata")

and the x "cache" is the L1: hits / misses of the global-load lookups
(`l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_{hit,miss}`; the NA
slot loads never allocate, so the hits are x's).  Units are 32-byte sectors,
B200's transaction granularity, instead of the model's 128-byte segments.

Library entry: ``simulate(...) -> dict`` (the reference's JSON document);
command line, like the reference's ``spmvkit simulate``:

    python -m paper_1012_2270_b200.simulate --case 27:128 --format rgcsr \
        --group-size 32 --precision double [--ordering descending] [--out report.json]

(needs ncu and a GPU: the counters come from one profiled SpMV launch).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KERNELS = {"rgcsr": "rgcsr_spmv", "ellpack": "hybrid_spmv|hybrid_ell", "csr": "csr_spmv|hybrid_spmv_dyn"}


def child(a):
    import torch

    from . import generators as gen
    from . import spmvkit as sk
    from ._lib import lib
    torch.cuda.set_device(0)
    assert lib().spmvk_init(0) == 0
    prec = 8 if a.precision == "double" else 4
    csr = load(a, sk, gen)
    if a.ordering == "descending":  # tools/main.cpp apply_ordering (reorder.cpp:35-61)
        csr = sk.apply_descending_permutation(csr)[0]
    if prec == 4:
        rp, col, val = csr.to_host()
        csr = sk.build_csr(sk.TripletMatrix(csr.num_rows, csr.num_cols, rp, col, val), 4)
    if a.format == "rgcsr":
        h = sk.build_rgcsr(csr, a.group_size, prec)
        fn = sk.spmv_rgcsr
        az = sk.fill_report(h).artificial_zeros
    elif a.format == "ellpack":  # Hybrid at K1 = max row length is plain ELLPACK
        h = sk.build_hybrid(csr, csr.row_length_range()[0], prec)
        fn = sk.spmv_hybrid
        az = sk.fill_report(h).artificial_zeros
    else:
        h, fn, az = csr, sk.spmv_csr, 0
    dt = torch.float64 if prec == 8 else torch.float32
    x = torch.from_numpy(gen.random_vector(csr.num_cols, a.seed)).cuda().to(dt)
    fn(h, x)  # ONE SpMV: every kernel it launches is profiled (ncu flushes caches)
    torch.cuda.synchronize()
    with open(a.meta, "w") as f:
        json.dump({"nnz": csr.nnz(), "artificial_zeros": az, "rows": csr.num_rows}, f)


def load(a, sk, gen):
    if a.mtx:
        return sk.load_matrix_market(a.mtx)
    kind, n = (int(v) for v in a.case.split(":"))
    if kind == 0:
        return sk.build_csr(gen.powerlaw(n, 7))
    return sk.CsrMatrix.stencil(kind, n)


def classify(rows, sv, meta_sectors=0):
    """Sum per-instruction sectors over every profiled kernel's section of the
    `--page source --csv` output (each section: a "Kernel Name" row, a header
    row, then one row per SASS instruction)."""
    out = {k: [0, 0] for k in ("values", "columns", "x", "output", "metadata", "na32")}
    ix, ix_inst, i = None, None, 0
    while i < len(rows):
        r = rows[i]
        i += 1
        if r and r[0] == "Kernel Name":
            h = rows[i]
            i += 1
            ix = {k: h.index(k) for k in ("Source", "Access Operation", "Access Size",
                                          "L2 Theoretical Sectors Global",
                                          "L2 Theoretical Sectors Global Ideal")}
            ix_inst = h.index("Instructions Executed") if "Instructions Executed" in h else None
            continue
        if ix is None or len(r) <= max(ix.values()):
            continue
        op = r[ix["Access Operation"]]
        if op not in ("Load", "Store"):
            continue
        src = r[ix["Source"]]
        size = int(r[ix["Access Size"]] or 0)
        sec = int(float(r[ix["L2 Theoretical Sectors Global"]] or 0))
        ideal = int(float(r[ix["L2 Theoretical Sectors Global Ideal"]] or 0))
        if op == "Store":
            key = "output"
        elif "LDG" not in src:
            continue
        elif ix_inst is not None and 0 < sec <= int(float(r[ix_inst] or 0)):
            # warp-uniform loads (one sector per warp instruction): the group
            # pointers and tile bounds, never a slot stream or an x gather
            key = "metadata"
        elif ".NA" in src:  # streamed slots (L1 no-allocate)
            if sv == 8:
                key = "values" if size == 64 else "columns"
            else:
                key = "na32"
        elif size == 8 * sv:
            key = "x"
        else:
            key = "metadata"
        out[key][0] += sec
        out[key][1] += ideal
    if sv == 4:  # fp32: values and columns share one index pattern and width
        s, i = out.pop("na32")
        out["values"] = [s // 2, i // 2]
        out["columns"] = [s - s // 2, i - i // 2]
        # the 32-bit L1-allocating loads are x gathers AND the per-row metadata
        # (row length, group pointer); move the metadata's coalesced sector count
        meta = min(meta_sectors, out["x"][0])
        out["x"] = [out["x"][0] - meta, max(0, out["x"][1] - meta)]
        out["metadata"] = [out["metadata"][0] + meta, out["metadata"][1] + meta]
    else:
        out.pop("na32")
    return out


def simulate(case: str = "27:128", mtx: str = None, format: str = "rgcsr",
             group_size: int = 32, precision: str = "double", ordering: str = "none",
             seed: int = 1, ncu: str = "ncu") -> dict:
    """The reference's `simulate` report (tools/main.cpp:304-317) for one SpMV
    of the matrix (``mtx`` Matrix Market path, or ``case`` "kind:n": 5/7/27-point
    stencil, 0 = power-law rows), filled from ncu counters of the B200 kernel."""
    if format not in KERNELS:
        raise ValueError(f"simulate supports csr, ellpack and rgcsr, not '{format}'")
    if precision not in ("single", "double"):
        raise ValueError(f"unknown precision '{precision}'")
    if ordering not in ("none", "descending"):
        raise ValueError(f"unknown ordering '{ordering}'")
    sv = 8 if precision == "double" else 4
    with tempfile.TemporaryDirectory() as d:
        rep, meta = os.path.join(d, "sim"), os.path.join(d, "meta.json")
        argv = [sys.executable, "-m", "paper_1012_2270_b200.simulate", "--child", "--meta", meta,
                "--format", format, "--group-size", str(group_size), "--precision", precision,
                "--seed", str(seed), "--ordering", ordering] + (
                    ["--mtx", mtx] if mtx else ["--case", case])
        env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
        subprocess.run([ncu, "--section", "SourceCounters", "--import-source", "on",
                        "--metrics", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,"
                        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum",
                        "--clock-control", "none", "-k", f"regex:{KERNELS[format]}",
                        "-o", rep] + argv, check=True, stdout=subprocess.DEVNULL, env=env)
        src = subprocess.run([ncu, "-i", rep + ".ncu-rep", "--page", "source", "--csv",
                              "--print-source", "sass"], capture_output=True, text=True,
                             check=True).stdout
        raw = subprocess.run([ncu, "-i", rep + ".ncu-rep", "--page", "raw", "--csv"],
                             capture_output=True, text=True, check=True).stdout
        m = json.load(open(meta))
    tx = classify(list(csv.reader(io.StringIO(src))), sv)
    rr = list(csv.reader(io.StringIO(raw)))
    hdr = rr[0]

    def total_of(metric):  # summed over the profiled kernels (one raw row each)
        j = hdr.index(metric)
        return sum(int(float(v[j].replace(",", ""))) for v in rr[2:] if len(v) > j and v[j])
    hits = total_of("l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum")
    miss_all = total_of("l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum")
    kernels = [v[hdr.index("Kernel Name")] for v in rr[2:] if len(v) > 1]
    total = sum(v[0] for v in tx.values())
    ideal = sum(v[1] for v in tx.values())
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bw, bw_kind = float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        bw, bw_kind = 6650.0, "fallback"
    bytes_per_nnz = 4 + sv  # x cached, as the reference's simulate (cached_x=true)
    doc = {"matrix": mtx or f"synthetic:{case}", "format": format,
           "precision": precision, "nnz": m["nnz"], "artificial_zeros": m["artificial_zeros"],
           "transactions": {k: tx[k][0] for k in ("values", "columns", "x", "output")},
           "min_possible": ideal, "efficiency": ideal / total if total else 1.0,
           "cache": {"hits": hits, "misses": max(0, tx["x"][0] - hits)},
           "peak": {"bytes_per_nnz": bytes_per_nnz, "gflops": 2.0 * bw / bytes_per_nnz},
           "metadata_sectors": tx["metadata"][0],
           "units": "32-byte L2 sectors per launch (ncu SourceCounters), B200; "
                    "cache = L1 global-load lookup hits of the x gathers",
           "peak_bandwidth": {"gbs": bw, "kind": bw_kind},
           "ordering": ordering,
           "all_load_lookup_misses": miss_all, "kernels": kernels}
    if format == "rgcsr":
        doc["group_size"] = group_size
    return doc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="27:128")
    ap.add_argument("--mtx")
    ap.add_argument("--format", default="rgcsr", choices=sorted(KERNELS))
    ap.add_argument("--group-size", type=int, default=32)
    ap.add_argument("--precision", default="double", choices=["single", "double"])
    ap.add_argument("--ordering", default="none", choices=["none", "descending"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--meta")
    a = ap.parse_args()
    if a.child:
        return child(a)
    doc = simulate(a.case, a.mtx, a.format, a.group_size, a.precision, a.ordering, a.seed)
    text = json.dumps(doc, indent=2)
    if a.out:
        open(a.out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
