"""ncu counters for every SURVEY 8d record (the "ncu counters are attached to
each record" clause): one SpMV launch per (config, format, G, precision)
under `ncu --metrics`, cases separated by a marker kernel, then the
per-case sums merged into the records .jsonl.

  ncu --metrics <METRICS> --csv --log-file gpurun_out/rec_ncu.csv \\
      -k regex:"rgcsr_spmv|hybrid_spmv|hybrid_ell_vec|csr_spmv|dot_partials" \
      python scripts/records_ncu.py run
  python scripts/records_ncu.py merge gpurun_out/rec_ncu.csv profiles/r01_records.jsonl

Counters per record: DRAM bytes read + written (summed over the case's SpMV
kernels), L2 sector hit rate and the average bytes used per global-load
sector (sector efficiency), both weighted by sectors."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,"
           "lts__t_sectors.sum,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,"
           "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
WORKLOADS = ("5pt-1024", "27pt-128", "powerlaw-8M")
FORMATS = ("csr", "rgcsr32", "rgcsr64", "rgcsr128", "rgcsr256", "hybrid")


def cases():
    for wl in WORKLOADS:
        for prec in (8, 4):
            for fmt in FORMATS:
                yield wl, prec, fmt


def run():
    import torch

    import bench
    from paper_1012_2270_b200 import generators as gen
    from paper_1012_2270_b200 import spmvkit as sk
    torch.cuda.set_device(0)
    import ctypes as C

    from paper_1012_2270_b200._lib import lib
    L = lib()
    assert L.spmvk_init(0) == 0
    mk = torch.ones(64, dtype=torch.float64, device="cuda")
    mo = torch.empty(1, dtype=torch.float64, device="cuda")

    def marker():  # case boundary in the kernel list: dot_partials (cg.cu)
        assert L.spmvk_dot_f64(C.c_void_p(mk.data_ptr()), C.c_void_p(mk.data_ptr()), 64,
                               C.c_void_p(mo.data_ptr()), None) == 0
        torch.cuda.synchronize()
    for wl in WORKLOADS:
        csr64 = bench.make_csr(wl)
        rows, cols = csr64.num_rows, csr64.num_cols
        xh = gen.random_vector(cols, 1)
        for prec in (8, 4):
            dt = torch.float64 if prec == 8 else torch.float32
            c = csr64 if prec == 8 else sk.build_csr(
                sk.TripletMatrix(rows, cols, *csr64.to_host()), 4)
            x = torch.from_numpy(xh).cuda().to(dt)
            y = torch.empty(rows, dtype=dt, device="cuda")
            for fmt in FORMATS:
                h = c if fmt == "csr" else (sk.build_hybrid(c, None, prec) if fmt == "hybrid"
                                            else sk.build_rgcsr(c, int(fmt[5:]), prec))
                torch.cuda.synchronize()
                marker()
                if fmt == "csr":
                    sk.spmv_csr(h, x, y)
                elif fmt == "hybrid":
                    sk.spmv_hybrid(h, x, y)
                else:
                    sk.spmv_rgcsr(h, x, y)
                torch.cuda.synchronize()
                print(json.dumps({"case": [wl, prec, fmt]}), flush=True)
    marker()


def merge(csv_path, records_path):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    hdr = rows[0]
    ik, iname, iv = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Value")
    imn = hdr.index("Metric Name")
    kern = {}
    for r in rows[1:]:
        k = kern.setdefault(int(r[ik]), {"name": r[iname]})
        k[r[imn]] = float(r[iv].replace(",", ""))
    groups, cur = [], None
    for kid in sorted(kern):
        k = kern[kid]
        if "dot_partials" in k["name"]:
            if cur is not None:
                groups.append(cur)
            cur = []
        elif cur is not None and "_fill" not in k["name"]:  # a builder kernel, not a SpMV
            cur.append(k)
    per = {}
    for (wl, prec, fmt), ks in zip(cases(), groups):
        sec = sum(k.get("lts__t_sectors.sum", 0) for k in ks) or 1
        lds = sum(k.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 0) for k in ks) or 1
        per[(wl, prec, fmt)] = {
            "ncu_kernels": [k["name"].split("(")[0].replace("void ", "") for k in ks],
            "ncu_dram_bytes": sum(k.get("dram__bytes_read.sum", 0) +
                                  k.get("dram__bytes_write.sum", 0) for k in ks),
            "ncu_l2_hit_pct": sum(k.get("lts__t_sector_hit_rate.pct", 0) *
                                  k.get("lts__t_sectors.sum", 0) for k in ks) / sec,
            "ncu_sector_efficiency_pct": sum(
                k.get("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct", 0) *
                k.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 0) for k in ks) / lds}
    out = []
    for line in open(records_path):
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        fmt = r["format_name"] if r["format_name"] != "rgcsr" else f"rgcsr{r['group_size']}"
        key = (r["matrix_name"], 8 if r["precision"] == "double" else 4, fmt)
        r.update(per.get(key, {}))
        out.append(r)
    with open(records_path, "w") as f:
        for r in out:
            f.write(json.dumps(r) + "\n")
    print(f"merged counters into {sum(1 for r in out if 'ncu_dram_bytes' in r)} of {len(out)} records")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        merge(sys.argv[2], sys.argv[3])
