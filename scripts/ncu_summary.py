"""Summarises ncu output for profiles/: a --set full report of one kernel
(speed-of-light, DRAM bytes, cache hit rates, occupancy, stall reasons) and a
launch list (per-kernel count and time share).

  python scripts/ncu_summary.py --rep gpurun_out/prof_X.ncu-rep \
      --launches gpurun_out/launches_X.csv --out profiles/r01_X.md [--traffic-key K]
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "smsp__inst_executed.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(hdr, units, vals)})
    return res


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    keep = []
    for r in rows[1:]:
        sec = r[h.index("Section Name")]
        if sec in ("GPU Speed Of Light Throughput", "Memory Workload Analysis",
                   "Warp State Statistics", "Occupancy", "Scheduler Statistics"):
            keep.append((sec, r[h.index("Metric Name")], r[h.index("Metric Value")],
                         r[h.index("Metric Unit")]))
    return keep


def launches(path):
    txt = open(path).read().splitlines()
    start = [i for i, l in enumerate(txt) if l.startswith('"ID"')][0]
    rows = list(csv.reader(io.StringIO("\n".join(txt[start:]))))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        n = r[ki].split("(")[0].replace("void ", "")
        agg[n][0] += 1
        agg[n][1] += float(r[vi].replace(",", ""))
    return sorted(agg.items(), key=lambda kv: -kv[1][1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    ap.add_argument("--traffic-key")
    args = ap.parse_args()
    lines = [f"# {args.title or os.path.basename(args.out)}", ""]
    if args.rep:
        for k in raw(args.rep):
            name = k.get("Kernel Name", ("?", ""))[0]
            lines += [f"## kernel `{name[:160]}`", "", "| metric | value | unit |", "|---|---|---|"]
            for key in KEYS:
                if key in k:
                    lines.append(f"| {key} | {k[key][0]} | {k[key][1]} |")
            # request-path utilisation (the floor of gather-bound kernels)
            for key in sorted(k):
                if ("xbar_req" in key or "l1tex__lsu_writeback" in key) and key not in KEYS:
                    lines.append(f"| {key} | {k[key][0]} | {k[key][1]} |")
            rd = float(k["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(k["dram__bytes_write.sum"][0].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic = rd * mult[k["dram__bytes_read.sum"][1]] + wr * mult[k["dram__bytes_write.sum"][1]]
            lines += ["", f"dram traffic per launch (read + write): **{traffic:,.0f} B**", ""]
            if args.traffic_key:
                tpath = os.path.join(os.path.dirname(args.out), "traffic.json")
                t = json.load(open(tpath)) if os.path.exists(tpath) else {}
                t[args.traffic_key] = traffic
                json.dump(t, open(tpath, "w"), indent=1, sort_keys=True)
        lines += ["### sections", "", "| section | metric | value | unit |", "|---|---|---|---|"]
        lines += [f"| {a} | {b} | {c} | {d} |" for a, b, c, d in stalls(args.rep)]
        lines.append("")
    if args.launches:
        ls = launches(args.launches)
        tot = sum(v[1] for _, v in ls)
        lines += ["## launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for n, (c, t) in ls:
            lines.append(f"| `{n[:90]}` | {c} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("wrote", args.out)


if __name__ == "__main__":
    main()
