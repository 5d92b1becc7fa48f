"""CPU test of scripts/records_ncu.py's merge: kernels between dot_partials
markers are attributed to the records in case order, DRAM bytes summed, hit
rate and sector efficiency sector-weighted."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import records_ncu as rn  # noqa: E402


def test_merge_attributes_kernels_to_cases(tmp_path):
    cases = list(rn.cases())
    rows = [["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "a", "b", "c",
             "d", "e", "f"]]
    kid = 0

    def kernel(name, metrics):
        nonlocal kid
        for m, v in metrics.items():
            rows.append([str(kid), name, m, "", str(v), "", "", "", "", "", ""])
        kid += 1

    for i, _ in enumerate(cases):
        kernel("void spmvk::dot_partials(...)", {"dram__bytes_read.sum": 1})
        kernel("void spmvk::rgcsr_spmv_grp<double>(...)",
               {"dram__bytes_read.sum": 100 + i, "dram__bytes_write.sum": 10,
                "lts__t_sector_hit_rate.pct": 50, "lts__t_sectors.sum": 10,
                "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct": 90,
                "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": 10})
        if i == 0:  # a second kernel in the first case (e.g. the long-row kernel)
            kernel("void spmvk::rgcsr_spmv_long_mixed<double>(...)",
                   {"dram__bytes_read.sum": 1000, "dram__bytes_write.sum": 0,
                    "lts__t_sector_hit_rate.pct": 0, "lts__t_sectors.sum": 30,
                    "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct": 10,
                    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": 30})
    kernel("void spmvk::dot_partials(...)", {"dram__bytes_read.sum": 1})
    p = tmp_path / "n.csv"
    with open(p, "w", newline="") as f:
        csv.writer(f).writerows(rows)
    recs = tmp_path / "r.jsonl"
    wl, prec, fmt = cases[0]
    wl1, prec1, fmt1 = cases[1]
    with open(recs, "w") as f:
        for w, pr, fm in ((wl, prec, fmt), (wl1, prec1, fmt1)):
            g = int(fm[5:]) if fm.startswith("rgcsr") else None
            f.write(json.dumps({"matrix_name": w, "precision": "double" if pr == 8 else "single",
                                "format_name": "rgcsr" if g else fm, "group_size": g}) + "\n")
    rn.merge(str(p), str(recs))
    r0, r1 = [json.loads(ln) for ln in open(recs)]
    assert r0["ncu_dram_bytes"] == 100 + 10 + 1000 and len(r0["ncu_kernels"]) == 2
    assert abs(r0["ncu_l2_hit_pct"] - 50 * 10 / 40) < 1e-9
    assert abs(r0["ncu_sector_efficiency_pct"] - (90 * 10 + 10 * 30) / 40) < 1e-9
    assert r1["ncu_dram_bytes"] == 101 + 10 and r1["ncu_l2_hit_pct"] == 50
