"""bench.py host-side pieces that need no GPU: the live-traffic ncu parse
(a faked ncu CSV), the reference-golden lookups, the config dicts both arms
print."""
import json
import os
import shutil
import subprocess
import types

import bench


def test_measured_traffic_parses_ncu_csv(monkeypatch):
    hdr = ('"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream",'
           '"Block Size","Grid Size","Device","CC","Section Name","Metric Name","Metric Unit",'
           '"Metric Value"')
    row = ('"0","1","python","h","void rgcsr_spmv_grp<double, 0, 8, 4>(unsigned int)","1","7",'
           '"(256, 1, 1)","(592, 1, 1)","0","10.0","Command line profiler metrics",'
           '"{m}","byte","{v}"')
    out = "\n".join(["==PROF== Connected", hdr,
                     row.format(m="dram__bytes_read.sum", v="689,547,008"),
                     row.format(m="dram__bytes_write.sum", v="6,174,464"), "ok"])
    monkeypatch.setattr(shutil, "which", lambda _: "/usr/bin/ncu")
    monkeypatch.delenv("CUDA_INJECTION64_PATH", raising=False)
    monkeypatch.setattr(subprocess, "run",
                        lambda *a, **k: types.SimpleNamespace(stdout=out, returncode=0))
    got = bench.measured_traffic("27pt-128")
    assert got["bytes"] == 689547008 + 6174464
    assert "rgcsr_spmv_grp" in got["kernel"]
    assert bench.measured_traffic("powerlaw-8M") is None  # only stencils are re-profiled


def test_measured_traffic_skips_under_a_profiler(monkeypatch):
    monkeypatch.setenv("CUDA_INJECTION64_PATH", "/x/libinject.so")
    assert bench.measured_traffic("27pt-128") is None


def test_golden_lookups_and_config_dicts():
    assert bench.golden_checksum("27pt-128") == 1674.3573800651031
    assert bench.golden_checksum("7pt-512") is None
    with open(os.path.join(bench.ROOT, "tests", "golden", "iterate_7pt512.json")) as f:
        g = json.load(f)
    assert int(g["bits_sum_int64_after"]["100"]) == -7592457614606409731
    c1 = bench.bench_config("27pt-128", 1)
    c8 = bench.bench_config("7pt-512", 8, "fused")
    assert c1["parallelism"] == "single GPU" and "x8" in c8["parallelism"]
    assert 90 < bench.PCIE_BIDIR_GBS < 110
