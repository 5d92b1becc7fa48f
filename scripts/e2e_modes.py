"""e2e host-span SpMV (bench.py's e2e leg) per workload: pinned host x/y
through spmvk_rgcsr_spmv_host_* (the chunked, graph-captured pipeline),
median of 30 calls; SPMVK_PIPE_CHUNKS / SPMVK_PIPE_MAPPED_Y select its
shapes."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

L = lib()
torch.cuda.set_device(0)
assert L.spmvk_init(0) == 0
for kind, n in ((27, 128), (7, 256), (5, 2048)):
    csr = sk.CsrMatrix.stencil(kind, n)
    for prec in (8, 4):
        a = sk.build_rgcsr(csr, 32, prec)
        dt = torch.float64 if prec == 8 else torch.float32
        xh = torch.from_numpy(gen.random_vector(a.num_cols, 1)).to(dt).pin_memory()
        yh = torch.empty(a.num_rows, dtype=dt).pin_memory()
        want = sk.spmv_rgcsr(a, xh.cuda()).cpu()
        f = L.spmvk_rgcsr_spmv_host_f64 if prec == 8 else L.spmvk_rgcsr_spmv_host_f32
        ts = []
        for i in range(35):
            t0 = time.perf_counter()
            assert f(a._h, xh.data_ptr(), a.num_cols, yh.data_ptr(), a.num_rows, None) == 0
            ts.append(time.perf_counter() - t0)
        ok = torch.equal(yh.view(torch.int64 if prec == 8 else torch.int32),
                         want.view(torch.int64 if prec == 8 else torch.int32))
        med = statistics.median(ts[5:])
        print(json.dumps({"chunks": os.environ.get("SPMVK_PIPE_CHUNKS", "ramp"),
                          "case": f"{kind}pt-{n}", "prec": prec, "ms": round(med * 1e3, 3),
                          "GBs_pcie": round((a.num_cols + a.num_rows) * prec / med / 1e9, 1),
                          "gflops": round(2 * a.nnz() / med / 1e9, 1), "bitwise": ok}), flush=True)
        del a
