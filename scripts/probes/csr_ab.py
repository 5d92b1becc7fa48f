"""spmv_csr back-to-back time per SPMVK_CSR_KERNEL setting (run once per
setting): stencils and the config-3 power-law, fp64 / fp32, best of 5 x 30,
y bit checksum."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from long_fused_ab import timed  # noqa: E402

torch.cuda.set_device(0)
assert lib().spmvk_init(0) == 0
tag = os.environ.get("SPMVK_CSR_KERNEL", "")
for name in ("27:128", "7:256", "5:2048", "0:8000000"):
    kind, n = (int(v) for v in name.split(":"))
    c64 = sk.CsrMatrix.stencil(kind, n) if kind else sk.build_csr(gen.powerlaw(n, 7))
    for prec in (8, 4):
        c = c64 if prec == 8 else sk.build_csr(
            sk.TripletMatrix(c64.num_rows, c64.num_cols, *c64.to_host()), 4)
        dt = torch.float64 if prec == 8 else torch.float32
        x = torch.from_numpy(gen.random_vector(c.num_cols, 1)).cuda().to(dt)
        y = torch.empty(c.num_rows, dtype=dt, device="cuda")
        us = timed(lambda: sk.spmv_csr(c, x, y), reps=30)
        iv = torch.int64 if prec == 8 else torch.int32
        print(json.dumps({"case": name, "prec": prec, "kernel": tag or "default", "us": round(us, 2),
                          "gflops": round(2 * c.nnz() / us / 1e3, 1),
                          "bits": int(y.view(iv).sum().item())}), flush=True)
        if prec == 4:
            del c
