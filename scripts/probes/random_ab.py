"""RgCSR on the sweep's random-class matrices (ragged rows, no long rows):
back-to-back time of the auto kernel vs named variants, fp64 / fp32."""
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

L = lib()
torch.cuda.set_device(0)
assert L.spmvk_init(0) == 0
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SPMVK_"))
for seed in (0, 3, 27, 48, 96, 138, 183):
    name, m = gen.sweep_case(seed)
    if not name.startswith("random"):
        continue
    csr = sk.build_csr(m)
    for prec in (8, 4):
        a = sk.build_rgcsr(csr, 32, prec)
        dt = torch.float64 if prec == 8 else torch.float32
        x = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda().to(dt)
        y = torch.empty(a.num_rows, dtype=dt, device="cuda")
        for v in os.environ.get("AB_VARIANTS", "auto,pipe,lite8").split(","):
            L.spmvk_set_rgcsr_kernel(v.encode())
            us = timed(lambda: sk.spmv_rgcsr(a, x, y), reps=20)
            iv = torch.int64 if prec == 8 else torch.int32
            print(json.dumps({"m": name, "prec": prec, "v": v, "us": round(us, 1),
                              "long": a.info.num_rows, "bits": int(y.view(iv).sum().item()),
                              "env": tag}), flush=True)
        L.spmvk_set_rgcsr_kernel(b"auto")
        del a
