"""Pure-ELL Hybrid kernels on the stencils: back-to-back time per variant
(AB_VARIANTS, default auto,vec), best of 5 x 50, y bit checksum."""
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
for kind, n in ((27, 128), (7, 256), (5, 2048)):
    csr = sk.CsrMatrix.stencil(kind, n)
    for prec in (8, 4):
        h = sk.build_hybrid(csr, None, prec)
        dt = torch.float64 if prec == 8 else torch.float32
        x = torch.from_numpy(gen.random_vector(h.num_cols, 1)).cuda().to(dt)
        y = torch.empty(h.num_rows, dtype=dt, device="cuda")
        for v in os.environ.get("AB_VARIANTS", "auto,vec").split(","):
            L.spmvk_set_hybrid_kernel(v.encode())
            us = timed(lambda: sk.spmv_hybrid(h, x, y), reps=50)
            iv = torch.int64 if prec == 8 else torch.int32
            print(json.dumps({"case": f"{kind}pt-{n}", "prec": prec, "variant": v,
                              "us": round(us, 2), "bits": int(y.view(iv).sum().item())}),
                  flush=True)
        L.spmvk_set_hybrid_kernel(b"auto")
        del h
