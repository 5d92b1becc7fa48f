"""Back-to-back SpMV time of the default RgCSR kernel on the stencil configs
(best of 5 x 50 launches, CUDA events on the launching stream) -- run once
per environment setting to A/B a kernel knob, e.g.
  SPMVK_GRP_DYN=1 python scripts/probes/stencil_ab.py
Prints one JSON line per (case, precision) with a bit checksum of y."""
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

CASES = [(27, 128), (7, 256), (7, 384), (5, 2048), (5, 1024), (7, 512)]


def main():
    torch.cuda.set_device(0)
    assert lib().spmvk_init(0) == 0
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SPMVK_"))
    for kind, n in CASES:
        csr = sk.CsrMatrix.stencil(kind, n)
        for prec in ((8,) if n == 512 else (8, 4)):
            a = sk.build_rgcsr(csr, 32, prec)
            dt = torch.float64 if prec == 8 else torch.float32
            x = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda().to(dt)
            y = torch.empty(a.num_rows, dtype=dt, device="cuda")
            us = timed(lambda: sk.spmv_rgcsr(a, x, y), reps=50 if n < 512 else 10)
            iv = torch.int64 if prec == 8 else torch.int32
            ck = int(y.view(iv).sum().item())
            print(json.dumps({"case": f"{kind}pt-{n}", "prec": prec, "us": round(us, 2),
                              "gflops": round(2 * a.nnz() / us / 1e3, 1), "bits": ck,
                              "env": tag}), flush=True)
            del a
        del csr


if __name__ == "__main__":
    main()
