"""A/B of the Hybrid kernels with a COO part on the config-3 power-law (8M
rows): the staged-tile default (litef / litefh + heavy-row launch) vs
hybrid_spmv_dyn, original and descending order, fp64 / fp32.  Best of 5 x 20
back-to-back launches.  usage: python scripts/probes/hybrid_dyn_ab.py [rows]"""
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


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    csr = sk.build_csr(gen.powerlaw(rows, 7))
    desc = sk.apply_descending_permutation(csr)[0]
    nnz = csr.nnz()
    for order, c in (("orig", csr), ("desc", desc)):
        for prec in (8, 4):
            h = sk.build_hybrid(c, None, prec)
            dt = torch.float64 if prec == 8 else torch.float32
            x = torch.from_numpy(gen.random_vector(h.num_cols, 1)).cuda().to(dt)
            y = torch.empty(h.num_rows, dtype=dt, device="cuda")
            ref = None
            for variant in os.environ.get("AB_VARIANTS", "auto,dyn").split(","):
                L.spmvk_set_hybrid_kernel(variant.encode())
                sk.spmv_hybrid(h, x, y)
                torch.cuda.synchronize()
                if ref is None:
                    ref = y.clone()
                iv = torch.int64 if prec == 8 else torch.int32
                same = bool(torch.equal(y.view(iv), ref.view(iv)))
                us = timed(lambda: sk.spmv_hybrid(h, x, y))
                print(json.dumps({"order": order, "prec": prec, "variant": variant,
                                  "heavy_warps": os.environ.get("SPMVK_HYB_HEAVY_WARPS", "2"),
                                  "us": round(us, 1), "gflops": round(2 * nnz / us / 1e3, 1),
                                  "bitwise_same": same}), flush=True)
            L.spmvk_set_hybrid_kernel(b"auto")
            del h


if __name__ == "__main__":
    main()
