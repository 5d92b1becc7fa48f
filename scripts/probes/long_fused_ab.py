"""A/B of the long-row handling on the config-3 power-law (8M rows): the long
rows fused into the tile kernel (dynamic items) vs the separate long-row
launch, original and descending order, fp64 / fp32, per K2 variant.  Best of
5 x 20 back-to-back launches (CUDA events on the launching stream).
usage: python scripts/probes/long_fused_ab.py [rows]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def timed(fn, reps=20, rounds=5):
    s = torch.cuda.current_stream()
    best = 1e30
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


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
            a = sk.build_rgcsr(c, 32, prec)
            dt = torch.float64 if prec == 8 else torch.float32
            x = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda().to(dt)
            y = torch.empty(a.num_rows, dtype=dt, device="cuda")
            ref = None
            for variant in os.environ.get("AB_VARIANTS", "auto,lite,lite8,lite8h,pipe").split(","):
                L.spmvk_set_rgcsr_kernel(variant.encode())
                for fused in (1, 0):
                    L.spmvk_set_long_fused(fused)
                    sk.spmv_rgcsr(a, x, y)
                    torch.cuda.synchronize()
                    if ref is None:
                        ref = y.clone()
                    same = bool(torch.equal(y.view(torch.int64 if prec == 8 else torch.int32),
                                            ref.view(torch.int64 if prec == 8 else torch.int32)))
                    us = timed(lambda: sk.spmv_rgcsr(a, x, y))
                    print(json.dumps({"order": order, "prec": prec, "variant": variant,
                                      "fused": fused, "us": round(us, 1),
                                      "long_warps": os.environ.get("SPMVK_LONG_WARPS", "2"),
                                      "gflops": round(2 * nnz / us / 1e3, 1),
                                      "bitwise_same": same}), flush=True)
            L.spmvk_set_rgcsr_kernel(b"auto")
            L.spmvk_set_long_fused(1)
            del a


if __name__ == "__main__":
    main()
