"""Golden bit checksum of the config-5 iterate (test infrastructure): the
UNMODIFIED reference (oracle/_ref, spmv_rgcsr over group-aligned row slabs on
all host threads, bitwise equal to one thread) runs BASELINE configs[4] --
7-point 512^3, fp64, G = 32 -- for 100 iterations of x <- (A x) * 2^-4 from
x0 = random_vector(N, seed 1), and the wrapping int64 sum of the final x's
raw bits is written to tests/golden/iterate_7pt512.json.  bench.py's N > 1
leg gates its distributed iterate on this number; test_config5 checks the
single-GPU and P = 1 fused iterates against the reference directly.
    python oracle/make_iterate_golden.py      (~3 min, ~40 GB of host memory)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as orc  # noqa: E402


def bits_sum(x):
    return int(np.ascontiguousarray(x, np.float64).view(np.int64).sum(dtype=np.int64))


def main():
    t0 = time.time()
    n, G, iters = 512, 32, 100
    om = orc.stencil(7, n)
    N = om.rows
    ref = orc.RefMatrix.from_csr(om)
    del om
    slabs = orc.RefSlabs(ref, fmt=1, G=G, prec=8)
    del ref
    x = orc.random_vector(N, 1)
    marks = {}
    for k in range(1, iters + 1):
        x = slabs.spmv(x) * 0.0625
        if k in (1, 10, 50, 100):
            marks[str(k)] = bits_sum(x)
    slabs.free()
    out = {"workload": "7pt-512", "rows": N, "group_size": G, "precision": "fp64",
           "x0": "random_vector(N, seed=1)", "step": "x <- spmv_rgcsr(A, x) * 2^-4",
           "bits_sum_int64_after": marks,
           "generated_by": "oracle/make_iterate_golden.py (unmodified reference, oracle/_ref)",
           "seconds": round(time.time() - t0, 1)}
    with open(os.path.join(ROOT, "tests", "golden", "iterate_7pt512.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
