"""CG iteration throughput (spmvk_cg_solve_f64, graph-replayed iterations) on
the 7-point stencils: time for a fixed iteration count (tol = 0), bytes per
iteration = the SpMV's B_fmt (p.q is fused into its epilogue) + the vector
traffic of the other kernels (update: x, p, r, q read, x, r written;
direction: r, p read, p written -> 9 N doubles), achieved GB/s vs the
measured copy peak."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

torch.cuda.set_device(0)
assert lib().spmvk_init(0) == 0
peak, _ = bench.peaks()
for n in (128, 256, 384):
    a = sk.build_rgcsr(sk.CsrMatrix.stencil(7, n), 32)
    N = a.num_rows
    b = torch.ones(N, dtype=torch.float64, device="cuda")
    def run(iters):
        torch.cuda.synchronize()
        t = time.perf_counter()
        x, it, rel = sk.cg(a, b, tol=0.0, max_iter=iters, check_every=50)
        torch.cuda.synchronize()
        return time.perf_counter() - t, it
    run(100)  # warm-up
    # per-iteration cost from the difference of two lengths (allocation,
    # capture and setup cancel), best of three pairs
    import statistics
    per = statistics.median((run(2000)[0] - run(400)[0]) / 1600 for _ in range(5))
    it = 1600
    dt = per * it
    B = bench.rg_bytes(a.info, 8) + 9 * 8 * N
    print(json.dumps({"case": f"7pt-{n}", "rows": N, "ms_per_iter": dt / it * 1e3,
                      "bytes_per_iter": B, "GBs": B / (dt / it) / 1e9,
                      "frac_of_copy_peak": B / (dt / it) / 1e9 / peak}),
          flush=True)
