"""Probe: the device SpMV entry point fed pinned HOST x and/or y (UVA mapped,
zero-copy over PCIe) -- does the L2 keep the gathered x after its first
PCIe read?  Compares device x/y, host x, host y, host x + y (27pt-128 fp64)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

L = lib()
torch.cuda.set_device(0)
assert L.spmvk_init(0) == 0
wl = sys.argv[1] if len(sys.argv) > 1 else "27:128"
kind, n = (int(v) for v in wl.split(":"))
a = sk.build_rgcsr(sk.CsrMatrix.stencil(kind, n), 32, 8)
xh = torch.from_numpy(gen.random_vector(a.num_cols, 1)).pin_memory()
yh = torch.empty(a.num_rows, dtype=torch.float64).pin_memory()
xd, yd = xh.cuda(), torch.empty(a.num_rows, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
want = sk.spmv_rgcsr(a, xd).cpu()


def timed(x, y, reps=20):
    fn = lambda: L.spmvk_rgcsr_spmv_f64(a._h, x.data_ptr(), a.num_cols, y.data_ptr(),  # noqa
                                        a.num_rows, s)
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name, x, y in (("device x, device y", xd, yd), ("host x, device y", xh, yd),
                   ("device x, host y", xd, yh), ("host x, host y", xh, yh)):
    us = timed(x, y)
    got = (y if y.is_cuda else y).cpu()
    print(f"{wl} {name:22s} {us:9.1f} us  {2 * a.nnz() / us / 1e3:7.1f} GFLOP/s  "
          f"bitwise={torch.equal(got.view(torch.int64), want.view(torch.int64))}", flush=True)
