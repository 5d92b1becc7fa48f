"""Time the fused dist step at world 1 (7pt-512 fp64) against the plain scaled
SpMV on the same slab: isolates the PeerEpi epilogue / window layout cost."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import partition as pt  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

L = lib()
torch.cuda.set_device(0)
assert L.spmvk_init(0) == 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
csr = sk.CsrMatrix.stencil(7, n)
a = sk.build_rgcsr(csr, 32, 8)
del csr
s = torch.cuda.current_stream().cuda_stream
x0 = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda()


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


y = torch.empty(a.num_rows, dtype=torch.float64, device="cuda")
xn = torch.empty_like(y)
xa = x0.clone()


def scaled():
    L.spmvk_rgcsr_spmv_scaled_f64(a._h, xa.data_ptr(), a.num_cols, y.data_ptr(), a.num_rows,
                                  xn.data_ptr(), 0.0625, s)


print("scaled_us", round(timed(scaled), 1))
sl = pt.Slab(0, 0, a.num_rows, a.num_rows)
win = pt.ExchangeWindow(a.num_rows, 8)
it = pt.FusedIteratedSpmv(sl, [(0, a.num_rows)], a, win, 1, s, local_windows=[win],
                          barrier=False)
it.set_x(x0)
print("fused_us", os.environ.get("SPMVK_WINDOW_PAD", "0"), round(timed(it.step), 1))
