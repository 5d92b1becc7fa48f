"""Builds the 27-pt 128^3 RgCSR (G = 32, fp64) three times -- for ncu of the
K1 kernels (ncu -k regex:rgcsr_scatter -s 2 -c 1 ...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

torch.cuda.set_device(0)
assert lib().spmvk_init(0) == 0
csr = sk.CsrMatrix.stencil(27, 128)
for _ in range(3):
    a = sk.build_rgcsr(csr, 32, 8)
    del a
torch.cuda.synchronize()
print("ok")
