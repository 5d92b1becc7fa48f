"""Minimal K2 runner for ncu: builds one stencil RgCSR and launches the chosen
variant `--launches` times (ncu -k regex:rgcsr_spmv -s <warm> -c 1 ...).
Also used for Hybrid: --format hybrid."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="27:128:32")
    ap.add_argument("--prec", type=int, default=8)
    ap.add_argument("--variant", default="pipe")
    ap.add_argument("--format", default="rgcsr")
    ap.add_argument("--hvariant", default="auto", help="Hybrid kernel variant")
    ap.add_argument("--launches", type=int, default=4)
    ap.add_argument("--reorder", action="store_true", help="descending row reordering first")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    assert L.spmvk_set_rgcsr_kernel(a.variant.encode()) == 0
    assert L.spmvk_set_hybrid_kernel(a.hvariant.encode()) == 0
    kind, n, G = (int(v) for v in a.case.split(":"))
    if kind == 0:
        csr = sk.build_csr(gen.powerlaw(n, 7), a.prec)
    else:
        csr = sk.CsrMatrix.stencil(kind, n)
    if a.reorder:
        csr = sk.apply_descending_permutation(csr)[0]
    h = sk.build_rgcsr(csr, G, a.prec) if a.format == "rgcsr" else sk.build_hybrid(csr, None, a.prec)
    del csr
    dt = torch.float64 if a.prec == 8 else torch.float32
    x = torch.from_numpy(gen.random_vector(h.num_cols, 1)).cuda().to(dt)
    y = torch.empty(h.num_rows, dtype=dt, device="cuda")
    fn = sk.spmv_rgcsr if a.format == "rgcsr" else sk.spmv_hybrid
    for _ in range(a.launches):
        fn(h, x, y)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
