"""Small end-to-end pass for compute-sanitizer (memcheck / racecheck /
synccheck): every default kernel family on small matrices, results checked
bitwise against the oracle.  Usage:
    compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as orc  # noqa: E402
from helpers import triplets  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402

torch.cuda.set_device(0)
mats = {"27pt-16": orc.stencil(27, 16), "5pt-64": orc.stencil(5, 64),
        "powerlaw-20k": orc.powerlaw(20000, 7)}
for name, om in mats.items():
    m = triplets(om)
    for prec, dt in ((8, np.float64), (4, np.float32)):
        x = orc.random_vector(om.cols, 1).astype(dt)
        xd = torch.from_numpy(x).cuda()
        for G in (32, 7):
            a = sk.build_rgcsr(m, G, prec)
            want = orc.spmv_rgcsr(orc.build_rgcsr(om, G, prec), x)[0]
            assert sk.spmv_rgcsr(a, xd).cpu().numpy().tobytes() == want.tobytes(), (name, G)
        h = sk.build_hybrid(m, None, prec)
        want = orc.spmv_hybrid(orc.build_hybrid(om, None, prec), x)
        assert sk.spmv_hybrid(h, xd).cpu().numpy().tobytes() == want.tobytes(), name
        c = sk.build_csr(m, prec)
        assert sk.spmv_csr(c, xd).cpu().numpy().tobytes() == orc.spmv_csr(om, x, prec).tobytes()
    c2, _ = sk.apply_descending_permutation(sk.build_csr(m))
    a2 = sk.build_rgcsr(c2, 32)
    rp, col, val = c2.to_host()
    o2 = orc.Csr(c2.num_rows, c2.num_cols, rp, col, val)
    x = orc.random_vector(om.cols, 1)
    want = orc.spmv_rgcsr(orc.build_rgcsr(o2, 32), x)[0]
    assert sk.spmv_rgcsr(a2, torch.from_numpy(x).cuda()).cpu().numpy().tobytes() == want.tobytes()
torch.cuda.synchronize()
print("sanitize pass ok")
