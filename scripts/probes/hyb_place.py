"""Placement sensitivity of the pure-ELL Hybrid kernel (27-pt 128^3 fp32):
allocate a pad of p MB (cudaMalloc through torch with caching disabled),
build the Hybrid (handle-array cache off), time back-to-back SpMVs, repeat for
several pads.  Run with PYTORCH_NO_CUDA_MEMORY_CACHING=1 SPMVK_ALLOC_CACHE_MB=0."""
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

L = lib()
torch.cuda.set_device(0)
assert L.spmvk_init(0) == 0
csr = sk.CsrMatrix.stencil(27, 128)
prec = int(os.environ.get("PREC", "4"))
dt = torch.float32 if prec == 4 else torch.float64
x = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda().to(dt)
y = torch.empty(csr.num_rows, dtype=dt, device="cuda")
for pad_mb in [int(v) for v in os.environ.get("PADS", "0,1,2,3,4,6,8,12,16,24,32,48,64").split(",")]:
    pad = torch.empty(pad_mb << 20, dtype=torch.uint8, device="cuda") if pad_mb else None
    h = sk.build_hybrid(csr, None, prec)
    us = timed(lambda: sk.spmv_hybrid(h, x, y), reps=50)
    print(json.dumps({"pad_mb": pad_mb, "prec": prec, "us": round(us, 2)}), flush=True)
    del h, pad
