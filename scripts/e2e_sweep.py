"""e2e host-span SpMV time per step vs pipeline chunk count (SPMVK_PIPE_CHUNKS)."""
import os
import subprocess
import sys

code = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_1012_2270_b200 import spmvkit as sk
from paper_1012_2270_b200._lib import lib
L = lib(); torch.cuda.set_device(0); assert L.spmvk_init(0) == 0
csr = sk.CsrMatrix.stencil(27, 128)
for prec, dt in ((8, torch.float64), (4, torch.float32)):
    a = sk.build_rgcsr(csr if prec == 8 else sk.build_csr(sk.TripletMatrix(csr.num_rows, csr.num_cols, *csr.to_host()), 4), 32, prec)
    f = L.spmvk_rgcsr_spmv_host_f64 if prec == 8 else L.spmvk_rgcsr_spmv_host_f32
    xp = torch.rand(csr.num_cols, dtype=dt).pin_memory(); yp = torch.empty(csr.num_rows, dtype=dt).pin_memory()
    for _ in range(5): f(a._h, xp.data_ptr(), csr.num_cols, yp.data_ptr(), csr.num_rows, None)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        for _ in range(50): f(a._h, xp.data_ptr(), csr.num_cols, yp.data_ptr(), csr.num_rows, None)
        ts.append((time.perf_counter() - t) / 50 * 1e3)
    print(sys.argv[1], prec, "ms/step min %.3f med %.3f" % (min(ts), sorted(ts)[2]), flush=True)
'''
for mapped in ("1", "0"):
    print("mapped_y", mapped, flush=True)
    subprocess.run([sys.executable, "-c", code, "ramp"], stderr=subprocess.DEVNULL,
                   env=dict(os.environ, SPMVK_PIPE_MAPPED_Y=mapped))
for mapped in ("1", "0"):
    for n in sys.argv[1:] or ["2", "4", "8", "16"]:
        print("mapped_y", mapped, flush=True)
        subprocess.run([sys.executable, "-c", code, n], stderr=subprocess.DEVNULL,
                       env=dict(os.environ, SPMVK_PIPE_CHUNKS=n, SPMVK_PIPE_MAPPED_Y=mapped))
