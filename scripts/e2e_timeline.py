"""CUPTI timeline (torch.profiler) of the pipelined host-span SpMV: per-op
start/end on each stream, to check that H2D, SpMV chunks and D2H overlap."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

L = lib()
torch.cuda.set_device(0)
assert L.spmvk_init(0) == 0
csr = sk.CsrMatrix.stencil(27, 128)
a = sk.build_rgcsr(csr, 32, 8)
if os.environ.get("E2E_HOST", "spmvk") == "torch":
    xpin = torch.from_numpy(np.random.default_rng(1).random(csr.num_cols)).pin_memory()
    ypin = torch.empty(csr.num_rows, dtype=torch.float64).pin_memory()
else:  # spmvk_host_alloc buffers (the bench default)
    xpin = torch.from_numpy(sk.host_array(csr.num_cols))
    xpin.numpy()[:] = np.random.default_rng(1).random(csr.num_cols)
    ypin = torch.from_numpy(sk.host_array(csr.num_rows))


def call():
    rc = L.spmvk_rgcsr_spmv_host_f64(a._h, xpin.data_ptr(), csr.num_cols, ypin.data_ptr(),
                                     csr.num_rows, None)
    assert rc == 0


for _ in range(3):
    call()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    call()
print("wall ms/step", (time.perf_counter() - t) / 20 * 1e3)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as p:
    for _ in range(3):
        call()
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
p.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy")]
gpu.sort(key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
for e in gpu[:int(os.environ.get('E2E_ROWS', '80'))]:
    print(f'{e["ts"]-t0:9.1f} {e["dur"]:7.1f} s{e["args"].get("stream")} {e["name"][:50]}')
