"""K1 converter timeline (CUPTI via torch.profiler): where the wall time of
spmvk_rgcsr_build goes on 27-pt 128^3 fp64 G=32 -- kernels, gaps, host API."""
import os, sys, time, statistics, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from torch.profiler import profile, ProfilerActivity
from paper_1012_2270_b200 import spmvkit as sk

csr = sk.CsrMatrix.stencil(27, 128)
s = torch.cuda.Stream()
for _ in range(3):
    a = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream); del a
torch.cuda.synchronize()
walls = []
for _ in range(7):
    torch.cuda.synchronize(); t = time.perf_counter()
    a = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream)
    walls.append((time.perf_counter() - t) * 1e6); del a
print("wall us", [round(w) for w in walls], "median", round(statistics.median(walls)))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        torch.cuda.synchronize()
        a = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream); del a
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name in ("CUDA", "CPU")]
ev.sort(key=lambda e: e.time_range.start)
t0 = None
for e in ev:
    if t0 is None: t0 = e.time_range.start
    print(f"{e.device_type.name:4s} {e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")
