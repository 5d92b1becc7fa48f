"""Hybrid converter at the wall (steady state): build_hybrid on 27-pt 128^3
fp64 and power-law 8M fp64, median of 7 after 3 warm builds, plus a CUPTI
timeline of one 27-pt build."""
import os, sys, time, statistics, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from torch.profiler import profile, ProfilerActivity
from paper_1012_2270_b200 import spmvkit as sk, generators as gen

s = torch.cuda.Stream()
for name, csr in (("27pt-128", sk.CsrMatrix.stencil(27, 128)),
                  ("powerlaw-8M", sk.build_csr(gen.powerlaw(8_000_000, 7)))):
    for prec in (8,):
        for _ in range(3):
            h = sk.build_hybrid(csr, None, prec, stream=s.cuda_stream); del h
        ts = []
        for _ in range(7):
            torch.cuda.synchronize(); t = time.perf_counter()
            h = sk.build_hybrid(csr, None, prec, stream=s.cuda_stream)
            ts.append((time.perf_counter() - t) * 1e6); del h
        print(name, prec, "hybrid build us", [round(v) for v in ts], "median", round(statistics.median(ts)))
        for _ in range(2):
            a = sk.build_rgcsr(csr, 32, prec, stream=s.cuda_stream); del a
        ts = []
        for _ in range(7):
            torch.cuda.synchronize(); t = time.perf_counter()
            a = sk.build_rgcsr(csr, 32, prec, stream=s.cuda_stream)
            ts.append((time.perf_counter() - t) * 1e6); del a
        print(name, prec, "rgcsr build us", [round(v) for v in ts], "median", round(statistics.median(ts)))
    if name == "27pt-128":
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            h = sk.build_hybrid(csr, None, 8, stream=s.cuda_stream); del h
            torch.cuda.synchronize()
        ev = sorted([e for e in prof.events()], key=lambda e: e.time_range.start)
        t0 = ev[0].time_range.start
        for e in ev:
            print(f"{e.device_type.name:4s} {e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")
