"""Power-law 8M fp64: RgCSR G=32 and Hybrid builds (for an ncu launch list)."""
import os, sys, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1012_2270_b200 import spmvkit as sk, generators as gen
csr = sk.build_csr(gen.powerlaw(8_000_000, 7))
s = torch.cuda.Stream()
for _ in range(2):
    a = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream); del a
    h = sk.build_hybrid(csr, None, 8, stream=s.cuda_stream); del h
torch.cuda.synchronize()
print("ok")
