"""Where the K1 converter's wall time goes (27-pt 128^3, fp64, G = 32): host
wall per build, and a torch.profiler (CUPTI) trace of the runtime API calls
and kernels of a few builds.  usage: python scripts/probes/convert_probe.py"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402


def main():
    torch.cuda.set_device(0)
    assert lib().spmvk_init(0) == 0
    csr = sk.CsrMatrix.stencil(27, 128)
    s = torch.cuda.Stream()
    keep = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream)
    for mode in ("del", "keep"):
        ts = []
        held = []
        for _ in range(6):
            torch.cuda.synchronize()
            t = time.perf_counter()
            a = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream)
            ts.append((time.perf_counter() - t) * 1e3)
            if mode == "keep":
                held.append(a)
            del a
        print(mode, "build ms:", " ".join("%.2f" % v for v in ts))
        del held
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
        for _ in range(3):
            torch.cuda.synchronize()
            a = sk.build_rgcsr(csr, 32, 8, stream=s.cuda_stream)
            torch.cuda.synchronize()
            del a
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in p.events():
        d = e.device_time if e.device_type.name == "CUDA" else e.cpu_time
        agg[(e.device_type.name, e.name)][0] += 1
        agg[(e.device_type.name, e.name)][1] += d
    for (dev, name), (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print("%-5s %6d %10.1f us  %s" % (dev, n, us / 3, name[:100]))
    del keep


if __name__ == "__main__":
    main()
