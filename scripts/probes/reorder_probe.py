"""Descending row reordering (f1) of the power-law 8M: wall time and the
CUDA API / kernel breakdown of one call."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

torch.cuda.set_device(0)
assert lib().spmvk_init(0) == 0
csr = sk.build_csr(gen.powerlaw(8_000_000, 7))
ts = []
for _ in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d, _ = sk.apply_descending_permutation(csr)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
    del d
print("reorder ms:", " ".join("%.2f" % v for v in ts))
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
    d, _ = sk.apply_descending_permutation(csr)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in p.events():
    dd = e.device_time if e.device_type.name == "CUDA" else e.cpu_time
    agg[(e.device_type.name, e.name)][0] += 1
    agg[(e.device_type.name, e.name)][1] += dd
for (dev, nm), (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print("  %-5s %6d %10.1f us  %s" % (dev, n, us, nm[:90]))
