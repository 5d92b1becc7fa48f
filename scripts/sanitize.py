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
    h2 = sk.build_hybrid(c2)  # reordered: walked tiles + heavy COO rows
    want = orc.spmv_hybrid(orc.build_hybrid(o2, None, 8), x)
    assert sk.spmv_hybrid(h2, torch.from_numpy(x).cuda()).cpu().numpy().tobytes() == want.tobytes()
# host-span pipeline (pinned x / y, graph-captured chunks), CG, fused dist step
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import partition as pt  # noqa: E402
csr = sk.CsrMatrix.stencil(7, 48)
a = sk.build_rgcsr(csr, 32)
xh = torch.from_numpy(orc.random_vector(a.num_cols, 2)).pin_memory()
yh = torch.empty(a.num_rows, dtype=torch.float64).pin_memory()
want = sk.spmv_rgcsr(a, xh.cuda()).cpu().numpy()
sk.spmv_rgcsr(a, xh.numpy(), yh.numpy())
assert yh.numpy().tobytes() == want.tobytes()
b = torch.ones(a.num_rows, dtype=torch.float64, device="cuda")
xs, it, rel = sk.cg(a, b, tol=1e-8, max_iter=200)
assert rel < 1e-8, rel
P, G = 3, 32
slabs = pt.slab_bounds(csr.num_rows, G, P)
import ctypes as C  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402
ranges = []
for sl in slabs:
    cr = (C.c_uint64 * 2)()
    sk._check(lib().spmvk_csr_column_range(csr._h, sl.row_begin, sl.row_end, cr))
    ranges.append((int(cr[0]), int(cr[1])))
recv = pt.fused_receive_ranges(slabs, ranges, "halo")
wins = [pt.ExchangeWindow(csr.num_rows, 8) for _ in slabs]
x0 = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda()
its = []
for sl in slabs:
    it = pt.FusedIteratedSpmv(sl, recv, sk.build_rgcsr(csr, G, 8, row_range=(sl.row_begin,
                                                                            sl.row_end)),
                              wins[sl.rank], P, torch.cuda.current_stream().cuda_stream,
                              local_windows=wins, barrier=False)
    it.set_x(x0)
    its.append(it)
for _ in range(3):
    for it in its:
        it.step()
torch.cuda.synchronize()
for it in its:
    it.close()
for w in wins:
    w.close()
# fused-exchange distributed CG on local windows (direction kernel -> peer stores)
wins = [pt.ExchangeWindow(csr.num_rows, 8) for _ in slabs]
s0 = torch.cuda.current_stream().cuda_stream
ranks = []
for sl in slabs:
    a_s = sk.build_rgcsr(csr, G, 8, row_range=(sl.row_begin, sl.row_end))
    f = pt.FusedIteratedSpmv(sl, recv, a_s, wins[sl.rank], P, s0, local_windows=wins,
                             barrier=False)
    ranks.append(pt.FusedCgRank(sl, a_s, f, b[sl.row_begin:sl.row_end], s0))


def all_reduce(ts):
    total = ts[0].clone()
    for t in ts[1:]:
        total += t
    for t in ts:
        t.copy_(total)


pt.fused_cg(ranks, all_reduce, float(torch.dot(b, b)), tol=0.0, max_iter=5, check_every=5,
            barrier=False)
torch.cuda.synchronize()
for rk in ranks:
    rk.f.close()
for w in wins:
    w.close()
torch.cuda.synchronize()
# round 2: every kept K2 variant (incl. the L2-hinted ones) and the Hybrid
# group-walk shapes on the same matrices, the empty-column shape, an offset
# (8-byte aligned) x view, the NCCL iterated product at world size 1, and the
# bounded barrier timing out on a missing peer
om = orc.powerlaw(20000, 7)
m = triplets(om)
for prec, dt in ((8, np.float64), (4, np.float32)):
    x = orc.random_vector(om.cols, 1).astype(dt)
    want = orc.spmv_rgcsr(orc.build_rgcsr(om, 32, prec), x)[0]
    a = sk.build_rgcsr(m, 32, prec)
    for v in ("liteh", "lite8h", "pipe", "lite8", "lite"):
        lib().spmvk_set_rgcsr_kernel(v.encode())
        assert sk.spmv_rgcsr(a, torch.from_numpy(x).cuda()).cpu().numpy().tobytes() == \
            want.tobytes(), v
    lib().spmvk_set_rgcsr_kernel(b"auto")
    for name, o2 in (("5pt", orc.stencil(5, 64)), ("27pt", orc.stencil(27, 16)), ("pl", om)):
        h = sk.build_hybrid(triplets(o2), None, prec)
        x2 = orc.random_vector(o2.cols, 1).astype(dt)
        want = orc.spmv_hybrid(orc.build_hybrid(o2, None, prec), x2)
        for v in ("g6", "g7", "g8", "g8r", "litefh", "auto"):
            lib().spmvk_set_hybrid_kernel(v.encode())
            assert sk.spmv_hybrid(h, torch.from_numpy(x2).cuda()).cpu().numpy().tobytes() == \
                want.tobytes(), (name, v)
    lib().spmvk_set_hybrid_kernel(b"auto")
e = sk.build_rgcsr(sk.TripletMatrix(100, 0, np.zeros(101, np.uint32), np.zeros(0, np.uint32),
                                    np.zeros(0)), 32)
assert not sk.spmv_rgcsr(e, torch.empty(0, dtype=torch.float64, device="cuda")).any()
o5 = orc.stencil(5, 64)
buf = torch.zeros(o5.cols + 1, dtype=torch.float64, device="cuda")
buf[1:] = torch.from_numpy(orc.random_vector(o5.cols, 1)).cuda()
want = orc.spmv_rgcsr(orc.build_rgcsr(o5, 32), orc.random_vector(o5.cols, 1))[0]
assert sk.spmv_rgcsr(sk.build_rgcsr(triplets(o5), 32), buf[1:]).cpu().numpy().tobytes() == \
    want.tobytes()
for mode in ("allgather", "halo"):
    comm = pt.NcclComm.init_rank(pt.NcclComm.unique_id(), 1, 0, 0)
    sl = pt.slab_bounds(csr.num_rows, 32, 1)[0]
    it = pt.NcclIteratedSpmv(comm, sl, sk.build_rgcsr(csr, 32, 8), csr.num_rows, mode,
                             torch.cuda.current_stream().cuda_stream)
    it.set_x(x0)
    for _ in range(3):
        it.step()
    torch.cuda.synchronize()
    it.close()
    comm.close()
wins = [pt.ExchangeWindow(csr.num_rows, 8) for _ in range(2)]
sl2 = pt.slab_bounds(csr.num_rows, 32, 2)
it = pt.FusedIteratedSpmv(sl2[0], [(0, csr.num_rows)] * 2,
                          sk.build_rgcsr(csr, 32, 8, row_range=(sl2[0].row_begin,
                                                                sl2[0].row_end)),
                          wins[0], 2, torch.cuda.current_stream().cuda_stream,
                          local_windows=wins, barrier=True)
lib().spmvk_dist_set_timeout_ms(it._d, 50)
it.step()
assert lib().spmvk_dist_status(it._d, None) == 4
it.close()
for w in wins:
    w.close()
torch.cuda.synchronize()
# round 2 (later): long rows fused into the row-pipelined kernel (dynamic
# items + dynamic row slices) and the separate launch, both orders, repeated
# launches on one stream (the per-stream counters reset themselves); the
# handle-array block cache reusing a released block under a queued SpMV
for order in ("orig", "desc"):
    c = sk.build_csr(m) if order == "orig" else sk.apply_descending_permutation(sk.build_csr(m))[0]
    rp, col, val = c.to_host()
    oc = orc.Csr(c.num_rows, c.num_cols, rp, col, val)
    for prec, dt in ((8, np.float64), (4, np.float32)):
        x = orc.random_vector(oc.cols, 1).astype(dt)
        want = orc.spmv_rgcsr(orc.build_rgcsr(oc, 32, prec), x)[0]
        a = sk.build_rgcsr(c, 32, prec)
        for fused in (1, 0):
            lib().spmvk_set_long_fused(fused)
            for v in ("pipe", "lite8", "lite8h", "auto"):
                lib().spmvk_set_rgcsr_kernel(v.encode())
                for _ in range(2):
                    assert sk.spmv_rgcsr(a, torch.from_numpy(x).cuda()).cpu().numpy().tobytes() \
                        == want.tobytes(), (order, prec, fused, v)
        lib().spmvk_set_long_fused(1)
        lib().spmvk_set_rgcsr_kernel(b"auto")
big = sk.CsrMatrix.stencil(27, 40)
xb = torch.from_numpy(orc.random_vector(big.num_cols, 1)).cuda()
a = sk.build_rgcsr(big, 32)
want = sk.spmv_rgcsr(a, xb).cpu().numpy()
yb = torch.empty_like(xb)
for _ in range(5):
    sk.spmv_rgcsr(a, xb, yb)
del a
a = sk.build_rgcsr(big, 32)
assert yb.cpu().numpy().tobytes() == want.tobytes()
assert sk.spmv_rgcsr(a, xb).cpu().numpy().tobytes() == want.tobytes()
torch.cuda.synchronize()
print("sanitize pass ok")
