"""CG around the RgCSR SpMV (not in the reference): converges
on SPD stencil systems and matches a direct sparse solve (scipy, test-only)."""
import numpy as np
import pytest
import torch

import oracle as orc
from helpers import triplets
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n", [(5, 64), (7, 24), (27, 16)])
def test_cg_solves_stencil_systems(cuda, kind, n):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    om = orc.stencil(kind, n)
    a = sk.build_rgcsr(triplets(om), 32)
    bh = orc.random_vector(om.rows, 3)
    b = torch.from_numpy(bh).cuda()
    x, iters, rel = sk.cg(a, b, tol=1e-10, max_iter=5000)
    assert rel <= 1e-10 and 0 < iters < 5000
    xh = x.cpu().numpy()
    # true residual with the reference-order SpMV
    r = bh - orc.spmv_rgcsr(orc.build_rgcsr(om, 32), xh)[0]
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(bh)
    A = sp.csr_matrix((om.val, om.col.astype(np.int64), om.rp.astype(np.int64)),
                      shape=(om.rows, om.cols))
    xs = spl.spsolve(A.tocsc(), bh)
    assert np.linalg.norm(xh - xs) <= 1e-7 * np.linalg.norm(xs)


def test_dot_is_deterministic(cuda):
    from paper_1012_2270_b200._lib import lib
    v = torch.from_numpy(orc.random_vector(1_000_003, 5)).cuda()
    w = torch.from_numpy(orc.random_vector(1_000_003, 6)).cuda()
    out = torch.empty(4, dtype=torch.float64, device="cuda")
    for i in range(4):
        assert lib().spmvk_dot_f64(v.data_ptr(), w.data_ptr(), v.numel(),
                                   out[i:].data_ptr(), None) == 0
    o = out.cpu().numpy()
    assert len(set(o.tobytes()[k:k + 8] for k in range(0, 32, 8))) == 1
    assert abs(o[0] - float(np.dot(v.cpu().numpy(), w.cpu().numpy()))) < 1e-9 * abs(o[0]) + 1e-9


def test_distributed_cg_world1_nccl_matches_single_gpu_solver(cuda, tmp_path):
    """partition.distributed_cg over NCCL at world size 1 runs the same kernels
    in the same order as spmvk_cg_solve_f64: after K iterations x is bitwise equal."""
    import torch.distributed as dist
    from paper_1012_2270_b200 import partition as part
    om = orc.stencil(7, 32)
    a = sk.build_rgcsr(triplets(om), 32)
    b = torch.from_numpy(orc.random_vector(om.rows, 3)).cuda()
    x1, it1, _ = sk.cg(a, b, tol=0.0, max_iter=25, check_every=1000)
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        s = torch.cuda.current_stream().cuda_stream
        slab = part.slab_bounds(om.rows, 32, 1)[0]
        x2, it2, _ = part.distributed_cg(
            slab, 1, om.cols, b, part.GpuCgOps(a, s),
            lambda o, i: dist.all_gather_into_tensor(o, i), lambda t: dist.all_reduce(t),
            tol=0.0, max_iter=25, check_every=1000)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    assert it1 == it2 == 25
    assert torch.equal(x1.view(torch.int64), x2.view(torch.int64))


def test_spmv_dot_fused(cuda):
    """spmvk_rgcsr_spmv_dot_f64: y bitwise the plain SpMV's, dot = x[off:].y to
    1e-12 (relative), bitwise repeatable; row slabs use x_offset; matrices with
    long rows take the unfused fallback."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_1012_2270_b200 import generators as gen
    from paper_1012_2270_b200 import spmvkit as sk
    from paper_1012_2270_b200._lib import lib
    L = lib()
    cases = [(sk.CsrMatrix.stencil(7, 40), None), (sk.CsrMatrix.stencil(5, 300), None),
             (sk.CsrMatrix.stencil(7, 40), (32 * 700, 32 * 1400)),
             (sk.build_csr(gen.powerlaw(30000, 7)), None)]
    for csr, rr in cases:
        a = sk.build_rgcsr(csr, 32, row_range=rr)
        x = torch.from_numpy(gen.random_vector(csr.num_cols, 3)).cuda()
        off = rr[0] if rr else 0
        want = sk.spmv_rgcsr(a, x).cpu().numpy()
        outs = []
        for _ in range(2):
            y = torch.empty(a.num_rows, dtype=torch.float64, device="cuda")
            d = torch.zeros(1, dtype=torch.float64, device="cuda")
            assert L.spmvk_rgcsr_spmv_dot_f64(a._h, x.data_ptr(), x.numel(), y.data_ptr(),
                                              y.numel(), off, d.data_ptr(), None) == 0
            torch.cuda.synchronize()
            assert y.cpu().numpy().tobytes() == want.tobytes()
            outs.append(d.item())
        ref = float(np.dot(x.cpu().numpy()[off:off + a.num_rows], want))
        assert outs[0] == outs[1]  # deterministic
        assert abs(outs[0] - ref) <= 1e-12 * max(1.0, abs(ref)), (outs[0], ref)
    bad = torch.zeros(1, dtype=torch.float64, device="cuda")
    assert L.spmvk_rgcsr_spmv_dot_f64(a._h, x.data_ptr(), x.numel(), y.data_ptr(), y.numel(),
                                      x.numel(), bad.data_ptr(), None) != 0  # offset too large


def test_cg_with_long_rows_graph_captured(cuda):
    """CG on an SPD matrix with rows past the long-row cut (three dense hub
    rows / columns on a 1-D Laplacian): its SpMV is the fused long-row kernel
    (work counters per stream), run eagerly once and then replayed from the
    CUDA graph CG captures -- the solution must match a direct solve."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    n = 20000
    hubs = [0, 7000, 15000]
    rng = np.random.default_rng(5)
    rows, cols, vals = [], [], []
    for i in range(n):  # 1-D Laplacian
        rows += [i]
        cols += [i]
        vals += [4.0]
        if i:
            rows += [i, i - 1]
            cols += [i - 1, i]
            vals += [-1.0, -1.0]
    for h in hubs:  # symmetric dense-ish hub row / column, diagonally dominated
        js = rng.choice(np.setdiff1d(np.arange(n), [h - 1, h, h + 1]), 600, replace=False)
        w = -rng.random(600) / 700.0
        rows += [h] * 600 + list(js)
        cols += list(js) + [h] * 600
        vals += list(w) + list(w)
    A = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    om = orc.Csr(n, n, A.indptr.astype(np.uint32), A.indices.astype(np.uint32), A.data)
    assert int(om.lens().max()) > 128
    a = sk.build_rgcsr(triplets(om), 32)
    bh = orc.random_vector(n, 9)
    x, iters, rel = sk.cg(a, torch.from_numpy(bh).cuda(), tol=1e-10, max_iter=2000)
    assert rel <= 1e-10 and 0 < iters < 2000
    xs = spl.spsolve(A.tocsc(), bh)
    assert np.linalg.norm(x.cpu().numpy() - xs) <= 1e-7 * np.linalg.norm(xs)
