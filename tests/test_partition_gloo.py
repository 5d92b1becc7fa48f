"""Multi-process (gloo, world_size 2 and 3) checks of the row-slab partitioner
and the iterated distributed SpMV loop (paper_1012_2270_b200.partition).
The per-slab SpMV is the oracle here (CPU); on the GPU it is K2 fused with the
x_{k+1} scale.  The distributed iterate must be bitwise the 1-process one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_1012_2270_b200 import partition as part


def slab_csr(m: orc.Csr, r0, r1) -> orc.Csr:
    b, e = int(m.rp[r0]), int(m.rp[r1])
    return orc.Csr(r1 - r0, m.cols, m.rp[r0:r1 + 1] - m.rp[r0], m.col[b:e], m.val[b:e])


def test_slab_bounds_cover_and_align():
    for n in (1, 31, 32, 33, 1000, 2097152):
        for G in (1, 32, 128):
            for P in (1, 2, 3, 4, 8):
                sl = part.slab_bounds(n, G, P)
                assert sl[0].row_begin == 0 and sl[-1].row_end == n
                for a, b in zip(sl, sl[1:]):
                    assert a.row_end == b.row_begin
                for s in sl:
                    assert s.row_begin % G == 0 or s.row_begin == n
                    assert s.rows <= s.pad_rows


def test_weighted_bounds_balance_slots():
    m = orc.powerlaw(50_000, 7)
    cuts = part.weighted_slab_bounds(m.lens(), 32, 4)
    assert cuts[0][0] == 0 and cuts[-1][1] == m.rows
    slots = []
    for r0, r1 in cuts:
        assert r0 % 32 == 0
        slots.append(orc.build_rgcsr(slab_csr(m, r0, r1), 32)["values"].size)
    assert max(slots) < 1.5 * (sum(slots) / len(slots))


def test_slab_rgcsr_is_global_slice():
    m = orc.stencil(27, 10)
    G = 32
    full = orc.build_rgcsr(m, G)
    gp = full["group_pointers"]
    for s in part.slab_bounds(m.rows, G, 3):
        a = orc.build_rgcsr(slab_csr(m, s.row_begin, s.row_end), G)
        g0, g1 = s.row_begin // G, (s.row_end + G - 1) // G
        assert np.array_equal(a["group_pointers"], gp[g0:g1 + 1] - gp[g0])
        assert np.array_equal(a["values"], full["values"][gp[g0]:gp[g1]])


def test_halo_plan_of_7pt_slabs():
    n = 16
    rows = n ** 3
    sl = part.slab_bounds(rows, 32, 4)
    s = sl[1]
    plan = part.halo_plan(s, s.row_begin - n * n, s.row_end - 1 + n * n, sl)
    assert [p[0] for p in plan] == [0, 2]
    assert sum(c1 - c0 for _, c0, c1 in plan) == 2 * n * n


def _worker(rank, world, port, steps, out, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = orc.stencil(7, 12)
    G = 32
    slabs = part.slab_bounds(m.rows, G, world)
    me = slabs[rank]
    a = orc.build_rgcsr(slab_csr(m, me.row_begin, me.row_end), G)

    def slab_spmv(x, y, xn):
        yy = orc.spmv_rgcsr(a, x.numpy())[0]
        y.copy_(torch.from_numpy(yy))
        xn.copy_(torch.from_numpy(yy * 0.0625))

    def all_gather(o, i):
        dist.all_gather_into_tensor(o, i)

    x0 = torch.from_numpy(orc.random_vector(m.cols, 1))
    if mode == "allgather":
        it = part.IteratedSpmv(me, m.cols, world, slab_spmv, all_gather, x0)
    else:
        sc = slab_csr(m, me.row_begin, me.row_end)
        mine = (int(sc.col.min()), int(sc.col.max())) if sc.nnz else (1, 0)
        ranges = [None] * world
        dist.all_gather_object(ranges, mine)
        it = part.HaloIteratedSpmv(me, slabs, ranges, m.cols, slab_spmv, part.torch_p2p, x0)
        # every entry the slab reads must be covered by its own rows + halos
        covered = set(range(me.row_begin, me.row_end))
        for _, c0, c1 in it.recv:
            covered |= set(range(c0, c1))
        assert set(np.unique(a["columns"][a["values"] != 0]).tolist()) <= covered
    it.set_x(x0)
    for _ in range(steps):
        it.step()
    x_now = it.x[: m.cols] if mode == "allgather" else it.x_current
    # gather full x on rank 0 to compare (halo ranks hold only their rows fresh)
    xs = [None] * world
    dist.all_gather_object(xs, (me.row_begin, me.row_end, x_now[me.row_begin:me.row_end].numpy()))
    if rank == 0:
        full = np.empty(m.cols)
        for r0, r1, v in xs:
            full[r0:r1] = v
        out.put(full.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["allgather", "halo"])
@pytest.mark.parametrize("world", [2, 3])
def test_iterated_distributed_equals_single_process(world, mode):
    steps = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, q, mode))
             for r in range(world)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=120), np.float64)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    m = orc.stencil(7, 12)
    full = orc.build_rgcsr(m, 32)
    x = orc.random_vector(m.cols, 1)
    for _ in range(steps):
        x = orc.spmv_rgcsr(full, x)[0] * 0.0625
    assert got.tobytes() == x.tobytes()


class NumpyCgOps:
    """CPU stand-in for the slab kernels of partition.distributed_cg."""

    def __init__(self, a):
        self.a = a

    def spmv(self, p_full, q):
        q.copy_(torch.from_numpy(orc.spmv_rgcsr(self.a, p_full.numpy())[0]))

    def dot(self, a, b, out):
        out.fill_(float(np.dot(a.numpy(), b.numpy())))

    def update(self, rr, pap, p, q, x, r, rrn):
        alpha = float(rr) / float(pap)
        x += alpha * p
        r -= alpha * q
        rrn.fill_(float(torch.dot(r, r)))

    def direction(self, r, p, rr, rrn):
        p.copy_(r + (float(rrn) / float(rr)) * p)
        rr.copy_(rrn)


def _cg_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = orc.stencil(7, 10)
    slabs = part.slab_bounds(m.rows, 32, world)
    me = slabs[rank]
    a = orc.build_rgcsr(slab_csr(m, me.row_begin, me.row_end), 32)
    b = torch.from_numpy(orc.random_vector(m.rows, 4)[me.row_begin:me.row_end].copy())
    x, iters, res = part.distributed_cg(
        me, world, m.cols, b, NumpyCgOps(a),
        lambda o, i: dist.all_gather_into_tensor(o, i), lambda t: dist.all_reduce(t),
        tol=1e-11, max_iter=500, check_every=1)
    xs = [None] * world
    dist.all_gather_object(xs, (me.row_begin, x.numpy(), iters, res))
    if rank == 0:
        full = np.empty(m.rows)
        for r0, v, _, _ in xs:
            full[r0:r0 + v.size] = v
        out.put((full.tobytes(), iters, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_cg_solves(world):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    xb, iters, res = q.get(timeout=180)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    x = np.frombuffer(xb, np.float64)
    m = orc.stencil(7, 10)
    A = sp.csr_matrix((m.val, m.col.astype(np.int64), m.rp.astype(np.int64)), shape=(m.rows, m.cols))
    bh = orc.random_vector(m.rows, 4)
    assert res <= 1e-11 and iters < 500
    assert np.linalg.norm(x - spl.spsolve(A.tocsc(), bh)) <= 1e-8 * np.linalg.norm(x)
