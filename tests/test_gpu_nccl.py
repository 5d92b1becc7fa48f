"""The multi-GPU boundary in host C++ (spmvk_plan_* / spmvk_comm_* /
spmvk_nccl_iter_*, csrc/nccl_dist.cu) driven through ctypes -- no
torch.distributed anywhere on the path.

World size 1 runs on any box (ncclCommInitRank with a fresh unique id, and
ncclCommInitAll over one device).  With >= 2 visible GPUs the same checks
run over ncclCommInitAll in one process (the per-rank calls of a step
bracketed by ncclGroupStart/End), and the fused peer-window step runs across
devices through spmvk_dist_open_local; they skip on a one-GPU box.
Bar: the iterate is bitwise the single-GPU iterate."""
import numpy as np
import pytest
import torch

from helpers import bitwise
from paper_1012_2270_b200 import generators as gen
from paper_1012_2270_b200 import partition as pt
from paper_1012_2270_b200 import spmvkit as sk
from paper_1012_2270_b200._lib import lib

pytestmark = pytest.mark.gpu
MODES = ["allgather", "halo"]


def single_gpu_iterate(csr, G, prec, x0, steps):
    a = sk.build_rgcsr(csr, G, prec)
    x = x0.clone()
    for _ in range(steps):
        x = sk.spmv_rgcsr(a, x) * 0.0625  # exact power-of-two scale
    return x


def as_prec(csr, prec):
    if prec == 8:
        return csr
    return sk.build_csr(sk.TripletMatrix(csr.num_rows, csr.num_cols, *csr.to_host()), 4)


def test_nccl_version(cuda):
    import ctypes as C
    v = C.c_int()
    assert lib().spmvk_nccl_version(C.byref(v)) == 0
    assert v.value >= 22700, v.value  # 2.27+


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("init", ["rank", "all"])
@pytest.mark.parametrize("name", ["7pt-24", "powerlaw"])
def test_world1_bitwise(cuda, mode, init, name):
    csr8 = sk.CsrMatrix.stencil(7, 24) if name == "7pt-24" else sk.build_csr(gen.powerlaw(6000, 7))
    G, steps = 32, 6
    for prec in (8, 4):
        csr = as_prec(csr8, prec)
        dt = torch.float64 if prec == 8 else torch.float32
        x0 = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda().to(dt)
        want = single_gpu_iterate(csr, G, prec, x0, steps)
        comm = (pt.NcclComm.init_rank(pt.NcclComm.unique_id(), 1, 0, 0) if init == "rank"
                else pt.NcclComm.init_all([0])[0])
        sl = pt.slab_bounds(csr.num_rows, G, 1)[0]
        a = sk.build_rgcsr(csr, G, prec, row_range=(sl.row_begin, sl.row_end))
        s = torch.cuda.current_stream().cuda_stream
        it = pt.NcclIteratedSpmv(comm, sl, a, csr.num_rows, mode, s)
        it.set_x(x0)
        for _ in range(steps):
            it.step()
        torch.cuda.synchronize()
        assert bitwise(it.x_current.cpu().numpy(), want.cpu().numpy()), (name, mode, prec)
        assert it.halo_entries() == 0
        it.close()
        comm.close()


def test_nccl_iter_argument_errors(cuda):
    import ctypes as C
    L = lib()
    comm = pt.NcclComm.init_all([0])[0]
    csr = sk.CsrMatrix.stencil(5, 40)
    a = sk.build_rgcsr(csr, 32, 8, row_range=(0, 1600))
    h = C.c_void_p()
    assert L.spmvk_nccl_iter_create(comm._h, a._h, 0, 1600, 1600, 1600, 7, C.byref(h)) == 1
    assert L.spmvk_nccl_iter_create(comm._h, a._h, 0, 1599, 1600, 1600, 0, C.byref(h)) == 1
    assert L.spmvk_nccl_iter_create(comm._h, a._h, 0, 1600, 1600, 1000, 1, C.byref(h)) == 1
    assert L.spmvk_nccl_iter_create(comm._h, a._h, 0, 1600, 1600, 1600, 1, C.byref(h)) == 0
    y = torch.empty(1600, dtype=torch.float32, device="cuda")
    assert L.spmvk_nccl_iter_step_f32(h, 0.5, y.data_ptr(), None) == 1  # fp64 slab
    L.spmvk_nccl_iter_destroy(h)
    comm.close()


ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
multi = pytest.mark.skipif(ndev < 2, reason="needs >= 2 GPUs in this process")


@multi
@pytest.mark.parametrize("mode", MODES)
def test_multi_device_nccl_bitwise(cuda, mode):
    P = min(ndev, 8)
    csr0 = sk.CsrMatrix.stencil(7, 32)
    G, steps, N = 32, 8, csr0.num_rows
    x0h = gen.random_vector(N, 1)
    want = single_gpu_iterate(csr0, G, 8, torch.from_numpy(x0h).cuda(), steps).cpu().numpy()
    slabs = pt.slab_bounds(N, G, P)
    comms = pt.NcclComm.init_all(list(range(P)))
    its, streams = [], []
    L = lib()
    for r in range(P):
        torch.cuda.set_device(r)
        assert L.spmvk_init(r) == 0
        csr = sk.CsrMatrix.stencil(7, 32)
        sl = slabs[r]
        a = sk.build_rgcsr(csr, G, 8, row_range=(sl.row_begin, sl.row_end))
        st = torch.cuda.Stream(device=r)
        streams.append(st)
        its.append((a, csr, st))
    # creation is collective and synchronous (it gathers the ranks' plans):
    # one host thread per rank
    import threading
    made, errs = [None] * P, []

    def create(r):
        try:
            torch.cuda.set_device(r)
            a, _, st = its[r]
            made[r] = pt.NcclIteratedSpmv(comms[r], slabs[r], a, N, mode, st.cuda_stream)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=create, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in range(P):
        torch.cuda.set_device(r)
        made[r].set_x(torch.from_numpy(x0h).cuda(r))
        torch.cuda.synchronize(r)
    for _ in range(steps):
        assert L.spmvk_nccl_group_start() == 0
        for r in range(P):
            torch.cuda.set_device(r)
            made[r].step()
        assert L.spmvk_nccl_group_end() == 0
    for r in range(P):
        torch.cuda.synchronize(r)
        sl = slabs[r]
        got = made[r].x_current.cpu().numpy()
        assert bitwise(got[sl.row_begin:sl.row_end], want[sl.row_begin:sl.row_end]), (r, mode)
    for m in made:
        m.close()
    for c in comms:
        c.close()
    torch.cuda.set_device(0)


@multi
def test_multi_device_fused_peer_windows(cuda):
    """The fused step across real devices in one process: peer stores into
    windows on other GPUs (cudaDeviceEnablePeerAccess) + the flag barrier."""
    P = min(ndev, 8)
    csr0 = sk.CsrMatrix.stencil(7, 32)
    G, steps, N = 32, 8, csr0.num_rows
    x0h = gen.random_vector(N, 1)
    want = single_gpu_iterate(csr0, G, 8, torch.from_numpy(x0h).cuda(), steps).cpu().numpy()
    slabs = pt.slab_bounds(N, G, P)
    import ctypes as C
    ranges = []
    for sl in slabs:
        cr = (C.c_uint64 * 2)()
        sk._check(lib().spmvk_csr_column_range(csr0._h, sl.row_begin, sl.row_end, cr))
        ranges.append((int(cr[0]), int(cr[1])))
    recv = pt.fused_receive_ranges(slabs, ranges, "halo")
    wins, its = [], []
    for r in range(P):
        torch.cuda.set_device(r)
        assert lib().spmvk_init(r) == 0
        wins.append(pt.ExchangeWindow(N, 8))
    for r in range(P):
        torch.cuda.set_device(r)
        csr = sk.CsrMatrix.stencil(7, 32)
        a = sk.build_rgcsr(csr, G, 8, row_range=(slabs[r].row_begin, slabs[r].row_end))
        st = torch.cuda.Stream(device=r)
        it = pt.FusedIteratedSpmv(slabs[r], recv, a, wins[r], P, st.cuda_stream,
                                  local_windows=wins, barrier=True)
        it.set_x(torch.from_numpy(x0h).cuda(r))
        its.append((it, a, st))
    for r in range(P):
        torch.cuda.synchronize(r)
    for _ in range(steps):
        for r in range(P):
            torch.cuda.set_device(r)
            its[r][0].step()
    for r in range(P):
        torch.cuda.synchronize(r)
        it = its[r][0]
        assert lib().spmvk_dist_status(it._d, None) == 0, sk._lib.last_error()
        lo, hi = recv[r]
        assert bitwise(it.x_current[lo:hi].cpu().numpy(), want[lo:hi]), r
    for it, _, _ in its:
        it.close()
    for w in wins:
        w.close()
    torch.cuda.set_device(0)
