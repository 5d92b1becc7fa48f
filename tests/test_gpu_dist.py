"""Fused distributed step over peer memory (spmvk_dist_*).

The SpMV's row epilogue stores x_{k+1} into the exchange windows of every
rank whose receive range covers the row; after any number of steps each
rank's window must hold the 1-GPU iterate bitwise on its receive range.

* test_local_ranks_*: P ranks in this process on one GPU (spmvk_dist_open_local),
  stepped in turn without the device barrier -- covers the epilogue routing for
  P = 1..8, both plans, fp64 / fp32, long rows (power-law tail kernel).
* test_two_processes_ipc_barrier: 2-3 processes on the same GPU exchange
  cudaIpcMemHandles over gloo and run the real path -- IPC-mapped peer stores
  plus the release/acquire flag barrier every step.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from helpers import bitwise
from paper_1012_2270_b200 import generators as gen
from paper_1012_2270_b200 import partition as pt
from paper_1012_2270_b200 import spmvkit as sk

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def as_prec(csr, prec):
    if prec == 8:
        return csr
    return sk.build_csr(sk.TripletMatrix(csr.num_rows, csr.num_cols, *csr.to_host()), 4)


def column_ranges(csr, slabs):
    import ctypes as C

    from paper_1012_2270_b200._lib import lib
    out = []
    for s in slabs:
        cr = (C.c_uint64 * 2)()
        sk._check(lib().spmvk_csr_column_range(csr._h, s.row_begin, s.row_end, cr))
        out.append((int(cr[0]), int(cr[1])))
    return out


def reference_iterates(csr, G, prec, x0, steps):
    a = sk.build_rgcsr(csr, G, prec)
    x, ys = x0.clone(), []
    for _ in range(steps):
        y = sk.spmv_rgcsr(a, x)
        ys.append(y)
        x = y * 0.0625  # exact power-of-two scale, as the kernel's epilogue
    return x, ys


MATRICES = {
    "7pt-24": lambda: sk.CsrMatrix.stencil(7, 24),
    "banded": lambda: sk.build_csr(gen.banded(5000, 7, 3)),
    "powerlaw": lambda: sk.build_csr(gen.powerlaw(6000, 7)),  # rows > 128: long-row kernel
}


@pytest.mark.parametrize("mode", ["allgather", "halo"])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name", sorted(MATRICES))
def test_local_ranks_match_single_gpu(cuda, name, P, mode):
    G, steps = 32, 5
    for prec in (8, 4):
        csr = as_prec(MATRICES[name](), prec)
        dt = torch.float64 if prec == 8 else torch.float32
        x0 = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda().to(dt)
        want_x, want_y = reference_iterates(csr, G, prec, x0, steps)
        slabs = pt.slab_bounds(csr.num_rows, G, P)
        recv = pt.fused_receive_ranges(slabs, column_ranges(csr, slabs), mode)
        n = max(csr.num_cols, slabs[-1].row_end)
        wins = [pt.ExchangeWindow(n, prec) for _ in slabs]
        s = torch.cuda.current_stream().cuda_stream
        its = []
        for sl in slabs:
            a = sk.build_rgcsr(csr, G, prec, row_range=(sl.row_begin, sl.row_end))
            it = pt.FusedIteratedSpmv(sl, recv, a, wins[sl.rank], P, s, local_windows=wins,
                                      barrier=False)
            it.set_x(x0)
            its.append(it)
        for k in range(steps):
            for it in its:
                it.step()
            for it in its:
                sl = it.slab
                assert bitwise(it.y[: sl.rows].cpu().numpy(),
                               want_y[k][sl.row_begin: sl.row_end].cpu().numpy()), (k, sl)
        torch.cuda.synchronize()
        for it in its:
            lo, hi = recv[it.slab.rank]
            got = it.window.x[it.cur][lo:hi].cpu().numpy()
            assert bitwise(got, want_x[lo:hi].cpu().numpy()), (name, P, mode, prec, it.slab)
            it.close()
        for w in wins:
            w.close()


def test_window_and_dist_argument_errors(cuda):
    import ctypes as C

    from paper_1012_2270_b200._lib import lib
    L = lib()
    h = C.c_void_p()
    assert L.spmvk_window_create(100, 3, C.byref(h)) != 0  # bad precision
    w = pt.ExchangeWindow(100, 8)
    d = C.c_void_p()
    arr = (C.c_void_p * 1)(w._h.value)
    assert L.spmvk_dist_open_local(arr, 1, 1, C.byref(d)) != 0  # rank outside world
    assert L.spmvk_dist_open_local(arr, 0, 9, C.byref(d)) != 0  # world > 8
    assert L.spmvk_dist_open_local(arr, 0, 1, C.byref(d)) == 0
    rr = (C.c_uint64 * 2)(0, 100)
    assert L.spmvk_dist_set_rows(d, 0, 101, rr) != 0  # past the window
    assert L.spmvk_dist_set_rows(d, 0, 64, rr) == 0
    a = sk.build_rgcsr(sk.CsrMatrix.stencil(5, 10), 32, 8)  # 100 rows != 64
    y = torch.empty(100, dtype=torch.float64, device="cuda")
    assert L.spmvk_dist_step_f64(d, a._h, 0.5, y.data_ptr(), 0, None) != 0
    assert "slab rows" in sk._lib.last_error()
    assert L.spmvk_dist_step_f32(d, a._h, 0.5, y.data_ptr(), 0, None) != 0  # precision
    L.spmvk_dist_destroy(d)
    w.close()


CHILD = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
from paper_1012_2270_b200 import generators as gen, partition as pt, spmvkit as sk
from paper_1012_2270_b200._lib import lib
from test_gpu_dist import column_ranges, reference_iterates, bitwise
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["PORT"],
                        rank=rank, world_size=world)
torch.cuda.set_device(0)
assert lib().spmvk_init(0) == 0
mode, steps, G = os.environ["MODE"], int(os.environ.get("STEPS", "12")), 32
csr = sk.CsrMatrix.stencil(7, 24)
x0 = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda()
want_x, _ = reference_iterates(csr, G, 8, x0, steps)
slabs = pt.slab_bounds(csr.num_rows, G, world)
me = slabs[rank]
recv = pt.fused_receive_ranges(slabs, column_ranges(csr, slabs), mode)
a = sk.build_rgcsr(csr, G, 8, row_range=(me.row_begin, me.row_end))
win = pt.ExchangeWindow(max(csr.num_cols, slabs[-1].row_end), 8)
hs = [None] * world
dist.all_gather_object(hs, win.ipc_handle())
s = torch.cuda.Stream()
it = pt.FusedIteratedSpmv(me, recv, a, win, world, s.cuda_stream, handles=hs)
with torch.cuda.stream(s):
    it.set_x(x0)
s.synchronize()
dist.barrier()
for _ in range(steps):
    it.step()
s.synchronize()
lo, hi = recv[rank]
ok = bitwise(it.window.x[it.cur][lo:hi].cpu().numpy(), want_x[lo:hi].cpu().numpy())
it.close()
dist.barrier()
win.close()
print("ok" if ok else "MISMATCH", flush=True)
'''


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return str(s.getsockname()[1])


@pytest.mark.parametrize("mode,world,steps", [("halo", 2, 12), ("allgather", 2, 12),
                                              ("halo", 3, 12), ("allgather", 4, 12),
                                              ("halo", 3, 150)])
def test_two_processes_ipc_barrier(cuda, mode, world, steps):
    port = free_port()
    procs = [subprocess.Popen([sys.executable, "-c", CHILD], cwd=ROOT, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True,
                              env=dict(os.environ, ROOT=ROOT, RANK=str(r), WORLD_SIZE=str(world),
                                       PORT=port, MODE=mode, STEPS=str(steps)))
             for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=240))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (out, err) in zip(procs, outs):
        assert p.returncode == 0 and out.strip().endswith("ok"), err[-3000:]


def _bench_json(world, workload, steps=6):
    """bench.py's N > 1 leg under torchrun with every rank on GPU 0
    (SPMVK_SHARE_GPU=1, gloo plumbing, fused exchange over CUDA IPC)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           "bench.py", "--gpus", str(world), "--workload", workload, "--steps", str(steps),
           "--warmup", "3", "--distributed"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, SPMVK_SHARE_GPU="1"))
    assert p.returncode == 0, p.stderr[-3000:]
    import json
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def _bench_ref_config(world, workload):
    """The config dict the reference arm prints for the same run."""
    sys.path.insert(0, ROOT)
    import bench
    return bench.bench_config(workload, world, "fused")


@pytest.mark.parametrize("workload", ["27pt-128"])
def test_bench_distributed_shared_gpu_bitwise(cuda, workload):
    """The driver's scaling run path (bench.py under torchrun, N ranks, fused
    exchange + flag barrier) on one GPU: after the same number of steps the
    final iterate's bit checksum is identical at 1, 2 and 3 ranks."""
    ref = _bench_json(1, workload)
    assert ref["n_gpus"] == 1 and ref["x_bits_checksum"] != 0
    for world in (2, 3):
        d = _bench_json(world, workload)
        assert d["n_gpus"] == world and d["exchange"]["exchange_fallback"] is None
        assert d["exchange"]["shared_gpu"]
        assert d["config"] == _bench_ref_config(world, workload)
        assert d["x_bits_checksum"] == ref["x_bits_checksum"], world
        assert d["e2e"]["value"] > 0 and d["gpu_launches"] == 2 * d["steps"]


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_fused_cg_local_ranks(cuda, P):
    """Distributed CG with the p exchange fused into the direction step
    (spmvk_dist_cg_direction_f64: p_new stored into the peers' windows, no
    all-gather), P ranks on one GPU stepped in turn.  P = 1 is bitwise the
    single-GPU solver (same kernels, same dots); P > 1 differs only in the
    dots' summation order."""
    csr = sk.CsrMatrix.stencil(7, 24)
    N, G, iters = csr.num_rows, 32, 40
    b = torch.from_numpy(gen.random_vector(N, 9)).cuda()
    a_full = sk.build_rgcsr(csr, G)
    x1, it1, _ = sk.cg(a_full, b, tol=0.0, max_iter=iters, check_every=10)
    assert it1 == iters
    slabs = pt.slab_bounds(N, G, P)
    recv = pt.fused_receive_ranges(slabs, column_ranges(csr, slabs), "halo")
    wins = [pt.ExchangeWindow(N, 8) for _ in slabs]
    s = torch.cuda.current_stream().cuda_stream
    ranks = []
    for sl in slabs:
        a = sk.build_rgcsr(csr, G, row_range=(sl.row_begin, sl.row_end))
        f = pt.FusedIteratedSpmv(sl, recv, a, wins[sl.rank], P, s, local_windows=wins,
                                 barrier=False)
        ranks.append(pt.FusedCgRank(sl, a, f, b[sl.row_begin:sl.row_end], s))

    def all_reduce(ts):
        total = ts[0].clone()
        for t in ts[1:]:
            total += t
        for t in ts:
            t.copy_(total)

    k, res = pt.fused_cg(ranks, all_reduce, float(torch.dot(b, b)), tol=0.0, max_iter=iters,
                         check_every=10, barrier=False)
    assert k == iters
    x = torch.cat([rk.x[: rk.slab.rows] for rk in ranks]).cpu().numpy()
    want = x1.cpu().numpy()
    if P == 1:
        assert bitwise(x, want)
    else:
        assert np.abs(x - want).max() <= 1e-10 * np.abs(want).max()
    for rk in ranks:
        rk.f.close()
    for w in wins:
        w.close()


CG_CHILD = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
from paper_1012_2270_b200 import generators as gen, partition as pt, spmvkit as sk
from paper_1012_2270_b200._lib import lib
from test_gpu_dist import column_ranges
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["PORT"],
                        rank=rank, world_size=world)
torch.cuda.set_device(0)
assert lib().spmvk_init(0) == 0
G, iters = 32, 30
csr = sk.CsrMatrix.stencil(7, 24)
N = csr.num_rows
b = torch.from_numpy(gen.random_vector(N, 9)).cuda()
x1, _, _ = sk.cg(sk.build_rgcsr(csr, G), b, tol=0.0, max_iter=iters, check_every=10)
slabs = pt.slab_bounds(N, G, world)
me = slabs[rank]
recv = pt.fused_receive_ranges(slabs, column_ranges(csr, slabs), "halo")
a = sk.build_rgcsr(csr, G, 8, row_range=(me.row_begin, me.row_end))
win = pt.ExchangeWindow(N, 8)
hs = [None] * world
dist.all_gather_object(hs, win.ipc_handle())
s = torch.cuda.Stream()
f = pt.FusedIteratedSpmv(me, recv, a, win, world, s.cuda_stream, handles=hs)
with torch.cuda.stream(s):
    rk = pt.FusedCgRank(me, a, f, b[me.row_begin:me.row_end], s.cuda_stream)
s.synchronize()
dist.barrier()

def all_reduce(ts):  # scalars through the host (gloo): rank-order sum
    s.synchronize()
    v = ts[0].cpu()
    dist.all_reduce(v)
    ts[0].copy_(v.cuda())

k, res = pt.fused_cg([rk], all_reduce, float(torch.dot(b, b)), tol=0.0, max_iter=iters,
                     check_every=10, barrier=True)
s.synchronize()
x = rk.x[: me.rows]
want = x1[me.row_begin:me.row_end]
ok = k == iters and float((x - want).abs().max()) <= 1e-10 * float(x1.abs().max())
f.close()
dist.barrier()
win.close()
print("ok" if ok else "MISMATCH", flush=True)
'''


@pytest.mark.parametrize("world", [2, 3])
def test_fused_cg_ipc_processes(cuda, world):
    """The fused-exchange CG across real processes: CUDA IPC peer windows,
    p_new stored by the direction kernel into the peers' windows, the flag
    barrier every iteration, dots all-reduced over gloo; x matches the
    single-GPU solver to 1e-10."""
    port = free_port()
    procs = [subprocess.Popen([sys.executable, "-c", CG_CHILD], cwd=ROOT, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True,
                              env=dict(os.environ, ROOT=ROOT, RANK=str(r), WORLD_SIZE=str(world),
                                       PORT=port))
             for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=300))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (out, err) in zip(procs, outs):
        assert p.returncode == 0 and out.strip().endswith("ok"), err[-3000:]
