"""Row-slab partitioner and the iterated, distributed SpMV (north_star item 4).

A is cut into P contiguous, group-aligned row slabs, one per GPU (one process
per GPU, torch.distributed over NCCL).  Because slab boundaries are
multiples of the group size G, each slab's RgCSR arrays are exactly the
global build's slice (group pointers rebased) — checked in
tests/test_gpu_rgcsr.py::test_row_slabs_equal_global_slices — so every row
accumulates in the reference's order and the distributed y is bitwise the
1-GPU y.  Columns stay global.

Iteration (a CG-style repeated product):
    y_k = A x_k ;  x_{k+1} = y_k * 2^-4
The scale is fused into the SpMV epilogue (spmvk_rgcsr_spmv_scaled_f64 writes
y and the rank's slab of x_{k+1} in one pass); the slabs are then exchanged
with an NCCL all-gather so every rank holds the whole x_{k+1}.  All slabs
have S = ceil(groups / P) * G rows (the last one is padded), so the
all-gather has equal counts; padding entries of x are never referenced.

The exchange is a real data dependency of the iterated product (every rank
needs every x entry its columns touch), so this is the one place the path
uses a collective.  A halo variant that exchanges only the column ranges a
slab actually reads (``halo_plan``) is the scaling path for banded matrices.
"""
from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass
from typing import Callable, List, Sequence

import numpy as np


@dataclass(frozen=True)
class Slab:
    rank: int
    row_begin: int
    row_end: int  # exclusive; real rows only
    pad_rows: int  # S: rows every slab reserves in the gathered x

    @property
    def rows(self) -> int:
        return self.row_end - self.row_begin


def _u64(values):
    import ctypes as C
    vals = list(values)
    return (C.c_uint64 * max(1, len(vals)))(*vals)


def _plan_check(rc):
    if rc:
        from . import spmvkit as sk
        sk._check(rc)


def slab_bounds(num_rows: int, group_size: int, parts: int) -> List[Slab]:
    """Equal, group-aligned slabs: S = ceil(groups / P) * G rows each
    (spmvk_plan_slabs, csrc/nccl_dist.cu)."""
    import ctypes as C

    from ._lib import lib
    if group_size <= 0 or parts <= 0:
        raise ValueError("group size and part count must be positive")
    b = _u64([0] * (parts + 1))
    S = C.c_uint64()
    _plan_check(lib().spmvk_plan_slabs(num_rows, group_size, parts, b, C.byref(S)))
    return [Slab(p, int(b[p]), int(b[p + 1]), int(S.value)) for p in range(parts)]


def weighted_slab_bounds(row_lengths: Sequence[int], group_size: int, parts: int) -> List[tuple]:
    """Group-aligned cuts balancing stored slots (for skewed matrices such as
    the power-law config): cut p sits at the first group boundary where the
    running slot count reaches p/P of the total (spmvk_plan_slabs_weighted).
    Returns [(r0, r1)]."""
    from ._lib import lib
    lens = np.ascontiguousarray(row_lengths, dtype=np.uint32)
    b = _u64([0] * (parts + 1))
    _plan_check(lib().spmvk_plan_slabs_weighted(lens.ctypes.data if lens.size else None,
                                                lens.size, group_size, parts, b))
    return [(int(b[p]), int(b[p + 1])) for p in range(parts)]


def halo_plan(slab: Slab, column_min: int, column_max: int, slabs: Sequence[Slab]):
    """Ranks whose x slab intersects [column_min, column_max] of this slab's
    columns and the intersecting ranges: [(rank, c0, c1)] excluding self
    (the receive list of spmvk_plan_halo)."""
    import ctypes as C

    from ._lib import lib
    P = len(slabs)
    bounds = _u64([s.row_begin for s in slabs] + [slabs[-1].row_end])
    ranges = [(1, 0)] * P
    ranges[slab.rank] = (column_min, column_max)
    cr = _u64([v for r in ranges for v in r])
    recv, send = _u64([0] * (3 * P)), _u64([0] * (3 * P))
    nr, ns = C.c_int(), C.c_int()
    _plan_check(lib().spmvk_plan_halo(slab.rank, P, bounds, cr, recv, C.byref(nr), send,
                                      C.byref(ns)))
    return [(int(recv[3 * k]), int(recv[3 * k + 1]), int(recv[3 * k + 2]))
            for k in range(nr.value)]


class IteratedSpmv:
    """The distributed iteration loop, independent of where the SpMV runs.

    ``slab_spmv(x_full, y_slab, x_next_slab)`` computes the rank's rows of
    y = A x and x_next = y * scale; ``all_gather(out_full, in_slab)`` is a
    torch.distributed all_gather_into_tensor.  Buffers are torch tensors
    (CUDA under NCCL, CPU under gloo in the tests)."""

    def __init__(self, slab: Slab, num_cols: int, world: int, slab_spmv: Callable,
                 all_gather: Callable, like):
        import torch
        self.slab, self.world = slab, world
        S = slab.pad_rows
        self.x = torch.zeros(S * world, dtype=like.dtype, device=like.device)
        self.x_next = torch.zeros(S, dtype=like.dtype, device=like.device)
        self.y = torch.zeros(S, dtype=like.dtype, device=like.device)
        self.num_cols = num_cols
        self.slab_spmv = slab_spmv
        self.all_gather = all_gather

    def set_x(self, x_full):
        self.x[: x_full.numel()].copy_(x_full)

    def step(self):
        """y_k = A x_k on this slab; x_{k+1} gathered from all slabs."""
        xv = self.x[: self.num_cols]
        self.slab_spmv(xv, self.y[: self.slab.rows], self.x_next[: self.slab.rows])
        self.all_gather(self.x, self.x_next)


class HaloIteratedSpmv:
    """Iterated SpMV exchanging only the x entries each slab reads.

    Each rank knows every slab's column range [cmin, cmax] (all-gathered once
    at setup).  Per step the rank's SpMV reads x_k from ``x[cur]`` and writes
    its own rows of x_{k+1} straight into ``x[nxt]`` (fused scale), then sends
    to every peer the part of its slab that the peer's range covers and
    receives the parts of the peers' slabs its own range covers (point-to-point
    sends/receives, NCCL on GPUs).  For the 7-point stencil a slab reads one
    n^2 plane from each neighbour: 2 * n^2 entries per step instead of the
    whole vector.  ``p2p(ops)`` runs a list of (kind, tensor, peer) with kind
    'send' | 'recv' and waits for them (torch.distributed.batch_isend_irecv)."""

    def __init__(self, slab: Slab, slabs: Sequence[Slab], ranges: Sequence[tuple], num_cols: int,
                 slab_spmv: Callable, p2p: Callable, like):
        import torch
        self.slab, self.num_cols = slab, num_cols
        n = max(num_cols, slabs[-1].row_end)
        self.x = [torch.zeros(n, dtype=like.dtype, device=like.device) for _ in range(2)]
        self.y = torch.zeros(max(slab.rows, 1), dtype=like.dtype, device=like.device)
        self.cur = 0
        self.slab_spmv, self.p2p = slab_spmv, p2p
        me = slab.rank
        cmin, cmax = ranges[me]
        self.recv = [] if cmin > cmax else halo_plan(slab, cmin, cmax, slabs)
        self.send = []
        for q in slabs:
            if q.rank == me or q.rows == 0:
                continue
            qmin, qmax = ranges[q.rank]
            if qmin > qmax:
                continue
            c0, c1 = max(qmin, slab.row_begin), min(qmax + 1, slab.row_end)
            if c0 < c1:
                self.send.append((q.rank, c0, c1))

    def halo_entries(self) -> int:
        return sum(c1 - c0 for _, c0, c1 in self.recv)

    def set_x(self, x_full):
        self.x[self.cur][: x_full.numel()].copy_(x_full)

    @property
    def x_current(self):
        return self.x[self.cur][: self.num_cols]

    def step(self):
        cur, nxt = self.x[self.cur], self.x[1 - self.cur]
        r0, r1 = self.slab.row_begin, self.slab.row_end
        self.slab_spmv(cur[: self.num_cols], self.y[: r1 - r0], nxt[r0:r1])
        ops = [("send", nxt[c0:c1], q) for q, c0, c1 in self.send]
        ops += [("recv", nxt[c0:c1], q) for q, c0, c1 in self.recv]
        if ops:
            self.p2p(ops)
        self.cur = 1 - self.cur


def distributed_cg(slab: Slab, world: int, num_cols: int, b, ops, all_gather, all_reduce,
                   tol: float = 1e-10, max_iter: int = 1000, check_every: int = 10):
    """Conjugate gradients over row slabs (SURVEY §8f-4 on top of the §8e
    partition): every rank owns its rows of A, x, r, p; p is all-gathered
    before each SpMV and the two dot products per iteration are all-reduced
    scalars that never leave the device.

    ``ops`` supplies the slab-local kernels (``spmv(p_full, q)``,
    ``dot(a, b, out)``, ``update(rr, pap, p, q, x, r, rr_new)``,
    ``direction(r, p, rr, rr_new)`` — GpuCgOps wraps the C-ABI; the gloo
    tests pass a numpy stand-in).  Returns (x_slab, iterations, rel_residual)."""
    import torch
    n = slab.rows
    S = slab.pad_rows
    dev, dt = b.device, b.dtype
    x = torch.zeros(max(n, 1), dtype=dt, device=dev)
    r = b.clone() if n else torch.zeros(1, dtype=dt, device=dev)
    p_local = torch.zeros(S, dtype=dt, device=dev)
    p_local[:n] = r[:n]
    p_full = torch.zeros(S * world, dtype=dt, device=dev)
    q = torch.zeros(max(n, 1), dtype=dt, device=dev)
    sc = torch.zeros(4, dtype=dt, device=dev)  # rr, pap, rr_new, bb
    rr, pap, rrn, bb = (sc[i:i + 1] for i in range(4))
    ops.dot(b[:n], b[:n], bb)
    ops.dot(r[:n], r[:n], rr)
    all_reduce(sc[0:1])
    all_reduce(sc[3:4])
    bnorm = float(bb.item()) ** 0.5
    res = (float(rr.item()) ** 0.5) / (bnorm or 1.0)
    k = 0
    while k < max_iter and res > tol:
        all_gather(p_full, p_local)
        if hasattr(ops, "spmv_dot"):  # q = A p with p.q fused into the SpMV epilogue
            ops.spmv_dot(p_full[:num_cols], q[:n], pap, slab.row_begin)
        else:
            ops.spmv(p_full[:num_cols], q[:n])
            ops.dot(p_local[:n], q[:n], pap)
        all_reduce(pap)
        ops.update(rr, pap, p_local[:n], q[:n], x[:n], r[:n], rrn)
        all_reduce(rrn)
        ops.direction(r[:n], p_local[:n], rr, rrn)
        k += 1
        if k % check_every == 0 or k == max_iter:
            res = (float(rr.item()) ** 0.5) / (bnorm or 1.0)
    return x[:n], k, res


class FusedCgRank:
    """One rank of the distributed CG whose p exchange is fused into the
    direction step (spmvk_dist_cg_direction_f64): p lives in the rank's
    exchange window, the direction kernel stores p_new into the next buffer
    of its own window and of every peer that reads the row (NVLink stores),
    then the flag barrier -- no all-gather.  The dots stay scalar all-reduces.
    ``a`` is the rank's slab RgCSR (columns global), ``fused`` its
    FusedIteratedSpmv-style dist handle (window + routing, set up by the
    caller), ``b`` its rows of the right-hand side."""

    def __init__(self, slab: Slab, a, fused, b, stream: int):
        import torch
        from ._lib import lib
        self.slab, self.a, self.f, self.s, self.L = slab, a, fused, stream or None, lib()
        n = slab.rows
        dev = self.dev = b.device
        # the setup runs on the stream the C calls use (ordered before them)
        with self._on_stream():
            self.x = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
            self.r = b.clone() if n else torch.zeros(1, dtype=torch.float64, device=dev)
            self.q = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
            # rr pap rrn bb | 1.0 0.0: the start step's beta = 0 / 1 (it copies
            # sc[5] into sc[4], so start() re-seeds both every time)
            self.sc = torch.zeros(6, dtype=torch.float64, device=dev)
        self.rr, self.pap, self.rrn, self.bb = (self.sc[i:i + 1] for i in range(4))

    def _on_stream(self):
        import contextlib
        import torch
        if not self.s:
            return contextlib.nullcontext()
        ext = torch.cuda.ExternalStream(self.s, device=self.dev)
        ext.wait_stream(torch.cuda.current_stream(self.dev))  # inputs made on torch's stream
        return torch.cuda.stream(ext)

    def _ok(self, rc):
        if rc:
            from . import spmvkit as sk
            sk._check(rc)

    def p_current(self):
        return self.f.window.x[self.f.cur]

    def start(self, barrier: bool):
        """p = r in every window that reads it (a direction step with beta = 0
        over a zeroed p_old), local dots r.r and b.b into rr / bb."""
        sl = self.slab
        with self._on_stream():
            self.p_current()[sl.row_begin:sl.row_end].zero_()
            self.sc[4].fill_(1.0)
            self.sc[5].fill_(0.0)
        self._ok(self.L.spmvk_dist_cg_direction_f64(
            self.f._d, self.r.data_ptr(), self.sc[4:5].data_ptr(), self.sc[5:6].data_ptr(),
            1 if barrier else 0, self.s))
        n = sl.rows
        self._ok(self.L.spmvk_dot_f64(self.r.data_ptr(), self.r.data_ptr(), n, self.rr.data_ptr(),
                                      self.s))

    def spmv_dot(self):
        sl = self.slab
        p = self.p_current()
        self._ok(self.L.spmvk_rgcsr_spmv_dot_f64(self.a._h, p.data_ptr(), self.a.num_cols,
                                                 self.q.data_ptr(), sl.rows, sl.row_begin,
                                                 self.pap.data_ptr(), self.s))

    def update(self):
        sl = self.slab
        p_local = self.p_current()[sl.row_begin:sl.row_end]
        self._ok(self.L.spmvk_cg_update_f64(sl.rows, self.rr.data_ptr(), self.pap.data_ptr(),
                                            p_local.data_ptr(), self.q.data_ptr(),
                                            self.x.data_ptr(), self.r.data_ptr(),
                                            self.rrn.data_ptr(), self.s))

    def direction(self, barrier: bool):
        self._ok(self.L.spmvk_dist_cg_direction_f64(self.f._d, self.r.data_ptr(),
                                                    self.rr.data_ptr(), self.rrn.data_ptr(),
                                                    1 if barrier else 0, self.s))


def fused_cg(ranks, all_reduce, b_dot, tol: float = 1e-10, max_iter: int = 1000,
             check_every: int = 10, barrier: bool = True):
    """Drives FusedCgRank objects through CG.  ``ranks`` are the ranks this
    process steps (one per process on a node; all of them, stepped in turn
    with barrier=False, when a test runs every rank on one GPU);
    ``all_reduce(tensors)`` sums the given per-rank 1-element tensors in rank
    order and writes the sum back into each; ``b_dot`` = global b.b.
    Returns (iterations, relative residual)."""
    bnorm = float(b_dot) ** 0.5 or 1.0
    for rk in ranks:
        rk.start(barrier)
    all_reduce([rk.rr for rk in ranks])
    res = float(ranks[0].rr.item()) ** 0.5 / bnorm
    k = 0
    while k < max_iter and res > tol:
        for rk in ranks:
            rk.spmv_dot()
        all_reduce([rk.pap for rk in ranks])
        for rk in ranks:
            rk.update()
        all_reduce([rk.rrn for rk in ranks])
        for rk in ranks:
            rk.direction(barrier)
        k += 1
        if k % check_every == 0 or k == max_iter:
            res = float(ranks[0].rr.item()) ** 0.5 / bnorm
    return k, res


class GpuCgOps:
    """distributed_cg's slab kernels through the C-ABI (fp64, one stream)."""

    def __init__(self, a, stream: int):
        from ._lib import lib
        from . import spmvkit as sk
        self.a, self.s, self.L, self.sk = a, stream or None, lib(), sk

    def _ok(self, rc):
        if rc:
            self.sk._check(rc)

    def spmv(self, p_full, q):
        self._ok(self.L.spmvk_rgcsr_spmv_f64(self.a._h, p_full.data_ptr(), p_full.numel(),
                                             q.data_ptr(), q.numel(), self.s))

    def spmv_dot(self, p_full, q, out, x_offset):
        self._ok(self.L.spmvk_rgcsr_spmv_dot_f64(self.a._h, p_full.data_ptr(), p_full.numel(),
                                                 q.data_ptr(), q.numel(), x_offset,
                                                 out.data_ptr(), self.s))

    def dot(self, a, b, out):
        self._ok(self.L.spmvk_dot_f64(a.data_ptr(), b.data_ptr(), a.numel(), out.data_ptr(),
                                      self.s))

    def update(self, rr, pap, p, q, x, r, rrn):
        self._ok(self.L.spmvk_cg_update_f64(p.numel(), rr.data_ptr(), pap.data_ptr(),
                                            p.data_ptr(), q.data_ptr(), x.data_ptr(),
                                            r.data_ptr(), rrn.data_ptr(), self.s))

    def direction(self, r, p, rr, rrn):
        self._ok(self.L.spmvk_cg_direction_f64(r.numel(), r.data_ptr(), p.data_ptr(),
                                               rr.data_ptr(), rrn.data_ptr(), self.s))


def torch_p2p(ops):
    """p2p callable for HaloIteratedSpmv over torch.distributed."""
    import torch.distributed as dist
    reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend if k == "send" else dist.irecv, t, p)
                                   for k, t, p in ops])
    for r in reqs:
        r.wait()


# ---------------------------------------------------------------- fused peer-memory step
def fused_receive_ranges(slabs: Sequence[Slab], ranges, mode: str) -> List[tuple]:
    """Global rows [lo, hi) each rank's window must receive every step of the
    fused path (spmvk_dist_set_rows): the whole x for "allgather"; for "halo"
    the span of its own slab and the columns its slab reads (``ranges[q]`` =
    (cmin, cmax), cmin > cmax for a slab without entries).  spmvk_plan_receive."""
    from ._lib import lib
    P = len(slabs)
    if mode not in ("allgather", "halo"):
        raise ValueError(f"unknown exchange mode {mode!r}")
    bounds = _u64([s.row_begin for s in slabs] + [slabs[-1].row_end if slabs else 0])
    cr = _u64([v for r in (ranges if mode == "halo" else [(1, 0)] * P) for v in r])
    out = _u64([0] * (2 * P))
    _plan_check(lib().spmvk_plan_receive(P, bounds, cr, 0 if mode == "allgather" else 1, out))
    return [(int(out[2 * q]), int(out[2 * q + 1])) for q in range(P)]


def simulate_fused_routing(slabs, receive, slab_matvec, x0, steps: int):
    """CPU model of the fused step's data movement (for the gloo-free unit
    tests): every rank owns two window buffers; step k reads its window's
    x[cur] and stores its slab of x_{k+1} into x[1-cur] of every window whose
    receive range covers the row.  ``slab_matvec(rank, x) -> x_next slab``.
    Returns the windows' current buffers."""
    n = max(x0.size, max(s.row_end for s in slabs))
    win = [[np.zeros(n, x0.dtype), np.zeros(n, x0.dtype)] for _ in slabs]
    for w in win:
        w[0][: x0.size] = x0
    cur = 0
    for _ in range(steps):
        for s in slabs:
            xn = slab_matvec(s.rank, win[s.rank][cur])
            for q, (lo, hi) in enumerate(receive):
                a, b = max(lo, s.row_begin), min(hi, s.row_end)
                if a < b:
                    win[q][1 - cur][a:b] = xn[a - s.row_begin: b - s.row_begin]
        cur = 1 - cur
    return [w[cur] for w in win]


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 2, "strides": None}


class ExchangeWindow:
    """This rank's exchange window (spmvk_window): two x buffers + flags."""

    def __init__(self, n: int, prec: int = 8):
        import ctypes as C

        import torch

        from . import spmvkit as sk
        from ._lib import lib
        self._L, self.n, self.prec = lib(), n, prec
        h = C.c_void_p()
        sk._check(self._L.spmvk_window_create(n, prec, C.byref(h)))
        self._h = h
        self.x = []
        for b in range(2):
            p = C.c_void_p()
            sk._check(self._L.spmvk_window_x(h, b, C.byref(p)))
            self.x.append(torch.as_tensor(_DevArray(p.value, n, "<f8" if prec == 8 else "<f4"),
                                          device="cuda"))

    def ipc_handle(self) -> bytes:
        import ctypes as C

        from . import spmvkit as sk
        buf = (C.c_ubyte * 64)()
        sk._check(self._L.spmvk_window_ipc_handle(self._h, buf))
        return bytes(buf)

    def close(self):
        if self._h:
            self.x = []
            self._L.spmvk_window_destroy(self._h)
            self._h = None


class FusedIteratedSpmv:
    """Iterated SpMV with the x exchange fused into the SpMV (spmvk_dist_*):
    the kernel's row epilogue stores x_{k+1} into every window whose receive
    range covers the row (peer windows over NVLink), then a device flag
    barrier ends the step.  ``handles`` = the 64-byte IPC handles of every
    rank's window in rank order (gathered by the caller), or ``local_windows``
    = the ExchangeWindow of every rank when all ranks live in this process
    (then ``barrier`` is usually False and the caller steps ranks in turn)."""

    def __init__(self, slab: Slab, receive: Sequence[tuple], a, window: ExchangeWindow,
                 world: int, stream: int, handles=None, local_windows=None, barrier=True,
                 scale: float = 0.0625):
        import ctypes as C

        import torch

        from . import spmvkit as sk
        from ._lib import lib
        self._L, self.slab, self.a, self.window, self.stream = lib(), slab, a, window, stream
        self.world, self.scale, self.barrier = world, scale, bool(barrier)
        self.num_cols = a.num_cols
        d = C.c_void_p()
        if local_windows is not None:
            arr = (C.c_void_p * world)(*[w._h.value for w in local_windows])
            sk._check(self._L.spmvk_dist_open_local(arr, slab.rank, world, C.byref(d)))
        else:
            blob = b"".join(handles) if handles else None
            sk._check(self._L.spmvk_dist_open(window._h, slab.rank, world, blob, C.byref(d)))
        self._d = d
        rr = (C.c_uint64 * (2 * world))(*[v for lo_hi in receive for v in lo_hi])
        sk._check(self._L.spmvk_dist_set_rows(d, slab.row_begin, slab.row_end, rr))
        dt = torch.float64 if window.prec == 8 else torch.float32
        self.y = torch.zeros(max(slab.rows, 1), dtype=dt, device="cuda")
        self._step = self._L.spmvk_dist_step_f64 if window.prec == 8 else \
            self._L.spmvk_dist_step_f32
        lo, hi = receive[slab.rank]  # entries received from peers per step
        self.halo = max(0, min(hi, slab.row_begin) - lo) + max(0, hi - max(lo, slab.row_end))

    @property
    def cur(self) -> int:
        import ctypes as C
        c = C.c_int()
        self._L.spmvk_dist_current(self._d, C.byref(c))
        return c.value

    @property
    def x(self):  # the two window buffers (HaloIteratedSpmv's x[cur] convention)
        return self.window.x

    @property
    def x_current(self):
        return self.window.x[self.cur][: self.num_cols]

    def set_x(self, x_full):
        self.window.x[self.cur][: x_full.numel()].copy_(x_full)

    def halo_entries(self) -> int:
        return self.halo

    def step(self):
        from . import spmvkit as sk
        sk._check(self._step(self._d, self.a._h, self.scale, self.y.data_ptr(),
                             1 if self.barrier else 0, self.stream))

    def status(self) -> tuple:
        """(0, "") while every flag barrier so far completed; else the
        SPMVK_ENCCL code and the message naming the rank that never arrived
        (spmvk_dist_status: synchronises the stream)."""
        import ctypes as C

        from ._lib import lib
        rc = self._L.spmvk_dist_status(self._d, C.c_void_p(self.stream))
        return rc, (lib().spmvk_last_error().decode() if rc else "")

    def close(self):
        if self._d:
            self._L.spmvk_dist_destroy(self._d)
            self._d = None


class NcclComm:
    """spmvk_comm: an NCCL communicator made by the C-ABI (ncclCommInitRank
    with the 128-byte unique id, or ncclCommInitAll via ``init_all``)."""

    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from . import spmvkit as sk
        from ._lib import lib
        buf = (C.c_ubyte * 128)()
        sk._check(lib().spmvk_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def init_rank(cls, uid: bytes, world: int, rank: int, device: int) -> "NcclComm":
        import ctypes as C

        from . import spmvkit as sk
        from ._lib import lib
        h = C.c_void_p()
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        sk._check(lib().spmvk_comm_init_rank(buf, world, rank, device, C.byref(h)))
        return cls(h)

    @classmethod
    def init_all(cls, devices) -> list:
        import ctypes as C

        from . import spmvkit as sk
        from ._lib import lib
        n = len(devices)
        hs = (C.c_void_p * n)()
        sk._check(lib().spmvk_comm_init_all(n, (C.c_int * n)(*devices), hs))
        return [cls(C.c_void_p(h)) for h in hs]

    def close(self):
        if self._h:
            from ._lib import lib
            lib().spmvk_comm_destroy(self._h)
            self._h = None


class NcclIteratedSpmv:
    """The iterated product with the x exchange over NCCL, all in the C-ABI
    (spmvk_nccl_iter_*, csrc/nccl_dist.cu): scaled slab SpMV, then an in-place
    ncclAllGather ("allgather", equal slabs) or grouped ncclSend/ncclRecv of
    the column ranges each slab reads ("halo").  Creating it is collective."""

    def __init__(self, comm: NcclComm, slab: Slab, a, n: int, mode: str, stream: int,
                 scale: float = 0.0625):
        import ctypes as C

        import torch

        from . import spmvkit as sk
        from ._lib import lib
        self._L, self.slab, self.a, self.stream, self.scale = lib(), slab, a, stream, scale
        self.num_cols = a.num_cols
        h = C.c_void_p()
        sk._check(self._L.spmvk_nccl_iter_create(comm._h, a._h, slab.row_begin, slab.row_end,
                                                 slab.pad_rows, n,
                                                 0 if mode == "allgather" else 1, C.byref(h)))
        self._h = h
        self.xbuf = []
        for b in range(2):
            p, ln = C.c_void_p(), C.c_uint64()
            sk._check(self._L.spmvk_nccl_iter_x(h, b, C.byref(p), C.byref(ln)))
            self.xbuf.append(torch.as_tensor(
                _DevArray(p.value, ln.value, "<f8" if a.precision == 8 else "<f4"), device="cuda"))
        dt = torch.float64 if a.precision == 8 else torch.float32
        self.y = torch.zeros(max(slab.rows, 1), dtype=dt, device="cuda")
        self._step = self._L.spmvk_nccl_iter_step_f64 if a.precision == 8 else \
            self._L.spmvk_nccl_iter_step_f32

    @property
    def cur(self) -> int:
        import ctypes as C
        c = C.c_int()
        self._L.spmvk_nccl_iter_current(self._h, C.byref(c))
        return c.value

    @property
    def x(self):
        return self.xbuf

    @property
    def x_current(self):
        return self.xbuf[self.cur][: self.num_cols]

    def set_x(self, x_full):
        self.xbuf[self.cur][: x_full.numel()].copy_(x_full)

    def halo_entries(self) -> int:
        import ctypes as C
        v = C.c_uint64()
        self._L.spmvk_nccl_iter_halo_entries(self._h, C.byref(v))
        return v.value

    def step(self):
        from . import spmvkit as sk
        sk._check(self._step(self._h, self.scale, self.y.data_ptr(), self.stream))

    def close(self):
        if self._h:
            self.xbuf = []
            self._L.spmvk_nccl_iter_destroy(self._h)
            self._h = None


# ---------------------------------------------------------------- bench (N > 1)
def bench_distributed(args, metric: str, workloads: dict, clock_cls=None, peaks=None,
                      rg_bytes=None, config_fn=None, cpu_fn=None, traffic=None):
    """bench.py leg for torchrun N > 1: strong scaling of the iterated SpMV.
    ``clock_cls`` / ``peaks`` / ``rg_bytes`` are bench.py's NVML clock sampler,
    measured HBM peak and algorithmic-bytes function; ``config_fn(n, exchange)``
    the config dict both bench arms print; ``cpu_fn()`` the CPU reference
    baseline (rank 0, after the GPU timing); ``traffic`` the committed ncu DRAM
    bytes of the single-GPU kernel on this workload."""
    import torch
    import torch.distributed as dist

    from . import generators as gen
    from . import spmvkit as sk
    from ._lib import lib

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    # SPMVK_SHARE_GPU=1: every rank on GPU 0 with gloo plumbing (the fused
    # exchange's data path is CUDA IPC + the device flag barrier, which works
    # between processes sharing a GPU) -- exercises the N > 1 bench path on a
    # one-GPU box; NCCL refuses two ranks on one device
    share = os.environ.get("SPMVK_SHARE_GPU") == "1"
    local = 0 if share else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    assert lib().spmvk_init(local) == 0, sk._lib.last_error()
    if share:
        if getattr(args, "exchange", "fused") != "fused":
            raise SystemExit("SPMVK_SHARE_GPU=1 supports --exchange fused only")
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cdev = "cpu" if share else "cuda"  # device of the plumbing tensors

    def gather_flat(t):  # all-gather of a small 1-D plumbing tensor, rank order
        t = t.to(cdev)
        if share:
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return torch.cat(parts)
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=cdev)
        dist.all_gather_into_tensor(out, t)
        return out

    def reduce_scalar(v, op, dtype=torch.float64):
        t = torch.tensor([v], dtype=dtype, device=cdev)
        dist.all_reduce(t, op=op)
        return t
    G = 32
    kind, a_, b_, desc = workloads[args.workload]
    csr = sk.CsrMatrix.stencil(a_, b_) if kind == "stencil" else sk.build_csr(gen.powerlaw(b_, 7))
    slabs = slab_bounds(csr.num_rows, G, world)
    me = slabs[rank]
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    a = sk.build_rgcsr(csr, G, 8, stream=sp, row_range=(me.row_begin, me.row_end))
    nnz_local = a.nnz()
    exchange = getattr(args, "exchange", "allgather")
    if exchange in ("halo", "fused"):
        import ctypes as C
        cr = (C.c_uint64 * 2)()
        sk._check(lib().spmvk_csr_column_range(csr._h, me.row_begin, me.row_end, cr))
        allr = gather_flat(torch.tensor([int(cr[0]), int(cr[1])], dtype=torch.int64))
        ranges = [tuple(allr[2 * r: 2 * r + 2].tolist()) for r in range(world)]
    del csr
    L = lib()
    x0 = torch.from_numpy(gen.random_vector(a.num_cols, 1)).cuda()

    def slab_spmv(x, y, xn):
        rc = L.spmvk_rgcsr_spmv_scaled_f64(a._h, x.data_ptr(), x.numel(), y.data_ptr(),
                                           y.numel(), xn.data_ptr(), 0.0625, sp)
        assert rc == 0, sk._lib.last_error()

    def all_gather(out, inp):
        with torch.cuda.stream(stream):
            dist.all_gather_into_tensor(out, inp)

    def p2p(ops):
        with torch.cuda.stream(stream):
            torch_p2p(ops)

    fallback = None
    if exchange == "fused":
        # peer windows need CUDA IPC + P2P between the GPUs; if any rank cannot
        # map them, every rank switches to the NCCL halo exchange (recorded)
        win = it = None
        try:
            win = ExchangeWindow(max(a.num_cols, slabs[-1].row_end), 8)
            handles = [None] * world
            dist.all_gather_object(handles, win.ipc_handle())
            recv = fused_receive_ranges(slabs, ranges, "halo")
            it = FusedIteratedSpmv(me, recv, a, win, world, sp, handles=handles,
                                   barrier=world > 1)
            ok, why = 1, ""
        except Exception as e:  # noqa: BLE001 -- reported, then the NCCL path runs
            ok, why = 0, f"rank {rank}: {e}"
        flag = reduce_scalar(ok, dist.ReduceOp.MIN, torch.int64)
        if not flag.item():
            reasons = [None] * world
            dist.all_gather_object(reasons, why)
            fallback = "; ".join(r for r in reasons if r) or "a peer could not map windows"
            if it is not None:
                it.close()
            dist.barrier()
            if win is not None:
                win.close()
            exchange = "halo"
    comm = None
    if exchange == "fused":
        pass
    elif share:  # gloo plumbing: the torch.distributed forms of the exchanges
        it = (HaloIteratedSpmv(me, slabs, ranges, a.num_cols, slab_spmv, p2p, x0)
              if exchange == "halo" else IteratedSpmv(me, a.num_cols, world, slab_spmv,
                                                      all_gather, x0))
    else:  # NCCL driven from the C-ABI (spmvk_comm_init_rank + spmvk_nccl_iter_*)
        uid = [NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = NcclComm.init_rank(uid[0], world, rank, local)
        it = NcclIteratedSpmv(comm, me, a, slabs[-1].row_end, exchange, sp)
    with torch.cuda.stream(stream):
        it.set_x(x0)
    stream.synchronize()
    dist.barrier()
    for _ in range(args.warmup):
        it.step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = clock_cls(local) if clock_cls else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.__enter__()
    e0.record(stream)
    for _ in range(args.steps):
        it.step()
    e1.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.__exit__(None, None, None)
    ms = reduce_scalar(e0.elapsed_time(e1), dist.ReduceOp.MAX)
    # a flag barrier that timed out makes every later step return at once: a
    # time measured across one is not a step time -- fail instead
    if exchange == "fused" and world > 1:
        rc, why = it.status()
        bad = reduce_scalar(1 if rc else 0, dist.ReduceOp.MAX, torch.int64)
        if bad.item():
            whys = [None] * world
            dist.all_gather_object(whys, f"rank {rank}: {why}" if rc else "")
            raise SystemExit("fused exchange failed: " + "; ".join(w for w in whys if w))
    # checksum of this rank's rows of the iterate after warmup + steps
    # iterations (bitwise across P: the slab arrays are global slices and
    # every row keeps the reference's order) -- taken before the e2e leg,
    # which re-uploads each rank's own x slab only
    xf = it.x[: a.num_cols] if isinstance(it, IteratedSpmv) else it.x_current
    # order-independent bit checksum: wrapping int64 sum of the raw bits
    part_sum = xf[me.row_begin:me.row_end].contiguous().view(torch.int64).sum().reshape(1)
    sums = gather_flat(part_sum)
    tot_nnz = reduce_scalar(float(nnz_local), dist.ReduceOp.SUM)

    # parity gate: from x0 again, exactly 100 iterations, and the wrapping
    # int64 sum of the iterate's raw bits over all ranks must equal the
    # unmodified reference's (tests/golden/iterate_7pt512.json, made by
    # oracle/make_iterate_golden.py) -- the P-GPU iterate bitwise the CPU one
    parity = None
    golden_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "tests", "golden", "iterate_7pt512.json")
    if args.workload == "7pt-512" and os.path.exists(golden_path):
        with open(golden_path) as f:
            want = int(json.load(f)["bits_sum_int64_after"]["100"])
        with torch.cuda.stream(stream):
            it.set_x(x0)
        stream.synchronize()
        dist.barrier()
        for _ in range(100):
            it.step()
        torch.cuda.synchronize()
        if exchange == "fused" and world > 1 and it.status()[0]:
            raise SystemExit(f"fused exchange failed in the parity pass: {it.status()[1]}")
        xp = it.x[: a.num_cols] if isinstance(it, IteratedSpmv) else it.x_current
        mine = xp[me.row_begin:me.row_end].contiguous().view(torch.int64).sum().reshape(1)
        got = int(gather_flat(mine).sum().item())
        got = (got + 2 ** 63) % 2 ** 64 - 2 ** 63
        parity = {"iterations": 100, "bits_sum_int64": got, "reference": want,
                  "bitwise": got == want, "golden": "tests/golden/iterate_7pt512.json"}
        if got != want:
            raise SystemExit(f"parity gate failed: {world}-GPU iterate bit sum {got} != "
                             f"reference {want}")

    # kernel-only time of this rank's slab SpMV (roofline of the dominant kernel)
    xs = (it.x[: a.num_cols] if isinstance(it, IteratedSpmv) else it.x_current).clone()
    ys = torch.empty(max(a.num_rows, 1), dtype=torch.float64, device="cuda")
    xn = torch.empty_like(ys)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 200))]
    for s_, e_ in kev:
        s_.record(stream)
        slab_spmv(xs, ys[: a.num_rows], xn[: a.num_rows])
        e_.record(stream)
    torch.cuda.synchronize()
    kern_ms = reduce_scalar(sum(s_.elapsed_time(e_) for s_, e_ in kev) / len(kev),
                            dist.ReduceOp.MAX)
    slab_bytes = (rg_bytes(a.info, 8) if rg_bytes else 0)

    # e2e: every step each rank uploads its x slab from pinned host memory,
    # runs the exchange + slab SpMV, and downloads its y slab
    # (page-locked 2 MB-page host buffers, spmvk_host_alloc: no slow first
    # calls, profiles/r02t_e2e_env.md)
    xs_h = sk.host_array(me.row_end - me.row_begin)
    xs_h[:] = gen.random_vector(a.num_cols, 1)[me.row_begin:me.row_end]
    xh = torch.from_numpy(xs_h)
    yh = torch.from_numpy(sk.host_array(max(a.num_rows, 1)))
    e2e_steps = max(3, min(args.steps, 50))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        with torch.cuda.stream(stream):
            cur = it.x if isinstance(it, IteratedSpmv) else it.x[it.cur]
            cur[me.row_begin:me.row_end].copy_(xh, non_blocking=True)
        it.step()
        with torch.cuda.stream(stream):
            yh[: a.num_rows].copy_(it.y[: a.num_rows], non_blocking=True)
        stream.synchronize()
    torch.cuda.synchronize()
    e2e_s = reduce_scalar((time.perf_counter() - t0) / e2e_steps, dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        step_ms = ms.item() / args.steps
        value = 2.0 * tot_nnz.item() / (step_ms * 1e-3) / 1e9
        halo = it.halo_entries() if hasattr(it, "halo_entries") else None
        k_s = kern_ms.item() * 1e-3
        achieved = slab_bytes / k_s / 1e9 if slab_bytes else None
        peak, peak_kind = peaks if peaks else (None, None)
        print(json.dumps({
            "metric": metric, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": (config_fn(world, getattr(args, "exchange", "fused")) if config_fn else
                       {"workload": args.workload, "description": desc}),
            "exchange": {"used": exchange,
                       "how": (f"row-slab x{world}, halo of x stored into peer windows "
                                       "by the SpMV epilogue (NVLink P2P) + device flag barrier"
                                       if exchange == "fused" else
                                       f"row-slab x{world}, NCCL {exchange} of x"),
                       "step": (f"fused slab SpMV + peer-window x_next stores"
                                f"{' + flag barrier' if world > 1 else ''}"
                                if exchange == "fused" else
                                f"slab SpMV (+fused x_next = y/16) + {exchange} exchange"),
                       "halo_entries_rank0": halo,
                       "exchange_fallback": fallback,
                       "shared_gpu": (f"SPMVK_SHARE_GPU=1: all {world} ranks on GPU 0 (gloo "
                                      "plumbing; a correctness run, not a scaling number)"
                                      if share else None)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved and peak else None,
                         "peak_kind": peak_kind, "bytes_per_launch": slab_bytes,
                         "kernel_us": k_s * 1e6, "scope": "rank-0 slab SpMV, max over ranks",
                         "traffic": traffic,
                         "traffic_note": ("ncu DRAM bytes per launch of the whole-matrix "
                                          "kernel at N = 1 (profiles/traffic.json); a slab "
                                          "moves ~1/N of it") if traffic else None},
            "cpu_baseline": cpu_fn() if cpu_fn else None,
            "e2e": {"value": 2.0 * tot_nnz.item() / e2e_s.item() / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 8 * me.rows * world,
                    "d2h_bytes_per_step": 8 * me.rows * world,
                    "ms_per_step": e2e_s.item() * 1e3,
                    "path": "per rank: pinned H2D of the x slab, exchange + slab SpMV, D2H of y"},
            "clocks": clocks.summary() if clocks else None,
            "gpu_launches": args.steps * (2 if exchange == "fused" and world > 1 else 1),
            "x_bits_checksum": int(sums.sum().item()),
            "parity": parity,
        }), flush=True)
    dist.barrier()  # the other ranks wait for rank 0's CPU baseline
    if hasattr(it, "close"):
        it.close()
    if comm is not None:
        comm.close()
    dist.destroy_process_group()
