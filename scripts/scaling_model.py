"""Config 5 (7-point 512^3, fp64, G = 32) strong-scaling model from one GPU.

gpurun offers one B200, so the P-GPU step is composed from measured parts:
for P in 1, 2, 4, 8 the group-aligned slab of rank 0 (one halo) and of an
interior rank (two halos) is built, and on the one GPU we time
  * the plain scaled slab SpMV (y, x_next = y/16), and
  * the fused step (spmvk_dist_step without the barrier): the same kernel
    with the PeerEpi epilogue storing each x_next row into every window whose
    receive range covers it -- local windows here, NVLink peer windows on a
    real node,
both as back-to-back launches.  The halo each rank receives per step and its
NVLink time at 700 GB/s (an assumption, not a measurement) are printed beside
them.  Predicted step time = max over ranks of the fused step (the halo
stores overlap the SpMV tile by tile) + the flag barrier (est. 8 us).
One JSON line per (P, rank)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1012_2270_b200 import generators as gen  # noqa: E402
from paper_1012_2270_b200 import partition as pt  # noqa: E402
from paper_1012_2270_b200 import spmvkit as sk  # noqa: E402
from paper_1012_2270_b200._lib import lib  # noqa: E402

NVLINK_GBS = 700.0
BARRIER_US = 8.0


def b2b(fn, stream, k=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / k


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    torch.cuda.set_device(0)
    L = lib()
    assert L.spmvk_init(0) == 0
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    csr = sk.CsrMatrix.stencil(7, n)
    N, G = csr.num_rows, 32
    x0 = torch.from_numpy(gen.random_vector(N, 1)).cuda()
    t1 = None
    for P in (1, 2, 4, 8):
        slabs = pt.slab_bounds(N, G, P)
        ranges = []
        for s in slabs:
            cr = (C.c_uint64 * 2)()
            sk._check(L.spmvk_csr_column_range(csr._h, s.row_begin, s.row_end, cr))
            ranges.append((int(cr[0]), int(cr[1])))
        recv = pt.fused_receive_ranges(slabs, ranges, "halo")
        wins = [pt.ExchangeWindow(N, 8) for _ in slabs]
        worst = 0.0
        for r in sorted({0, min(1, P - 1)}):
            sl = slabs[r]
            a = sk.build_rgcsr(csr, G, 8, stream=sp, row_range=(sl.row_begin, sl.row_end))
            y = torch.empty(sl.rows, dtype=torch.float64, device="cuda")
            xn = torch.empty_like(y)
            plain = b2b(lambda: L.spmvk_rgcsr_spmv_scaled_f64(a._h, x0.data_ptr(), N, y.data_ptr(),
                                                              sl.rows, xn.data_ptr(), 0.0625, sp),
                        stream)
            it = pt.FusedIteratedSpmv(sl, recv, a, wins[r], P, sp, local_windows=wins,
                                      barrier=False)
            with torch.cuda.stream(stream):
                it.set_x(x0)
            fused = b2b(it.step, stream)
            halo = it.halo_entries()
            nvl_us = halo * 8 / (NVLINK_GBS * 1e3)
            # slab bytes: its stored slots + group pointers / row lengths, the x
            # entries it reads (own rows + halo), y and x_next written
            B = bench.rg_bytes(a.info, 8) - 8 * a.num_cols + 8 * (sl.rows + halo) + 8 * sl.rows
            worst = max(worst, fused)
            print(json.dumps({"P": P, "rank": r, "slab_rows": sl.rows, "plain_us": round(plain, 1),
                              "fused_step_us": round(fused, 1),
                              "slab_GBs": round(B / plain / 1e3, 1),
                              "halo_entries": halo, "halo_nvlink_us_at_700GBs": round(nvl_us, 1)}),
                  flush=True)
            it.close()
            del a
        step = worst + (BARRIER_US if P > 1 else 0.0)
        t1 = t1 or step
        print(json.dumps({"P": P, "predicted_step_us": round(step, 1),
                          "predicted_speedup": round(t1 / step, 2),
                          "predicted_efficiency": round(t1 / step / P, 3)}), flush=True)
        for w in wins:
            w.close()


if __name__ == "__main__":
    main()
