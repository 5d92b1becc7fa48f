import sys, torch, numpy as np
sys.path.insert(0, '.')
import bench
from paper_1012_2270_b200 import spmvkit as sk, generators as gen
from paper_1012_2270_b200._lib import lib
L = lib(); torch.cuda.set_device(0); L.spmvk_init(0)
csr = sk.CsrMatrix.stencil(27, 128)
stream = torch.cuda.Stream(); sp = stream.cuda_stream
x = torch.from_numpy(gen.random_vector(csr.num_cols, 1)).cuda().to(torch.float32)
y = torch.empty(csr.num_rows, dtype=torch.float32, device='cuda')
h64 = sk.build_hybrid(csr, None, 4, stream=sp)
c32 = sk.build_csr(sk.TripletMatrix(csr.num_rows, csr.num_cols, *csr.to_host()), 4)
h32 = sk.build_hybrid(c32, None, 4)
for name, h in (("from f64 csr", h64), ("from f32 csr", h32)):
    for v in (b"auto", b"g7", b"litef"):
        L.spmvk_set_hybrid_kernel(v)
        _, per = bench.time_launches(lambda: L.spmvk_hybrid_spmv_f32(h._h, x.data_ptr(), h.num_cols, y.data_ptr(), h.num_rows, sp), stream, 300, 10)
        _, per2 = bench.time_launches(lambda: L.spmvk_hybrid_spmv_f32(h._h, x.data_ptr(), h.num_cols, y.data_ptr(), h.num_rows, None), torch.cuda.current_stream(), 300, 10)
        print(name, v, round(per*1e3,2), round(per2*1e3,2), h.slots_per_row, h.coo_nnz())
