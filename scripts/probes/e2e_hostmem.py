"""e2e host-span SpMV (27-pt 128^3 fp64) vs how the pinned host x / y were
allocated: torch pin_memory (cudaHostAlloc via the caching host allocator),
or an anonymous mmap advised to transparent huge pages (MADV_HUGEPAGE),
touched, then page-locked with cudaHostRegister (portable | mapped).  Each
mode in fresh processes, 7 rounds x 10 back-to-back calls, median round."""
import os, sys, time, statistics, subprocess, json, ctypes
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

def thp_buffer(nbytes):
    import numpy as np, mmap
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    libc.mmap.restype = ctypes.c_void_p
    libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
    libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    align = 2 << 20
    size = (nbytes + align - 1) // align * align
    raw = libc.mmap(None, size + align, mmap.PROT_READ | mmap.PROT_WRITE,
                    mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    p = (raw + align - 1) // align * align
    assert libc.madvise(p, size, 14) == 0  # MADV_HUGEPAGE
    buf = (ctypes.c_char * size).from_address(p)
    ctypes.memset(p, 0, size)
    import torch
    rc = torch.cuda.cudart().cudaHostRegister(p, size, 1 | 2)  # portable | mapped
    assert int(rc) == 0, rc
    return p, size

if len(sys.argv) > 1 and sys.argv[1] == "child":
    mode = sys.argv[2]
    import numpy as np, torch
    from paper_1012_2270_b200 import spmvkit as sk, generators as gen
    from paper_1012_2270_b200._lib import lib
    L = lib(); assert L.spmvk_init(0) == 0
    csr = sk.CsrMatrix.stencil(27, 128)
    a = sk.build_rgcsr(csr, 32, 8)
    xh = gen.random_vector(a.num_cols, 1)
    if mode == "torch":
        xp = torch.from_numpy(xh).pin_memory(); yp = torch.empty(a.num_rows, dtype=torch.float64).pin_memory()
        xa, ya = xp.data_ptr(), yp.data_ptr()
    else:
        xa, _ = thp_buffer(8 * a.num_cols); ya, _ = thp_buffer(8 * a.num_rows)
        ctypes.memmove(xa, xh.ctypes.data, 8 * a.num_cols)
    for _ in range(10):
        L.spmvk_rgcsr_spmv_host_f64(a._h, xa, a.num_cols, ya, a.num_rows, None)
    rounds = []
    for _ in range(7):
        t = time.perf_counter()
        for _ in range(10):
            rc = L.spmvk_rgcsr_spmv_host_f64(a._h, xa, a.num_cols, ya, a.num_rows, None)
        torch.cuda.synchronize()
        rounds.append((time.perf_counter() - t) / 10 * 1e3)
    assert rc == 0
    y = np.ctypeslib.as_array((ctypes.c_double * a.num_rows).from_address(ya))
    ysum = float(np.cumsum(y)[-1])
    hp = open("/proc/meminfo").read().split("AnonHugePages:")[1].split("\n")[0].strip()
    print(json.dumps({"mode": mode, "ms": [round(r, 4) for r in rounds],
                      "median": round(statistics.median(rounds), 4), "ysum": ysum, "AnonHugePages": hp}))
    sys.exit(0)

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
for rep in range(3):
    for mode in ("torch", "thp"):
        r = subprocess.run([sys.executable, __file__, "child", mode], capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-800:])
