"""e2e host-span SpMV (27-pt 128^3 fp64) vs the host CPU / NUMA placement of
the process and its pinned buffers: prints the topology, then times the
C-ABI span call with the process bound to each NUMA node's CPUs (pinned
buffers allocated after binding, so first touch places them there)."""
import os, sys, time, statistics, subprocess, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

def topo():
    nodes = sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
    out = {}
    for n in nodes:
        out[n] = open(f"/sys/devices/system/node/{n}/cpulist").read().strip()
    return out

def cpus(lst):
    s = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-"); s.update(range(int(a), int(b) + 1))
        elif part:
            s.add(int(part))
    return s

if len(sys.argv) > 1 and sys.argv[1] == "child":
    cs = cpus(sys.argv[2]) if sys.argv[2] != "all" else None
    if cs: os.sched_setaffinity(0, cs)
    import torch
    from paper_1012_2270_b200 import spmvkit as sk, generators as gen
    from paper_1012_2270_b200._lib import lib
    L = lib(); assert L.spmvk_init(0) == 0
    csr = sk.CsrMatrix.stencil(27, 128)
    a = sk.build_rgcsr(csr, 32, 8)
    xh = gen.random_vector(a.num_cols, 1)
    xpin = torch.from_numpy(xh).pin_memory()
    ypin = torch.empty(a.num_rows, dtype=torch.float64).pin_memory()
    for _ in range(10):
        L.spmvk_rgcsr_spmv_host_f64(a._h, xpin.data_ptr(), a.num_cols, ypin.data_ptr(), a.num_rows, None)
    rounds = []
    for _ in range(7):
        t = time.perf_counter()
        for _ in range(10):
            L.spmvk_rgcsr_spmv_host_f64(a._h, xpin.data_ptr(), a.num_cols, ypin.data_ptr(), a.num_rows, None)
        torch.cuda.synchronize()
        rounds.append((time.perf_counter() - t) / 10 * 1e3)
    print(json.dumps({"cpus": sys.argv[2], "ms": [round(r, 4) for r in rounds],
                      "median": round(statistics.median(rounds), 4)}))
    sys.exit(0)

t = topo()
print("numa nodes:", t)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    mask = pynvml.nvmlDeviceGetCpuAffinity(h, 4)
    print("nvml cpu affinity mask:", [hex(m) for m in mask])
except Exception as e:
    print("nvml:", e)
sets = ["all"] + list(t.values())
for rep in range(2):
    for s in sets:
        r = subprocess.run([sys.executable, __file__, "child", s], capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-500:])
