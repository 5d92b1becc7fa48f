"""HBM calibration on the GPU box: read-only and copy bandwidth with torch
kernels (sum reduction over 8 GiB; copy of 4 GiB), CUDA-event timed, best of
10.  Gives the read-dominated ceiling next to MEASURED_PEAKS.json's copy
figure.  Prints one JSON line."""
import json

import torch


def best_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    n = 1 << 30  # 1 Gi doubles = 8 GiB
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    out = {}
    ms = best_ms(lambda: x.sum())
    out["read_sum_f64_GBs"] = 8 * n / ms / 1e6
    xf = x[: n // 2].view(torch.float32)  # 4 GiB of floats (reinterpret)
    ms = best_ms(lambda: xf.sum())
    out["read_sum_f32_GBs"] = 4 * n / ms / 1e6
    a = x[: n // 2]
    b = torch.empty_like(a)
    ms = best_ms(lambda: b.copy_(a))
    out["copy_GBs_read_plus_write"] = 2 * 8 * (n // 2) / ms / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
