"""Pinned host<->device copy probe for the e2e leg: whole-buffer and chunked
H2D / D2H, alone and concurrent, with and without a pipeline dependency."""
import json
import torch

n = 16 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for s in (s1, s2):
            s.wait_stream(main)
        fn()
        for s in (s1, s2):
            main.wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(chunks, up=True, down=True, dep=0):
    c = n // chunks
    ev = [torch.cuda.Event() for _ in range(chunks)]

    def f():
        for k in range(chunks):
            if up:
                with torch.cuda.stream(s1):
                    d1[k * c:(k + 1) * c].copy_(h1[k * c:(k + 1) * c], non_blocking=True)
                    ev[k].record(s1)
        for k in range(chunks):
            if down:
                with torch.cuda.stream(s2):
                    if up and dep:
                        s2.wait_event(ev[min(chunks - 1, k + dep - 1)])
                    h2[k * c:(k + 1) * c].copy_(d2[k * c:(k + 1) * c], non_blocking=True)
    return f


out = {}
for chunks in (1, 4, 16, 64):
    for name, kw in (("h2d", dict(down=False)), ("d2h", dict(up=False)), ("both", {}),
                     ("both_dep", dict(dep=2))):
        ms = timed(run(chunks, **kw))
        out[f"{name}_x{chunks}"] = round(ms * 1e3, 1)
print(json.dumps(out, indent=0))
