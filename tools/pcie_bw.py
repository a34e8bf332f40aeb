"""Pinned host <-> device copy bandwidth (the e2e ceiling): H2D, D2H, both."""
import torch

n = 335 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


ms = t(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {n / ms / 1e6:.1f} GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {n / ms / 1e6:.1f} GB/s")
ms = t(both)
print(f"H2D+D2H concurrent {2 * n / ms / 1e6:.1f} GB/s total")
