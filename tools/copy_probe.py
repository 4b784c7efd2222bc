"""Pinned host<->device copy bandwidth alone and concurrently (diagnostics)."""
import time
import torch

n = 1 << 30  # 1 GiB
h_up = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def up():
    with torch.cuda.stream(s1):
        d_a.copy_(h_up, non_blocking=True)


def dn():
    with torch.cuda.stream(s2):
        h_dn.copy_(d_b, non_blocking=True)


def both():
    up()
    dn()


for name, fn in [("h2d", up), ("d2h", dn), ("both", both)]:
    t = timed(fn)
    print(f"{name}: {t * 1e3:.1f} ms per GiB each -> {n / t / 1e9:.1f} GB/s per direction")
