"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone, both at once
(the ceiling of bench.py's e2e leg, which moves 512 MiB each way per step).

    python tools/pcie_bw.py
"""
import torch

dev = torch.device("cuda", 0)
nb = 128 << 20
h = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(8)]
d = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(8)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        for i in range(4):
            d[i].copy_(h[i], non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for i in range(4):
            h[4 + i].copy_(d[4 + i], non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d 512 MiB", h2d), ("d2h 512 MiB", d2h), ("both (512 MiB each way)", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.2f} ms, {(4 * nb if name[0] != 'b' else 8 * nb) / ms / 1e6:.1f} GB/s")
