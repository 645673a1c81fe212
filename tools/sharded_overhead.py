"""Host cost of the sequence-sharded step (sharded_forward + sharded_backward) on one GPU, world = 1:
eager device time per step vs the plain race_forward / race_backward step, and the host submit time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_04008_b200 as rb  # noqa: E402
from paper_2510_04008_b200.sharded import sharded_backward, sharded_forward  # noqa: E402

dev = torch.device("cuda", 0)
cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=True)
w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
p = cfg.params()
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, do = (torch.randn(1, 4, 131072, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))


def plain():
    o, den, st = rb.race_forward(q, k, v, w, p)
    return rb.race_backward(q, k, v, w, do, p, state=st)


def sharded():
    o, den, st = sharded_forward(q, k, v, w, p)
    return sharded_backward(q, k, v, w, do, p, st)


for name, fn in (("plain", plain), ("sharded", sharded)):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        fn()
    host = (time.perf_counter() - t0) / 100 * 1e6
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(50):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{name}: {ev[0].elapsed_time(ev[1]) / 50 * 1e3:.1f} us/step device, host submit {host:.1f} us/step")
