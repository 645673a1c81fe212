"""One warm-up + 2 fwd+bwd steps of a grouped (several tcgen05 passes) sketch, for ncu launch lists.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
        python tools/profile_grouped.py --P 2 --L 4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_04008_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--L", type=int, default=4)
ap.add_argument("--n", type=int, default=131072)
args = ap.parse_args()
dev = torch.device("cuda", 0)
cfg = rb.SketchConfig(hyperplanes=args.P, tables=args.L, seed=0, causal=True)
w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
p = cfg.params()
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, do = (torch.randn(1, 4, args.n, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
for _ in range(3):
    o, den, st = rb.race_forward(q, k, v, w, p)
    rb.race_backward(q, k, v, w, do, p, state=st)
torch.cuda.synchronize()
print("ok")
