"""One warm-up + N fwd+bwd steps of the bench workload, for ncu captures.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py
    ncu --set full --clock-control none --import-source on -k regex:k_bwd_causal_k \
        -s 1 -c 1 -o gpurun_out/prof python tools/profile_step.py
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_04008_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--noncausal", action="store_true")
ap.add_argument("--dtype", default="bf16")
args = ap.parse_args()
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=not args.noncausal)
w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
p = cfg.params()
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, do = (torch.randn(1, 4, args.n, 128, generator=g, device=dev).to(dt) for _ in range(4))
for _ in range(args.steps):
    o, den, st = rb.race_forward(q, k, v, w, p)
    dq, dk, dv = rb.race_backward(q, k, v, w, do, p, state=st)
torch.cuda.synchronize()
print("ok", float(o.float().abs().mean()), float(dq.float().abs().mean()))
