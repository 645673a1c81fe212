"""Bitwise run-to-run determinism of the causal headline layer (fwd state/outputs, bwd grads).

    python tools/det_check.py [--reps 5] [--n 131072]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_04008_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--noncausal", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(1)
q, k, v, g = (torch.randn(1, 4, args.n, 128, generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=not args.noncausal)
w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
p = cfg.params()
ref = rb.race_forward(q, k, v, w, p)
gref = rb.race_backward(q, k, v, w, g, p, ref[2])
bad = 0
for r in range(args.reps):
    a = rb.race_forward(q, k, v, w, p)
    ga = rb.race_backward(q, k, v, w, g, p, a[2])
    diffs = {n: int((x != y).sum()) for n, x, y in zip(("o", "den", "state", "dq", "dk", "dv"), a + ga, ref + gref)}
    if any(diffs.values()):
        bad += 1
        st = a[2]
        print("rep", r, diffs)
        if diffs["state"]:
            idx = (st != ref[2]).nonzero().flatten()
            print("  first state diffs at", idx[:10].tolist(), "of", st.numel())
print("reps with differences:", bad, "of", args.reps, "| env:", {k_: os.environ.get(k_) for k_ in ("RACE_NO_PDL", "RACE_SEG_TARGET")})
