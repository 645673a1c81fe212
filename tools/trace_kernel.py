"""Per-chunk timeline of CTA 0 of one fast-path kernel (RACE_TRACE slots).

    RACE_DEBUG_PROGRESS=1 python tools/trace_kernel.py [--kernel fwd|bq|bk] [--n 131072]

Prints, for the first chunks CTA 0 processes, the clock() value of every
traced event relative to the first, in microseconds at the measured SM clock.
"""
import argparse
import ctypes
import os
import sys

os.environ["RACE_DEBUG_PROGRESS"] = "2"  # device-memory trace buffer
_k = [sys.argv[i + 1] for i, x in enumerate(sys.argv[:-1]) if x == "--kernel"]
os.environ["RACE_TRACE_KERNEL"] = _k[0] if _k else "fwd"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_04008_b200 as rb  # noqa: E402
from paper_2510_04008_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--kernel", default="fwd")
ap.add_argument("--events", type=int, default=16)
ap.add_argument("--mhz", type=float, default=1965.0)
ap.add_argument("--cta-table", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=True)
w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
p = cfg.params()
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, do = (torch.randn(1, 4, args.n, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
L = _lib.lib()
L.race_debug_progress_buffer.restype = ctypes.c_void_p
L.race_debug_progress_clear.restype = None
o, den, st = rb.race_forward(q, k, v, w, p)
torch.cuda.synchronize()
for rep in range(3):
    L.race_debug_progress_clear()
    torch.cuda.synchronize()
    if args.kernel == "fwd":
        o, den, st = rb.race_forward(q, k, v, w, p)
    else:  # RACE_TRACE_KERNEL (set above) picks which backward kernel writes the trace
        rb.race_backward(q, k, v, w, do, p, state=st)
    torch.cuda.synchronize()
buf = (ctypes.c_uint * (148 * 256)).from_address(L.race_debug_progress_buffer())
vals = [[buf[e * 32 + c] for c in range(32)] for e in range(args.events)]
base = min(x for row in vals for x in row if x) if any(any(r) for r in vals) else 0
print("chunk " + " ".join(f"  ev{e:<3d}" for e in range(args.events)))
cta = [(buf[148 * 256 - 296 + 2 * b], buf[148 * 256 - 296 + 2 * b + 1]) for b in range(148)]
if any(x for x, _ in cta):
    t0 = min(x for x, _ in cta)
    ends = sorted(((e - t0) & 0xffffffff) / 1e3 for _, e in cta)
    starts = sorted(((s_ - t0) & 0xffffffff) / 1e3 for s_, _ in cta)
    print(f"CTA start spread {starts[-1]:.2f} us; end: min {ends[0]:.2f} median {ends[74]:.2f} max {ends[-1]:.2f} us; "
          f"CTA0 {((cta[0][1] - t0) & 0xffffffff) / 1e3:.2f}")
    if args.cta_table:
        from paper_2510_04008_b200.functional import Problem
        pr = Problem(q, k, v, w, p)
        items = pr.bh * pr.nseg
        grid = min(items, 148)
        rows = []
        for b in range(grid):
            i0, i1 = b * items // grid, (b + 1) * items // grid
            ch = sum(-(-(min((it % pr.nseg + 1) * pr.seg_tokens, pr.n) - (it % pr.nseg) * pr.seg_tokens) // 128)
                     for it in range(i0, i1))
            bhs = len({it // pr.nseg for it in range(i0, i1)})
            dur = ((cta[b][1] - cta[b][0]) & 0xffffffff) / 1e3
            rows.append((ch, bhs, dur, ((cta[b][0] - t0) & 0xffffffff) / 1e3, b))
        import collections
        by = collections.defaultdict(list)
        for ch, bhs, dur, st0, b in rows:
            by[(ch, bhs)].append(dur)
        for key in sorted(by):
            d = sorted(by[key])
            print(f"  chunks {key[0]:3d} seqs {key[1]}: n={len(d):3d} dur min {d[0]:.1f} med {d[len(d)//2]:.1f} max {d[-1]:.1f} us"
                  f"  -> {d[len(d)//2] / key[0]:.2f} us/chunk")
        slow = sorted(rows, key=lambda x: -x[2])[:8]
        print("  slowest CTAs (chunks, seqs, dur, start, id):", [(a_, b_, round(c_, 1), round(d_, 2), e_) for a_, b_, c_, d_, e_ in slow])
for c in range(32):
    cells = []
    for e in range(args.events):
        x = vals[e][c]
        cells.append(f"{((x - base) & 0xffffffff) / args.mhz:7.2f}" if x else "      -")
    print(f"{c:5d} " + " ".join(cells))
