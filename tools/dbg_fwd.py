import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2510_04008_b200 as rb
dev = torch.device("cuda", 0)
for (H, n) in [(1, 130), (1, 128), (1, 256), (1, 1000), (4, 4096), (4, 131072)]:
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=True)
    w = rb.head_hyperplanes(cfg, H, 128).to(dev)
    p = cfg.params()
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = (torch.randn(1, H, n, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    try:
        o, den, st = rb.race_forward(q, k, v, w, p)
        torch.cuda.synchronize()
        print("fwd ok", H, n, flush=True)
        dq, dk, dv = rb.race_backward(q, k, v, w, do, p, state=st)
        torch.cuda.synchronize()
        print("bwd ok", H, n, flush=True)
    except Exception as e:
        print("FAIL", H, n, e, flush=True)
        break
