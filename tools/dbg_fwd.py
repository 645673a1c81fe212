import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2510_04008_b200 as rb
dev = torch.device("cuda", 0)
sizes = [int(x) for x in sys.argv[1:]] or [130, 1000, 16666, 16667, 131072]
for n in sizes:
    H = 4
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=True)
    w = rb.head_hyperplanes(cfg, H, 128).to(dev)
    p = cfg.params()
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = (torch.randn(1, H, n, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    try:
        o, den, st = rb.race_forward(q, k, v, w, p)
        torch.cuda.synchronize()
        print("fwd ok", n, flush=True)
        dq, dk, dv = rb.race_backward(q, k, v, w, do, p, state=st)
        torch.cuda.synchronize()
        print("ok", n, flush=True)
    except Exception as e:
        print("FAIL", n, str(e)[:200], flush=True)
        break
