"""Small generic-path (fp32, d=64) fwd+bwd, causal and not, for compute-sanitizer (memcheck / racecheck clean)."""
import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2510_04008_b200 as rb
dev = torch.device('cuda', 0)
for causal in (True, False):
    for P, L in ((2, 2), (3, 3)):
        cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=0, causal=causal)
        w = rb.head_hyperplanes(cfg, 2, 64).to(dev)
        q, k, v, g = (torch.randn(1, 2, 300, 64, device=dev) for _ in range(4))
        o, den, st = rb.race_forward(q, k, v, w, cfg.params())
        dq, dk, dv = rb.race_backward(q, k, v, w, g, cfg.params(), state=st)
torch.cuda.synchronize()
print("ok")
