"""Small fast-path fwd+bwd (causal and not, ragged N, with and without saved state) for
compute-sanitizer:  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_step.py"""
import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2510_04008_b200 as rb
dev = torch.device('cuda', 0)
for causal in (True, False):
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, 2, 128).to(dev)
    q, k, v, g = (torch.randn(1, 2, 4099, 128, device=dev).to(torch.bfloat16) for _ in range(4))
    o, den, st = rb.race_forward(q, k, v, w, cfg.params())
    dq, dk, dv = rb.race_backward(q, k, v, w, g, cfg.params(), state=st)
    dq2 = rb.race_backward(q, k, v, w, g, cfg.params())
    # strided [B, N, H, d] operands (4-D TMA maps) and a narrow head width
    qkv = torch.randn(1, 1000, 3 * 2 * 64, device=dev).to(torch.bfloat16)
    qs, ks, vs = (x.view(1, 1000, 2, 64).transpose(1, 2) for x in qkv.split(128, dim=-1))
    w64 = rb.head_hyperplanes(cfg, 2, 64).to(dev)
    o, den, st = rb.race_forward(qs, ks, vs, w64, cfg.params())
    rb.race_backward(qs, ks, vs, w64, o, cfg.params(), state=st)
# grouped tcgen05 passes (table groups and corner groups) with their pass buffers and pass states
for P, L in ((2, 4), (4, 2)):
    for causal in (True, False):
        cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=0, causal=causal)
        w = rb.head_hyperplanes(cfg, 2, 128).to(dev)
        q, k, v, g = (torch.randn(1, 2, 1500, 128, device=dev).to(torch.bfloat16) for _ in range(4))
        o, den, st = rb.race_forward(q, k, v, w, cfg.params())
        rb.race_backward(q, k, v, w, g, cfg.params(), state=st)
        rb.race_backward(q, k, v, w, g, cfg.params())
torch.cuda.synchronize()
print("ok")
