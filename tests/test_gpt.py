"""GPT-style model with RACE attention in every layer (BASELINE configs[4]).

* d=64 heads on the tcgen05 kernels (native width: TMA zero-fills the tile columns
  beyond 64) equal the generic CUDA-core kernels and the float64 oracle;
* a small RaceGPT trains: finite loss, gradients reach every parameter, and
  the loss drops on a fixed batch.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2510_04008_b200 as rb
from conftest import rel_err
from oracle import race_oracle as ro

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    return torch.device("cuda", 0)


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
def test_d64_heads_fast_path_matches_generic_and_oracle(causal):
    import os

    from paper_2510_04008_b200 import _lib
    from paper_2510_04008_b200.functional import Problem

    dev = _cuda()
    heads, n, d = 3, 1000, 64
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=4, causal=causal)
    layer = rb.RaceAttention(heads, d, cfg).to(dev)
    g = torch.Generator(device=dev).manual_seed(2)
    q, k, v, do = (torch.randn(1, heads, n, d, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    assert _lib.fast_path(Problem(q, k, v, layer.w, layer.params_).desc)
    outs = []
    for generic in (False, True):
        if generic:
            os.environ["RACE_DISABLE_FAST_PATH"] = "1"
        try:
            qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
            o = layer(qq, kk, vv)
            o.backward(do)
            outs.append([o.detach().float().cpu()] + [t.grad.float().cpu() for t in (qq, kk, vv)])
        finally:
            os.environ.pop("RACE_DISABLE_FAST_PATH", None)
    for a, b in zip(*outs):
        assert rel_err(a, b.numpy()) <= TOL_BF16
    qh, kh, vh, gh = (t[0, 1].double().cpu().numpy() for t in (q, k, v, do))
    wh = layer.w[1].double().cpu().numpy()
    o_r, _, _ = ro.forward(qh, kh, vh, wh, cfg.beta, causal)
    grads = ro.vjp(qh, kh, vh, wh, cfg.beta, gh, causal)
    assert rel_err(outs[0][0][0, 1], o_r) <= TOL_BF16
    for got, ref in zip(outs[0][1:], grads):
        assert rel_err(got[0, 1], ref) <= TOL_BF16


def test_race_gpt_trains():
    from paper_2510_04008_b200.gpt import GPTConfig, RaceGPT, train_step

    dev = _cuda()
    torch.manual_seed(0)
    cfg = GPTConfig(vocab=512, seq_len=1024, layers=2, d_model=256, heads=4)
    model = RaceGPT(cfg).to(dev)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-3, fused=True)
    idx = torch.randint(0, cfg.vocab, (2, cfg.seq_len), device=dev)
    tgt = torch.roll(idx, -1, dims=1)
    losses = [float(train_step(model, opt, idx, tgt)) for _ in range(25)]
    assert all(np.isfinite(losses))
    assert min(losses[-5:]) < losses[0] - 0.5, losses  # memorising a fixed batch
    # every parameter received a gradient on the last step (before zero_grad)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = torch.nn.functional.cross_entropy(model(idx).float().view(-1, cfg.vocab), tgt.view(-1))
    loss.backward()
    assert all(p.grad is not None and torch.isfinite(p.grad).all() for p in model.parameters())
