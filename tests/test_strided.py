"""Strided operands: [B, N, H, d]-ordered q, k, v, dO (views of a fused projection's output) run in
place on the one-pass tcgen05 path through 4-D TMA maps (race_fwd_layout / race_bwd_layout), with
results identical to the contiguous run of the same values; everything else falls back to
contiguous copies.  Also the CPU-side layout detection and the ABI's rejection of strided grouped
problems."""

from __future__ import annotations

import ctypes

import pytest
import torch

import paper_2510_04008_b200 as rb
from paper_2510_04008_b200 import _lib
from paper_2510_04008_b200.functional import Problem, _strides


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _qkv_views(b, n, h, d, dtype, dev, seed=0):
    """q, k, v as [B, H, N, d] views of one [B, N, 3*H*d] projection output (no copies)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    qkv = torch.randn(b, n, 3 * h * d, generator=g, device=dev).to(dtype)
    q, k, v = (t.view(b, n, h, d).transpose(1, 2) for t in qkv.split(h * d, dim=-1))
    return qkv, q, k, v


def test_stride_detection_cpu():
    x = torch.zeros(2, 100, 3 * 4 * 64, dtype=torch.bfloat16)
    q = x[..., : 4 * 64].view(2, 100, 4, 64).transpose(1, 2)
    assert _strides(q) == (3 * 4 * 64, 64, 100 * 3 * 4 * 64)
    assert _strides(q.contiguous()) is None                      # contiguous: the default layout
    assert _strides(torch.zeros(2, 4, 100, 64)[..., :32]) == (64, 6400, 25600)  # width 32 at row pitch 64
    assert _strides(torch.zeros(2, 4, 100, 64).transpose(2, 3)) is None  # rows not contiguous


def test_layout_struct_matches_header():
    assert ctypes.sizeof(_lib.RaceStride) == 24
    assert ctypes.sizeof(_lib.RaceLayout) == 8 * 24


@pytest.mark.gpu
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("d", [64, 128])
def test_strided_equals_contiguous(causal, d):
    dev = _cuda()
    b, n, h = 2, 1000, 3
    _, q, k, v = _qkv_views(b, n, h, d, torch.bfloat16, dev)
    gen = torch.Generator(device=dev).manual_seed(1)
    do = torch.randn(b, n, h * d, generator=gen, device=dev).to(torch.bfloat16).view(b, n, h, d).transpose(1, 2)
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=3, causal=causal)
    w = rb.head_hyperplanes(cfg, h, d).to(dev)
    p = cfg.params()
    assert Problem(q, k, v, w, p).one_pass_fast
    n0 = _lib.lib().race_launch_count()
    o, den, st = rb.race_forward(q, k, v, w, p)
    dq, dk, dv = rb.race_backward(q, k, v, w, do, p, state=st)
    assert _lib.lib().race_launch_count() > n0
    # outputs come back in the inputs' [B, N, H, d] storage order: the transpose back is a free view
    for t in (o, dq, dk, dv):
        assert t.transpose(1, 2).is_contiguous()
    qc, kc, vc, doc = (t.contiguous() for t in (q, k, v, do))
    o2, den2, st2 = rb.race_forward(qc, kc, vc, w, p)
    dq2, dk2, dv2 = rb.race_backward(qc, kc, vc, w, doc, p, state=st2)
    torch.cuda.synchronize()
    for a, c in ((o, o2), (den, den2), (dq, dq2), (dk, dk2), (dv, dv2)):
        assert torch.equal(a, c)


@pytest.mark.gpu
def test_strided_mixed_and_autograd():
    """Strided q, k with a contiguous v, through the autograd layer; the GPT block's pattern."""
    dev = _cuda()
    b, n, h, d = 1, 777, 4, 64
    qkv, q, k, _ = _qkv_views(b, n, h, d, torch.bfloat16, dev, seed=5)
    v = torch.randn(b, h, n, d, device=dev).to(torch.bfloat16)
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=True)
    layer = rb.RaceAttention(h, d, cfg).to(dev)
    qkv = qkv.detach().requires_grad_(True)
    vv = v.detach().requires_grad_(True)
    q, k, _ = (t.view(b, n, h, d).transpose(1, 2) for t in qkv.split(h * d, dim=-1))
    out = layer(q, k, vv)
    g = torch.randn_like(out)
    out.backward(g)
    qc = q.detach().contiguous().requires_grad_(True)
    kc = k.detach().contiguous().requires_grad_(True)
    vc = v.detach().clone().requires_grad_(True)
    out2 = layer(qc, kc, vc)
    out2.backward(g)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    assert torch.equal(qkv.grad[..., : h * d].view(b, n, h, d).transpose(1, 2), qc.grad)
    assert torch.equal(qkv.grad[..., h * d: 2 * h * d].view(b, n, h, d).transpose(1, 2), kc.grad)
    assert torch.equal(vv.grad, vc.grad)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tables", [(torch.float32, 2), (torch.bfloat16, 4)])
def test_strided_fallback_paths(dtype, tables):
    """fp32 (CUDA-core kernels) and a grouped bf16 sketch take contiguous copies: same results."""
    dev = _cuda()
    b, n, h, d = 1, 600, 2, 64
    _, q, k, v = _qkv_views(b, n, h, d, dtype, dev, seed=7)
    cfg = rb.SketchConfig(hyperplanes=2, tables=tables, seed=0, causal=True)
    w = rb.head_hyperplanes(cfg, h, d).to(dev)
    p = cfg.params()
    assert not Problem(q, k, v, w, p).one_pass_fast
    o, den, st = rb.race_forward(q, k, v, w, p)
    o2, den2, _ = rb.race_forward(q.contiguous(), k.contiguous(), v.contiguous(), w, p)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(den, den2)


@pytest.mark.gpu
def test_layout_abi_rejects_grouped():
    dev = _cuda()
    b, n, h, d = 1, 256, 2, 64
    _, q, k, v = _qkv_views(b, n, h, d, torch.bfloat16, dev)
    cfg = rb.SketchConfig(hyperplanes=2, tables=4, seed=0, causal=True)  # F = 16: two passes
    w = rb.head_hyperplanes(cfg, h, d).to(dev)
    pr = Problem(q, k, v, w, cfg.params())
    lay = _lib.RaceLayout()
    lay.q.token, lay.q.head, lay.q.batch = _strides(q)
    o = torch.empty(b, h, n, d, dtype=torch.bfloat16, device=dev)
    den = torch.empty(b, h, n, device=dev)
    ws = pr.ws()
    rc = _lib.lib().race_fwd_layout(pr.dref, ctypes.byref(lay), q.data_ptr(), k.contiguous().data_ptr(),
                                    v.contiguous().data_ptr(), pr.w.data_ptr(), o.data_ptr(), den.data_ptr(), None,
                                    ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.RACE_EUNSUPPORTED
    assert b"tcgen05" in _lib.lib().race_last_error()
