"""GPU parity: the CUDA path (through the C-ABI) against the reference.

Tolerances (BASELINE.json north_star): rel err <= 1e-3 for fp32 inputs and
<= 1e-2 for bf16 inputs, metric max|a-b|/max|b| (ra/acceptance.py:89-91).
For gradients the denominator is floored at 5% of the call's largest
reference gradient, so components that vanish in exact arithmetic (d = 1,
N = 1) are judged on the natural gradient scale rather than on 1e-17 noise.

* golden fixtures (tests/golden, produced by the real reference): every case
  through the drop-in numpy API (fp32 on device), and the bf16-valued cases
  again as bf16 tensors;
* config-1 shapes (B=1, H=4, d=128, N=4096, P=2, L=2) against the oracle on
  the same (upcast) inputs, fp32 and bf16, causal and non-causal;
* size-independent properties at the BASELINE sizes (N=131072 bf16 causal):
  constant V, determinism, causal prefix consistency, sequence sharding.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2510_04008_b200 as rb
from conftest import grad_errs, load_golden, rel_err
from oracle import race_oracle as ro
from paper_2510_04008_b200 import _lib
from paper_2510_04008_b200.sharded import sharded_backward, sharded_forward

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-3
TOL_BF16 = 1e-2
GRAD_FLOOR = 0.05

CASES = load_golden()


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _is_bf16_valued(a):
    f = np.asarray(a, dtype=np.float32)
    return np.array_equal(f.view(np.uint32) & 0xFFFF, np.zeros_like(f.view(np.uint32)))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['index']:03d}-{c['tag']}")
def test_golden_fp32(case):
    _cuda()
    cfg = rb.SketchConfig(**case.cfg_kwargs)
    inp = rb.AttnInputs(case["q"], case["k"], case["v"])
    out = rb.race_attention(inp, cfg)  # P = 11 cases run as corner groups (factored form)
    assert out.o.dtype == np.float64 and out.den.dtype == np.float64
    assert rel_err(out.o, case["o"]) <= TOL_F32
    assert rel_err(out.den, case["den"]) <= TOL_F32
    flags = np.zeros(inp.n, dtype=bool)
    flags[list(out.degenerate_rows)] = True
    assert np.array_equal(flags, case["degenerate"])
    g = rb.race_attention_vjp(inp, cfg, case["d_out"])
    errs = grad_errs((g.dq, g.dk, g.dv), (case["dq"], case["dk"], case["dv"]), GRAD_FLOOR)
    assert max(errs) <= TOL_F32, errs


BF16_CASES = [c for c in CASES if all(_is_bf16_valued(c[x]) for x in ("q", "k", "v", "d_out"))]


@pytest.mark.parametrize("case", BF16_CASES, ids=lambda c: f"{c['index']:03d}-{c['tag']}")
def test_golden_bf16(case):
    dev = _cuda()
    cfg = rb.SketchConfig(**case.cfg_kwargs)
    t = {x: torch.from_numpy(case[x].astype(np.float32)).to(dev, torch.bfloat16) for x in ("q", "k", "v", "d_out")}
    inp = rb.AttnInputs(t["q"], t["k"], t["v"])
    out = rb.race_attention(inp, cfg)
    assert out.o.dtype == torch.bfloat16
    assert rel_err(out.o.float().cpu(), case["o"]) <= TOL_BF16
    assert rel_err(out.den.cpu(), case["den"]) <= TOL_F32  # den is kept in fp32
    g = rb.race_attention_vjp(inp, cfg, t["d_out"])
    errs = grad_errs([x.float().cpu().numpy() for x in (g.dq, g.dk, g.dv)],
                     (case["dq"], case["dk"], case["dv"]), GRAD_FLOOR)
    assert max(errs) <= TOL_BF16, errs


# ---------------------------------------------------------------------------
# config-1 shapes vs the oracle on identical inputs
# ---------------------------------------------------------------------------
def _layer_inputs(n, d, heads, dtype, seed=0):
    per_head = ro.head_inputs(seed, n, d, heads, np.float32)
    dev = _cuda()
    stack = [np.stack([h[i] for h in per_head])[None] for i in range(4)]  # [1, H, N, d]
    q, k, v, g = (torch.from_numpy(a).to(dev, dtype) for a in stack)
    return q, k, v, g


def _oracle_layer(q, k, v, g, w, beta, causal):
    """Per-head oracle in float64 on the device's exact input values."""
    outs = []
    for h in range(q.shape[1]):
        qh, kh, vh, gh = (t[0, h].double().cpu().numpy() for t in (q, k, v, g))
        wh = w[h].double().cpu().numpy()
        o, den, _ = ro.forward(qh, kh, vh, wh, beta, causal)
        dq, dk, dv = ro.vjp(qh, kh, vh, wh, beta, gh, causal)
        outs.append((o, den, dq, dk, dv))
    return outs


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("n", [4096, 1000])
def test_config1_layer(dtype, causal, n):
    q, k, v, g = _layer_inputs(n, 128, 4, dtype)
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=causal)
    layer = rb.RaceAttention(4, 128, cfg).to(q.device)
    p = layer.params_
    o, den, state = rb.race_forward(q, k, v, layer.w, p)
    dq, dk, dv = rb.race_backward(q, k, v, layer.w, g, p, state=state)
    ref = _oracle_layer(q, k, v, g, layer.w, cfg.beta, causal)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    for h, (o_r, den_r, dq_r, dk_r, dv_r) in enumerate(ref):
        assert rel_err(o[0, h].float().cpu(), o_r) <= tol
        assert rel_err(den[0, h].cpu(), den_r) <= TOL_F32
        errs = grad_errs([t[0, h].float().cpu().numpy() for t in (dq, dk, dv)], (dq_r, dk_r, dv_r), GRAD_FLOOR)
        assert max(errs) <= tol, (h, errs)
    # backward without saved state (reference-style recompute) is bit-identical
    dq2, dk2, dv2 = rb.race_backward(q, k, v, layer.w, g, p, state=None)
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)


def test_autograd_matches_vjp():
    q, k, v, g = _layer_inputs(777, 64, 2, torch.float32, seed=3)
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=9, causal=True)
    layer = rb.RaceAttention(2, 64, cfg).to(q.device)
    qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
    o = layer(qq, kk, vv)
    (o * g).sum().backward()
    dq, dk, dv = rb.race_backward(q, k, v, layer.w, g, layer.params_)
    assert torch.equal(qq.grad, dq) and torch.equal(kk.grad, dk) and torch.equal(vv.grad, dv)


# ---------------------------------------------------------------------------
# properties at the BASELINE size (config 2: causal N=131072 bf16, H=4)
# ---------------------------------------------------------------------------
def _big(n=131072, dtype=torch.bfloat16, causal=True, seed=1):
    dev = _cuda()
    gen = torch.Generator(device=dev).manual_seed(seed)
    shape = (1, 4, n, 128)
    q, k, v, g = (torch.randn(shape, generator=gen, device=dev).to(dtype) for _ in range(4))
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
    return q, k, v, g, w, cfg.params()


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
def test_constant_values_give_constant_output(causal):
    q, k, v, g, w, p = _big(causal=causal)
    c = torch.randn(128, device=q.device).to(torch.bfloat16)
    vc = c.expand_as(v).contiguous()
    o, den, _ = rb.race_forward(q, k, vc, w, p, want_state=False)
    assert rel_err(o.float().cpu(), c.float().expand_as(o).cpu()) <= 1e-2
    assert bool((den > 0).all())


def test_determinism_bitwise():
    q, k, v, g, w, p = _big()
    a = rb.race_forward(q, k, v, w, p)
    b = rb.race_forward(q, k, v, w, p)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    ga = rb.race_backward(q, k, v, w, g, p, a[2])
    gb = rb.race_backward(q, k, v, w, g, p, b[2])
    assert all(torch.equal(x, y) for x, y in zip(ga, gb))


def test_causal_prefix_consistency():
    """Criterion 2 (ra/acceptance.py:167-196): causal row t == non-causal on keys 0..t."""
    q, k, v, g, w, p = _big(n=20000, dtype=torch.float32)
    o, _, _ = rb.race_forward(q, k, v, w, p, want_state=False)
    pn = rb.SketchParams(p.hyperplanes, p.tables, p.beta, False)
    for t in (0, 1, 127, 128, 4095, 12345, 19999):
        on, _, _ = rb.race_forward(q[:, :, :t + 1], k[:, :, :t + 1], v[:, :, :t + 1], w, pn, want_state=False)
        assert rel_err(o[0, :, t].cpu(), on[0, :, t].cpu()) <= TOL_F32, t


def test_mass_conservation():
    """Criterion 8 (ra/acceptance.py:383-416): column dv of S sums to N*T; colsum of B = T*colsum V."""
    q, k, v, g, w, p = _big(n=65536, dtype=torch.float32, causal=False)
    _, _, state = rb.race_forward(q, k, v, w, p)
    s = state.double()
    n = q.shape[2]
    assert torch.allclose(s[..., -1].sum(-1), torch.full((4,), float(n * p.tables), dtype=torch.float64,
                                                          device=s.device), rtol=1e-5)
    colsum = s[..., :-1].sum(1)
    assert rel_err(colsum.cpu(), (p.tables * v[0].double().sum(1)).cpu()) <= 1e-4


class _EmuComm:
    """Single-process stand-in for torch.distributed: rank `r` of `world`."""

    def __init__(self, rank, totals, record):
        self.rank, self.totals, self.record = rank, totals, record

    def allreduce(self, local):
        self.record.append(local.clone())
        return sum(self.totals) if self.totals else local.clone()

    def carry(self, local, direction):
        self.record.append(local.clone())
        if not self.totals:
            return torch.zeros_like(local)
        idx = range(self.rank) if direction == "prefix" else range(len(self.totals) - 1, self.rank, -1)
        out = torch.zeros_like(local)
        for r in idx:
            out += self.totals[r]
        return out


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_sequence_sharding_matches_single_gpu(causal, dtype):
    """Split-phase C-ABI + exchange algebra with 3 emulated ranks
    (f32: generic kernels; bf16: the tcgen05 fast path)."""
    q, k, v, g, w, p = _big(n=50000, dtype=dtype, causal=causal)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    o1, den1, st1 = rb.race_forward(q, k, v, w, p)
    dq1, dk1, dv1 = rb.race_backward(q, k, v, w, g, p, st1)
    world = 3
    bounds = [rb.shard_bounds(q.shape[2], world, r) for r in range(world)]
    sl = [(q[:, :, a:b], k[:, :, a:b], v[:, :, a:b], g[:, :, a:b]) for a, b in bounds]
    # pass 1: record local totals; pass 2: run with the true exchange
    rec = [[] for _ in range(world)]
    for r in range(world):
        sharded_forward(*sl[r][:3], w, p, comm=_EmuComm(r, None, rec[r]))
    totals = [rec[r][0] for r in range(world)]
    outs = [sharded_forward(*sl[r][:3], w, p, comm=_EmuComm(r, totals, [])) for r in range(world)]
    o = torch.cat([x[0] for x in outs], dim=2)
    den = torch.cat([x[1] for x in outs], dim=2)
    assert rel_err(o.float().cpu(), o1.float().cpu()) <= tol and rel_err(den.cpu(), den1.cpu()) <= 1e-4
    rec = [[] for _ in range(world)]
    for r in range(world):
        q_, k_, v_, g_ = sl[r]
        sharded_backward(q_, k_, v_, w, g_, p, outs[r][2], comm=_EmuComm(r, None, rec[r]))
    dtot = [rec[r][0] for r in range(world)]
    grads = [sharded_backward(sl[r][0], sl[r][1], sl[r][2], w, sl[r][3], p, outs[r][2], comm=_EmuComm(r, dtot, []))
             for r in range(world)]
    for i, ref in enumerate((dq1, dk1, dv1)):
        got = torch.cat([x[i] for x in grads], dim=2)
        assert rel_err(got.float().cpu(), ref.float().cpu()) <= tol, i


def test_n1_output_is_v_and_empty():
    dev = _cuda()
    cfg = rb.SketchConfig(hyperplanes=2, tables=2)
    v = np.random.default_rng(0).standard_normal((1, 16)).astype(np.float32)
    out = rb.race_attention(rb.AttnInputs(v[:, :8], v[:, 8:], v), cfg)
    assert np.allclose(out.o, v, rtol=1e-6, atol=1e-6)
    e = np.zeros((0, 8), np.float32)
    out = rb.race_attention(rb.AttnInputs(e, e, e), cfg)
    assert out.o.shape == (0, 8) and out.degenerate_rows == ()
    assert dev.type == "cuda"


def test_bad_d_out_raises():
    _cuda()
    rng = np.random.default_rng(0)
    inp = rb.AttnInputs(*(rng.standard_normal((8, 4)) for _ in range(3)))
    with pytest.raises(ValueError):
        rb.race_attention_vjp(inp, rb.SketchConfig(hyperplanes=2, tables=2), np.ones((8, 3)))


def test_workers_invariance():
    """Criterion 9: identical results for any `workers` value."""
    _cuda()
    rng = np.random.default_rng(19)
    inp = rb.AttnInputs(*(rng.standard_normal((33, 6)) for _ in range(2)), rng.standard_normal((33, 5)))
    cfg = rb.SketchConfig(hyperplanes=2, tables=3, ensembles=2, seed=777, causal=True)
    a, b = rb.race_attention(inp, cfg), rb.race_attention(inp, cfg, workers=4)
    assert np.array_equal(a.o, b.o) and np.array_equal(a.den, b.den)


# ---------------------------------------------------------------------------
# sm_100a fast path (tcgen05/TMA) against the generic CUDA kernels and the oracle
# ---------------------------------------------------------------------------
def _both_paths(fn):
    import os

    os.environ["RACE_DISABLE_FAST_PATH"] = "1"
    try:
        slow = fn()
    finally:
        os.environ.pop("RACE_DISABLE_FAST_PATH", None)
    fast = fn()
    return fast, slow


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("n", [128, 1000, 4096, 4099, 16666, 70000])  # incl. N % 4 != 0 (TMA row pitch)
@pytest.mark.parametrize("pl", [(2, 2), (1, 3), (3, 1)], ids=["P2L2", "P1L3", "P3L1"])
def test_fast_path_forward(causal, n, pl):
    q, k, v, g, w, p = _big(n=n, causal=causal)
    P, L = pl
    cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=3, causal=causal)
    w = rb.head_hyperplanes(cfg, 4, 128).to(q.device)
    p = cfg.params()
    from paper_2510_04008_b200.functional import Problem

    assert _lib.fast_path(Problem(q, k, v, w, p).desc)
    (o_f, den_f, st_f), (o_s, den_s, st_s) = _both_paths(lambda: rb.race_forward(q, k, v, w, p))
    if causal:  # carries, and the row norms of the sketch rows (the generic path leaves the projections 0)
        pr = Problem(q, k, v, w, p)
        (car_f, rows_f), (car_s, rows_s) = pr.split_causal_state(st_f), pr.split_causal_state(st_s)
        assert rel_err(car_f.cpu(), car_s.cpu()) <= 1e-4
        assert rel_err(rows_f[..., [7, 15]].cpu(), rows_s[..., [7, 15]].cpu()) <= 1e-4
    else:
        assert rel_err(st_f.cpu(), st_s.cpu()) <= 1e-4
    assert rel_err(den_f.cpu(), den_s.cpu()) <= 1e-4
    assert rel_err(o_f.float().cpu(), o_s.float().cpu()) <= TOL_BF16
    if n <= 4096:  # and against the oracle, head 0
        qh, kh, vh = (t[0, 0].double().cpu().numpy() for t in (q, k, v))
        o_r, den_r, _ = ro.forward(qh, kh, vh, w[0].double().cpu().numpy(), cfg.beta, causal)
        assert rel_err(o_f[0, 0].float().cpu(), o_r) <= TOL_BF16
        assert rel_err(den_f[0, 0].cpu(), den_r) <= TOL_F32


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("n", [128, 1000, 4096, 4099, 16666, 70000])  # incl. N % 4 != 0 (TMA row pitch)
@pytest.mark.parametrize("pl", [(2, 2), (1, 3), (3, 1)], ids=["P2L2", "P1L3", "P3L1"])
def test_fast_path_backward(causal, n, pl):
    q, k, v, g, w, p = _big(n=n, causal=causal)
    P, L = pl
    cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=5, causal=causal)
    w = rb.head_hyperplanes(cfg, 4, 128).to(q.device)
    p = cfg.params()

    def run():
        o, den, st = rb.race_forward(q, k, v, w, p)
        return rb.race_backward(q, k, v, w, g, p, state=st)

    fast, slow = _both_paths(run)
    for x, y in zip(fast, slow):
        assert rel_err(x.float().cpu(), y.float().cpu()) <= TOL_BF16
    if n <= 4096:
        qh, kh, vh, gh = (t[0, 1].double().cpu().numpy() for t in (q, k, v, g))
        ref = ro.vjp(qh, kh, vh, w[1].double().cpu().numpy(), cfg.beta, gh, causal)
        errs = grad_errs([t[0, 1].float().cpu().numpy() for t in fast], ref, GRAD_FLOOR)
        assert max(errs) <= TOL_BF16, errs


def test_long_context_prefix_and_oracle():
    """BASELINE configs[2] scale: a 16 Mi-token causal layer (bf16, ~140 GB resident).

    Causal outputs of the first 4096 tokens depend on those tokens only, so O,
    den and dQ of that prefix must match (a) the same layer run on the prefix
    alone and (b) the float64 oracle; the tail must be finite.  This covers the
    long-sequence carry chain (many segments per head, carries over 16M tokens)."""
    n, n0 = 1 << 24, 4096
    dev = _cuda()
    free, _ = torch.cuda.mem_get_info(dev)
    if free < n * 8700:
        pytest.skip("needs ~145 GB of free HBM")
    gen = torch.Generator(device=dev).manual_seed(11)
    shape = (1, 4, n, 128)
    q, k, v, g = (torch.randn(shape, generator=gen, device=dev, dtype=torch.bfloat16) for _ in range(4))
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=True)
    w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
    p = cfg.params()
    o, den, st = rb.race_forward(q, k, v, w, p)
    dq, dk, dv = rb.race_backward(q, k, v, w, g, p, state=st)
    o0, den0, dq0 = o[:, :, :n0].clone(), den[:, :, :n0].clone(), dq[:, :, :n0].clone()
    tail_ok = all(bool(torch.isfinite(t[:, :, -4096:].float()).all()) for t in (o, dq, dk, dv))
    qp, kp, vp, gp = (t[:, :, :n0].clone() for t in (q, k, v, g))
    del q, k, v, g, o, den, st, dq, dk, dv
    torch.cuda.empty_cache()
    assert tail_ok
    op, denp, stp = rb.race_forward(qp, kp, vp, w, p)
    dqp, _, _ = rb.race_backward(qp, kp, vp, w, gp, p, state=stp)
    assert rel_err(o0.float().cpu(), op.float().cpu().numpy()) <= TOL_BF16
    assert rel_err(den0.cpu(), denp.cpu().numpy()) <= 1e-4
    assert rel_err(dq0.float().cpu(), dqp.float().cpu().numpy()) <= TOL_BF16
    qh, kh, vh, gh = (t[0, 0].double().cpu().numpy() for t in (qp, kp, vp, gp))
    o_r, den_r, _ = ro.forward(qh, kh, vh, w[0].double().cpu().numpy(), cfg.beta, True)
    dq_r, _, _ = ro.vjp(qh, kh, vh, w[0].double().cpu().numpy(), cfg.beta, gh, True)
    assert rel_err(o0[0, 0].float().cpu(), o_r) <= TOL_BF16
    assert rel_err(den0[0, 0].cpu(), den_r) <= TOL_F32
    assert rel_err(dq0[0, 0].float().cpu(), dq_r) <= TOL_BF16


@pytest.mark.parametrize("n", [1000, 4099, 70000])
@pytest.mark.parametrize("pl", [(2, 2), (1, 3), (3, 1)], ids=["P2L2", "P1L3", "P3L1"])
def test_causal_forward_from_kside_rows(n, pl):
    """race_kside_partials_rows + race_fwd_causal_krows (k projections taken from the rows the
    aggregation wrote; K not re-read) == race_kside_partials + race_fwd_causal."""
    from paper_2510_04008_b200.functional import Problem, _stream, _vp

    q, k, v, g, w, p = _big(n=n, causal=True)
    P, L = pl
    cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=7, causal=True)
    w = rb.head_hyperplanes(cfg, 4, 128).to(q.device)
    p = cfg.params()
    pr = Problem(q, k, v, w, p)
    lib, S, ws = _lib.lib(), _stream(), pr.ws()
    outs = []
    for krows in (False, True):
        part = torch.empty((pr.bh, pr.nseg, pr.table_elems), device=q.device)
        state = torch.full(pr.state_shape(), float("nan"), device=q.device)
        car, rows = pr.split_causal_state(state)
        o, den = torch.empty_like(v), torch.empty((1, 4, n), device=q.device)
        if krows:
            _lib.check(lib.race_kside_partials_rows(pr.dref, _vp(k), _vp(v), _vp(pr.w), _vp(part), _vp(rows),
                                                    _vp(ws), S), "kside_rows")
        else:
            _lib.check(lib.race_kside_partials(pr.dref, _vp(k), _vp(v), _vp(pr.w), _vp(part), _vp(ws), S), "kside")
        _lib.check(lib.race_combine(pr.dref, _lib.COMBINE_PREFIX, _vp(part), None, _vp(car), S), "combine")
        fn = lib.race_fwd_causal_krows if krows else lib.race_fwd_causal
        _lib.check(fn(pr.dref, _vp(q), _vp(k), _vp(v), _vp(pr.w), _vp(car), _vp(o), _vp(den), _vp(rows), _vp(ws), S),
                   "fwd")
        torch.cuda.synchronize()
        # carries + sketch rows (not the alignment gap between them, race_state_elems)
        outs.append((o.float().cpu(), den.cpu(), torch.cat([car.flatten(), rows.flatten()]).cpu()))
    (o0, d0, s0), (o1, d1, s1) = outs
    assert torch.isfinite(s1).all()
    assert rel_err(s1, s0) <= 1e-6
    assert rel_err(d1, d0) <= 1e-5
    assert rel_err(o1, o0) <= 1e-2


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("shape", [(300, 16, 16, 2, 300), (130, 128, 64, 3, 40)], ids=["L300", "P3L40"])
def test_table_groups_match_oracle(causal, shape):
    """F beyond one kernel pass (the reference's own criteria 4/5 use P=2 with up to 2048 tables):
    tables run in groups whose numerators, denominators and gradients are summed."""
    n, d, dv, P, L = shape
    dev = _cuda()
    rng = np.random.default_rng(5)
    q, k, v, g = (rng.standard_normal((n, x)) for x in (d, d, dv, dv))
    cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=9, causal=causal)
    from paper_2510_04008_b200.functional import Problem

    t = [torch.tensor(x, dtype=torch.float32, device=dev)[None] for x in (q, k, v, g)]
    w = torch.tensor(rb.all_hyperplanes(cfg, d), dtype=torch.float32, device=dev)
    pr = Problem(t[0], t[1], t[2], w, cfg.params())
    assert pr.grouped and pr.state_shape() == (n * (dv + 1),)  # grouped: the summed num / den are the state
    o, den, st = rb.race_forward(t[0], t[1], t[2], w, cfg.params())
    dq, dk, dvv = rb.race_backward(t[0], t[1], t[2], w, t[3], cfg.params(), state=st)
    # the saved sums give exactly the recomputing backward's gradients (ra/backward.py:200 recomputes)
    for a, b in zip((dq, dk, dvv), rb.race_backward(t[0], t[1], t[2], w, t[3], cfg.params())):
        assert torch.equal(a, b)
    wr = rb.all_hyperplanes(cfg, d)
    o_r, den_r, _ = ro.forward(q, k, v, wr, cfg.beta, causal)
    assert rel_err(o[0].cpu(), o_r) <= TOL_F32
    assert rel_err(den[0].cpu(), den_r) <= TOL_F32
    ref = ro.vjp(q, k, v, wr, cfg.beta, g, causal)
    errs = grad_errs([x[0].cpu().numpy() for x in (dq, dk, dvv)], ref, GRAD_FLOOR)
    assert max(errs) <= TOL_F32, errs
    # the drop-in API runs the same configs (ra/acceptance.py criteria 4-5 use L up to 2048)
    out = rb.race_attention(rb.AttnInputs(q, k, v), cfg, w=wr)
    assert rel_err(out.o, o_r) <= TOL_F32


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("kind", ["fast", "generic", "groups"])
def test_inplace_backward_matches(causal, kind):
    """race_bwd with dq, dk, dv aliasing q, k, v gives the allocating backward's results bit for bit."""
    dev = _cuda()
    n = 5000
    if kind == "fast":
        q, k, v, g, w, p = _big(n=n, causal=causal)
    else:
        d = 32
        P, L = (2, 2) if kind == "generic" else (2, 300)
        gen = torch.Generator(device=dev).manual_seed(3)
        q, k, v, g = (torch.randn(1, 2, n if kind == "generic" else 300, d, generator=gen, device=dev)
                      for _ in range(4))
        cfg = rb.SketchConfig(hyperplanes=P, tables=L, seed=1, causal=causal)
        w = rb.head_hyperplanes(cfg, 2, d).to(dev)
        p = cfg.params()
    o, den, st = rb.race_forward(q, k, v, w, p)
    ref = rb.race_backward(q, k, v, w, g, p, state=st)
    qc, kc, vc = q.clone(), k.clone(), v.clone()
    got = rb.race_backward(qc, kc, vc, w, g, p, state=st, inplace=True)
    assert got[0].data_ptr() == qc.data_ptr() and got[2].data_ptr() == vc.data_ptr()
    for a, b in zip(got, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("dims", [(64, 64), (96, 128), (128, 32), (8, 8), (40, 72)],
                         ids=["d64", "d96dv128", "dv32", "d8", "d40dv72"])
def test_narrow_bf16_heads_run_natively_on_fast_path(causal, dims):
    """bf16 heads narrower than 128 run on the tcgen05 kernels at their own width (TMA zero-fills the
    tile columns beyond d, clips the stores; tables use the dv + 1 row stride); results match the
    generic path and the oracle."""
    dev = _cuda()
    d, dv = dims
    n = 3000
    gen = torch.Generator(device=dev).manual_seed(11)
    q, k = (torch.randn(1, 2, n, d, generator=gen, device=dev).to(torch.bfloat16) for _ in range(2))
    v, g = (torch.randn(1, 2, n, dv, generator=gen, device=dev).to(torch.bfloat16) for _ in range(2))
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=4, causal=causal)
    w = rb.head_hyperplanes(cfg, 2, d).to(dev)
    p = cfg.params()
    from paper_2510_04008_b200.functional import Problem

    assert _lib.fast_path(Problem(q, k, v, w, p).desc)

    def run():
        o, den, st = rb.race_forward(q, k, v, w, p)
        return (o, den) + tuple(rb.race_backward(q, k, v, w, g, p, state=st))

    fast, slow = _both_paths(run)
    assert fast[0].shape == (1, 2, n, dv) and fast[1].shape == (1, 2, n)
    for x, y in zip(fast, slow):
        assert rel_err(x.float().cpu(), y.float().cpu()) <= TOL_BF16
    qh, kh, vh, gh = (t[0, 1].double().cpu().numpy() for t in (q, k, v, g))
    wh = w[1].double().cpu().numpy()
    o_r, _, _ = ro.forward(qh, kh, vh, wh, cfg.beta, causal)
    assert rel_err(fast[0][0, 1].float().cpu(), o_r) <= TOL_BF16
    ref = ro.vjp(qh, kh, vh, wh, cfg.beta, gh, causal)
    errs = grad_errs([t[0, 1].float().cpu().numpy() for t in fast[2:]], ref, GRAD_FLOOR)
    assert max(errs) <= TOL_BF16, errs
    qc, kc, vc = q.clone(), k.clone(), v.clone()
    st = rb.race_forward(q, k, v, w, p)[2]
    got = rb.race_backward(qc, kc, vc, w, g, p, state=st, inplace=True)
    assert got[0] is qc and torch.equal(qc, fast[2])


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
@pytest.mark.parametrize("shape", [(2, 3, 777), (3, 1, 129), (1, 7, 2560), (5, 2, 1)], ids=lambda s: "x".join(map(str, s)))
def test_fast_path_batch_head_layouts(causal, shape):
    """B > 1, odd head counts (per-head hyperplanes picked by bh % H), ragged and tiny N: the
    tcgen05 path matches the generic path, forward and backward."""
    dev = _cuda()
    B, H, n = shape
    gen = torch.Generator(device=dev).manual_seed(B * 100 + H * 10 + n)
    q, k, v, g = (torch.randn(B, H, n, 128, generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=21, causal=causal)
    w = rb.head_hyperplanes(cfg, H, 128).to(dev)
    p = cfg.params()

    def run():
        o, den, st = rb.race_forward(q, k, v, w, p)
        return (o, den) + tuple(rb.race_backward(q, k, v, w, g, p, state=st))

    fast, slow = _both_paths(run)
    for x, y in zip(fast[:2], slow[:2]):
        assert x.shape == y.shape
        assert rel_err(x.float().cpu(), y.float().cpu()) <= TOL_BF16
    # gradients: denominator floored at 5% of the call's largest gradient (N = 1: dq = dk = 0 exactly)
    scale = max(float(t.float().abs().max()) for t in slow[2:])
    for x, y in zip(fast[2:], slow[2:]):
        assert x.shape == y.shape
        err = float((x.float() - y.float()).abs().max()) / max(float(y.float().abs().max()), GRAD_FLOOR * scale)
        assert err <= TOL_BF16, err
