"""Exact quadratic attention references on the GPU (mirror of ra/exact.py).

* ``angular_similarity``        ra/exact.py:96-113   (two vectors; host scalar math)
* ``angular_kernel_matrix``     ra/exact.py:116-125  -> race_aux_angular_kernel
* ``angular_attention``         ra/exact.py:128-166  -> race_aux_angular_fwd
* ``angular_attention_vjp``     ra/exact.py:169-218  -> race_aux_angular_fwd + race_aux_angular_bwd
* ``softmax_attention[_vjp]``   ra/exact.py:54-93    (float64 torch ops on the device; library GEMMs)

The angular kernels (csrc/race_aux.cu) are tiled fp64 flash-style passes:
no N x N matrix is materialised, so the accuracy reference reaches N far
beyond the reference's CPU limits, and results match it to ~1e-12.
Outputs follow the reference's dtype rules (input dtype).
"""

from __future__ import annotations

import math
import warnings

import numpy as np
import torch

from . import _aux
from .attention import DEGENERATE_DEN_EPS, AttnInputs, _as_matrix


def _check_gamma(gamma) -> int:
    if not (isinstance(gamma, (int, np.integer)) and not isinstance(gamma, bool) and gamma >= 1):
        raise ValueError(f"gamma must be a positive integer, got {gamma!r}")
    return int(gamma)


def _nonzero_rows(*ts: torch.Tensor) -> None:
    for t in ts:
        if t.shape[0] and bool((t.double().norm(dim=1) == 0).any()):
            raise ValueError("zero-norm rows are not allowed")


def angular_similarity(q, k, gamma: int) -> float:
    """(1 - theta/pi)^gamma between two vectors, dot clamped to [-1, 1] (ra/exact.py:96-113)."""
    gamma = _check_gamma(gamma)
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    k = np.asarray(k, dtype=np.float64).reshape(-1)
    if q.shape != k.shape:
        raise ValueError("q and k must have equal length")
    nq, nk = math.sqrt(float(q @ q)), math.sqrt(float(k @ k))
    if nq == 0.0 or nk == 0.0:
        raise ValueError("angular_similarity requires nonzero vectors")
    rho = min(1.0, max(-1.0, float(q @ k) / (nq * nk)))
    return (1.0 - math.acos(rho) / math.pi) ** gamma


def angular_kernel_matrix(q, k, gamma: int):
    """Dense S[i, j] = angular_similarity(q_i, k_j, gamma), float64 (ra/exact.py:116-125)."""
    q = _as_matrix(q, "q")
    k = _as_matrix(k, "k")
    gamma = _check_gamma(gamma)
    if q.shape[1] != k.shape[1]:
        raise ValueError("q and k must share the embedding dimension")
    dev = _aux.device()
    qd, kd = _aux.same_dtype(_aux.to_dev(q, dev), _aux.to_dev(k, dev))
    _nonzero_rows(qd, kd)
    out = torch.empty((qd.shape[0], kd.shape[0]), dtype=torch.float64, device=dev)
    _aux.check(_aux.lib().race_aux_angular_kernel(_aux.code(qd), qd.shape[0], kd.shape[0], qd.shape[1], _aux._vp(qd),
                                                  _aux._vp(kd), gamma, _aux._vp(out), _aux._stream()),
               "angular_kernel_matrix")
    return _aux.back(out, q)


def _angular_forward(inp: AttnInputs, gamma: int, causal: bool):
    dev = _aux.device()
    q, k, v = _aux.same_dtype(*(_aux.to_dev(x, dev) for x in (inp.q, inp.k, inp.v)))
    _nonzero_rows(q, k)
    n, d, dv = inp.n, inp.dim, inp.dim_v
    o = torch.empty((n, dv), dtype=torch.float64, device=dev)
    den = torch.empty((n,), dtype=torch.float64, device=dev)
    _aux.check(_aux.lib().race_aux_angular_fwd(_aux.code(q), n, d, dv, _aux._vp(q), _aux._vp(k), _aux._vp(v), gamma,
                                               int(causal), _aux._vp(o), _aux._vp(den), _aux._stream()),
               "angular_attention")
    return (q, k, v), o, den


def angular_attention(inp: AttnInputs, gamma: int, causal: bool = False):
    """Row-normalised attention under the sharpened angular kernel (ra/exact.py:128-166).

    Degenerate rows (similarity sum <= 1e-30) are zeroed and reported through a RuntimeWarning.
    """
    gamma = _check_gamma(gamma)
    _, o, den = _angular_forward(inp, gamma, causal)
    deg = torch.nonzero(den <= DEGENERATE_DEN_EPS).flatten().tolist()
    if deg:
        warnings.warn(f"angular_attention: {len(deg)} degenerate row(s) zeroed: "
                      f"{deg[:8]}{'...' if len(deg) > 8 else ''}", RuntimeWarning, stacklevel=2)
    return _aux.back(o, inp.q)


def angular_attention_vjp(inp: AttnInputs, gamma: int, d_out, causal: bool = False):
    """(dq, dk, dv) of angular_attention (ra/exact.py:169-218); pairs clamped at |rho| >= 1 pass no gradient."""
    gamma = _check_gamma(gamma)
    d_out = _as_matrix(d_out, "d_out")
    if tuple(d_out.shape) != (inp.n, inp.dim_v):
        raise ValueError(f"d_out shape {tuple(d_out.shape)} does not match output shape {(inp.n, inp.dim_v)}")
    (q, k, v), o, den = _angular_forward(inp, gamma, causal)
    g = _aux.to_dev(d_out, q.device).to(q.dtype).contiguous()
    n, d, dv = inp.n, inp.dim, inp.dim_v
    dq = torch.empty((n, d), dtype=torch.float64, device=q.device)
    dk = torch.empty_like(dq)
    dvv = torch.empty((n, dv), dtype=torch.float64, device=q.device)
    _aux.check(_aux.lib().race_aux_angular_bwd(_aux.code(q), n, d, dv, _aux._vp(q), _aux._vp(k), _aux._vp(v),
                                               _aux._vp(g), _aux._vp(o), _aux._vp(den), gamma, int(causal),
                                               _aux._vp(dq), _aux._vp(dk), _aux._vp(dvv), _aux._stream()),
               "angular_attention_vjp")
    return _aux.back(dq, inp.q), _aux.back(dk, inp.k), _aux.back(dvv, inp.v)


def _softmax_parts(inp: AttnInputs, causal: bool):
    dev = _aux.device()
    q, k, v = (_aux.to_dev(x, dev).double() for x in (inp.q, inp.k, inp.v))
    scale = 1.0 / math.sqrt(inp.dim)
    scores = (q @ k.T) * scale
    if causal:
        mask = torch.ones((inp.n, inp.n), dtype=torch.bool, device=dev).triu(1)
        scores = scores.masked_fill(mask, float("-inf"))
    return q, k, v, torch.softmax(scores, dim=1), scale


def softmax_attention(inp: AttnInputs, causal: bool = False):
    """softmax(Q K^T / sqrt(d)) V with optional causal masking (ra/exact.py:54-65)."""
    _, _, v, wts, _ = _softmax_parts(inp, causal)
    return _aux.back(wts @ v, inp.q)


def softmax_attention_vjp(inp: AttnInputs, d_out, causal: bool = False):
    """(dq, dk, dv) of softmax_attention (ra/exact.py:68-93)."""
    d_out = _as_matrix(d_out, "d_out")
    q, k, v, wts, scale = _softmax_parts(inp, causal)
    g = _aux.to_dev(d_out, q.device).double()
    d_v = wts.T @ g
    dw = g @ v.T
    ds = wts * (dw - (dw * wts).sum(1, keepdim=True))
    return _aux.back((ds @ k) * scale, inp.q), _aux.back((ds.T @ q) * scale, inp.k), _aux.back(d_v, inp.v)
