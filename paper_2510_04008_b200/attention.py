"""Drop-in mirror of the reference package's hot-path API.

Same names, dataclasses, argument meaning and error behaviour as
``race_attention`` (``/root/reference/pkg/src/race_attention``):

* ``SketchConfig``                ra/core.py:45-90
* ``derive_table_rng``            ra/core.py:93-104
* ``gaussian_matrix``             ra/core.py:107-111
* ``table_hyperplanes``           ra/forward.py:54-57
* ``AttnInputs``                  ra/exact.py:19-51
* ``RaceOutput``                  ra/forward.py:38-44
* ``RaceGradients``               ra/backward.py:46-50
* ``race_attention``              ra/forward.py:147-164
* ``race_attention_vjp``          ra/backward.py:184-235
* ``accumulate_num_den``          ra/forward.py:124-144
* ``row_normalize``               ra/core.py:114-123
* ``row_normalize_vjp``           ra/core.py:126-139

The compute runs on the GPU through the C-ABI (``functional.py``); there is no
CPU path.  Additions (keyword-only, optional): ``w=`` passes the random
projection tensor explicitly ([T, P, d], tables in (m, l) order) so results are
comparable across implementations; otherwise it is derived from ``cfg.seed``
exactly as the reference does.  ``workers`` is accepted for signature
compatibility; the result is identical for any value (the reference's
worker-invariance contract, ra/acceptance.py:419-450).

numpy inputs give numpy outputs (o in the input dtype, den float64, as the
reference).  float64 inputs are computed in float32 on the device (the B200
path is fp32-accumulate, rel err ~1e-6 against the reference's float64, inside
the 1e-3 fp32 tolerance but not the reference's own 1e-10 self-consistency
bound); each such call emits a ``PrecisionWarning``.  torch
inputs (float32 / bfloat16) give torch outputs on the input's device.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from .functional import SketchParams, race_backward, race_forward

# ra/core.py:14-22
ZERO_ROW_EPS = 1e-12
DEGENERATE_DEN_EPS = 1e-30
MAX_HYPERPLANES = 20


@dataclass(frozen=True)
class SketchConfig:
    """Hyperparameters of the sketched attention estimator (ra/core.py:45-90)."""

    hyperplanes: int
    tables: int
    ensembles: int = 1
    beta: float = 8.0
    seed: int = 0
    causal: bool = False
    normalize_inputs: bool = True
    block_size: int = 4096

    def __post_init__(self):
        if not (1 <= self.hyperplanes <= MAX_HYPERPLANES):
            raise ValueError(f"hyperplanes must be in [1, {MAX_HYPERPLANES}], got {self.hyperplanes}")
        if self.tables < 1:
            raise ValueError("tables must be >= 1")
        if self.ensembles < 1:
            raise ValueError("ensembles must be >= 1")
        if not (math.isfinite(self.beta) and self.beta > 0):
            raise ValueError("beta must be positive and finite")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")

    @property
    def n_buckets(self) -> int:
        return 1 << self.hyperplanes

    @property
    def total_tables(self) -> int:
        return self.ensembles * self.tables

    def params(self, causal: bool | None = None, normalize: bool | None = None) -> SketchParams:
        return SketchParams(self.hyperplanes, self.total_tables, float(self.beta),
                            self.causal if causal is None else causal,
                            self.normalize_inputs if normalize is None else normalize)


def derive_table_rng(seed: int, ensemble: int, table: int) -> np.random.Generator:
    """numpy Generator for one (ensemble, table) slot (ra/core.py:93-104)."""
    if ensemble < 0 or table < 0:
        raise ValueError("ensemble and table indices must be non-negative")
    ss = np.random.SeedSequence(entropy=int(seed) & 0xFFFFFFFFFFFFFFFF, spawn_key=(ensemble, table))
    return np.random.default_rng(ss)


def gaussian_matrix(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """rows x cols i.i.d. standard normals, float64 (ra/core.py:107-111)."""
    if rows < 1 or cols < 1:
        raise ValueError("rows and cols must be >= 1")
    return rng.standard_normal((rows, cols))


def table_hyperplanes(cfg: SketchConfig, dim: int, ensemble: int, table: int) -> np.ndarray:
    """Gaussian hyperplanes (P, d) float64 for one slot (ra/forward.py:54-57)."""
    return gaussian_matrix(derive_table_rng(cfg.seed, ensemble, table), cfg.hyperplanes, dim)


def all_hyperplanes(cfg: SketchConfig, dim: int) -> np.ndarray:
    """(T, P, d) float64 stack in the reference's (m, l) task order (ra/forward.py:128)."""
    return np.stack([table_hyperplanes(cfg, dim, m, l)
                     for m in range(cfg.ensembles) for l in range(cfg.tables)])


def _as_matrix(x, name: str):
    """2-D finite float validation (ra/core.py:27-42) for numpy or torch input."""
    if isinstance(x, torch.Tensor):
        if x.dim() != 2:
            raise ValueError(f"{name} must be 2-D, got shape {tuple(x.shape)}")
        if not x.is_floating_point():
            x = x.to(torch.float64 if not x.is_cuda else torch.float32)
        if x.numel() and not bool(torch.isfinite(x).all()):
            raise ValueError(f"{name} contains non-finite entries")
        return x
    a = np.asarray(x)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{name} contains non-finite entries")
    return a


@dataclass(frozen=True)
class AttnInputs:
    """Per-head Q, K (N x d) and V (N x dv) (ra/exact.py:19-51)."""

    q: object
    k: object
    v: object

    def __post_init__(self):
        object.__setattr__(self, "q", _as_matrix(self.q, "q"))
        object.__setattr__(self, "k", _as_matrix(self.k, "k"))
        object.__setattr__(self, "v", _as_matrix(self.v, "v"))
        if tuple(self.q.shape) != tuple(self.k.shape):
            raise ValueError(f"q and k shapes differ: {tuple(self.q.shape)} vs {tuple(self.k.shape)}")
        if self.v.shape[0] != self.q.shape[0]:
            raise ValueError(f"v has {self.v.shape[0]} rows but q/k have {self.q.shape[0]}")

    @property
    def n(self) -> int:
        return int(self.q.shape[0])

    @property
    def dim(self) -> int:
        return int(self.q.shape[1])

    @property
    def dim_v(self) -> int:
        return int(self.v.shape[1])


@dataclass(frozen=True)
class RaceOutput:
    """Estimator output, averaged denominators, degenerate-row flags (ra/forward.py:38-44)."""

    o: object
    den: object
    degenerate_rows: tuple


@dataclass(frozen=True)
class RaceGradients:
    """(dq, dk, dv) in the input dtypes (ra/backward.py:46-50)."""

    dq: object
    dk: object
    dv: object


def row_normalize(x):
    """Rows scaled to unit norm; rows with norm < 1e-12 unchanged (ra/core.py:114-123).

    Runs on the GPU in float64 (race_aux_row_normalize); the result has x's container and dtype.
    On the hot path this step is fused into the kernels (proj(x^) = x W^T / ||x||)."""
    from . import _aux

    x = _as_matrix(x, "x")
    xd = _aux.to_dev(x)
    out = torch.empty(xd.shape, dtype=torch.float64, device=xd.device)
    _aux.check(_aux.lib().race_aux_row_normalize(_aux.code(xd), xd.shape[0], xd.shape[1], _aux._vp(xd), None,
                                                 _aux._vp(out), _aux._stream()), "row_normalize")
    return _aux.back(out, x)


def row_normalize_vjp(x_raw, grad_normalized):
    """Cotangent on row_normalize(x_raw) pulled back to x_raw (ra/core.py:126-139), float64."""
    from . import _aux

    x = _as_matrix(x_raw, "x_raw")
    g = _as_matrix(grad_normalized, "grad_normalized")
    if tuple(g.shape) != tuple(x.shape):
        raise ValueError(f"grad shape {tuple(g.shape)} does not match x {tuple(x.shape)}")
    xd, gd = _aux.same_dtype(_aux.to_dev(x), _aux.to_dev(g))
    out = torch.empty(xd.shape, dtype=torch.float64, device=xd.device)
    _aux.check(_aux.lib().race_aux_row_normalize(_aux.code(xd), xd.shape[0], xd.shape[1], _aux._vp(xd),
                                                 _aux._vp(gd), _aux._vp(out), _aux._stream()), "row_normalize_vjp")
    return _aux.back(out, x, dtype=np.float64) if not isinstance(x, torch.Tensor) else out.to(x.device)


class PrecisionWarning(UserWarning):
    """float64 inputs were computed in float32 on the device."""


def _warn_f64(*xs) -> None:
    if any((isinstance(x, torch.Tensor) and x.dtype == torch.float64) or
           (not isinstance(x, torch.Tensor) and np.asarray(x).dtype == np.float64) for x in xs):
        warnings.warn("float64 inputs are computed in float32 on the B200 path (fp32 accumulate; "
                      "rel err ~1e-6 vs the reference's float64)", PrecisionWarning, stacklevel=3)


# ---------------------------------------------------------------------------
def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("race_attention (B200 path) needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x, dev):
    if isinstance(x, torch.Tensor):
        t = x.to(dev)
        return t if t.dtype in (torch.float32, torch.bfloat16) else t.to(torch.float32)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)


def _back(t: torch.Tensor, like):
    """Return t in the container/dtype convention of `like`."""
    if isinstance(like, torch.Tensor):
        return t.to(device=like.device, dtype=like.dtype)
    return t.float().cpu().numpy().astype(like.dtype, copy=False)


def _w_tensor(cfg: SketchConfig, dim: int, w, dev) -> torch.Tensor:
    if w is None:
        w = all_hyperplanes(cfg, dim)
    if isinstance(w, torch.Tensor):
        return w.to(device=dev, dtype=torch.float32)
    return torch.from_numpy(np.asarray(w, dtype=np.float32)).to(dev)


def race_attention(inp: AttnInputs, cfg: SketchConfig, workers: int = 1, *, w=None) -> RaceOutput:
    """Sketched attention estimate O = Num / Den (ra/forward.py:147-164).

    Rows whose averaged denominator is <= 1e-30 are zeroed and flagged.
    """
    dev = _device()
    _warn_f64(inp.q, inp.k, inp.v)
    q, k, v = (_to_dev(x, dev) for x in (inp.q, inp.k, inp.v))
    if not (q.dtype == k.dtype == v.dtype):
        q, k, v = q.float(), k.float(), v.float()
    o, den, _ = race_forward(q, k, v, _w_tensor(cfg, inp.dim, w, dev), cfg.params(), want_state=False)
    deg = torch.nonzero(den <= DEGENERATE_DEN_EPS).flatten().tolist()
    if isinstance(inp.q, torch.Tensor):
        den_out = den.to(device=inp.q.device, dtype=torch.float64)
    else:
        den_out = den.double().cpu().numpy()
    return RaceOutput(o=_back(o, inp.q), den=den_out, degenerate_rows=tuple(int(i) for i in deg))


def race_attention_vjp(inp: AttnInputs, cfg: SketchConfig, d_out, workers: int = 1, *, w=None) -> RaceGradients:
    """(dq, dk, dv) of race_attention against cotangent d_out (ra/backward.py:184-235)."""
    d_out = _as_matrix(d_out, "d_out")
    if tuple(d_out.shape) != (inp.n, inp.dim_v):
        raise ValueError(f"d_out shape {tuple(d_out.shape)} does not match output shape {(inp.n, inp.dim_v)}")
    dev = _device()
    _warn_f64(inp.q, inp.k, inp.v, d_out)
    q, k, v, g = (_to_dev(x, dev) for x in (inp.q, inp.k, inp.v, d_out))
    if not (q.dtype == k.dtype == v.dtype == g.dtype):
        q, k, v, g = q.float(), k.float(), v.float(), g.float()
    dq, dk, dv = race_backward(q, k, v, _w_tensor(cfg, inp.dim, w, dev), g, cfg.params())
    return RaceGradients(dq=_back(dq, inp.q), dk=_back(dk, inp.k), dv=_back(dv, inp.v))


def accumulate_num_den(q, k, v, cfg: SketchConfig, workers: int = 1, *, w=None):
    """Averaged (num [N, dv], den [N]) float64 on already-prepared q, k (ra/forward.py:124-144).

    One device pass (no row normalisation, as the reference's caller has prepared q, k) gives
    O = num / den and den; num is recovered as O * den in float64 from the fp32 O, so it is the
    numerator to fp32 rounding.  Rows whose den is <= 1e-30 have |num| <= max|v| * den (phi >= 0),
    i.e. |num| <= 1e-30 max|v|, and are returned as 0."""
    inp = AttnInputs(q, k, v)
    dev = _device()
    _warn_f64(inp.q, inp.k, inp.v)
    qd, kd, vd = (_to_dev(x, dev) for x in (inp.q, inp.k, inp.v))
    if not (qd.dtype == kd.dtype == vd.dtype):
        qd, kd, vd = qd.float(), kd.float(), vd.float()
    o, den, _ = race_forward(qd, kd, vd, _w_tensor(cfg, inp.dim, w, dev), cfg.params(normalize=False),
                             want_state=False)
    den64 = den.double()
    num = o.double() * den64[:, None]
    if isinstance(inp.q, torch.Tensor):
        return num.to(inp.q.device), den64.to(inp.q.device)
    return num.cpu().numpy(), den64.cpu().numpy()
