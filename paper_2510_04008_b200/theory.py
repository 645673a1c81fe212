"""Estimator-theory functions on the GPU (mirror of ra/theory.py and race_kernel).

* ``race_kernel``               ra/forward.py:167-212  (soft features of every table + their Gram, fp64)
* ``hard_race_attention``       ra/theory.py:205-227   (hard sign-hash buckets, fp64)
* ``kernel_deviation``          ra/theory.py:230-241
* ``kernel_variance_bound``     ra/theory.py:244-246
* ``variance_sweep``            ra/theory.py:92-136    (RACE on the B200 path vs GPU angular attention)
* ``bias_sweep``                ra/theory.py:139-202
* ``collision_identity_check``  ra/theory.py:271-318   (hyperplanes drawn with the caller's numpy rng, as the
                                                        reference; sign tests on the device)
* ``row_sum_stability``         ra/theory.py:333-360
* ``output_rms_error``, ``ScalingExperiment``, ``CollisionReport``, ``RowSumReport``

Each function keeps the reference's arguments, validation and return types.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _aux
from .attention import (
    DEGENERATE_DEN_EPS,
    AttnInputs,
    RaceOutput,
    SketchConfig,
    _as_matrix,
    all_hyperplanes,
    race_attention,
)
from .exact import angular_attention, angular_kernel_matrix
from .sketch import _codes, _features

KERNEL_MAX_ROWS = 2048  # ra/forward.py:35
BIAS_LINEAR_CONSTANT = 4.0 / math.sqrt(2.0 * math.pi)
BIAS_EXP_RATE = 2.0 * math.tanh(1.0)
DEFAULT_DELTA = 0.01
COLLISION_ANGLES = (math.pi / 6, math.pi / 3, math.pi / 2, 2 * math.pi / 3)


def race_kernel(q, k, cfg: SketchConfig, *, table_batch: int = 256):
    """Averaged sketch kernel S^[i, j] = (1/T) sum_tables phi(q_i) . phi(k_j), entries in [0, 1] (ra/forward.py:167-202).

    Quadratic by construction, so limited to N <= KERNEL_MAX_ROWS like the reference.
    ``table_batch`` is accepted for signature compatibility (all tables run in one launch).
    """
    q = _as_matrix(q, "q")
    k = _as_matrix(k, "k")
    if q.shape[1] != k.shape[1]:
        raise ValueError("q and k must share the embedding dimension")
    if max(q.shape[0], k.shape[0]) > KERNEL_MAX_ROWS:
        raise ValueError(f"race_kernel is limited to N <= {KERNEL_MAX_ROWS}")
    dev = _aux.device()
    qd, kd = _aux.same_dtype(_aux.to_dev(q, dev), _aux.to_dev(k, dev))
    w = all_hyperplanes(cfg, q.shape[1])
    T, P = cfg.total_tables, cfg.hyperplanes
    fq = _features(qd, w, cfg.beta, T, P, cfg.normalize_inputs)
    fk = _features(kd, w, cfg.beta, T, P, cfg.normalize_inputs)
    n, m = fq.shape[0], fk.shape[0]
    out = torch.empty((n, m), dtype=torch.float64, device=dev)
    _aux.check(_aux.lib().race_aux_feature_gram(n, m, fq.shape[1], _aux._vp(fq), _aux._vp(fk), 1.0 / T, _aux._vp(out),
                                                _aux._stream()), "race_kernel")
    return out if isinstance(q, torch.Tensor) else out.cpu().numpy()


def hard_race_attention(inp: AttnInputs, cfg: SketchConfig) -> RaceOutput:
    """The estimator with hard sign-hash buckets; non-causal only (ra/theory.py:205-227)."""
    if cfg.causal:
        raise NotImplementedError("hard-bucket reference is non-causal only")
    dev = _aux.device()
    q, k, v = _aux.same_dtype(*(_aux.to_dev(x, dev) for x in (inp.q, inp.k, inp.v)))
    T, P = cfg.total_tables, cfg.hyperplanes
    w = all_hyperplanes(cfg, inp.dim)
    cq = _codes(q, w, T, P, cfg.normalize_inputs)
    ck = _codes(k, w, T, P, cfg.normalize_inputs)
    L = _aux.lib()
    n, dv = inp.n, inp.dim_v
    ws = torch.empty((max(1, L.race_aux_hard_workspace_bytes(dv, P, T)),), dtype=torch.uint8, device=dev)
    o = torch.empty((n, dv), dtype=torch.float64, device=dev)
    den = torch.empty((n,), dtype=torch.float64, device=dev)
    _aux.check(L.race_aux_hard_attention(_aux.code(v), n, dv, _aux._vp(cq), _aux._vp(ck), _aux._vp(v), P, T,
                                         _aux._vp(o), _aux._vp(den), _aux._vp(ws), _aux._stream()),
               "hard_race_attention")
    deg = torch.nonzero(den <= DEGENERATE_DEN_EPS).flatten().tolist()
    if isinstance(inp.q, torch.Tensor):
        return RaceOutput(o=o, den=den, degenerate_rows=tuple(deg))
    return RaceOutput(o=o.cpu().numpy(), den=den.cpu().numpy(), degenerate_rows=tuple(int(i) for i in deg))


def kernel_deviation(q, k, cfg: SketchConfig, gamma: int) -> float:
    """Frobenius distance between the averaged sketch kernel and the exact angular kernel (ra/theory.py:230-241)."""
    if int(gamma) != cfg.hyperplanes:
        raise ValueError("kernel_deviation requires gamma == cfg.hyperplanes")
    q = _as_matrix(q, "q")
    k = _as_matrix(k, "k")
    if max(q.shape[0], k.shape[0]) > 1024:
        raise ValueError("kernel_deviation is limited to N <= 1024")
    s_hat = torch.as_tensor(race_kernel(q, k, cfg))
    s_exact = torch.as_tensor(angular_kernel_matrix(q, k, gamma)).to(s_hat.device, torch.float64)
    return float(torch.linalg.norm(s_hat - s_exact))


def kernel_variance_bound(n: int, tables: int, delta: float = DEFAULT_DELTA) -> float:
    """High-probability variance term of the kernel deviation bound (ra/theory.py:244-246)."""
    return 4.0 * n / math.sqrt(tables) * math.sqrt(math.log(2.0 * n / delta))


def output_rms_error(o_hat, o) -> float:
    """sqrt(mean_i ||o_hat_i - o_i||^2) (ra/theory.py:38-45)."""
    o_hat = _as_matrix(o_hat, "o_hat")
    o = _as_matrix(o, "o")
    if tuple(o_hat.shape) != tuple(o.shape):
        raise ValueError(f"shape mismatch: {tuple(o_hat.shape)} vs {tuple(o.shape)}")
    a = torch.as_tensor(o_hat).double()
    b = torch.as_tensor(o).double().to(a.device)
    return float(((a - b) ** 2).sum(1).mean().sqrt())


@dataclass(frozen=True)
class ScalingExperiment:
    """One sweep: grid, seed-averaged errors, their standard errors and a log-log fit (ra/theory.py:48-70)."""

    name: str
    grid: np.ndarray
    errors: np.ndarray
    std_errors: np.ndarray
    seed_count: int
    fit_slope: float
    fit_r2: float

    def __post_init__(self):
        grid = np.asarray(self.grid, dtype=np.float64)
        errors = np.asarray(self.errors, dtype=np.float64)
        if np.any(np.diff(grid) <= 0):
            raise ValueError("grid must be strictly increasing")
        if np.any(errors <= 0):
            raise ValueError("errors must be positive")
        object.__setattr__(self, "grid", grid)
        object.__setattr__(self, "errors", errors)
        object.__setattr__(self, "std_errors", np.asarray(self.std_errors, dtype=np.float64))


def _loglog_fit(grid, errors) -> tuple[float, float]:
    x, y = np.log(np.asarray(grid, float)), np.log(np.asarray(errors, float))
    slope, icpt = np.polyfit(x, y, 1)
    ss_res = float(np.sum((y - (slope * x + icpt)) ** 2))
    ss_tot = float(np.sum((y - y.mean()) ** 2))
    return float(slope), 1.0 if ss_tot == 0 else 1.0 - ss_res / ss_tot


def _check_grid(grid, name: str, min_points: int = 3) -> list:
    grid = list(grid)
    if len(grid) < min_points:
        raise ValueError(f"{name} needs at least {min_points} points, got {len(grid)}")
    if any(b <= a for a, b in zip(grid, grid[1:])):
        raise ValueError(f"{name} must be strictly increasing")
    return grid


def _sweep(inp, name, grid, n_seeds, make_cfg, reference) -> tuple[list, list]:
    means, stds = [], []
    for gv in grid:
        errs = np.asarray([output_rms_error(race_attention(inp, make_cfg(gv, s)).o, reference)
                           for s in range(n_seeds)])
        means.append(errs.mean())
        stds.append(errs.std(ddof=1) / math.sqrt(n_seeds))
    return means, stds


def variance_sweep(inp: AttnInputs, hyperplanes: int, beta: float, l_grid, *, n_seeds: int = 20,
                   base_seed: int = 0) -> ScalingExperiment:
    """RMS error vs table count at fixed beta with a log-log fit (slope about -1/2), ra/theory.py:92-136."""
    l_grid = _check_grid(l_grid, "l_grid")
    if n_seeds < 2:
        raise ValueError("n_seeds must be >= 2")
    reference = angular_attention(inp, gamma=hyperplanes)
    means, stds = _sweep(inp, "variance", l_grid, n_seeds,
                         lambda L, s: SketchConfig(hyperplanes=hyperplanes, tables=int(L), beta=beta,
                                                   seed=base_seed + s), reference)
    slope, r2 = _loglog_fit(l_grid, means)
    return ScalingExperiment("variance_vs_tables", np.asarray(l_grid, float), np.asarray(means), np.asarray(stds),
                             n_seeds, slope, r2)


def bias_sweep(inp: AttnInputs, hyperplanes: int, tables: int, beta_grid, *, n_seeds: int = 8, base_seed: int = 0,
               check_monotone: bool = True) -> ScalingExperiment:
    """Seed-averaged RMS error vs beta at a fixed table count; strictly decreasing (ra/theory.py:139-202)."""
    beta_grid = _check_grid(beta_grid, "beta_grid")
    if beta_grid[-1] / beta_grid[0] < 10.0:
        raise ValueError("beta_grid should span at least one decade")
    if n_seeds < 2:
        raise ValueError("n_seeds must be >= 2")
    reference = angular_attention(inp, gamma=hyperplanes)
    means, stds = _sweep(inp, "bias", beta_grid, n_seeds,
                         lambda b, s: SketchConfig(hyperplanes=hyperplanes, tables=tables, beta=float(b),
                                                   seed=base_seed + s), reference)
    if check_monotone:
        for i in range(1, len(means)):
            if not means[i] < means[i - 1]:
                raise ValueError("seed-averaged error is not strictly decreasing in beta: "
                                 f"err({beta_grid[i - 1]}) = {means[i - 1]:.6g} <= "
                                 f"err({beta_grid[i]}) = {means[i]:.6g}")
    slope, r2 = _loglog_fit(beta_grid, means)
    return ScalingExperiment("bias_vs_beta", np.asarray(beta_grid, float), np.asarray(means), np.asarray(stds),
                             n_seeds, slope, r2)


@dataclass(frozen=True)
class CollisionCheckRow:
    angle: float
    p_hat: float
    p_exact: float
    std_err: float
    z_score: float
    passed: bool


@dataclass(frozen=True)
class CollisionReport:
    hyperplanes: int
    trials: int
    band: float
    rows: tuple

    @property
    def all_passed(self) -> bool:
        return all(r.passed for r in self.rows)


def collision_identity_check(hyperplanes: int, trials: int, rng: np.random.Generator, *, angles=COLLISION_ANGLES,
                             dim: int = 8, band: float = 4.0) -> CollisionReport:
    """Monte-Carlo hard-hash collision rate vs (1 - theta/pi)^p (ra/theory.py:271-318).

    The hyperplane stacks come from `rng` in the reference's draw order, so the
    report is identical to the reference's for the same generator state.
    """
    if trials < 10_000:
        raise ValueError("trials must be >= 10000")
    if hyperplanes < 1:
        raise ValueError("hyperplanes must be >= 1")
    dev = _aux.device()
    rows = []
    for theta in angles:
        x = np.zeros((2, dim))
        x[0, 0] = 1.0
        x[1, 0], x[1, 1] = math.cos(theta), math.sin(theta)
        w = rng.standard_normal((trials, hyperplanes, dim))
        # codes of both vectors under every stack: trials "tables" of P hyperplanes each
        codes = _codes(_aux.to_dev(x, dev), w.reshape(trials * hyperplanes, dim), trials, hyperplanes, False)
        p_hat = float((codes[:, 0] == codes[:, 1]).double().mean())
        p_exact = (1.0 - theta / math.pi) ** hyperplanes
        se = math.sqrt(p_exact * (1.0 - p_exact) / trials)
        z = (p_hat - p_exact) / se if se > 0 else 0.0
        rows.append(CollisionCheckRow(angle=float(theta), p_hat=p_hat, p_exact=p_exact, std_err=se, z_score=z,
                                      passed=abs(p_hat - p_exact) <= band * se))
    return CollisionReport(hyperplanes=hyperplanes, trials=trials, band=band, rows=tuple(rows))


@dataclass(frozen=True)
class RowSumReport:
    """Stability margins of the normalising denominators on one instance (ra/theory.py:321-330)."""

    n: int
    min_row_sum: float
    min_den: float
    ratio: float
    all_positive: bool
    near_degenerate: bool


def row_sum_stability(q, k, cfg: SketchConfig) -> RowSumReport:
    """Exact-kernel row-sum floor vs the sketched denominators (ra/theory.py:333-360)."""
    q = _as_matrix(q, "q")
    k = _as_matrix(k, "k")
    row_sums = torch.as_tensor(angular_kernel_matrix(q, k, cfg.hyperplanes)).double().sum(1)
    den = torch.as_tensor(race_kernel(q, k, cfg)).sum(1)
    if bool((den <= 0).any()):
        raise RuntimeError("sketched denominators must be strictly positive")
    mn_rs, mn_den = float(row_sums.min()), float(den.min())
    return RowSumReport(n=int(q.shape[0]), min_row_sum=mn_rs, min_den=mn_den,
                        ratio=mn_den / mn_rs if mn_rs > 0 else float("inf"), all_positive=True,
                        near_degenerate=mn_rs < 0.01 * k.shape[0])
