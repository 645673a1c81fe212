"""GPU scaling harness with the reference's CSV schema (mirror of ra/bench.py).

``bench_scaling(lengths, methods, ...)`` times one forward (or forward +
backward) pass of a multi-head attention layer over a grid of sequence
lengths, exactly like ``ra/bench.py:189-284`` (median of repeats after one
warm-up, ``time_guard`` for quadratic methods whose projected cost exceeds
the budget, ``oom_guard`` above a memory limit, guarded rows still emitted),
but on the B200:

* ``race``           -> the sm_100a RACE layer (all heads in one call,
                        head h hashed with seed + h as ra/bench.py:175);
* ``angular_exact``  -> the fp64 angular attention kernels (race_aux.cu);
* ``softmax_exact``  -> torch scaled_dot_product_attention (library).

Timing is device time (CUDA events around the pass, inputs resident in HBM).
The CSV keeps the reference's columns (``BENCH_CSV_COLUMNS``) and, with
``extended=True``, appends ``threads`` (as the reference) plus ``gpus``,
``dtype``, ``tokens_per_s`` and ``roofline_frac`` (SURVEY.md section 8(d):
(7d + 5dv) e + 8 algorithmic bytes per token-head over the measured HBM peak).
"""

from __future__ import annotations

import json
import math
import os
import statistics
from dataclasses import dataclass

import numpy as np
import torch

from .attention import AttnInputs, SketchConfig
from .exact import angular_attention, angular_attention_vjp
from .functional import race_backward, race_forward
from .module import head_hyperplanes

METHODS = ("race", "softmax_exact", "angular_exact")
PASS_KINDS = ("forward", "forward_backward")
BENCH_CSV_COLUMNS = ("method", "N", "d", "heads", "P", "L", "M", "beta", "causal", "pass_kind", "wall_seconds",
                     "peak_bytes", "seed", "status")
EXTENDED_COLUMNS = ("threads", "gpus", "dtype", "tokens_per_s", "roofline_frac")
_SCALING_EXPONENT = {"race": 1.0, "softmax_exact": 2.0, "angular_exact": 2.0}
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@dataclass(frozen=True)
class BenchMethod:
    """One benchmarked configuration (ra/bench.py:59-79)."""

    method: str
    sketch: SketchConfig | None = None
    gamma: int = 8
    causal: bool = False

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.method == "race" and self.sketch is None:
            raise ValueError("race method needs a SketchConfig")

    @property
    def is_causal(self) -> bool:
        return self.sketch.causal if self.method == "race" else self.causal


@dataclass(frozen=True)
class BenchRecord:
    """One CSV row (ra/bench.py:81-127) plus the GPU columns."""

    method: str
    n: int
    dim: int
    heads: int
    hyperplanes: int | None
    tables: int | None
    ensembles: int | None
    beta: float | None
    causal: bool
    pass_kind: str
    wall_seconds: float | None
    peak_bytes: int
    seed: int
    status: str
    threads: int = 1
    gpus: int = 1
    dtype: str = "float32"
    tokens_per_s: float | None = None
    roofline_frac: float | None = None

    def to_csv_row(self, extended: bool = False) -> str:
        def fmt(x):
            if x is None:
                return ""
            if isinstance(x, bool):
                return "true" if x else "false"
            if isinstance(x, float):
                return f"{x:.6g}"
            return str(x)

        vals = [self.method, self.n, self.dim, self.heads, self.hyperplanes, self.tables, self.ensembles, self.beta,
                self.causal, self.pass_kind, self.wall_seconds, self.peak_bytes, self.seed, self.status]
        if extended:
            vals += [self.threads, self.gpus, self.dtype, self.tokens_per_s, self.roofline_frac]
        return ",".join(fmt(v) for v in vals)


def bench_csv_header(extended: bool = False) -> str:
    return ",".join(BENCH_CSV_COLUMNS + (EXTENDED_COLUMNS if extended else ()))


def records_to_csv(records, extended: bool = False) -> str:
    return "\n".join([bench_csv_header(extended)] + [r.to_csv_row(extended) for r in records]) + "\n"


def _itemsize(dtype) -> int:
    if isinstance(dtype, torch.dtype):
        return torch.empty((), dtype=dtype).element_size()
    return np.dtype(dtype).itemsize


def estimate_peak_bytes(method: str, n: int, dim: int, dtype, sketch: SketchConfig | None, heads: int = 1) -> int:
    """Device working set of one pass (used by the memory guard).

    race: q, k, v, o, d_out and three gradients per head plus the causal
    sketch rows (64 B per token-head); exact methods stream tiles, so their
    footprint is linear too (softmax via SDPA, angular via fp64 tiles).
    """
    e = _itemsize(dtype)
    base = 8 * n * dim * e * heads
    if method == "race":
        return int(base + (64 * n * heads if sketch is not None and sketch.causal else 0) + (16 << 20))
    if method == "angular_exact":
        return int(base + 5 * n * dim * 8 * heads)
    return int(base + 4 * n * heads * 4)


def _hbm_peak_gbs() -> float:
    try:
        return float(json.load(open(os.path.join(_ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 7672.0  # B200_PROFILING.md fallback


def _make_inputs(n: int, dim: int, dtype: torch.dtype, heads: int, seed: int, dev) -> list[torch.Tensor]:
    """q, k, v, d_out [1, H, N, d], N(0, 1).  Up to 131072 tokens the values are drawn on the
    host in the reference's order (ra/bench.py:161-169) so a CPU run sees identical inputs."""
    if n <= 131072:
        rng = np.random.default_rng(np.random.SeedSequence(seed & 0xFFFFFFFFFFFFFFFF, spawn_key=(n,)))
        per = [[rng.standard_normal((n, dim)) for _ in range(4)] for _ in range(heads)]
        return [torch.from_numpy(np.stack([per[h][i] for h in range(heads)])[None].astype(np.float32)).to(dev, dtype)
                for i in range(4)]
    gen = torch.Generator(device=dev).manual_seed((seed * 1_000_003 + n) & 0x7FFFFFFFFFFFFFFF)
    return [torch.randn((1, heads, n, dim), generator=gen, device=dev).to(dtype) for _ in range(4)]


def _runner(spec: BenchMethod, x: list[torch.Tensor], pass_kind: str):
    q, k, v, g = x
    heads, dim = q.shape[1], q.shape[3]
    if spec.method == "race":
        w = head_hyperplanes(spec.sketch, heads, dim).to(q.device)
        p = spec.sketch.params()

        def run():
            o, den, st = race_forward(q, k, v, w, p, want_state=pass_kind == "forward_backward")
            if pass_kind == "forward_backward":
                race_backward(q, k, v, w, g, p, state=st)
        return run
    if spec.method == "softmax_exact":
        qq, kk, vv = (t.detach().clone().requires_grad_(pass_kind == "forward_backward") for t in (q, k, v))

        def run():
            o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=spec.causal)
            if pass_kind == "forward_backward":
                torch.autograd.grad(o, (qq, kk, vv), g)
        return run

    def run():
        for h in range(heads):
            inp = AttnInputs(q[0, h], k[0, h], v[0, h])
            if pass_kind == "forward_backward":
                angular_attention_vjp(inp, spec.gamma, g[0, h], causal=spec.causal)
            else:
                angular_attention(inp, spec.gamma, causal=spec.causal)
    return run


def _time(run, repeats: int) -> float:
    run()  # warm-up (discarded, ra/bench.py:268)
    times = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    return statistics.median(times)


def bench_scaling(lengths, methods, repeats: int = 3, time_budget_s: float = 120.0, *, dim: int = 128,
                  heads: int = 4, dtype=torch.bfloat16, pass_kind: str = "forward_backward",
                  mem_limit_bytes: int | None = None, seed: int = 0, workers: int = 1) -> list[BenchRecord]:
    """Median-of-repeats device times over a grid of sequence lengths (ra/bench.py:189-284)."""
    lengths = list(lengths)
    if not lengths or any(b <= a for a, b in zip(lengths, lengths[1:])):
        raise ValueError("lengths must be a non-empty increasing sequence")
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    if pass_kind not in PASS_KINDS:
        raise ValueError(f"pass_kind must be one of {PASS_KINDS}")
    tdt = {np.float32: torch.float32, np.float64: torch.float64}.get(dtype, dtype)
    if not isinstance(tdt, torch.dtype):
        tdt = torch.float32
    dev = torch.device("cuda", torch.cuda.current_device())
    peak = _hbm_peak_gbs()
    e = _itemsize(tdt)
    records: list[BenchRecord] = []
    for spec in methods:
        sk = spec.sketch
        last = None
        for n in lengths:
            common = dict(method=spec.method, n=n, dim=dim, heads=heads,
                          hyperplanes=sk.hyperplanes if sk else None, tables=sk.tables if sk else None,
                          ensembles=sk.ensembles if sk else None, beta=sk.beta if sk else None,
                          causal=spec.is_causal, pass_kind=pass_kind, seed=seed, threads=workers,
                          dtype=str(tdt).replace("torch.", ""))
            est = estimate_peak_bytes(spec.method, n, dim, tdt, sk, heads)
            if mem_limit_bytes is not None and est > mem_limit_bytes:
                records.append(BenchRecord(**common, wall_seconds=None, peak_bytes=est, status="oom_guard"))
                continue
            if last is not None and last[1] * (n / last[0]) ** _SCALING_EXPONENT[spec.method] > time_budget_s:
                records.append(BenchRecord(**common, wall_seconds=None, peak_bytes=int(torch.cuda.max_memory_allocated()),
                                           status="time_guard"))
                continue
            torch.cuda.reset_peak_memory_stats()
            try:
                x = _make_inputs(n, dim, tdt, heads, seed, dev)
                t = _time(_runner(spec, x, pass_kind), repeats)
            except torch.cuda.OutOfMemoryError:
                del x
                torch.cuda.empty_cache()
                records.append(BenchRecord(**common, wall_seconds=None, peak_bytes=est, status="oom"))
                continue
            last = (n, t)
            tps = n / t
            per_tok = ((7 if pass_kind == "forward_backward" else 3) * dim
                       + (5 if pass_kind == "forward_backward" else 1) * dim) * e + 8
            frac = tps * heads * per_tok / (peak * 1e9) if spec.method == "race" else None
            records.append(BenchRecord(**common, wall_seconds=t, peak_bytes=int(torch.cuda.max_memory_allocated()),
                                       status="ok", tokens_per_s=tps, roofline_frac=frac))
            del x
    return records


def median_time(records, method: str, n: int) -> float:
    for r in records:
        if r.method == method and r.n == n and r.status == "ok":
            return r.wall_seconds
    raise KeyError(f"no ok record for method={method} N={n}")


def demo_kernel_heatmap(gamma_list, resolution: int):
    """Rescaled exponential vs sharpened angular kernels on rho in [-1, 1] (ra/bench.py:294-317)."""
    if resolution < 8:
        raise ValueError("resolution must be >= 8")
    gammas = [int(g) for g in gamma_list]
    if not gammas or any(g < 1 for g in gammas):
        raise ValueError("gamma_list must contain positive integers")
    rho = np.linspace(-1.0, 1.0, resolution)
    ex = (np.exp(rho) - math.exp(-1.0)) / (math.exp(1.0) - math.exp(-1.0))
    base = 1.0 - np.arccos(np.clip(rho, -1.0, 1.0)) / np.pi
    header = ["rho", "exp_rescaled"] + [f"angular_gamma{g}" for g in gammas]
    return header, [[float(rho[i]), float(ex[i])] + [float(base[i] ** g) for g in gammas] for i in range(resolution)]


def heatmap_csv_text(header, rows) -> str:
    return "\n".join([",".join(header)] + [",".join(f"{x:.12g}" for x in r) for r in rows]) + "\n"
