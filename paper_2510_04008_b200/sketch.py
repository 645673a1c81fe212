"""Soft / hard LSH feature maps on the GPU (mirror of ra/sketch.py).

Same names, arguments and errors as the reference module:

* ``HashTable``, ``make_hash_table``        ra/sketch.py:22-49
* ``corner_vector``, ``corner_matrix``      ra/sketch.py:52-74 (host index helpers)
* ``soft_features``                         ra/sketch.py:87-129
* ``dominant_corner_mass``                  ra/sketch.py:132-140
* ``hard_hash``                             ra/sketch.py:143-149
* ``BucketStats``, ``bucket_stats``         ra/sketch.py:152-171

The per-row work runs in ``race_aux_soft_features`` / ``race_aux_hard_hash``
(csrc/race_aux.cu) in float64, so results match the reference to ~1e-15.
The two evaluation ``method``s of the reference (explicit corner softmax and
the factored per-bit form) are the same function; the kernel evaluates the
factored form for every P, and ``method`` is validated exactly as the
reference does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _aux
from .attention import MAX_HYPERPLANES, _as_matrix, gaussian_matrix

EXPLICIT_CORNER_LIMIT = 10  # ra/sketch.py:19


@dataclass(frozen=True)
class HashTable:
    """One table's Gaussian projection stack (n_bits x dim), ra/sketch.py:22-45."""

    w: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "w", _as_matrix(self.w, "w"))
        if not (1 <= self.w.shape[0] <= MAX_HYPERPLANES):
            raise ValueError(f"hash table needs 1..{MAX_HYPERPLANES} hyperplanes, got {self.w.shape[0]}")

    @property
    def n_bits(self) -> int:
        return int(self.w.shape[0])

    @property
    def n_buckets(self) -> int:
        return 1 << self.n_bits

    @property
    def dim(self) -> int:
        return int(self.w.shape[1])


def make_hash_table(rng: np.random.Generator, n_bits: int, dim: int) -> HashTable:
    return HashTable(gaussian_matrix(rng, n_bits, dim))


def corner_vector(index: int, n_bits: int) -> np.ndarray:
    """Corner of {+1, -1}^n_bits for bucket `index` (bit t: 0 -> +1, 1 -> -1)."""
    if n_bits < 1:
        raise ValueError("n_bits must be >= 1")
    if not 0 <= index < (1 << n_bits):
        raise ValueError(f"index {index} out of range for {n_bits} bits")
    return np.array([-1.0 if (index >> t) & 1 else 1.0 for t in range(n_bits)])


def corner_matrix(n_bits: int) -> np.ndarray:
    """All corners stacked in bucket-index order (n_bits <= EXPLICIT_CORNER_LIMIT)."""
    if not 1 <= n_bits <= EXPLICIT_CORNER_LIMIT:
        raise ValueError(f"explicit corner matrix limited to {EXPLICIT_CORNER_LIMIT} bits")
    r = np.arange(1 << n_bits)[:, None]
    return np.where((r >> np.arange(n_bits)[None, :]) & 1, -1.0, 1.0)


def _features(x_dev: torch.Tensor, w, beta: float, tables: int, hyperplanes: int, normalize: bool) -> torch.Tensor:
    """phi [n, tables * 2^P] float64 on the device (race_aux_soft_features)."""
    dev = x_dev.device
    wd = _aux.w64(w, dev)
    n, d = x_dev.shape
    if wd.shape != (tables * hyperplanes, d):
        raise ValueError(f"hyperplanes shape {tuple(wd.shape)} does not match {(tables * hyperplanes, d)}")
    phi = torch.empty((n, tables << hyperplanes), dtype=torch.float64, device=dev)
    _aux.check(_aux.lib().race_aux_soft_features(_aux.code(x_dev), n, d, _aux._vp(x_dev), _aux._vp(wd), hyperplanes,
                                                 tables, float(beta), int(normalize), _aux._vp(phi), _aux._stream()),
               "soft_features")
    return phi


def _codes(x_dev: torch.Tensor, w, tables: int, hyperplanes: int, normalize: bool) -> torch.Tensor:
    """hard_hash codes [tables, n] int32 on the device (race_aux_hard_hash)."""
    wd = _aux.w64(w, x_dev.device)
    n, d = x_dev.shape
    codes = torch.empty((tables, n), dtype=torch.int32, device=x_dev.device)
    _aux.check(_aux.lib().race_aux_hard_hash(_aux.code(x_dev), n, d, _aux._vp(x_dev), _aux._vp(wd), hyperplanes, tables,
                                             int(normalize), _aux._vp(codes), _aux._stream()), "hard_hash")
    return codes


def soft_features(x, table: HashTable, beta: float, *, method: str = "auto"):
    """Row-stochastic soft assignment of each row of x to the 2^P corners (ra/sketch.py:87-129)."""
    x = _as_matrix(x, "x")
    if not (math.isfinite(beta) and beta > 0):
        raise ValueError("beta must be positive and finite")
    if method not in ("auto", "corners", "factored"):
        raise ValueError(f"unknown method {method!r}")
    if method == "corners" and table.n_bits > EXPLICIT_CORNER_LIMIT:
        corner_matrix(table.n_bits)  # raises the reference's ValueError
    if x.shape[1] != table.dim:
        raise ValueError(f"x has dim {x.shape[1]} but the table has dim {table.dim}")
    phi = _features(_aux.to_dev(x), table.w, beta, 1, table.n_bits, False)
    return _aux.back(phi, x)


def hard_hash(x, table: HashTable):
    """Bucket index of the sign corner of W x per row; zero projections tie to +1 (ra/sketch.py:143-149)."""
    x = _as_matrix(x, "x")
    codes = _codes(_aux.to_dev(x), table.w, 1, table.n_bits, False)[0].long()
    return codes if isinstance(x, torch.Tensor) else codes.cpu().numpy()


def dominant_corner_mass(x, table: HashTable, beta: float):
    """Mass each row puts on its own sign corner = prod_t sigmoid(2 beta |tanh(w_t . x)|) (ra/sketch.py:132-140)."""
    x = _as_matrix(x, "x")
    xd = _aux.to_dev(x)
    phi = _features(xd, table.w, beta, 1, table.n_bits, False)
    codes = _codes(xd, table.w, 1, table.n_bits, False)[0].long()
    mass = phi.gather(1, codes[:, None])[:, 0]
    return mass if isinstance(x, torch.Tensor) else mass.cpu().numpy()


@dataclass(frozen=True)
class BucketStats:
    """Per-table soft bucket mass a (R) and value sums b (R x dv), ra/sketch.py:152-160."""

    a: np.ndarray
    b: np.ndarray

    def __post_init__(self):
        if self.a.ndim != 1 or self.b.ndim != 2 or self.a.shape[0] != self.b.shape[0]:
            raise ValueError("a must be length R and b must be R x d_v")


def bucket_stats(phi_k, v) -> BucketStats:
    """a = Phi^T 1, b = Phi^T V (ra/sketch.py:163-171), float64 on the device."""
    phi_k = _as_matrix(phi_k, "phi_k")
    v = _as_matrix(v, "v")
    if phi_k.shape[0] != v.shape[0]:
        raise ValueError(f"phi_k has {phi_k.shape[0]} rows but v has {v.shape[0]}")
    dev = _aux.device()
    p = _aux.to_dev(phi_k, dev).double()
    vd = _aux.to_dev(v, dev).double()
    return BucketStats(a=p.sum(0).cpu().numpy(), b=(p.T @ vd).cpu().numpy())
