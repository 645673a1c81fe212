"""Shared fixtures: golden vectors from the real reference + tolerance helpers."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_race.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


class Case(dict):
    """One golden instance (inputs, hyperplanes, cfg, reference outputs)."""

    @property
    def cfg_kwargs(self):
        return dict(hyperplanes=int(self["P"]), tables=int(self["L"]), ensembles=int(self["M"]),
                    beta=float(self["beta"]), seed=int(self["seed"]), causal=bool(self["causal"]),
                    normalize_inputs=bool(self["normalize"]), block_size=int(self["block_size"]))

    def __repr__(self):
        return (f"Case({self['tag']} n={self['q'].shape[0]} d={self['q'].shape[1]} dv={self['v'].shape[1]} "
                f"P={int(self['P'])} L={int(self['L'])} M={int(self['M'])} beta={float(self['beta'])} "
                f"causal={bool(self['causal'])})")


def load_golden() -> list[Case]:
    z = np.load(GOLDEN)
    out = []
    for i in range(int(z["count"])):
        pre = f"{i:03d}_"
        c = Case({k[len(pre):]: z[k] for k in z.files if k.startswith(pre)})
        c["tag"] = str(c["tag"])
        c["index"] = i
        out.append(c)
    return out


@pytest.fixture(scope="session")
def golden():
    return load_golden()


def rel_err(a, b, floor: float = 1e-30) -> float:
    """The reference's metric max|a-b| / max|b| (ra/acceptance.py:89-91) with a
    scale floor for tensors that are identically ~0 in exact arithmetic."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), floor)


def grad_errs(got, ref, rel_floor: float):
    """rel_err of (dq, dk, dv) with the floor rel_floor * max|ref grads| (so
    components that vanish exactly, e.g. d=1 or N=1 dq/dk, are judged on the
    call's natural gradient scale)."""
    scale = max(float(np.max(np.abs(np.asarray(r, dtype=np.float64)))) if np.asarray(r).size else 0.0
                for r in ref)
    floor = max(rel_floor * scale, 1e-30)
    return [rel_err(g, r, floor) for g, r in zip(got, ref)]


GOLDEN_EXTRA = os.path.join(ROOT, "tests", "golden", "golden_extra.npz")


def load_num_den_golden() -> list[dict]:
    """accumulate_num_den cases of tests/golden/make_extra_golden.py (real reference outputs)."""
    z = np.load(GOLDEN_EXTRA)
    out = []
    for i in range(int(z["nd_count"])):
        pre = f"nd{i:02d}_"
        c = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
        c["index"] = i
        c["cfg_kwargs"] = dict(hyperplanes=int(c["P"]), tables=int(c["L"]), ensembles=int(c["M"]),
                               beta=float(c["beta"]), seed=int(c["seed"]), causal=bool(c["causal"]))
        out.append(c)
    return out


def load_row_normalize_golden() -> dict:
    z = np.load(GOLDEN_EXTRA)
    return {k[3:]: z[k] for k in z.files if k.startswith("rn_")}


def record_parity(test: str, **errs) -> None:
    """Append the measured worst errors of a parity test as one JSON line to $RACE_PARITY_LOG
    (set by the GPU runs whose logs are committed under profiles/); no-op otherwise."""
    path = os.environ.get("RACE_PARITY_LOG")
    if not path:
        return
    import json

    with open(path, "a") as f:
        f.write(json.dumps({"test": test, **{k: (float(v) if isinstance(v, (int, float, np.floating)) else v)
                                             for k, v in errs.items()}}) + "\n")
