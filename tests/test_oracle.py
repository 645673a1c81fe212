"""Pin the CPU oracle (oracle/race_oracle.py) to the REAL reference's outputs.

tests/golden/golden_race.npz was produced by tests/golden/make_golden.py, which
imports the reference package itself; here the restatement must reproduce
every fixture to the reference's own 1e-10 tolerance (ra/acceptance.py:36).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import grad_errs, load_golden, rel_err
from oracle import race_oracle as ro

CASES = load_golden()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['index']:03d}-{c['tag']}")
def test_oracle_matches_reference(case):
    q, k, v, g, w = case["q"], case["k"], case["v"], case["d_out"], case["w"]
    kw = case.cfg_kwargs
    # the hyperplanes are re-derived exactly (ra/core.py:93-111)
    w2 = ro.stacked_hyperplanes(kw["seed"], kw["hyperplanes"], kw["tables"], kw["ensembles"], q.shape[1])
    assert np.array_equal(w2, w)
    o, den, deg = ro.forward(q, k, v, w, kw["beta"], kw["causal"], kw["normalize_inputs"], kw["block_size"])
    assert rel_err(o, case["o"]) <= 1e-10
    assert rel_err(den, case["den"]) <= 1e-10
    flags = np.zeros(q.shape[0], dtype=bool)
    flags[list(deg)] = True
    assert np.array_equal(flags, case["degenerate"])
    grads = ro.vjp(q, k, v, w, kw["beta"], g, kw["causal"], kw["normalize_inputs"], kw["block_size"])
    errs = grad_errs(grads, (case["dq"], case["dk"], case["dv"]), 1e-4)
    assert max(errs) <= 1e-10, errs


def test_known_answers():
    """SPEC known answers: N=1 -> O=V; constant V -> constant O (ra/acceptance.py:383-416)."""
    rng = np.random.default_rng(0)
    w = ro.stacked_hyperplanes(3, 2, 2, 1, 8)
    q, k, v = rng.standard_normal((1, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 5))
    o, _, _ = ro.forward(q, k, v, w, 8.0)
    assert np.allclose(o, v, atol=1e-12)
    q, k = rng.standard_normal((40, 8)), rng.standard_normal((40, 8))
    c = rng.standard_normal(5)
    for causal in (False, True):
        o, _, _ = ro.forward(q, k, np.tile(c, (40, 1)), w, 8.0, causal)
        assert np.max(np.abs(o - c)) <= 1e-10
    # feature rows are stochastic (criterion 8)
    phi = ro.features(q, w, 8.0)
    assert np.allclose(phi.reshape(40, 2, 4).sum(-1), 1.0, atol=1e-12)


def test_factored_equals_corners():
    """The P>10 factored branch equals the corner softmax (ra/sketch.py:97-100)."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((7, 5))
    w = rng.standard_normal((3, 5))
    phi_c, _ = ro.table_features(x, w, 4.0)
    pos = ro._logistic(2 * 4.0 * np.tanh(x @ w.T))
    neg = ro._logistic(-2 * 4.0 * np.tanh(x @ w.T))
    phi = np.ones((7, 1))
    for t in range(3):
        phi = np.hstack([phi * pos[:, t:t + 1], phi * neg[:, t:t + 1]])
    assert np.allclose(phi, phi_c, atol=1e-14)
