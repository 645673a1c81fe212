"""Pin the oracle's num/den and row normalisation to the real reference's
accumulate_num_den (ra/forward.py:124-144), race_attention degenerate rows
(ra/forward.py:157-163) and row_normalize[_vjp] (ra/core.py:114-139), from
tests/golden/golden_extra.npz (tests/golden/make_extra_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_num_den_golden, load_row_normalize_golden, rel_err
from oracle import race_oracle as ro

ND = load_num_den_golden()


@pytest.mark.parametrize("case", ND, ids=lambda c: f"nd{c['index']}")
def test_oracle_num_den_matches_reference(case):
    kw = case["cfg_kwargs"]
    w = ro.stacked_hyperplanes(kw["seed"], kw["hyperplanes"], kw["tables"], kw["ensembles"], case["q"].shape[1])
    num, den = ro.num_den(case["q"], case["k"], case["v"], w, kw["beta"], kw["causal"])
    assert rel_err(num, case["num"]) <= 1e-10
    assert rel_err(den, case["den"]) <= 1e-10
    o, den2, deg = ro.forward(case["q"], case["k"], case["v"], w, kw["beta"], kw["causal"])
    assert rel_err(o, case["o"]) <= 1e-10
    assert list(deg) == list(case["degenerate"])


def test_degenerate_fixture_is_degenerate():
    deg = [c for c in ND if len(c["degenerate"])]
    assert len(deg) == 2 and all(np.all(c["den"][c["degenerate"]] == 0.0) for c in deg)


def test_oracle_row_normalize_matches_reference():
    g = load_row_normalize_golden()
    assert rel_err(ro.unit_rows(g["x"]), g["y"]) <= 1e-15
    assert rel_err(ro.unit_rows_vjp(g["x"], g["g"]), g["dx"]) <= 1e-12
