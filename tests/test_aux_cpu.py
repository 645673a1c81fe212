"""CPU checks of the validation-side host code: the bench harness keeps the
reference's CSV schema byte for byte (golden strings from ra/bench.py)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2510_04008_b200 import benchmark as bm
from paper_2510_04008_b200 import sketch

Z = np.load(os.path.join(ROOT, "tests", "golden", "golden_aux.npz"))


def _recs():
    return [bm.BenchRecord("race", 4096, 128, 4, 2, 2, 1, 8.0, True, "forward_backward", 0.123456789, 1234, 0, "ok",
                           threads=8),
            bm.BenchRecord("angular_exact", 65536, 128, 4, None, None, None, None, False, "forward", None, 99, 3,
                           "time_guard")]


def test_csv_matches_reference():
    assert bm.records_to_csv(_recs()) == str(Z["csv"])
    ref_ext = str(Z["csv_ext"]).splitlines()
    ours = bm.records_to_csv(_recs(), extended=True).splitlines()
    for a, b in zip(ours, ref_ext):  # the reference's extended columns come first, then the GPU ones
        assert a.startswith(b)


def test_heatmap_matches_reference():
    assert bm.heatmap_csv_text(*bm.demo_kernel_heatmap([1, 2, 8], 9)) == str(Z["heatmap"])


def test_bench_validation():
    with pytest.raises(ValueError):
        bm.BenchMethod("flash")
    with pytest.raises(ValueError):
        bm.BenchMethod("race")
    with pytest.raises(ValueError):
        bm.bench_scaling([8, 4], [])
    with pytest.raises(ValueError):
        bm.bench_scaling([4], [], pass_kind="backward")


def test_corner_helpers():
    assert sketch.corner_vector(5, 3).tolist() == [-1.0, 1.0, -1.0]
    cm = sketch.corner_matrix(3)
    assert cm.shape == (8, 3) and cm[0].tolist() == [1, 1, 1] and cm[7].tolist() == [-1, -1, -1]
    with pytest.raises(ValueError):
        sketch.corner_matrix(11)
    with pytest.raises(ValueError):
        sketch.corner_vector(8, 3)
