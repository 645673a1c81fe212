"""CPU checks of the C-ABI library: it loads, exports every symbol
include/race_b200.h declares, and its host-side queries/validation behave
(no kernel is launched here)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

from paper_2510_04008_b200 import _lib

HEADER = os.path.join(ROOT, "include", "race_b200.h")
AUX_HEADER = os.path.join(ROOT, "include", "race_aux.h")


def declared_symbols(header=HEADER):
    src = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(race_\w+)\s*\(", src, flags=re.M)))


def test_header_matches_binding():
    assert set(declared_symbols()) == set(_lib.EXPORTS)
    assert set(declared_symbols(AUX_HEADER)) == set(_lib.AUX_EXPORTS)


def test_library_exports_every_symbol():
    so = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols() + declared_symbols(AUX_HEADER):
        assert hasattr(so, name), name
    assert _lib.lib().race_abi_version() == _lib.ABI_VERSION


def test_aux_validation_without_gpu():
    L = _lib.lib()
    # bad shapes are rejected on the host before any launch
    assert L.race_aux_soft_features(0, 4, 8, None, None, 0, 1, 8.0, 1, None, None) == _lib.RACE_EBADSHAPE
    assert L.race_aux_soft_features(0, 4, 8, None, None, 2, 1, 0.0, 1, None, None) == _lib.RACE_EBADSHAPE
    assert L.race_aux_angular_fwd(0, 4, 512, 8, None, None, None, 2, 0, None, None, None) == _lib.RACE_EUNSUPPORTED
    assert L.race_aux_hard_attention(0, 4, 8, None, None, None, 2, 1, None, None, None, None) == _lib.RACE_EBADSHAPE
    assert L.race_aux_hard_workspace_bytes(8, 2, 3) == 8 * 3 * 4 * 9


def _desc(**kw):
    base = dict(dtype=_lib.RACE_BF16, batch_heads=4, heads=4, n=131072, dim=128, dim_v=128,
                hyperplanes=2, tables=2, beta=8.0, causal=True, normalize=True, w_per_head=True)
    base.update(kw)
    return _lib.make_desc(**base)


def test_segmentation_and_sizes():
    d = _desc()
    nseg, seg = _lib.segments(d)
    assert seg % 128 == 0 and nseg * seg >= 131072 > (nseg - 1) * seg
    # carries (padded to 64 floats: the sketch rows start 256-byte aligned) + sketch rows
    assert _lib.state_elems(d) == ((4 * nseg * 8 * 129 + 63) // 64) * 64 + 16 * 4 * 131072
    assert _lib.state_elems(_desc(causal=False)) == 4 * 8 * 129
    assert _lib.workspace_bytes(d) >= 4 * 4 * nseg * 8 * 129
    assert _lib.segments(_desc(n=1)) == (1, 128)
    assert _lib.segments(_desc(n=0))[0] == 1


@pytest.mark.parametrize("kw, exc", [
    (dict(hyperplanes=0), ValueError),
    (dict(hyperplanes=21), ValueError),
    (dict(tables=0), ValueError),
    (dict(beta=0.0), ValueError),
    (dict(beta=float("inf")), ValueError),
    (dict(dim=0), ValueError),
    (dict(batch_heads=6, heads=4), ValueError),
    (dict(dim=4096), _lib.RaceUnsupported),
])
def test_validation(kw, exc):
    with pytest.raises(exc):
        _lib.segments(_desc(**kw))


@pytest.mark.parametrize("P", [8, 10, 11, 16, 20])
def test_wide_sketches_plan_corner_groups(P):
    """P beyond one kernel pass (and every P in [11, 20], which the reference accepts, ra/core.py:71)
    runs as table / corner groups: valid sizes; the state is the summed numerators [BH, N, dv] and
    denominators [BH, N] the backward takes its normalisers from."""
    d = _desc(hyperplanes=P, tables=2)
    assert _lib.segments(d)[0] >= 1
    assert _lib.workspace_bytes(d) > 0
    assert _lib.state_elems(d) == 4 * 131072 * 129
    plan = _lib.group_plan(d)
    assert plan["passes"] > 1 and plan["corner_bits"] <= 10


def test_state_rows_offset_is_aligned():
    for P, L, n, bh in ((1, 1, 128, 1), (1, 3, 300, 1), (2, 2, 4099, 3)):
        d = _desc(hyperplanes=P, tables=L, n=n, batch_heads=bh, heads=bh)
        nseg, _ = _lib.segments(d)
        carries = bh * nseg * (L << P) * 129
        assert _lib.state_elems(d) - 16 * bh * n == ((carries + 63) // 64) * 64


def test_bad_abi_version():
    d = _desc()
    d.abi_version = 99
    with pytest.raises(ValueError):
        _lib.segments(d)


@pytest.mark.gpu  # the plan depends on the tcgen05 path being available (a driver entry point)
@pytest.mark.parametrize("causal", [True, False])
def test_table_group_state_keeps_pass_states(causal):
    """bf16 table groups on the tcgen05 path: the grouped state is the summed numerators / denominators
    (padded to 64 floats) followed by every pass's own forward state (carries + sketch rows, or
    tables), which the grouped backward reuses instead of re-aggregating each pass."""
    d = _desc(tables=4, causal=causal)  # F = 16: two passes of two tables
    plan = _lib.group_plan(d)
    assert plan["passes"] == 2 and plan["fast"] and plan["tables_per_pass"] == 2
    one = _lib.state_elems(_desc(tables=2, causal=causal))  # one pass of two tables
    head = ((4 * 131072 * 129 + 63) // 64) * 64
    assert _lib.state_elems(d) == head + 2 * ((one + 63) // 64) * 64


def _busiest_cta_chunks(bh, n, nseg, seg, grid=148):
    """Chunks (128 tokens) of the busiest CTA when `bh * nseg` items are split evenly by count over the
    persistent grid (cta_range in tc_fast.cuh)."""
    items = bh * nseg
    g = min(items, grid)
    cps = -(-n // 128)
    load = 0
    for b in range(g):
        tot = 0
        for i in range(b * items // g, (b + 1) * items // g):
            s = i % nseg
            tot += seg // 128 if s + 1 < nseg else cps - s * (seg // 128)
        load = max(load, tot)
    return load


@pytest.mark.parametrize("bh,n", [(4, 131072), (12, 16384), (1, 131072), (8, 65536), (4, 20971520), (3, 5000)])
def test_fast_segmentation_balances_the_persistent_grid(bh, n):
    """The tcgen05 path's segment length (fast_segment in race_abi.cu): the busiest CTA gets no more
    128-token chunks than under the old fixed ~8-segments-per-CTA policy, with no more segments."""
    d = _desc(batch_heads=bh, heads=bh, n=n)
    nseg, seg = _lib.segments(d)
    target = -(-(148 * 8) // bh)
    old_seg = max(128, -(-(-(-n // target)) // 128) * 128)
    old_nseg = -(-n // old_seg)
    assert _busiest_cta_chunks(bh, n, nseg, seg) <= _busiest_cta_chunks(bh, n, old_nseg, old_seg)
    assert nseg <= old_nseg
    if (bh, n) == (4, 131072):  # the headline: one 28-chunk segment per CTA
        assert (nseg, seg) == (37, 3584)
