"""Host-side behaviour of the drop-in API that needs no GPU: config and input
validation (same ValueErrors as the reference), hyperplane derivation, and
the no-fallback rule."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2510_04008_b200 as rb
from conftest import load_golden


@pytest.mark.parametrize("kw", [dict(hyperplanes=0, tables=1), dict(hyperplanes=21, tables=1),
                                dict(hyperplanes=2, tables=0), dict(hyperplanes=2, tables=1, ensembles=0),
                                dict(hyperplanes=2, tables=1, beta=-1.0), dict(hyperplanes=2, tables=1, beta=np.nan),
                                dict(hyperplanes=2, tables=1, block_size=0)])
def test_sketch_config_validation(kw):
    with pytest.raises(ValueError):
        rb.SketchConfig(**kw)


def test_sketch_config_properties():
    c = rb.SketchConfig(hyperplanes=3, tables=2, ensembles=2)
    assert c.n_buckets == 8 and c.total_tables == 4
    assert c.params().tables == 4 and c.params().hyperplanes == 3


def test_attn_inputs_validation():
    rng = np.random.default_rng(0)
    with pytest.raises(ValueError):
        rb.AttnInputs(rng.standard_normal((4, 3)), rng.standard_normal((4, 2)), rng.standard_normal((4, 3)))
    with pytest.raises(ValueError):
        rb.AttnInputs(rng.standard_normal((4, 3)), rng.standard_normal((4, 3)), rng.standard_normal((5, 3)))
    with pytest.raises(ValueError):
        rb.AttnInputs(rng.standard_normal(4), rng.standard_normal(4), rng.standard_normal(4))
    bad = rng.standard_normal((4, 3))
    bad[1, 1] = np.inf
    with pytest.raises(ValueError):
        rb.AttnInputs(bad, bad, bad)
    inp = rb.AttnInputs(rng.standard_normal((4, 3)), rng.standard_normal((4, 3)), rng.standard_normal((4, 5)))
    assert (inp.n, inp.dim, inp.dim_v) == (4, 3, 5)
    ti = rb.AttnInputs(torch.ones(3, 2), torch.ones(3, 2), torch.ones(3, 4))
    assert ti.dim_v == 4


def test_hyperplanes_match_reference():
    for case in load_golden()[:20]:
        cfg = rb.SketchConfig(**case.cfg_kwargs)
        assert np.array_equal(rb.all_hyperplanes(cfg, case["q"].shape[1]), case["w"])


def test_head_hyperplanes_seed_plus_h():
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=5)
    w = rb.head_hyperplanes(cfg, 3, 16)
    assert tuple(w.shape) == (3, 2, 2, 16)
    for h in range(3):
        ref = rb.all_hyperplanes(rb.SketchConfig(hyperplanes=2, tables=2, seed=5 + h), 16)
        assert np.array_equal(w[h].numpy(), ref.astype(np.float32))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    rng = np.random.default_rng(0)
    inp = rb.AttnInputs(*(rng.standard_normal((8, 4)) for _ in range(3)))
    cfg = rb.SketchConfig(hyperplanes=2, tables=2)
    with pytest.raises(RuntimeError):
        rb.race_attention(inp, cfg)
    with pytest.raises(RuntimeError):
        rb.race_attention_vjp(inp, cfg, np.ones((8, 4)))
    with pytest.raises(ValueError):
        rb.race_forward(torch.ones(1, 4, 8), torch.ones(1, 4, 8), torch.ones(1, 4, 8),
                        torch.ones(2, 2, 8), rb.SketchParams(2, 2, 8.0))
