"""``torch.nn.Module`` front end: a multi-head RACE attention layer.

Hyperplanes are frozen (the reference treats W as a constant)
and derived per head with seed + h, as the reference's benchmark does
(ra/bench.py:175), so a layer built here reproduces the reference's per-head
calls exactly.
"""

from __future__ import annotations

import numpy as np
import torch

from .attention import SketchConfig, all_hyperplanes
from .functional import SketchParams, race_attention_torch


def head_hyperplanes(cfg: SketchConfig, heads: int, dim: int) -> torch.Tensor:
    """[H, T, P, d] float32: head h uses SketchConfig(seed=cfg.seed + h) (ra/bench.py:175)."""
    ws = []
    for h in range(heads):
        c = SketchConfig(cfg.hyperplanes, cfg.tables, cfg.ensembles, cfg.beta, cfg.seed + h,
                         cfg.causal, cfg.normalize_inputs, cfg.block_size)
        ws.append(all_hyperplanes(c, dim))
    return torch.from_numpy(np.stack(ws).astype(np.float32))


class RaceAttention(torch.nn.Module):
    """O = RACE(Q, K, V) on [B, H, N, d] CUDA tensors (fp32 or bf16), differentiable.

    bf16 heads of width up to 128 (e.g. the d=64 heads of a d_model=768, 12-head GPT) run on the
    tcgen05 kernels at their own width (no padded copies); fp32 inputs and other widths run on
    the CUDA-core kernels.  ``pad_head_dim`` is kept for compatibility and has no effect."""

    pad = False  # narrow heads are no longer zero-padded (gpt.py checks this)

    def __init__(self, heads: int, dim: int, cfg: SketchConfig, pad_head_dim: bool = True):
        super().__init__()
        self.cfg = cfg
        self.heads = heads
        self.dim = dim
        self.pad_head_dim = pad_head_dim
        self.params_ = SketchParams(cfg.hyperplanes, cfg.total_tables, float(cfg.beta), cfg.causal,
                                    cfg.normalize_inputs)
        w = head_hyperplanes(cfg, heads, dim)
        self.register_buffer("w", w, persistent=True)

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        return race_attention_torch(q, k, v, self.w, self.params_)
