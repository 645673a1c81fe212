"""GPT-style causal language model with RACE attention in every layer
(BASELINE configs[4]: 6 layers, d_model=768, 12 heads, sequence 16K).

The reference package has no model code; this is the "next" row
of SURVEY §8(f): a plain pre-LayerNorm decoder whose attention is
``RaceAttention`` (causal, the reference's P=2, L=2, beta=8 sketch, per-head
hyperplanes with seed + h as ``ra/bench.py:175``).  Everything except the
attention is standard PyTorch (cuBLAS GEMMs, bf16 autocast, fused AdamW).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from .attention import SketchConfig
from .module import RaceAttention


@dataclass(frozen=True)
class GPTConfig:
    vocab: int = 50304
    seq_len: int = 16384
    layers: int = 6
    d_model: int = 768
    heads: int = 12
    mlp_ratio: int = 4
    hyperplanes: int = 2
    tables: int = 2
    beta: float = 8.0


class Block(nn.Module):
    def __init__(self, cfg: GPTConfig, layer: int):
        super().__init__()
        self.heads = cfg.heads
        self.ln1 = nn.LayerNorm(cfg.d_model)
        self.qkv = nn.Linear(cfg.d_model, 3 * cfg.d_model, bias=False)
        self.proj = nn.Linear(cfg.d_model, cfg.d_model, bias=False)
        sk = SketchConfig(hyperplanes=cfg.hyperplanes, tables=cfg.tables, beta=cfg.beta,
                          seed=1000 * layer, causal=True)
        self.attn = RaceAttention(cfg.heads, cfg.d_model // cfg.heads, sk)
        self.ln2 = nn.LayerNorm(cfg.d_model)
        self.fc = nn.Linear(cfg.d_model, cfg.mlp_ratio * cfg.d_model, bias=False)
        self.out = nn.Linear(cfg.mlp_ratio * cfg.d_model, cfg.d_model, bias=False)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        b, n, c = x.shape
        q, k, v = self.qkv(self.ln1(x)).split(c, dim=-1)
        # [B, H, N, d] views of the projection's [B, N, H*d] columns: the tcgen05 kernels read them in
        # place (4-D TMA maps, race_fwd_layout) and write O in [B, N, H, d] order, so neither the
        # transposes here nor the one below copy
        q, k, v = (t.view(b, n, self.heads, c // self.heads).transpose(1, 2) for t in (q, k, v))
        o = self.attn(q, k, v)
        x = x + self.proj(o.transpose(1, 2).reshape(b, n, c))
        return x + self.out(F.gelu(self.fc(self.ln2(x)), approximate="tanh"))


class RaceGPT(nn.Module):
    def __init__(self, cfg: GPTConfig):
        super().__init__()
        self.cfg = cfg
        self.tok = nn.Embedding(cfg.vocab, cfg.d_model)
        self.pos = nn.Embedding(cfg.seq_len, cfg.d_model)
        self.blocks = nn.ModuleList(Block(cfg, i) for i in range(cfg.layers))
        self.ln = nn.LayerNorm(cfg.d_model)
        self.head = nn.Linear(cfg.d_model, cfg.vocab, bias=False)
        self.head.weight = self.tok.weight  # tied embeddings
        for m in self.modules():
            if isinstance(m, nn.Linear):
                nn.init.normal_(m.weight, std=0.02)
            elif isinstance(m, nn.Embedding):
                nn.init.normal_(m.weight, std=0.02)
        for blk in self.blocks:
            nn.init.normal_(blk.proj.weight, std=0.02 / math.sqrt(2 * cfg.layers))
            nn.init.normal_(blk.out.weight, std=0.02 / math.sqrt(2 * cfg.layers))

    def forward(self, idx: torch.Tensor) -> torch.Tensor:
        n = idx.shape[1]
        x = self.tok(idx) + self.pos(torch.arange(n, device=idx.device))
        for blk in self.blocks:
            x = blk(x)
        return self.head(self.ln(x))


def train_step(model: RaceGPT, opt: torch.optim.Optimizer, idx: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
    """One optimiser step (bf16 autocast, fp32 master weights); returns the loss (device tensor).

    The cross-entropy runs outside autocast on the bf16 logits (its softmax reductions accumulate in
    fp32): autocast would first materialise an fp32 copy of the [N, vocab] logits and its gradient,
    2.9 of the ~19.6 ms of the 16k-token step."""
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(idx)
    loss = F.cross_entropy(logits.view(-1, logits.shape[-1]), targets.view(-1))
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)
    return loss.detach()
