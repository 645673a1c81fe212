"""Sequence sharding with REAL processes on the GPU.

Two ranks (torch.distributed, gloo for the small table exchange since this
box has one GPU; the kernels and the exchange code are those NCCL runs use)
each own half of a bf16 causal / non-causal sequence, run sharded_forward /
sharded_backward on the tcgen05 kernels, and must reproduce the single-GPU
result on their slice.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, rel_err

pytestmark = pytest.mark.gpu
N, H, D = 16384, 4, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(dev):
    g = torch.Generator(device=dev).manual_seed(9)
    return [torch.randn(1, H, N, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(4)]


def _worker(rank, world, port, causal, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2510_04008_b200 as rb
    from paper_2510_04008_b200.sharded import sharded_backward, sharded_forward, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v, g = _inputs(dev)
        cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=causal)
        w = rb.head_hyperplanes(cfg, H, D).to(dev)
        p = cfg.params()
        lo, hi = shard_bounds(N, world, rank)
        sl = [t[:, :, lo:hi].contiguous() for t in (q, k, v, g)]
        o, den, st = sharded_forward(sl[0], sl[1], sl[2], w, p)
        dq, dk, dv = sharded_backward(sl[0], sl[1], sl[2], w, sl[3], p, st)
        torch.cuda.synchronize()
        for name, t in (("o", o), ("den", den), ("dq", dq), ("dk", dk), ("dv", dv)):
            np.save(os.path.join(out_dir, f"{name}{rank}.npy"), t.float().cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
def test_two_process_sharding_matches_single_gpu(causal, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_2510_04008_b200 as rb

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), causal, str(tmp_path)), nprocs=world, join=True)
    dev = torch.device("cuda", 0)
    q, k, v, g = _inputs(dev)
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, H, D).to(dev)
    p = cfg.params()
    o, den, st = rb.race_forward(q, k, v, w, p)
    dq, dk, dv = rb.race_backward(q, k, v, w, g, p, state=st)
    ref = {"o": o, "den": den, "dq": dq, "dk": dk, "dv": dv}
    for name, full in ref.items():
        got = np.concatenate([np.load(tmp_path / f"{name}{r}.npy") for r in range(world)], axis=2)
        tol = 1e-4 if name == "den" else 1e-2
        assert rel_err(got, full.float().cpu().numpy()) <= tol, name
