"""Multi-rank logic of the sequence-sharded path, on CPU with gloo (world 2 and 3).

Each rank owns a contiguous token slice; its local bucket tables are computed
with the oracle's feature map (numpy), then exchanged with the SAME helpers the
GPU path uses (paper_2510_04008_b200.sharded.allreduce_tables / rank_carry).
The results must reproduce the single-process oracle: non-causal outputs from
the all-reduced tables, causal outputs from the exclusive prefix carry, and the
backward suffix carry for dS.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(n=97, d=12, dv=7, seed=5):
    from oracle import race_oracle as ro

    rng = np.random.default_rng(seed)
    q, k, v, g = (rng.standard_normal((n, x)) for x in (d, d, dv, dv))
    w = ro.stacked_hyperplanes(seed, 2, 2, 1, d)
    return q, k, v, g, w


def _worker(rank, world, port, causal, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import race_oracle as ro
    from paper_2510_04008_b200.sharded import allreduce_tables, rank_carry, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v, g, w = _problem()
        beta, T = 8.0, w.shape[0]
        lo, hi = shard_bounds(q.shape[0], world, rank)
        qn, kn = ro.unit_rows(q[lo:hi]), ro.unit_rows(k[lo:hi])
        pk = ro.features(kn, w, beta)
        pq = ro.features(qn, w, beta)
        vx = np.hstack([v[lo:hi], np.ones((hi - lo, 1))])
        local = torch.from_numpy(pk.T @ vx)  # S_r = phi(K_r)^T [V_r | 1]
        if not causal:
            s = allreduce_tables(local).numpy()
            nd = pq @ s
            o = nd[:, :-1] / nd[:, -1:]
        else:
            carry = rank_carry(local, "prefix").numpy()
            cum = carry[None] + np.cumsum(pk[:, :, None] * vx[:, None, :], axis=0)
            nd = np.einsum("tf,tfc->tc", pq, cum)
            o = nd[:, :-1] / nd[:, -1:]
            # backward suffix carry: dS_r = phi(Q_r)^T G_r with G = [dO | 1] (any fixed G works)
            gx = np.hstack([g[lo:hi], np.ones((hi - lo, 1))])
            dloc = torch.from_numpy(pq.T @ gx)
            dcarry = rank_carry(dloc, "suffix").numpy()
            np.save(os.path.join(out_dir, f"dcarry{rank}.npy"), dcarry)
            np.save(os.path.join(out_dir, f"dloc{rank}.npy"), dloc.numpy())
        np.save(os.path.join(out_dir, f"o{rank}.npy"), o)
        np.save(os.path.join(out_dir, f"den{rank}.npy"), nd[:, -1] / T)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("causal", [False, True], ids=["noncausal", "causal"])
def test_gloo_exchange_reproduces_single_process(world, causal, tmp_path):
    from oracle import race_oracle as ro

    mp.spawn(_worker, args=(world, _free_port(), causal, str(tmp_path)), nprocs=world, join=True)
    q, k, v, g, w = _problem()
    o_ref, den_ref, _ = ro.forward(q, k, v, w, 8.0, causal)
    o = np.concatenate([np.load(tmp_path / f"o{r}.npy") for r in range(world)])
    den = np.concatenate([np.load(tmp_path / f"den{r}.npy") for r in range(world)])
    assert np.allclose(o, o_ref, rtol=1e-12, atol=1e-12)
    assert np.allclose(den, den_ref, rtol=1e-12, atol=1e-12)
    if causal:
        dl = [np.load(tmp_path / f"dloc{r}.npy") for r in range(world)]
        for r in range(world):
            want = sum((dl[x] for x in range(r + 1, world)), np.zeros_like(dl[0]))
            assert np.allclose(np.load(tmp_path / f"dcarry{r}.npy"), want, rtol=1e-14, atol=1e-14)


def test_shard_bounds_partition():
    from paper_2510_04008_b200.sharded import shard_bounds

    for n in (0, 1, 7, 100, 131072):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(hi - lo for lo, hi in b) - min(hi - lo for lo, hi in b) <= 1


def test_single_process_exchange_is_identity():
    from paper_2510_04008_b200.sharded import allreduce_tables, rank_carry

    t = torch.randn(2, 8, 5)
    assert torch.equal(allreduce_tables(t), t)
    assert torch.equal(rank_carry(t, "prefix"), torch.zeros_like(t))
