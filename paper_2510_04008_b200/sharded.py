"""Sequence-sharded RACE attention across GPUs (one process per GPU).

Rank r owns the contiguous token slice r of every (b, h) sequence (rank order
= sequence order).  Q/K/V/dO never move; only the bucket tables
(BH x F x (dv+1) fp32, 16.5 KB at B=1 H=4 P=2 L=2) cross NVLink:

* non-causal fwd: local S_r = phi(K_r)^T[V_r|1] -> all_gather + fixed-order sum -> readout.
* causal fwd:     local totals -> all_gather -> carry_r = sum_{r'<r} S_r'
                  (fixed order) -> per-segment exclusive prefix -> chunked scan.
* non-causal bwd: local dS_r -> all_gather + fixed-order sum -> key side.
* causal bwd:     local dS totals -> all_gather -> carry_r = sum_{r'>r} dS_r'
                  -> per-segment exclusive suffix -> reverse scan.

This is the exact algebra of SURVEY Appendix A.4 (the reference itself is
single-process: its only carry is the in-process block carry of
ra/forward.py:105-120 / ra/backward.py:139-180, which this generalises).
The exchange helpers below are device-agnostic torch code, so the multi-rank
logic is unit-tested with the gloo backend on CPU (tests/test_sharded_cpu.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .functional import Problem, SketchParams, _c, _check_device, _on_q_device, _stream, _vp


# ---------------------------------------------------------------------------
# exchange steps (pure torch; work on any backend)
# ---------------------------------------------------------------------------
class TorchDistComm:
    """The exchange used between phases: torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group

    def allreduce(self, local: torch.Tensor) -> torch.Tensor:
        return allreduce_tables(local, self.group)

    def carry(self, local_total: torch.Tensor, direction: str) -> torch.Tensor:
        return rank_carry(local_total, direction, self.group)


def allreduce_tables(local: torch.Tensor, group=None) -> torch.Tensor:
    """Global S (or dS) = sum over ranks of the local tables (non-causal).

    all_gather + a local sum in rank order 0..G-1 rather than all_reduce: NCCL's reduction order
    depends on the algorithm it picks (ring / tree / NVLS), so the result could differ in the last
    bits between runs or world sizes; this keeps the reference's bit-determinism
    (ra/acceptance.py:419-450) for the price of G x 16.5 KB per call."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return local.clone()
    world = dist.get_world_size(group)
    gathered = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(gathered, local.contiguous(), group=group)
    out = gathered[0].clone()
    for r in range(1, world):
        out += gathered[r]
    return out


def rank_carry(local_total: torch.Tensor, direction: str, group=None) -> torch.Tensor:
    """Exclusive prefix ('prefix': sum of ranks < r) or suffix ('suffix': ranks > r)
    of the per-rank totals, summed in a fixed rank order (deterministic)."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return torch.zeros_like(local_total)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gathered = [torch.empty_like(local_total) for _ in range(world)]
    dist.all_gather(gathered, local_total.contiguous(), group=group)
    carry = torch.zeros_like(local_total)
    ranks = range(rank) if direction == "prefix" else range(world - 1, rank, -1)
    for r in ranks:
        carry += gathered[r]
    return carry


# ---------------------------------------------------------------------------
# sharded passes
# ---------------------------------------------------------------------------
def _combine(pr: Problem, mode: int, part, carry, out):
    _lib.check(_lib.lib().race_combine(pr.dref, mode, _vp(part), _vp(carry), _vp(out), _stream()),
               "race_combine")


@_on_q_device
def sharded_forward(q, k, v, w, p: SketchParams, group=None, comm=None):
    """(o, den, state) for this rank's sequence shard; state feeds sharded_backward."""
    comm = comm or TorchDistComm(group)
    q, k, v = _c(q), _c(k), _c(v)
    pr = Problem(q, k, v, w, p)
    L = _lib.lib()
    dev = pr.device
    E = pr.table_elems
    o = torch.empty_like(v)
    den = torch.empty(pr.lead + (pr.n,), dtype=torch.float32, device=dev)
    ws = pr.ws()
    part = torch.empty((pr.bh, pr.nseg, E), dtype=torch.float32, device=dev)
    local = torch.zeros((pr.bh, E), dtype=torch.float32, device=dev)
    if pr.grouped or pr.state_shape() is None:
        raise _lib.RaceUnsupported("sequence sharding needs all F buckets in one kernel pass (no table groups)")
    if p.causal:
        state = torch.empty(pr.state_shape(), dtype=torch.float32, device=dev)
        carries, norms = pr.split_causal_state(state)
    if pr.n:
        if p.causal:  # the aggregation also writes the k halves of the sketch rows
            _lib.check(L.race_kside_partials_rows(pr.dref, _vp(k), _vp(v), _vp(pr.w), _vp(part), _vp(norms),
                                                  _vp(ws), _stream()), "race_kside_partials_rows")
        else:
            _lib.check(L.race_kside_partials(pr.dref, _vp(k), _vp(v), _vp(pr.w), _vp(part), _vp(ws), _stream()),
                       "race_kside_partials")
        _combine(pr, _lib.COMBINE_TOTAL, part, None, local)
    if not p.causal:
        tables = comm.allreduce(local)
        if pr.n:
            _lib.check(L.race_fwd_readout(pr.dref, _vp(q), _vp(pr.w), _vp(tables), _vp(o), _vp(den), _vp(ws),
                                          _stream()), "race_fwd_readout")
        return o, den, tables.view(pr.state_shape())
    carry = comm.carry(local, "prefix")
    if pr.n:
        _combine(pr, _lib.COMBINE_PREFIX, part, carry, carries)
        _lib.check(L.race_fwd_causal_krows(pr.dref, _vp(q), _vp(k), _vp(v), _vp(pr.w), _vp(carries), _vp(o), _vp(den),
                                     _vp(norms), _vp(ws), _stream()), "race_fwd_causal_krows")
    return o, den, state


@_on_q_device
def sharded_backward(q, k, v, w, d_o, p: SketchParams, state, group=None, comm=None):
    """(dq, dk, dv) for this rank's shard given sharded_forward's state."""
    comm = comm or TorchDistComm(group)
    q, k, v, d_o, state = _c(q), _c(k), _c(v), _c(d_o), _c(state)
    pr = Problem(q, k, v, w, p)
    _check_device(pr.device, d_o=d_o, state=state)
    L = _lib.lib()
    dev = pr.device
    E = pr.table_elems
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = pr.ws()
    dpart = torch.empty((pr.bh, pr.nseg, E), dtype=torch.float32, device=dev)
    local = torch.zeros((pr.bh, E), dtype=torch.float32, device=dev)
    if not p.causal:
        if pr.n:
            _lib.check(L.race_bwd_qside(pr.dref, _vp(q), _vp(d_o), _vp(pr.w), _vp(state), _vp(dq), _vp(dpart),
                                        _vp(ws), _stream()), "race_bwd_qside")
            _combine(pr, _lib.COMBINE_TOTAL, dpart, None, local)
        dtables = comm.allreduce(local)
        if pr.n:
            _lib.check(L.race_bwd_kside(pr.dref, _vp(k), _vp(v), _vp(pr.w), _vp(dtables), _vp(dk), _vp(dv),
                                        _vp(ws), _stream()), "race_bwd_kside")
        return dq, dk, dv
    rden = torch.empty((pr.bh, max((pr.n + 3) // 4 * 4, 4)), dtype=torch.float32, device=dev)  # row pitch: N up to x4
    gden = torch.empty_like(rden)
    carries, norms = pr.split_causal_state(state)
    if pr.n:
        _lib.check(L.race_bwd_causal_q(pr.dref, _vp(q), _vp(k), _vp(v), _vp(d_o), _vp(pr.w), _vp(carries),
                                       _vp(norms), _vp(dq), _vp(rden), _vp(gden), _vp(dpart), _vp(ws), _stream()),
                   "race_bwd_causal_q")
        _combine(pr, _lib.COMBINE_TOTAL, dpart, None, local)
    carry = comm.carry(local, "suffix")
    if pr.n:
        dcar = torch.empty((pr.bh, pr.nseg, E), dtype=torch.float32, device=dev)
        _combine(pr, _lib.COMBINE_SUFFIX, dpart, carry, dcar)
        _lib.check(L.race_bwd_causal_k(pr.dref, _vp(q), _vp(k), _vp(v), _vp(d_o), _vp(pr.w), _vp(rden),
                                       _vp(gden), _vp(dcar), _vp(norms), _vp(dk), _vp(dv), _vp(ws), _stream()),
                   "race_bwd_causal_k")
    return dq, dk, dv


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous token range [lo, hi) of rank `rank` (balanced, rank order = sequence order)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


__all__ = ["TorchDistComm", "allreduce_tables", "rank_carry", "sharded_forward", "sharded_backward", "shard_bounds"]
