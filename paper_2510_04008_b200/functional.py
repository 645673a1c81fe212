"""Device-tensor entry points over the C-ABI (the layer the drop-in API,
the autograd Function and the sharded path all call).

Tensors are torch CUDA tensors; the C library sees only raw device pointers,
sizes and the current stream (include/race_b200.h).  Layout: q, k are
``[..., N, d]`` and v, o, d_o are ``[..., N, dv]``; the leading dimensions are
flattened to ``BH`` rows, the last of which is the head index ``h`` used to
pick that head's hyperplanes (``bh % H``).

Hyperplanes ``w`` (float32 on the device) are either shared ``[T, P, d]`` /
``[T*P, d]`` or per head ``[H, T, P, d]`` / ``[H, T*P, d]``; tables are in the
reference's (m, l) task order (``ra/forward.py:128``).
"""

from __future__ import annotations

import ctypes
import functools
import os
from dataclasses import dataclass

import torch

from . import _lib

_DTYPES = {torch.float32: _lib.RACE_F32, torch.bfloat16: _lib.RACE_BF16}


@dataclass(frozen=True)
class SketchParams:
    """The estimator hyper-parameters the kernels need (SketchConfig minus RNG)."""

    hyperplanes: int
    tables: int  # total tables T = M * L
    beta: float
    causal: bool = False
    normalize: bool = True


# ---------------------------------------------------------------------------
# workspace cache: one growing buffer per (device, stream), so calls on different streams never
# share scratch (allocate before graph capture)
# ---------------------------------------------------------------------------
_WS: dict[tuple[int, int], torch.Tensor] = {}


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = (idx, torch.cuda.current_stream(idx).cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _vp(t: torch.Tensor | None) -> ctypes.c_void_p | None:
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device: torch.device | None = None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def prepare_w(w: torch.Tensor, p: SketchParams, d: int, device) -> tuple[torch.Tensor, bool, int]:
    """Return (w contiguous fp32 [H?, T*P, d], per_head, heads)."""
    w = w.to(device=device, dtype=torch.float32)
    tp = p.tables * p.hyperplanes
    shared3 = w.dim() == 3 and w.shape[0] == p.tables and w.shape[1] == p.hyperplanes
    if w.dim() == 4 or (w.dim() == 3 and not shared3):
        w = w.reshape(w.shape[0], tp, d)
        per_head, heads = True, w.shape[0]
    elif w.dim() in (2, 3):
        w = w.reshape(tp, d)
        per_head, heads = False, 1
    else:
        raise ValueError(f"hyperplane tensor has unsupported shape {tuple(w.shape)}")
    if w.shape[-1] != d or w.shape[-2] != tp:
        raise ValueError(f"hyperplanes {tuple(w.shape)} do not match T*P={tp}, d={d}")
    return w.contiguous(), per_head, heads


class _Meta:
    """Per-shape facts from the library (descriptor, segments, workspace and state sizes), queried
    once per distinct problem: an eager layer call then makes no sizing calls across the C-ABI."""

    __slots__ = ("desc", "dref", "nseg", "seg_tokens", "ws_bytes", "state_elems", "fast", "grouped", "fast_plan")

    def __init__(self, desc):
        self.desc = desc
        self.dref = _lib.ref(desc)
        self.nseg, self.seg_tokens = _lib.segments(desc)
        self.ws_bytes = _lib.workspace_bytes(desc)
        self.state_elems = _lib.state_elems(desc)
        self.fast = _lib.fast_path(desc)
        plan = _lib.group_plan(desc)
        self.grouped = plan["passes"] > 1
        self.fast_plan = plan["fast"]


_META: dict[tuple, _Meta] = {}


def _meta(**kw) -> _Meta:
    # the fast-path switch is part of the key: tests flip RACE_DISABLE_FAST_PATH at run time
    key = (tuple(sorted(kw.items())), os.environ.get("RACE_DISABLE_FAST_PATH"), torch.cuda.current_device())
    m = _META.get(key)
    if m is None:
        m = _META[key] = _Meta(_lib.make_desc(**kw))
    return m


def _check_device(dev: torch.device, **tensors) -> None:
    for name, t in tensors.items():
        if t is not None and t.device != dev:
            raise ValueError(f"{name} is on {t.device} but q is on {dev}; all tensors must be on one device")


class Problem:
    """Validated shapes + descriptor for one call."""

    def __init__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, w: torch.Tensor,
                 p: SketchParams):
        if not q.is_cuda:
            raise ValueError("the RACE B200 path needs CUDA tensors (there is no CPU fallback)")
        if q.dtype not in _DTYPES:
            raise ValueError(f"unsupported dtype {q.dtype}; use float32 or bfloat16")
        if k.dtype != q.dtype or v.dtype != q.dtype:
            raise ValueError("q, k, v must share one dtype")
        _check_device(q.device, k=k, v=v)
        if q.shape != k.shape:
            raise ValueError(f"q and k shapes differ: {tuple(q.shape)} vs {tuple(k.shape)}")
        if q.dim() < 2 or v.dim() != q.dim() or v.shape[:-1] != q.shape[:-1]:
            raise ValueError(f"v shape {tuple(v.shape)} does not match q {tuple(q.shape)}")
        self.lead = tuple(q.shape[:-2])
        self.n, self.d, self.dv = q.shape[-2], q.shape[-1], v.shape[-1]
        bh = 1
        for s in self.lead:
            bh *= s
        self.bh = bh
        self.p = p
        self.device = q.device
        self.dtype = q.dtype
        self.w, per_head, heads = prepare_w(w, p, self.d, q.device)
        if per_head and (len(self.lead) == 0 or self.lead[-1] != heads):
            raise ValueError(f"per-head hyperplanes for {heads} heads but inputs have lead dims {self.lead}")
        # desc heads = the operands' head dimension (W indexing uses it only when per_head; strided
        # operands are addressed as [B, H, N, w] through it)
        if not per_head and self.lead:
            heads = max(self.lead[-1], 1)
        m = _meta(dtype=_DTYPES[q.dtype], batch_heads=max(bh, 1), heads=heads, n=self.n, dim=self.d,
                  dim_v=self.dv, hyperplanes=p.hyperplanes, tables=p.tables, beta=float(p.beta),
                  causal=p.causal, normalize=p.normalize, w_per_head=per_head)
        self.desc, self.dref = m.desc, m.dref
        self.nseg, self.seg_tokens = m.nseg, m.seg_tokens
        self._ws_bytes, self._state_elems = m.ws_bytes, m.state_elems
        self.grouped = m.grouped
        self.one_pass_fast = bool(m.fast) and not m.grouped
        self.table_elems = (p.tables << p.hyperplanes) * (self.dv + 1)

    def ws(self) -> torch.Tensor:
        return workspace(self._ws_bytes, self.device)

    def carry_elems(self) -> int:
        """Floats of the causal carries [BH, nseg, F, dv+1], rounded up to 64 so the sketch rows that
        follow them start on a 256-byte boundary (race_state_elems, include/race_b200.h)."""
        return (self.bh * self.nseg * self.table_elems + 63) & ~63

    def state_shape(self) -> tuple[int, ...] | None:
        """Non-causal: the global tables [BH, F, dv+1].  Causal: a flat buffer holding the
        per-segment carries [BH, nseg, F, dv+1] (padded to 64 floats) then the q/k sketch rows
        [BH, N, 16] (projections x^.w_j and ||x||^2 of every q and k row, include/race_b200.h).
        Sketches run as table / corner groups (F beyond one kernel pass): a flat buffer of the
        summed numerators [BH, N, dv] then denominators [BH, N] (race_state_elems)."""
        if self._state_elems == 0:
            return None
        if self.grouped:
            return (self._state_elems,)
        f = self.p.tables << self.p.hyperplanes
        if self.p.causal:
            return (self.carry_elems() + 16 * self.bh * self.n,)
        return (self.bh, f, self.dv + 1)

    def split_causal_state(self, state: torch.Tensor):
        """(carries [BH, nseg, F, dv+1], sketch rows [BH, N, 16]) views of a causal state buffer."""
        nc = self.bh * self.nseg * self.table_elems
        off = self.carry_elems()
        return (state[:nc].view(self.bh, self.nseg, self.table_elems),
                state[off:].view(self.bh, max(self.n, 0), 16))


def _c(t: torch.Tensor) -> torch.Tensor:
    """Contiguous and 16-byte aligned (TMA tensor maps and the vector loads need aligned bases; a view
    starting mid-allocation gets copied)."""
    if t.is_contiguous() and t.data_ptr() % 16 == 0:
        return t
    return t.clone(memory_format=torch.contiguous_format) if t.is_contiguous() else t.contiguous()


def _strides(t: torch.Tensor):
    """(token, head, batch) element strides of a non-contiguous [B, H, N, w] view the tcgen05 kernels can
    read in place through their 4-D TMA maps (rows contiguous, 16-byte aligned base and strides), e.g.
    ``x.view(B, N, H, d).transpose(1, 2)`` of a [B, N, H*d] projection; None otherwise."""
    if t.dim() != 4 or t.is_contiguous() or t.stride(-1) != 1 or t.data_ptr() % 16:
        return None
    sb, sh, sn = t.stride(0), t.stride(1), t.stride(2)
    if sb % 8 or sh % 8 or sn % 8 or min(sb, sh, sn) < 0:
        return None
    return sn, sh, sb


def _bnhd(like: torch.Tensor, width: int) -> torch.Tensor:
    """An uninitialised [B, H, N, width] tensor stored as [B, N, H, width] (the layout of ``like``'s
    producer), so the caller's transpose back to [B, N, H*width] is a free view."""
    b, h, n = like.shape[:3]
    return torch.empty((b, n, h, width), dtype=like.dtype, device=like.device).transpose(1, 2)


def _layout(**tensors):
    """RaceLayout of the given operands (contiguous ones keep token stride 0)."""
    lay = _lib.RaceLayout()
    for name, t in tensors.items():
        st = _strides(t) if t is not None else None
        if st is not None:
            getattr(lay, name).token, getattr(lay, name).head, getattr(lay, name).batch = st
    return lay


def _strided_ok(pr: "Problem", *ts) -> bool:
    """Use the strided path: some operand is a readable strided view and the problem runs as one tcgen05
    pass (everything else takes contiguous copies)."""
    return pr.one_pass_fast and any(_strides(t) is not None for t in ts) and \
        all((t.is_contiguous() and t.data_ptr() % 16 == 0) or _strides(t) is not None for t in ts)


def _race_forward(q, k, v, w, p: SketchParams, *, want_state: bool = True):
    """race_forward at the tensors' own width.  [B, N, H, d]-strided q, k, v views (a fused projection's
    output) run in place on the one-pass tcgen05 path, and O is then returned in the same
    [B, N, H, dv] storage order."""
    pr = Problem(q, k, v, w, p)
    strided = _strided_ok(pr, q, k, v)
    if not strided:
        q, k, v = _c(q), _c(k), _c(v)
    o = _bnhd(v, pr.dv) if strided and _strides(v) is not None else torch.empty_like(v, memory_format=torch.contiguous_format)
    den = torch.empty(pr.lead + (pr.n,), dtype=torch.float32, device=pr.device)
    shape = pr.state_shape() if want_state else None
    state = torch.empty(shape, dtype=torch.float32, device=pr.device) if shape is not None else None
    if pr.n == 0 or pr.bh == 0:
        if state is not None:
            state.zero_()
        return o, den, state
    ws = pr.ws()
    if strided:
        lay = _layout(q=q, k=k, v=v, o=o)
        _lib.check(_lib.lib().race_fwd_layout(pr.dref, ctypes.byref(lay), _vp(q), _vp(k), _vp(v), _vp(pr.w),
                                              _vp(o), _vp(den), _vp(state), _vp(ws), _stream()), "race_fwd_layout")
    else:
        _lib.check(_lib.lib().race_fwd(pr.dref, _vp(q), _vp(k), _vp(v), _vp(pr.w), _vp(o), _vp(den),
                                       _vp(state), _vp(ws), _stream()), "race_fwd")
    return o, den, state


def _race_backward(q, k, v, w, d_o, p: SketchParams, state=None, *, inplace: bool = False):
    """race_backward at the tensors' own width."""
    if inplace and not (q.is_contiguous() and k.is_contiguous() and v.is_contiguous()):
        raise ValueError("inplace backward needs contiguous q, k, v")
    pr = Problem(q, k, v, w, p)
    _check_device(pr.device, d_o=d_o, state=state)
    if d_o.shape != v.shape or d_o.dtype != v.dtype:
        raise ValueError(f"d_out shape {tuple(d_o.shape)} does not match output shape {tuple(v.shape)}")
    strided = not inplace and _strided_ok(pr, q, k, v, d_o)
    if not strided:
        q, k, v, d_o = _c(q), _c(k), _c(v), _c(d_o)
    if inplace:
        dq, dk, dv = q, k, v
    else:  # gradients in their inputs' storage order (a strided q gets a [B, N, H, d]-ordered dq)
        dq, dk, dv = (_bnhd(x, x.shape[-1]) if strided and _strides(x) is not None
                      else torch.empty_like(x, memory_format=torch.contiguous_format) for x in (q, k, v))
    if pr.n == 0 or pr.bh == 0:
        return dq, dk, dv
    if state is not None:
        state = _c(state)
        if tuple(state.shape) != pr.state_shape() or state.dtype != torch.float32:
            raise ValueError("state does not match this problem")
    ws = pr.ws()
    if strided:
        lay = _layout(q=q, k=k, v=v, d_o=d_o, dq=dq, dk=dk, dv=dv)
        _lib.check(_lib.lib().race_bwd_layout(pr.dref, ctypes.byref(lay), _vp(q), _vp(k), _vp(v), _vp(pr.w),
                                              _vp(d_o), _vp(state), _vp(dq), _vp(dk), _vp(dv), _vp(ws), _stream()),
                   "race_bwd_layout")
    else:
        _lib.check(_lib.lib().race_bwd(pr.dref, _vp(q), _vp(k), _vp(v), _vp(pr.w), _vp(d_o), _vp(state),
                                       _vp(dq), _vp(dk), _vp(dv), _vp(ws), _stream()), "race_bwd")
    return dq, dk, dv


FAST_DIM = 128  # maximum head width of the sm_100a tcgen05 kernels (narrower bf16 heads run natively)


def _on_q_device(fn):
    """Run fn with q's GPU as the current device: the C library launches on the current device's
    stream (cudaGetDevice), so a call on cuda:1 tensors while cuda:0 is current must switch."""

    @functools.wraps(fn)
    def wrapped(q, *args, **kw):
        if isinstance(q, torch.Tensor) and q.is_cuda and q.device.index != torch.cuda.current_device():
            with torch.cuda.device(q.device):
                return fn(q, *args, **kw)
        return fn(q, *args, **kw)

    return wrapped


@_on_q_device
def race_forward(q, k, v, w, p: SketchParams, *, want_state: bool = True, pad: bool = True):
    """O, den (float32, the reference's averaged den) and the backward state.

    One fwd pass = key-side aggregation -> fixed-order combine -> readout
    (non-causal) or chunked scan (causal); see race_fwd in race_b200.h.  bf16 heads of any width
    d, dv <= 128 (multiples of 8) run on the tcgen05 kernels natively: the TMA maps zero-fill the
    tile columns beyond d and clip the stores, so no padded copies are made.  ``pad`` is accepted
    for compatibility with round-1 callers and ignored."""
    del pad
    return _race_forward(q, k, v, w, p, want_state=want_state)


@_on_q_device
def race_backward(q, k, v, w, d_o, p: SketchParams, state=None, *, inplace: bool = False, pad: bool = True):
    """(dq, dk, dv).  ``state`` from race_forward avoids re-aggregating K/V.

    ``inplace=True`` writes the gradients over q, k, v (which must be contiguous) and returns
    those tensors: the inputs are dead after the backward, so the layer holds 4 instead of 7
    N x d tensors (race_bwd allows dq, dk, dv to alias q, k, v).  ``pad`` is ignored."""
    del pad
    return _race_backward(q, k, v, w, d_o, p, state=state, inplace=inplace)


class RaceAttentionFunction(torch.autograd.Function):
    """Autograd wrapper: saves the tiny bucket-table state instead of phi."""

    @staticmethod
    def forward(ctx, q, k, v, w, hyperplanes, tables, beta, causal, normalize, pad=True):
        p = SketchParams(hyperplanes, tables, beta, causal, normalize)
        o, den, state = race_forward(q, k, v, w, p, want_state=True, pad=pad)
        ctx.p = p
        ctx.pad = pad
        ctx.save_for_backward(q, k, v, w, state)
        ctx.mark_non_differentiable(den)
        return o, den

    @staticmethod
    def backward(ctx, d_o, d_den):
        q, k, v, w, state = ctx.saved_tensors
        dq, dk, dv = race_backward(q, k, v, w, d_o, ctx.p, state=state, pad=ctx.pad)
        return dq, dk, dv, None, None, None, None, None, None, None


def race_attention_torch(q, k, v, w, p: SketchParams, pad: bool = True):
    """Differentiable RACE attention on ``[..., N, d]`` CUDA tensors; returns O."""
    o, _ = RaceAttentionFunction.apply(q, k, v, w, p.hyperplanes, p.tables, float(p.beta),
                                       bool(p.causal), bool(p.normalize), bool(pad))
    return o
