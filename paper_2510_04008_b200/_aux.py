"""Host glue for the validation-side kernels of include/race_aux.h.

Moves numpy / torch matrices to the GPU without changing their precision
(float64 stays float64: those kernels compute in fp64, like the reference),
calls the C-ABI and hands results back in the caller's container.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .functional import _stream, _vp

_CODES = {torch.float32: _lib.RACE_F32, torch.bfloat16: _lib.RACE_BF16, torch.float64: _lib.RACE_F64}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(x, dev: torch.device | None = None) -> torch.Tensor:
    """Contiguous device copy of a 2-D matrix, float32 / bfloat16 / float64 kept as is."""
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        t = x.to(dev)
        if t.dtype not in _CODES:
            t = t.to(torch.float64)
        return t.contiguous()
    a = np.asarray(x)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def code(t: torch.Tensor) -> int:
    return _CODES[t.dtype]


def same_dtype(*ts: torch.Tensor) -> list[torch.Tensor]:
    """Promote to one element type (float64 wins, then float32)."""
    dts = {t.dtype for t in ts}
    if len(dts) == 1:
        return list(ts)
    tgt = torch.float64 if torch.float64 in dts else torch.float32
    return [t.to(tgt) for t in ts]


def back(t: torch.Tensor, like, dtype=None):
    """t in the container of `like` (numpy -> numpy of `dtype` or like's dtype; torch -> torch)."""
    if isinstance(like, torch.Tensor):
        return t.to(device=like.device, dtype=dtype or like.dtype)
    arr = t.detach().cpu().numpy()
    dt = dtype if dtype is not None else np.asarray(like).dtype
    if dt not in (np.float32, np.float64):
        dt = np.float64
    return arr.astype(dt, copy=False)


def w64(w, dev: torch.device) -> torch.Tensor:
    """Hyperplanes as a contiguous float64 device tensor ([..., d] -> [rows, d])."""
    if isinstance(w, torch.Tensor):
        t = w.to(device=dev, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(w, dtype=np.float64))).to(dev)
    return t.reshape(-1, t.shape[-1]).contiguous()


def lib():
    return _lib.lib()


def check(rc: int, what: str) -> None:
    _lib.check(rc, what)


__all__ = ["back", "check", "code", "device", "lib", "same_dtype", "to_dev", "w64", "_stream", "_vp"]
