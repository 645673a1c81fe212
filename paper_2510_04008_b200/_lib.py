"""ctypes binding of the C-ABI in ``include/race_b200.h``.

The shared library ``librace_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``).
There is deliberately no fallback: if the library is missing or a call fails,
this module raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# RACE_LIB_PATH lets a benchmark A/B two in-tree builds of the same library
LIB_PATH = os.environ.get("RACE_LIB_PATH") or os.path.join(_HERE, "librace_b200.so")

ABI_VERSION = 1
RACE_OK, RACE_EBADSHAPE, RACE_EUNSUPPORTED, RACE_ECUDA = 0, 1, 2, 3
RACE_F32, RACE_BF16 = 0, 1
COMBINE_TOTAL, COMBINE_PREFIX, COMBINE_SUFFIX = 0, 1, 2

# Every symbol include/race_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "race_abi_version", "race_last_error", "race_launch_count", "race_fast_path", "race_segments",
    "race_workspace_bytes", "race_state_elems", "race_fwd", "race_bwd",
    "race_kside_partials", "race_combine", "race_fwd_readout", "race_fwd_causal",
    "race_bwd_qside", "race_bwd_kside", "race_bwd_causal_q", "race_bwd_causal_k",
    "race_kside_partials_rows", "race_fwd_causal_krows", "race_group_plan",
    "race_fwd_layout", "race_bwd_layout",
)


class RaceDesc(ctypes.Structure):
    """Mirror of ``race_desc_t``."""

    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("batch_heads", ctypes.c_int64),
        ("heads", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("dim", ctypes.c_int32),
        ("dim_v", ctypes.c_int32),
        ("hyperplanes", ctypes.c_int32),
        ("tables", ctypes.c_int32),
        ("beta", ctypes.c_float),
        ("causal", ctypes.c_int32),
        ("normalize", ctypes.c_int32),
        ("w_per_head", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 4),
    ]


class RaceStride(ctypes.Structure):
    """Mirror of ``race_stride_t``: element strides (token, head, batch); token 0 = contiguous."""

    _fields_ = [("token", ctypes.c_int64), ("head", ctypes.c_int64), ("batch", ctypes.c_int64)]


class RaceLayout(ctypes.Structure):
    """Mirror of ``race_layout_t``."""

    _fields_ = [(n, RaceStride) for n in ("q", "k", "v", "o", "d_o", "dq", "dk", "dv")]


class RaceError(RuntimeError):
    """A CUDA-side failure (status RACE_ECUDA)."""


class RaceUnsupported(ValueError):
    """A valid configuration the CUDA path does not implement (RACE_EUNSUPPORTED)."""


_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_SIGS = {
    "race_abi_version": ([], ctypes.c_int),
    "race_last_error": ([], ctypes.c_char_p),
    "race_launch_count": ([], ctypes.c_int64),
    "race_fast_path": ([_P], ctypes.c_int),
    "race_segments": ([_P, _P, _P], ctypes.c_int),
    "race_group_plan": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "race_workspace_bytes": ([_P, _P], ctypes.c_int),
    "race_state_elems": ([_P, _P], ctypes.c_int),
    "race_fwd": ([_P] * 10, ctypes.c_int),
    "race_bwd": ([_P] * 12, ctypes.c_int),
    "race_kside_partials": ([_P] * 7, ctypes.c_int),
    "race_combine": ([_P, ctypes.c_int32, _P, _P, _P, _P], ctypes.c_int),
    "race_fwd_readout": ([_P] * 8, ctypes.c_int),
    "race_fwd_causal": ([_P] * 11, ctypes.c_int),
    "race_bwd_qside": ([_P] * 9, ctypes.c_int),
    "race_bwd_kside": ([_P] * 9, ctypes.c_int),
    "race_bwd_causal_q": ([_P] * 14, ctypes.c_int),
    "race_bwd_causal_k": ([_P] * 14, ctypes.c_int),
    "race_kside_partials_rows": ([_P] * 8, ctypes.c_int),
    "race_fwd_causal_krows": ([_P] * 11, ctypes.c_int),
    "race_fwd_layout": ([_P] * 11, ctypes.c_int),
    "race_bwd_layout": ([_P] * 13, ctypes.c_int),
}
_I32, _I64, _F64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
# include/race_aux.h (validation-side GPU functions; float64 compute)
RACE_F64 = 2
AUX_SIGS = {
    "race_aux_row_normalize": ([_I32, _I64, _I32, _P, _P, _P, _P], ctypes.c_int),
    "race_aux_soft_features": ([_I32, _I64, _I32, _P, _P, _I32, _I32, _F64, _I32, _P, _P], ctypes.c_int),
    "race_aux_hard_hash": ([_I32, _I64, _I32, _P, _P, _I32, _I32, _I32, _P, _P], ctypes.c_int),
    "race_aux_feature_gram": ([_I64, _I64, _I32, _P, _P, _F64, _P, _P], ctypes.c_int),
    "race_aux_hard_workspace_bytes": ([_I32, _I32, _I32], ctypes.c_size_t),
    "race_aux_hard_attention": ([_I32, _I64, _I32, _P, _P, _P, _I32, _I32, _P, _P, _P, _P], ctypes.c_int),
    "race_aux_angular_kernel": ([_I32, _I64, _I64, _I32, _P, _P, _I32, _P, _P], ctypes.c_int),
    "race_aux_angular_fwd": ([_I32, _I64, _I32, _I32, _P, _P, _P, _I32, _I32, _P, _P, _P], ctypes.c_int),
    "race_aux_angular_bwd": ([_I32, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P],
                             ctypes.c_int),
}
AUX_EXPORTS = tuple(AUX_SIGS)
_SIGS.update(AUX_SIGS)


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()'). "
                    "There is no CPU fallback.")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = res
            if handle.race_abi_version() != ABI_VERSION:
                raise RuntimeError("librace_b200.so ABI version mismatch; rebuild it")
            _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc == RACE_OK:
        return
    msg = f"{what}: {lib().race_last_error().decode(errors='replace')}"
    if rc == RACE_EBADSHAPE:
        raise ValueError(msg)
    if rc == RACE_EUNSUPPORTED:
        raise RaceUnsupported(msg)
    raise RaceError(msg)


def make_desc(*, dtype: int, batch_heads: int, heads: int, n: int, dim: int, dim_v: int,
              hyperplanes: int, tables: int, beta: float, causal: bool, normalize: bool,
              w_per_head: bool) -> RaceDesc:
    d = RaceDesc()
    d.abi_version = ABI_VERSION
    d.dtype = dtype
    d.batch_heads = batch_heads
    d.heads = heads
    d.n = n
    d.dim = dim
    d.dim_v = dim_v
    d.hyperplanes = hyperplanes
    d.tables = tables
    d.beta = beta
    d.causal = 1 if causal else 0
    d.normalize = 1 if normalize else 0
    d.w_per_head = 1 if w_per_head else 0
    return d


def ref(desc: RaceDesc) -> ctypes.c_void_p:
    return ctypes.cast(ctypes.pointer(desc), ctypes.c_void_p)


def segments(desc: RaceDesc) -> tuple[int, int]:
    nseg, seg = ctypes.c_int64(), ctypes.c_int64()
    check(lib().race_segments(ref(desc), ctypes.byref(nseg), ctypes.byref(seg)), "race_segments")
    return nseg.value, seg.value


def workspace_bytes(desc: RaceDesc) -> int:
    b = ctypes.c_size_t()
    check(lib().race_workspace_bytes(ref(desc), ctypes.byref(b)), "race_workspace_bytes")
    return b.value


def state_elems(desc: RaceDesc) -> int:
    e = ctypes.c_int64()
    check(lib().race_state_elems(ref(desc), ctypes.byref(e)), "race_state_elems")
    return e.value


def fast_path(desc: RaceDesc) -> bool:
    return bool(lib().race_fast_path(ref(desc)))


def group_plan(desc: RaceDesc) -> dict:
    """{passes, tables_per_pass, corner_bits, fast}: how race_fwd / race_bwd split this sketch."""
    n, t, c, f = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    check(lib().race_group_plan(ref(desc), ctypes.byref(n), ctypes.byref(t), ctypes.byref(c), ctypes.byref(f)),
          "race_group_plan")
    return {"passes": n.value, "tables_per_pass": t.value, "corner_bits": c.value, "fast": bool(f.value)}
