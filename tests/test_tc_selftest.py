"""Device check of the tcgen05 operand layouts the fast path relies on.

libtc_selftest.so builds each canonical UMMA layout (K-/MN-major, SW128 /
SW64 / SW32) in shared memory, runs one tcgen05.mma chain and reads D back
from TMEM; the result must equal A @ B^T (bf16 products are exact in fp32).
"""

from __future__ import annotations

import ctypes
import os

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu
LIB = os.path.join(ROOT, "paper_2510_04008_b200", "libtc_selftest.so")

# (N, K, a_mn, b_mn, a_sw, b_sw): the operand pairings of the fast-path kernels
COMBOS = [
    (16, 128, 0, 0, 128, 128),   # projection: X tile (TMA SW128) x W' (K-major)
    (32, 128, 1, 1, 128, 64),    # state update: V^T (MN-major) x Phi (MN-major SW64)
    (128, 32, 0, 0, 64, 64),     # Phi_q Phi_k^T and Phi_q x S-operand
    (128, 128, 0, 1, 128, 128),  # P~ x V (B MN-major SW128)
    (128, 16, 0, 1, 32, 128),    # dproj x W (bwd)
    (128, 128, 0, 0, 128, 128),  # dO V^T (bwd)
    (32, 128, 1, 1, 128, 128),   # dO^T x Phi~ with Phi in SW128 rows
    (64, 64, 1, 0, 128, 128),
    (128, 128, 0, 1, 0, 128),    # P~ (A from TMEM) x V (causal forward, tcgen05.mma [d], [a], b)
    (128, 32, 0, 0, 0, 64),      # A from TMEM x K-major SW64 B
]


@pytest.mark.parametrize("combo", COMBOS, ids=lambda c: "N%d_K%d_a%s%s_b%s%d" % (
    c[0], c[1], "MN" if c[2] else "K", c[4] or "tmem", "MN" if c[3] else "K", c[5]))
def test_umma_layouts(combo):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    n, k, a_mn, b_mn, a_sw, b_sw = combo
    lib = ctypes.CDLL(LIB)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(n * 1000 + k)
    a = torch.randn(128, k, generator=g, device=dev).to(torch.bfloat16)
    b = torch.randn(n, k, generator=g, device=dev).to(torch.bfloat16)
    d = torch.full((128, n), float("nan"), device=dev)
    rc = lib.tc_selftest_gemm(128, n, k, a_mn, b_mn, a_sw, b_sw, ctypes.c_void_p(a.data_ptr()),
                              ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(d.data_ptr()),
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ref = a.double() @ b.double().T
    err = (d.double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("ts", [0, 1], ids=["smemA", "tmemA"])
@pytest.mark.parametrize("nk", [(128, 128), (32, 64), (16, 128)], ids=lambda x: "N%dK%d" % x)
def test_umma_m64_two_chains_share_columns(nk, ts):
    """Two M=64 accumulators in the same TMEM columns at DP offsets 0 and 16 (half-subpartition
    layout, CUTLASS TmemAllocMode::Interleaved), A from smem or from TMEM at the chain's offset."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    n, k = nk
    lib = ctypes.CDLL(LIB)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(n * 7 + k + ts)
    a = torch.randn(128, k, generator=g, device=dev).to(torch.bfloat16)
    b = torch.randn(n, k, generator=g, device=dev).to(torch.bfloat16)
    d = torch.full((128, n), float("nan"), device=dev)
    rc = lib.tc_selftest_m64(n, k, ts, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                             ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ref = a.double() @ b.double().T
    err = (d.double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("lane_off", [0, 16])
@pytest.mark.parametrize("shape", [64, 128, 256])
def test_tmem_ld16_layout_probe(shape, lane_off, tmp_path):
    """Record (and check self-consistency of) what tcgen05.ld.16x{64,128,256}b returns per thread:
    every value is a (dp, col) of the warp's quarter at DP offset lane_off..lane_off+15, every cell
    of those 16 DPs x 64 columns... read exactly once.  The mapping is logged for the kernels."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    lib = ctypes.CDLL(LIB)
    out = torch.zeros(128 * 8, dtype=torch.int32, device="cuda")
    assert lib.tc_ld16_probe(shape, lane_off, ctypes.c_void_p(out.data_ptr()),
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    torch.cuda.synchronize()
    v = out.view(4, 32, 8).cpu()
    dp, col = v // 1024, v % 1024
    lines = []
    for w in range(4):
        base = 32 * w + lane_off
        assert bool(((dp[w] >= base) & (dp[w] < base + 16)).all()), (w, dp[w])
        cells = {(int(a), int(b)) for a, b in zip(dp[w].flatten(), col[w].flatten())}
        assert len(cells) == 32 * 8  # no cell twice
    for t in range(32):
        lines.append(f"t{t}: " + " ".join(f"({int(dp[0, t, j]) - lane_off},{int(col[0, t, j])})" for j in range(8)))
    path = os.environ.get("RACE_PARITY_LOG")
    if path:
        with open(path.replace(".jsonl", f"_ld16x{shape}b_off{lane_off}.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
