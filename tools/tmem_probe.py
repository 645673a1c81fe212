"""TMEM read bandwidth and tcgen05.mma issue rates on this B200 (libtc_selftest.so probes).

    python tools/tmem_probe.py

tcgen05.ld: bytes per SM-cycle for 4..16 warps doing two 32-column loads per iteration;
tcgen05.mma: cycles per instruction of M = 128, K = 16 bf16 MMAs with N in {16, 32, 128}, A from shared
memory (SS) or from TMEM (TS) -- the shapes of the causal kernels' Z / S / dS / dV MMAs."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2510_04008_b200", "libtc_selftest.so"))
dev = torch.device("cuda", 0)
out = torch.zeros(256, dtype=torch.int64, device=dev)
s = torch.cuda.current_stream().cuda_stream
mhz = 1965.0
print("tcgen05.ld 32x32b.x32 (two per iteration), 1 CTA and 148 CTAs:")
for ctas in (1, 148):
    for warps in (4, 8, 12, 16):
        iters = 2000
        assert lib.tc_tmem_ld_rate(ctas, warps, iters, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s)) == 0
        torch.cuda.synchronize()
        cyc = out[:ctas].double().mean().item()
        nbytes = warps * iters * 2 * 32 * 32 * 4
        print(f"  ctas {ctas:3d} warps {warps:2d}: {nbytes / cyc:6.1f} B/cycle per SM ({cyc / iters:7.1f} cycles per iteration)")
print("tcgen05.mma M=128 K=16 bf16, cycles per instruction (64 per commit):")
for n in (16, 32, 128):
    for ts in (0, 1):
        assert lib.tc_mma_rate(n, ts, 64, 6, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s)) == 0
        torch.cuda.synchronize()
        cyc = out[0].item()
        print(f"  N={n:3d} {'TS' if ts else 'SS'}: {cyc / 64:6.1f} cycles per MMA (commit round {cyc} cycles)")
