#!/usr/bin/env python
"""RACE attention layer fwd+bwd throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the metric's config): causal RACE
attention layer, B=1, H=4, d=dv=128, N=131072 tokens per GPU, bf16, sketch
P=2, L=2, M=1, beta=8 (the reference defaults, ra/cli.py:71-76).  One step =
forward + backward of the whole layer over synthetic Q, K, V, dO resident in
HBM (512 MiB per step > 126 MB L2, so no L2 flush is needed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU over NCCL: each rank owns an
N-token slice of one N*world-token sequence (weak scaling); the bucket tables
cross NVLink through the causal exclusive scan (sharded.py).

--impl reference times the reference's CPU algorithm (the numpy port in
oracle/, since the reference is pure Python and cannot travel to the box) on
the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd tokens/s, RACE layer B=1 H=4 d=128; max context at 1/8 B200"
HEADS, DIM, P_, L_, BETA = 4, 128, 2, 2, 8.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=131072, help="tokens per GPU")
    ap.add_argument("--noncausal", action="store_true")
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-max-context", action="store_true")
    ap.add_argument("--n-total", type=int, default=0,
                    help="BASELINE configs[3] mode: tokens of the whole sharded sequence (strong scaling; "
                         "each rank owns n_total / world); default: --n tokens per GPU (weak scaling)")
    ap.add_argument("--sharded-64m-total", type=int, default=64 << 20,
                    help="sequence length of the sharded configs[3] run appended to multi-GPU lines")
    args = ap.parse_args()
    if args.n_total:
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        args.n = args.n_total // world
    return args


def _config(args, world):
    return {
        "workload": f"{'non-causal' if args.noncausal else 'causal'} RACE attention layer fwd+bwd, "
                    f"B=1 H={HEADS} d={DIM} N={args.n * world} ({args.n} per GPU), {args.dtype}",
        "batch": 1, "heads": HEADS, "head_dim": DIM, "seq_len": args.n * world, "tokens_per_gpu": args.n,
        "P": P_, "L": L_, "M": 1, "beta": BETA, "causal": not args.noncausal,
        "parallelism": f"sequence-sharded x{world}" if world > 1 else "single GPU",
        "scaling_mode": "strong (fixed total sequence, --n-total)" if args.n_total else "weak (fixed tokens per GPU)",
        "l2": "inputs (Q,K,V,dO = 4 x H*N*d) exceed the 126 MB L2; no flush needed",
    }


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (numpy port) on the host cores
# ---------------------------------------------------------------------------
def cpu_reference_step(n_sample, causal, seed=0):
    import numpy as np

    from oracle import race_oracle as ro

    per_head = ro.head_inputs(seed, n_sample, DIM, HEADS, np.float32)
    t0 = time.perf_counter()
    for h, (q, k, v, g) in enumerate(per_head):
        w = ro.stacked_hyperplanes(seed + h, P_, L_, 1, DIM)  # seed + h per head (ra/bench.py:175)
        ro.forward(q, k, v, w, BETA, causal)
        ro.vjp(q, k, v, w, BETA, g, causal)
    return time.perf_counter() - t0


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        blas = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(blas) if blas else os.cpu_count()
    except Exception:
        return os.cpu_count()


_BLAS_LIMIT = None


def _host_facts():
    """CPU model, core count, numpy / BLAS versions of this host."""
    import platform

    import numpy as np

    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info

        blas = [{"api": i.get("internal_api"), "version": i.get("version"), "threads": i.get("num_threads")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def _reference_package():
    """The UNMODIFIED reference from baseline/_ref (pip-installed there), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "race_attention")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import race_attention

        return race_attention
    except Exception:
        return None


def reference_step(ra, n_sample, causal, seed=0):
    """One fwd+bwd of the H=4 layer through the reference's public API, exactly as its own
    benchmark runs a RACE row (ra/bench.py:172-178: per head race_attention + race_attention_vjp with
    seed + head), on inputs drawn as ra/bench.py:161-169 draws them (float32, ra/bench.py:197)."""
    import dataclasses

    import numpy as np

    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(n_sample,)))
    per_head = []
    for _ in range(HEADS):
        q, k, v, g = (rng.standard_normal((n_sample, DIM)).astype(np.float32) for _ in range(4))
        per_head.append((ra.AttnInputs(q, k, v), g))
    sketch = ra.SketchConfig(hyperplanes=P_, tables=L_, beta=BETA, seed=0, causal=causal)
    t0 = time.perf_counter()
    for h, (inp, g) in enumerate(per_head):
        cfg = dataclasses.replace(sketch, seed=sketch.seed + h)
        ra.race_attention(inp, cfg)
        ra.race_attention_vjp(inp, cfg, g)
    return time.perf_counter() - t0


def run_reference(args, world, rank):
    if rank != 0:
        return
    # torchrun pins OMP_NUM_THREADS=1 per worker; the reference arm (rank 0 alone) gets every host core
    try:
        import numpy  # noqa: F401  (loads BLAS so threadpoolctl can see it)
        from threadpoolctl import threadpool_limits

        global _BLAS_LIMIT
        _BLAS_LIMIT = threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")  # held for the run
    except Exception:
        pass
    causal = not args.noncausal
    n_sample = 4096 if causal else 16384
    ra = _reference_package()
    if ra is not None:
        kind, what = "reference", "the unmodified reference package (baseline/_ref, race_attention 0.1.0) public API"
        fn = lambda i: reference_step(ra, n_sample, causal, seed=i)  # noqa: E731
    else:
        kind, what = "port", "oracle/race_oracle.py (numpy restatement; baseline/_ref not installed)"
        fn = lambda i: cpu_reference_step(n_sample, causal, seed=i)  # noqa: E731
    times = []
    for i in range(args.warmup + args.steps):
        dt = fn(i)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = n_sample * len(times) / tot
    cores = cpu_threads()
    config = _config(args, world)
    config["timed_sample_tokens"] = n_sample
    config["sample_note"] = (f"each step times a {n_sample}-token sequence of the same layer (CPU RACE cost is "
                             f"linear in N: the reference's own bench gives equal tokens/s at 4096 and 131072, "
                             f"BASELINE.md section 2); the declared N would take minutes per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) Q,K,V,dO (ra/bench.py:161-169 order)", "config": config,
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": f"{n_sample}-token {'causal' if causal else 'non-causal'} fwd+bwd, "
                                   f"H={HEADS}, d={DIM}, f32, per step, through {what}"},
        "host": _host_facts(),
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        self.thread.join(timeout=1)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# max context (BASELINE configs[2]): largest N whose fwd+bwd runs on this GPU
# ---------------------------------------------------------------------------
def max_context(dev, causal, dtype, inplace=False):
    """Largest N (multiple of 2^20) whose RACE layer fwd+bwd (B=1, H=4, d=128)
    completes on one GPU with every tensor resident in HBM, and its speed.

    allocating: Q, K, V, dO, O, dQ, dK, dV all live (~8.4 KB per token in bf16
    with den / sketch rows / normaliser terms).  inplace: the layer as a
    training step runs it -- O is handed on after the forward (dropped here)
    and the backward writes dQ, dK, dV over the dead Q, K, V (race_bwd allows
    the aliasing), so the peak is the forward's Q, K, V, dO, O (~5.7 KB per
    token).  Starts from the free-memory estimate and steps down 1 Mi tokens
    on each out-of-memory."""
    import torch

    import paper_2510_04008_b200 as rb

    cfg = rb.SketchConfig(hyperplanes=P_, tables=L_, beta=BETA, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, HEADS, DIM).to(dev)
    p = cfg.params()
    e = 2 if dtype == torch.bfloat16 else 4
    per_token = HEADS * ((5 if inplace else 8) * DIM * e + (170 if inplace else 96))
    free, _ = torch.cuda.mem_get_info(dev)
    n = int(free * 0.97 / per_token) >> 20 << 20
    gen = torch.Generator(device=dev).manual_seed(7)

    def step(q, k, v, g):
        o, den, st = rb.race_forward(q, k, v, w, p)
        if inplace:
            del o
            grads = rb.race_backward(q, k, v, w, g, p, state=st, inplace=True)
        else:
            grads = rb.race_backward(q, k, v, w, g, p, state=st)
            del o
        del den, st
        return grads

    q = k = v = g = grads = None
    while n >= 1 << 20:
        tensors = []
        try:
            shape = (1, HEADS, n, DIM)
            q, k, v, g = (torch.randn(shape, generator=gen, device=dev, dtype=dtype) for _ in range(4))
            tensors = [q, k, v, g]
            grads = step(q, k, v, g)  # warm-up (in-place: q, k, v now hold gradients)
            del grads
            if inplace:
                for t in (q, k, v):
                    t.normal_(generator=gen)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            grads = step(q, k, v, g)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            ok = bool(torch.isfinite(grads[0][0, 0, -1].float()).all())
            del q, k, v, g, tensors, grads
            torch.cuda.empty_cache()
            return {"tokens": n, "causal": causal, "dtype": "bf16" if e == 2 else "f32",
                    "mode": "inplace" if inplace else "allocating", "ms_fwd_bwd": ms,
                    "tokens_per_s": n / (ms / 1e3), "finite": ok, "hbm_gb_used_est": round(n * per_token / 1e9, 1)}
        except torch.cuda.OutOfMemoryError:
            q = k = v = g = grads = None
            tensors = []
            torch.cuda.empty_cache()
            n -= 1 << 20
    return {"tokens": 0, "causal": causal, "error": "nothing fits"}


def scale_sweep(dev, dtype, sizes=(1 << 20, 1 << 21, 1 << 22, 1 << 23, 12 << 20, 1 << 24)):
    """BASELINE configs[2]: fwd+bwd tokens/s of the H=4, d=128 layer for N from 1 Mi to
    16 Mi tokens (1, 2, 4, 8, 12, 16 Mi) on one GPU, causal and non-causal (inputs resident in HBM, 2 timed reps)."""
    import torch

    import paper_2510_04008_b200 as rb

    out = []
    gen = torch.Generator(device=dev).manual_seed(5)
    for causal in (True, False):
        cfg = rb.SketchConfig(hyperplanes=P_, tables=L_, beta=BETA, seed=0, causal=causal)
        w = rb.head_hyperplanes(cfg, HEADS, DIM).to(dev)
        p = cfg.params()
        for n in sizes:
            try:
                q, k, v, g = (torch.randn((1, HEADS, n, DIM), generator=gen, device=dev, dtype=dtype) for _ in range(4))
                o, den, st = rb.race_forward(q, k, v, w, p)
                rb.race_backward(q, k, v, w, g, p, state=st)
                del o, den, st
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record()
                for _ in range(2):
                    o, den, st = rb.race_forward(q, k, v, w, p)
                    rb.race_backward(q, k, v, w, g, p, state=st)
                    del o, den, st
                ev[1].record()
                torch.cuda.synchronize()
                ms = ev[0].elapsed_time(ev[1]) / 2
                out.append({"tokens": n, "causal": causal, "ms_fwd_bwd": round(ms, 3),
                            "tokens_per_s": n / (ms / 1e3)})
                del q, k, v, g
            except torch.cuda.OutOfMemoryError:
                out.append({"tokens": n, "causal": causal, "error": "out of memory"})
            torch.cuda.empty_cache()
    return out


def sketch_sweep(dev, dtype, n=131072):
    """SURVEY 8(d)'s optional sketch sweep: the headline layer with larger sketches.  One tcgen05
    pass covers F <= 8 buckets; larger bf16 sketches run as several tcgen05 passes (table groups for
    P <= 3, corner groups for P = 4, 5; race_group_plan), the rest on the CUDA-core kernels."""
    import torch

    import paper_2510_04008_b200 as rb
    from paper_2510_04008_b200 import _lib
    from paper_2510_04008_b200.functional import Problem

    out = []
    gen = torch.Generator(device=dev).manual_seed(9)
    q, k, v, g = (torch.randn((1, HEADS, n, DIM), generator=gen, device=dev, dtype=dtype) for _ in range(4))
    for P, L in ((2, 2), (3, 1), (1, 4), (2, 4), (2, 8), (3, 4), (4, 4), (5, 2)):
        cfg = rb.SketchConfig(hyperplanes=P, tables=L, beta=BETA, seed=0, causal=True)
        w = rb.head_hyperplanes(cfg, HEADS, DIM).to(dev)
        p = cfg.params()
        plan = _lib.group_plan(Problem(q, k, v, w, p).desc)
        fast = plan["fast"]
        for _ in range(3):
            o, den, st = rb.race_forward(q, k, v, w, p)
            rb.race_backward(q, k, v, w, g, p, state=st)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(3):
            o, den, st = rb.race_forward(q, k, v, w, p)
            rb.race_backward(q, k, v, w, g, p, state=st)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 3
        out.append({"P": P, "L": L, "F": L << P, "causal": True, "tokens": n, "fast_path": bool(fast),
                    "passes": plan["passes"],
                    "ms_fwd_bwd": round(ms, 3), "tokens_per_s": n / (ms / 1e3)})
    return out


def gpt_train_step(dev, steps=5, warmup=3):
    """BASELINE configs[4]: one training step (fwd + bwd + fused AdamW, bf16 autocast) of a
    6-layer, d_model=768, 12-head GPT with causal RACE attention in every layer, on a
    16K-token synthetic sequence (random init, random tokens).  Device-timed."""
    import torch

    from paper_2510_04008_b200.gpt import GPTConfig, RaceGPT, train_step

    torch.manual_seed(0)
    cfg = GPTConfig()
    model = RaceGPT(cfg).to(dev)
    opt = torch.optim.AdamW(model.parameters(), lr=3e-4, fused=True)
    g = torch.Generator(device=dev).manual_seed(3)
    idx = torch.randint(0, cfg.vocab, (1, cfg.seq_len), device=dev, generator=g)
    tgt = torch.roll(idx, -1, dims=1)
    for _ in range(warmup):
        train_step(model, opt, idx, tgt)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(steps):
        loss = train_step(model, opt, idx, tgt)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    return {"model": "RaceGPT 6 layers, d_model 768, 12 heads (d=64 heads on the tcgen05 kernels at their own width, q, k, v read in place from the projection)",
            "params_M": round(sum(p.numel() for p in model.parameters()) / 1e6, 1), "seq_len": cfg.seq_len,
            "batch": 1, "ms_per_step": round(ms, 3), "tokens_per_s": cfg.seq_len / (ms / 1e3),
            "loss": float(loss), "data": "synthetic random tokens", "dtype": "bf16 autocast, fp32 master, cross-entropy on the bf16 logits (fp32 reductions)"}


# ---------------------------------------------------------------------------
# our GPU path
# ---------------------------------------------------------------------------
# algorithmic bytes per token-head of each kernel (e = element bytes)
def kernel_bytes(e, causal):
    """(compulsory, intermediate) bytes per token-head of each launched kernel.

    compulsory = the kernel's share of the layer's N x d tensors and den (Q, K, V, O, dO
    read / O, dQ, dK, dV, den written); intermediate = what our decomposition adds: the 64-byte causal
    sketch row per token (16 fp32: q and k projections + norms, which let each backward pass skip
    one of the N x d operands) and the 1/D, -rho/D normaliser terms.  Re-reads of an input by a
    second kernel (V in the causal forward) count as that kernel's compulsory input."""
    d = dv = DIM
    rows = 64
    if causal:
        return {"kside_partials": ((d + dv) * e, rows // 2),                    # read K, V; write k half rows
                "fwd_causal": ((d + dv) * e + dv * e + 4, rows + rows // 2),    # read Q, V, rows; write O, den, q half
                "bwd_causal_q": ((d + 2 * dv) * e + d * e, rows + 8),           # read Q, V, dO, rows; write dQ, rden, gden
                "bwd_causal_k": ((d + 2 * dv) * e + (d + dv) * e, rows + 8)}    # read K, V, dO, rows, rden, gden; write dK, dV
    return {"kside_partials": ((d + dv) * e, 0), "fwd_readout": (d * e + dv * e + 4, 0),
            "bwd_qside": ((d + dv) * e + d * e, 0), "bwd_kside": (2 * (d + dv) * e, 0)}


def sharded_run(dev, world, n_total, dtype, causal=True, steps=3):
    """BASELINE configs[3]: one causal fwd+bwd of a B=1, H=4, d=128 layer over an n_total-token
    sequence sequence-sharded across the world (rank r owns tokens [r n/G, (r+1) n/G)), bucket
    tables exchanged by all_gather + fixed-order exclusive prefix / suffix (sharded.py).  Device
    time, max over ranks.  Every rank first reserves the step's memory and the ranks agree on it
    (all_reduce of an OOM flag) before any collective, so an out-of-memory rank cannot strand
    the others in a collective."""
    import torch
    import torch.distributed as dist

    import paper_2510_04008_b200 as rb
    from paper_2510_04008_b200.sharded import TorchDistComm, shard_bounds, sharded_backward, sharded_forward

    rank = dist.get_rank()
    lo, hi = shard_bounds(n_total, world, rank)
    n = hi - lo
    e = 2 if dtype == torch.bfloat16 else 4
    cfg = rb.SketchConfig(hyperplanes=P_, tables=L_, beta=BETA, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, HEADS, DIM).to(dev)
    p = cfg.params()
    comm = TorchDistComm()
    bad = torch.zeros(1, device=dev)
    tensors = []
    try:
        gen = torch.Generator(device=dev).manual_seed(77 + rank)
        tensors = [torch.randn((1, HEADS, n, DIM), generator=gen, device=dev, dtype=dtype) for _ in range(4)]
        # the step's own allocations (O, dQ, dK, dV + den / state / workspace) reserved up front
        reserve = torch.empty(int(n * HEADS * (4 * DIM * e + 160)), dtype=torch.uint8, device=dev)
        del reserve
    except torch.cuda.OutOfMemoryError:
        bad.fill_(1)
    dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    if bad.item():
        del tensors
        torch.cuda.empty_cache()
        return {"tokens_total": n_total, "world": world, "tokens_per_gpu": n, "error": "out of memory on a rank"}
    q, k, v, g = tensors

    def step():
        o, den, st = sharded_forward(q, k, v, w, p, comm=comm)
        del o
        return sharded_backward(q, k, v, w, g, p, st, comm=comm)

    step()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(steps):
        grads = step()
    ev[1].record()
    torch.cuda.synchronize()
    ms = torch.tensor([ev[0].elapsed_time(ev[1]) / steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    finite = torch.tensor([float(all(bool(torch.isfinite(t[0, :, -1].float()).all()) for t in grads))], device=dev)
    dist.all_reduce(finite, op=dist.ReduceOp.MIN)
    del q, k, v, g, tensors, grads
    torch.cuda.empty_cache()
    msf = float(ms.item())
    return {"tokens_total": n_total, "world": world, "tokens_per_gpu": n, "causal": causal,
            "ms_fwd_bwd": round(msf, 3), "tokens_per_s": n_total / (msf / 1e3), "finite": bool(finite.item()),
            "exchange": "all_gather of H x F x (dv+1) fp32 totals + fixed-order exclusive prefix / suffix"}


def sharded_max_context(dev, world, dtype):
    """Largest total sequence (multiple of world x 1 Mi) whose sharded causal fwd+bwd runs, stepping
    down 1 Mi tokens per rank from the free-memory estimate (the ranks agree on each attempt)."""
    import torch
    import torch.distributed as dist

    e = 2 if dtype == torch.bfloat16 else 4
    free, _ = torch.cuda.mem_get_info(dev)
    per = torch.tensor([int(free * 0.95 / (HEADS * (8 * DIM * e + 160))) >> 20], device=dev)
    dist.all_reduce(per, op=dist.ReduceOp.MIN)
    m = int(per.item())
    while m >= 1:
        r = sharded_run(dev, world, (m << 20) * world, dtype, steps=1)
        if "error" not in r:
            return r
        m -= 1
    return {"tokens_total": 0, "error": "nothing fits"}


def run_ours(args, world, rank, local_rank):
    import torch

    import paper_2510_04008_b200 as rb
    from paper_2510_04008_b200 import _lib
    from paper_2510_04008_b200.functional import Problem, _stream, _vp
    from paper_2510_04008_b200.sharded import TorchDistComm, sharded_backward, sharded_forward

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    e = 2 if dtype == torch.bfloat16 else 4
    causal = not args.noncausal
    n = args.n
    cfg = rb.SketchConfig(hyperplanes=P_, tables=L_, beta=BETA, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, HEADS, DIM).to(dev)
    p = cfg.params()
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    shape = (1, HEADS, n, DIM)
    q, k, v, g = (torch.randn(shape, generator=gen, device=dev, dtype=torch.float32).to(dtype) for _ in range(4))
    dist = None
    if world > 1:
        import torch.distributed as dist
    comm = TorchDistComm() if world > 1 else None

    def step():
        if world > 1:
            o, den, st = sharded_forward(q, k, v, w, p, comm=comm)
            return sharded_backward(q, k, v, w, g, p, st, comm=comm)
        o, den, st = rb.race_forward(q, k, v, w, p)
        return rb.race_backward(q, k, v, w, g, p, state=st)

    L = _lib.lib()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    c0 = L.race_launch_count()
    step()
    torch.cuda.synchronize()
    launches = L.race_launch_count() - c0

    graph = None
    if world == 1 and not args.no_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()

    def run():
        if graph is not None:
            graph.replay()
        else:
            step()

    # settle clocks, then time exactly K steps
    sampler = ClockSampler(local_rank)
    sampler.start()
    t_settle = time.perf_counter()
    while time.perf_counter() - t_settle < 0.5:
        run()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        run()
    ev1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    tokens = n * world
    value = tokens / (ms_step / 1e3)

    # per-kernel breakdown (split-phase entries, events on the launching stream)
    pr = Problem(q, k, v, w, p)
    E = pr.table_elems
    ws = pr.ws()
    part = torch.empty((pr.bh, pr.nseg, E), device=dev)
    tabs = torch.empty_like(part)
    dpart = torch.empty_like(part)
    dtabs = torch.empty_like(part)
    o = torch.empty_like(v)
    den = torch.empty((1, HEADS, n), device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    rden = torch.empty((pr.bh, (n + 3) // 4 * 4), device=dev)  # row pitch N rounded up to 4 (race_b200.h)
    gden = torch.empty_like(rden)
    norms = torch.empty((pr.bh, n, 16), device=dev)  # sketch rows
    S = _stream()
    ptr = _vp
    if causal:
        calls = [
            ("kside_partials", lambda: L.race_kside_partials_rows(pr.dref, ptr(k), ptr(v), ptr(pr.w), ptr(part),
                                                                  ptr(norms), ptr(ws), S)),
            ("combine", lambda: L.race_combine(pr.dref, 1, ptr(part), None, ptr(tabs), S)),
            ("fwd_causal", lambda: L.race_fwd_causal_krows(pr.dref, ptr(q), ptr(k), ptr(v), ptr(pr.w), ptr(tabs), ptr(o),
                                                     ptr(den), ptr(norms), ptr(ws), S)),
            ("bwd_causal_q", lambda: L.race_bwd_causal_q(pr.dref, ptr(q), ptr(k), ptr(v), ptr(g), ptr(pr.w), ptr(tabs),
                                                         ptr(norms), ptr(dq), ptr(rden), ptr(gden), ptr(dpart),
                                                         ptr(ws), S)),
            ("combine_d", lambda: L.race_combine(pr.dref, 2, ptr(dpart), None, ptr(dtabs), S)),
            ("bwd_causal_k", lambda: L.race_bwd_causal_k(pr.dref, ptr(q), ptr(k), ptr(v), ptr(g), ptr(pr.w), ptr(rden),
                                                         ptr(gden), ptr(dtabs), ptr(norms), ptr(dk), ptr(dv),
                                                         ptr(ws), S)),
        ]
    else:
        calls = [
            ("kside_partials", lambda: L.race_kside_partials(pr.dref, ptr(k), ptr(v), ptr(pr.w), ptr(part), ptr(ws), S)),
            ("combine", lambda: L.race_combine(pr.dref, 0, ptr(part), None, ptr(tabs), S)),
            ("fwd_readout", lambda: L.race_fwd_readout(pr.dref, ptr(q), ptr(pr.w), ptr(tabs), ptr(o), ptr(den),
                                                       ptr(ws), S)),
            ("bwd_qside", lambda: L.race_bwd_qside(pr.dref, ptr(q), ptr(g), ptr(pr.w), ptr(tabs), ptr(dq), ptr(dpart),
                                                   ptr(ws), S)),
            ("combine_d", lambda: L.race_combine(pr.dref, 0, ptr(dpart), None, ptr(dtabs), S)),
            ("bwd_kside", lambda: L.race_bwd_kside(pr.dref, ptr(k), ptr(v), ptr(pr.w), ptr(dtabs), ptr(dk), ptr(dv),
                                                   ptr(ws), S)),
        ]
    reps = 10
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(calls) + 1)] for _ in range(reps)]
    for r in range(reps):
        evs[r][0].record()
        for i, (name, fn) in enumerate(calls):
            _lib.check(fn(), name)
            evs[r][i + 1].record()
    torch.cuda.synchronize()
    per = {name: statistics.median(evs[r][i].elapsed_time(evs[r][i + 1]) for r in range(reps))
           for i, (name, _) in enumerate(calls)}
    kb = kernel_bytes(e, causal)
    dom = max(kb, key=lambda nm: per[nm])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    # (tools/ncu_summary.py traffic; same workload: N=131072 per GPU, H=4, bf16)
    ncu_names = {"kside_partials": "k_aggregate2", "fwd_causal": "k_causal_fwd8", "bwd_causal_q": "k_bwd_causal_q8",
                 "bwd_causal_k": "k_bwd_causal_k8", "fwd_readout": "k_readout8", "bwd_qside": "k_bwd_q8",
                 "bwd_kside": "k_bwd_k8", "combine": "k_combine", "combine_d": "k_combine"}
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        if n == 131072 and dtype == torch.bfloat16 and ncu_names[dom] in tr:
            traffic = tr[ncu_names[dom]]["dram_bytes"]
    except Exception:
        pass
    kernels = {}
    for nm, ms_k in per.items():
        io, inter = kb.get(nm, (0, 0))
        io_b, inter_b = io * HEADS * n, inter * HEADS * n
        kernels[nm] = {"ms": round(ms_k, 4), "compulsory_bytes": io_b, "intermediate_bytes": inter_b,
                       "frac": round(io_b / (ms_k / 1e3) / 1e9 / peak, 4) if io_b else None,
                       "frac_with_intermediates": round((io_b + inter_b) / (ms_k / 1e3) / 1e9 / peak, 4) if io_b else None}
    dom_bytes = kb[dom][0] * HEADS * n
    achieved = dom_bytes / (per[dom] / 1e3) / 1e9
    step_bytes = ((7 * DIM + 5 * DIM) * e + 8) * HEADS * n   # (7d+5dv)e+8 per token-head
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write per launch)", "peak_source": peak_src,
                "algorithmic_bytes_per_launch": dom_bytes,
                "algorithmic_note": "compulsory bytes only (the kernel's N x d reads/writes + den); "
                                    "kernels[].frac_with_intermediates adds sketch rows / normaliser terms",
                "kernels": kernels,
                "kernel_ms": {k2: round(v2, 4) for k2, v2 in per.items()},
                "step_algorithmic_GBps": step_bytes / (ms_step / 1e3) / 1e9,
                "step_frac": step_bytes / (ms_step / 1e3) / 1e9 / peak}

    # e2e through the public module API with pinned host buffers
    e2e = None
    if not args.no_e2e and world == 1:
        layer = rb.RaceAttention(HEADS, DIM, cfg).to(dev)
        hq, hk, hv, hg = (t.cpu().pin_memory() for t in (q, k, v, g))
        outs = [torch.empty(shape, dtype=dtype).pin_memory() for _ in range(4)]

        # Three streams: uploads (into one of two device buffer sets), compute, read-back.  Step i+1's
        # upload overlaps step i's compute and step i's read-back overlaps step i+1's upload (PCIe is
        # full duplex), so the step approaches the link's duplex time for 1 GiB.  Every step still
        # uploads its own inputs and reads back its own results inside the timed region.
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        bufs = [[torch.empty(shape, dtype=dtype, device=dev) for _ in range(4)] for _ in range(2)]
        up_done = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]

        def upload(b):
            with torch.cuda.stream(h2d):
                h2d.wait_event(used[b])  # the compute that last read buffer set b has finished
                for dst, src in zip(bufs[b], (hq, hk, hv, hg)):
                    dst.copy_(src, non_blocking=True)
                up_done[b].record(h2d)

        def compute(i):
            b = i % 2
            cur = torch.cuda.current_stream()
            cur.wait_event(up_done[b])
            q_, k_, v_ = (x.detach().requires_grad_(True) for x in bufs[b][:3])
            out = layer(q_, k_, v_)
            out.backward(bufs[b][3])
            used[b].record(cur)
            res = (out.detach(), q_.grad, k_.grad, v_.grad)
            d2h.wait_stream(cur)
            with torch.cuda.stream(d2h):
                for dst, src in zip(outs, res):
                    dst.copy_(src, non_blocking=True)
                    src.record_stream(d2h)

        def run_steps(k_steps):
            upload(0)
            for i in range(k_steps):
                if i + 1 < k_steps:
                    upload((i + 1) % 2)
                compute(i)
            torch.cuda.current_stream().wait_stream(d2h)  # the last read-back is inside the timed region

        run_steps(2)
        torch.cuda.synchronize()
        k_e2e = max(3, min(args.steps, 30))  # the pipeline fill (first upload, last read-back) amortised
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        run_steps(k_e2e)
        a1.record()
        torch.cuda.synchronize()
        ems = a0.elapsed_time(a1) / k_e2e
        nb = q.numel() * e
        e2e = {"value": n / (ems / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": 4 * nb,
               "d2h_bytes_per_step": 4 * nb, "ms_per_step": ems,
               "api": "RaceAttention (nn.Module) forward+backward from pinned host buffers: each step uploads its "
                      "Q, K, V, dO and reads back O, dQ, dK, dV; uploads, compute and read-backs on three streams "
                      "(step i+1's upload overlaps step i's compute and read-back)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = 8192 if causal else 32768
        ra = _reference_package()
        if ra is not None:
            dt = reference_step(ra, n_s, causal)
            kind, what = "reference", "the unmodified reference package (baseline/_ref) public API"
        else:
            dt = cpu_reference_step(n_s, causal)
            kind, what = "port", "oracle/race_oracle.py, the reference algorithm"
        cpu = {"value": n_s / dt, "unit": "tokens/s", "cores": cpu_threads(), "kind": kind,
               "sample": f"{n_s}-token {'causal' if causal else 'non-causal'} fwd+bwd, H={HEADS}, d={DIM}, f32 "
                         f"({what}), {dt:.1f} s", "host": _host_facts()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.n_total else "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic N(0,1) Q,K,V,dO resident in HBM",
            "config": _config(args, world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "cuda_graph": not args.no_graph and world == 1, "clocks": clocks,
            "fast_path": bool(_lib.fast_path(pr.desc)),
        }
        return line
    return None


def _relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` outside torchrun: re-exec as N ranks (one per GPU) so the line
    never reports one rank for N requested."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world if launched else args.gpus, rank)
        return
    if not launched and args.gpus > 1:
        sys.exit(_relaunch_under_torchrun(args))
    if launched and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU", file=sys.stderr)
        sys.exit(2)
    if os.environ.get("RACE_BENCH_ONE_GPU") == "1":  # test hook: every rank on cuda:0 over gloo
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if os.environ.get("RACE_BENCH_ONE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        line = run_ours(args, world, rank, local_rank)
        if world > 1 and not args.no_max_context:
            import torch
            import torch.distributed as dist

            dev = torch.device("cuda", local_rank)
            dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
            torch.cuda.empty_cache()
            s64 = sharded_run(dev, world, args.sharded_64m_total, dt)
            smax = sharded_max_context(dev, world, dt)
            if line is not None:
                line["sharded_configs3"] = s64
                line["max_context_sharded"] = smax
                line["comm"] = {"backend": dist.get_backend(), "world": world,
                                "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))
                                if dist.get_backend() == "nccl" else None}
        if line is not None:
            if world == 1 and not args.no_max_context:
                import torch

                torch.cuda.empty_cache()
                dev = torch.device("cuda", local_rank)
                dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
                line["max_context"] = [max_context(dev, c, dt) for c in (True, False)] + [
                    max_context(dev, True, dt, inplace=True)]
                line["scale_sweep"] = scale_sweep(dev, dt)
                line["sketch_sweep"] = sketch_sweep(dev, dt)
                line["gpt_train_step"] = gpt_train_step(dev)
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
