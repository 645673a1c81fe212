"""Eager (python API per call) vs CUDA-graph replay of the bench step, device time per step.
Measures the host overhead of the public entry points (race_forward / race_backward)."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_04008_b200 as rb  # noqa: E402

dev = torch.device("cuda", 0)
for causal in (True, False):
    cfg = rb.SketchConfig(hyperplanes=2, tables=2, seed=0, causal=causal)
    w = rb.head_hyperplanes(cfg, 4, 128).to(dev)
    p = cfg.params()
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = (torch.randn(1, 4, 131072, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))

    def step():
        o, den, st = rb.race_forward(q, k, v, w, p)
        return rb.race_backward(q, k, v, w, do, p, state=st)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        step()
    cpu_us = (time.perf_counter() - t0) / 200 * 1e6  # host submission time per step (queue not full)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(50):
        step()
    ev[1].record()
    torch.cuda.synchronize()
    eager = ev[0].elapsed_time(ev[1]) / 50
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(50):
        gr.replay()
    ev[1].record()
    torch.cuda.synchronize()
    graph = ev[0].elapsed_time(ev[1]) / 50
    print(f"{'causal' if causal else 'noncausal'}: eager {eager*1e3:.1f} us/step, graph {graph*1e3:.1f} us/step, "
          f"eager/graph {eager/graph:.3f}, host submit ~{cpu_us:.1f} us/step")
