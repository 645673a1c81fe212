"""Generate golden vectors from the REAL reference implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``race_attention`` from ``/root/reference/pkg/src`` and records,
per instance, the inputs, the hyperplanes the reference derived
(``ra/forward.py:54-57``), the forward outputs (``race_attention``,
``ra/forward.py:147``) and the VJP (``race_attention_vjp``,
``ra/backward.py:184``).  The resulting ``golden_*.npz`` files are committed;
nothing on the GPU box reads ``/root/reference``.

Instance grid:
* ``grid``: the reference's own acceptance grid (``ra/acceptance.py:108-133``,
  criterion 1), all 54 instances, float64, plus a seeded d_out for the VJP;
* ``gradcheck``: the criterion-6 instances (``ra/acceptance.py:281-297``),
  causal and non-causal;
* ``edge``: N=1, zero rows, large beta, M=2, P=11 (factored path), small
  ``block_size`` so block carries are exercised, d=64/128 shapes, and inputs
  whose values are exactly bf16-representable.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 (RNE) and return them as float64."""
    f = x.astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def main() -> None:
    sys.path.insert(0, REF)
    import race_attention as ra  # noqa: E402  (the reference, read-only)
    from race_attention.acceptance import gradcheck_instances, oracle_instances
    from race_attention.forward import table_hyperplanes

    def run(tag, q, k, v, g, cfg):
        d = q.shape[1]
        w = np.stack([table_hyperplanes(cfg, d, m, l)
                      for m in range(cfg.ensembles) for l in range(cfg.tables)])
        inp = ra.AttnInputs(q, k, v)
        out = ra.race_attention(inp, cfg)
        grads = ra.race_attention_vjp(inp, cfg, g)
        deg = np.zeros(q.shape[0], dtype=bool)
        deg[list(out.degenerate_rows)] = True
        return {
            "tag": np.array(tag),
            "q": q, "k": k, "v": v, "d_out": g, "w": w,
            "P": np.int64(cfg.hyperplanes), "L": np.int64(cfg.tables),
            "M": np.int64(cfg.ensembles), "beta": np.float64(cfg.beta),
            "seed": np.int64(cfg.seed), "causal": np.bool_(cfg.causal),
            "normalize": np.bool_(cfg.normalize_inputs),
            "block_size": np.int64(cfg.block_size),
            "o": out.o, "den": out.den, "degenerate": deg,
            "dq": grads.dq, "dk": grads.dk, "dv": grads.dv,
        }

    cases = []
    # --- criterion-1 grid (ra/acceptance.py:108-164) -----------------------
    for spec in oracle_instances():
        rng = np.random.default_rng(spec["seed"])
        q = rng.standard_normal((spec["n"], spec["d"]))
        k = rng.standard_normal((spec["n"], spec["d"]))
        v = rng.standard_normal((spec["n"], spec["dv"]))
        g = rng.standard_normal((spec["n"], spec["dv"]))
        cfg = ra.SketchConfig(hyperplanes=spec["hyperplanes"], tables=spec["tables"],
                              ensembles=spec["ensembles"], beta=spec["beta"],
                              seed=spec["seed"], causal=spec["causal"])
        cases.append(run("grid", q, k, v, g, cfg))
    # --- criterion-6 instances (ra/acceptance.py:281-326) ------------------
    for spec in gradcheck_instances():
        rng = np.random.default_rng(spec["seed"])
        q = rng.standard_normal((spec["n"], spec["d"]))
        k = rng.standard_normal((spec["n"], spec["d"]))
        v = rng.standard_normal((spec["n"], spec["dv"]))
        g = 1e-3 * rng.standard_normal((spec["n"], spec["dv"]))
        for causal in (False, True):
            cfg = ra.SketchConfig(hyperplanes=spec["hyperplanes"], tables=spec["tables"],
                                  ensembles=spec["ensembles"], beta=spec["beta"],
                                  seed=spec["seed"], causal=causal)
            cases.append(run("gradcheck", q, k, v, g, cfg))
    # --- edge cases ---------------------------------------------------------
    rng = np.random.default_rng(20251004)
    edge_specs = [
        # n, d, dv, P, L, M, beta, causal, block, zero_rows, bf16
        (1, 128, 128, 2, 2, 1, 8.0, False, 4096, 0, False),
        (1, 128, 128, 2, 2, 1, 8.0, True, 4096, 0, False),
        (37, 16, 8, 2, 2, 1, 8.0, False, 4096, 3, False),
        (37, 16, 8, 2, 2, 1, 8.0, True, 4096, 3, False),
        (64, 128, 128, 2, 2, 1, 8.0, False, 16, 0, False),
        (64, 128, 128, 2, 2, 1, 8.0, True, 16, 0, False),
        (130, 128, 128, 2, 2, 1, 8.0, True, 4096, 0, True),
        (130, 128, 128, 2, 2, 1, 8.0, False, 4096, 0, True),
        (97, 64, 64, 2, 2, 1, 8.0, True, 4096, 0, True),
        (97, 64, 64, 2, 2, 1, 8.0, False, 4096, 0, True),
        (64, 128, 128, 4, 4, 1, 8.0, True, 4096, 0, True),
        (64, 128, 128, 4, 4, 1, 8.0, False, 4096, 0, True),
        (65, 32, 48, 3, 2, 2, 16.0, True, 16, 0, False),
        (65, 32, 48, 3, 2, 2, 16.0, False, 16, 0, False),
        (48, 8, 8, 2, 1, 1, 64.0, False, 4096, 0, False),
        (48, 8, 8, 2, 1, 1, 64.0, True, 4096, 0, False),
        (20, 12, 5, 11, 1, 1, 2.0, False, 4096, 0, False),
        (20, 12, 5, 11, 1, 1, 2.0, True, 4096, 0, False),
        (40, 128, 128, 1, 3, 1, 0.5, True, 4096, 0, False),
        (40, 128, 128, 1, 3, 1, 0.5, False, 4096, 0, False),
    ]
    for i, (n, d, dv, p, l, m, beta, causal, block, zr, bf) in enumerate(edge_specs):
        q = rng.standard_normal((n, d))
        k = rng.standard_normal((n, d))
        v = rng.standard_normal((n, dv))
        g = rng.standard_normal((n, dv))
        if zr:
            q[:zr] = 0.0
            k[1:1 + zr] = 0.0
        if bf:
            q, k, v, g = (_bf16_round(a) for a in (q, k, v, g))
        cfg = ra.SketchConfig(hyperplanes=p, tables=l, ensembles=m, beta=beta,
                              seed=4242 + i, causal=causal, block_size=block)
        cases.append(run("edge", q, k, v, g, cfg))
    # unnormalised variant (normalize_inputs=False, ra/core.py:67)
    for causal in (False, True):
        q = 0.2 * rng.standard_normal((40, 16))
        k = 0.2 * rng.standard_normal((40, 16))
        v = rng.standard_normal((40, 16))
        g = rng.standard_normal((40, 16))
        cfg = ra.SketchConfig(hyperplanes=2, tables=2, beta=8.0, seed=77, causal=causal,
                              normalize_inputs=False)
        cases.append(run("edge", q, k, v, g, cfg))

    blob = {}
    for i, c in enumerate(cases):
        for key, val in c.items():
            blob[f"{i:03d}_{key}"] = val
    blob["count"] = np.int64(len(cases))
    blob["numpy_version"] = np.array(np.__version__)
    path = os.path.join(HERE, "golden_race.npz")
    np.savez_compressed(path, **blob)
    print(f"wrote {len(cases)} cases to {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
