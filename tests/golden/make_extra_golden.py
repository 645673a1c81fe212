"""Golden vectors (round 2) from the REAL reference implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_extra_golden.py

Writes ``golden_extra.npz`` with

* ``nd_*``: ``accumulate_num_den`` (``ra/forward.py:124-144``) on already
  prepared q, k -- the raw averaged float64 numerator and denominator --
  non-causal and causal, including one instance built so that some query rows
  have an exactly zero denominator (every key sits in the opposite corner of
  the single P=1 table at beta=1000, so exp(-2 beta |u|) underflows): those
  rows are ``degenerate_rows`` of ``race_attention`` (``ra/forward.py:157-163``);
* ``rn_*``: ``row_normalize`` / ``row_normalize_vjp`` (``ra/core.py:114-139``)
  with zero and tiny rows.

Nothing on the GPU box reads ``/root/reference``; the npz is committed.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import race_attention as ra  # noqa: E402  (the reference, read-only)
    from race_attention.core import row_normalize, row_normalize_vjp
    from race_attention.forward import accumulate_num_den, table_hyperplanes

    blob = {}
    rng = np.random.default_rng(20261017)
    nd = []
    # n, d, dv, P, L, M, beta, causal, seed
    for spec in [(300, 32, 16, 2, 2, 1, 8.0, False, 1), (300, 32, 16, 2, 2, 1, 8.0, True, 2),
                 (257, 128, 128, 3, 1, 2, 4.0, True, 3), (257, 128, 128, 1, 3, 1, 16.0, False, 4)]:
        n, d, dv, p, l, m, beta, causal, seed = spec
        cfg = ra.SketchConfig(hyperplanes=p, tables=l, ensembles=m, beta=beta, seed=seed, causal=causal)
        q = row_normalize(rng.standard_normal((n, d)))
        k = row_normalize(rng.standard_normal((n, d)))
        v = rng.standard_normal((n, dv))
        nd.append((cfg, q, k, v))
    # degenerate rows: P=1, L=1, beta=1000; keys all on the negative side of the hyperplane,
    # the first 5 queries on the positive side with |u| large -> den underflows to exactly 0
    for causal in (False, True):
        cfg = ra.SketchConfig(hyperplanes=1, tables=1, beta=1000.0, seed=5, causal=causal)
        d = 16
        w = table_hyperplanes(cfg, d, 0, 0)[0]
        wu = w / np.linalg.norm(w)

        def side(x, sign):
            x = x - np.outer(x @ wu, wu)  # drop the component along w, then put it on one side
            x = x / np.linalg.norm(x, axis=1, keepdims=True)
            return row_normalize(x * 0.6 + sign * 0.8 * wu[None, :])

        n = 40
        k = side(rng.standard_normal((n, d)), -1.0)
        q = np.vstack([side(rng.standard_normal((5, d)), 1.0), side(rng.standard_normal((n - 5, d)), -1.0)])
        v = rng.standard_normal((n, 8))
        nd.append((cfg, q, k, v))
    for i, (cfg, q, k, v) in enumerate(nd):
        num, den = accumulate_num_den(q, k, v, cfg)
        out = ra.race_attention(ra.AttnInputs(q, k, v), cfg)
        pre = f"nd{i:02d}_"
        blob.update({pre + "q": q, pre + "k": k, pre + "v": v, pre + "num": num, pre + "den": den,
                     pre + "o": out.o, pre + "degenerate": np.array(out.degenerate_rows, dtype=np.int64),
                     pre + "P": np.int64(cfg.hyperplanes), pre + "L": np.int64(cfg.tables),
                     pre + "M": np.int64(cfg.ensembles), pre + "beta": np.float64(cfg.beta),
                     pre + "seed": np.int64(cfg.seed), pre + "causal": np.bool_(cfg.causal)})
    blob["nd_count"] = np.int64(len(nd))
    # row_normalize / row_normalize_vjp with zero and tiny rows
    x = rng.standard_normal((50, 24))
    x[3] = 0.0
    x[7] = 1e-14
    x[11] *= 1e6
    g = rng.standard_normal((50, 24))
    blob.update({"rn_x": x, "rn_g": g, "rn_y": row_normalize(x), "rn_dx": row_normalize_vjp(x, g),
                 "rn_x32": x.astype(np.float32), "rn_y32": row_normalize(x.astype(np.float32))})
    blob["numpy_version"] = np.array(np.__version__)
    path = os.path.join(HERE, "golden_extra.npz")
    np.savez_compressed(path, **blob)
    print(f"wrote {len(nd)} num/den cases + row_normalize to {path} ({os.path.getsize(path) / 1e6:.2f} MB)")
    for i, (cfg, q, k, v) in enumerate(nd):
        print(i, cfg.causal, "degenerate rows:", list(blob[f"nd{i:02d}_degenerate"]))


if __name__ == "__main__":
    main()
