"""Golden vectors for the validation-side functions, from the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_aux_golden.py

Records inputs and outputs of ``soft_features`` / ``hard_hash`` /
``dominant_corner_mass`` (ra/sketch.py), ``race_kernel`` (ra/forward.py:167),
``hard_race_attention`` / ``kernel_deviation`` / ``row_sum_stability`` /
``collision_identity_check`` (ra/theory.py) and ``angular_kernel_matrix`` /
``angular_attention`` / ``angular_attention_vjp`` (ra/exact.py) into
``golden_aux.npz``.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import math
import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import race_attention as ra  # noqa: E402  (the reference, read-only)
    from race_attention import exact, sketch, theory
    from race_attention.forward import race_kernel

    out: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(20251004)

    # soft / hard hashing: P across the explicit-corner limit (10) and the factored path
    for P, n, d, beta in ((1, 64, 16, 8.0), (2, 200, 128, 8.0), (3, 130, 64, 2.5), (11, 40, 32, 1.0)):
        x = rng.standard_normal((n, d))
        x[3] = 0.0  # zero row
        table = sketch.make_hash_table(rng, P, d)
        tag = f"sf_P{P}"
        out[f"{tag}_x"], out[f"{tag}_w"] = x, table.w
        out[f"{tag}_beta"] = np.array(beta)
        out[f"{tag}_phi"] = sketch.soft_features(x, table, beta)
        out[f"{tag}_hard"] = sketch.hard_hash(x, table)
        out[f"{tag}_dom"] = sketch.dominant_corner_mass(x, table, beta)

    # race_kernel, kernel_deviation, row_sum_stability, hard_race_attention
    for i, (P, L, M, n, d, beta) in enumerate(((2, 2, 1, 96, 128, 8.0), (3, 4, 2, 150, 32, 4.0), (1, 8, 1, 64, 8, 16.0))):
        cfg = ra.SketchConfig(hyperplanes=P, tables=L, ensembles=M, beta=beta, seed=11 + i)
        q, k, v = rng.standard_normal((n, d)), rng.standard_normal((n, d)), rng.standard_normal((n, d))
        tag = f"th{i}"
        out[f"{tag}_cfg"] = np.array([P, L, M, beta, 11 + i])
        out[f"{tag}_q"], out[f"{tag}_k"], out[f"{tag}_v"] = q, k, v
        out[f"{tag}_kernel"] = race_kernel(q, k, cfg)
        out[f"{tag}_kdev"] = np.array(theory.kernel_deviation(q, k, cfg, P))
        rs = theory.row_sum_stability(q, k, cfg)
        out[f"{tag}_rowsum"] = np.array([rs.min_row_sum, rs.min_den, rs.ratio, float(rs.near_degenerate)])
        h = theory.hard_race_attention(ra.AttnInputs(q, k, v), cfg)
        out[f"{tag}_hard_o"], out[f"{tag}_hard_den"] = h.o, h.den
        out[f"{tag}_hard_deg"] = np.array(h.degenerate_rows, dtype=np.int64)

    # exact angular attention (+ VJP), causal and not, several gammas and shapes
    for i, (n, d, dv, gamma, causal) in enumerate(((50, 16, 16, 2, False), (77, 128, 128, 8, True),
                                                   (130, 64, 96, 3, False), (33, 200, 24, 1, True),
                                                   (64, 8, 8, 40, False))):
        q, k, v, g = (rng.standard_normal((n, dd)) for dd in (d, d, dv, dv))
        if i == 0:
            k[5] = q[5] * 3.0  # exactly aligned pair: clamped, no gradient through it
        inp = exact.AttnInputs(q, k, v)
        tag = f"ang{i}"
        out[f"{tag}_meta"] = np.array([gamma, int(causal)])
        out[f"{tag}_q"], out[f"{tag}_k"], out[f"{tag}_v"], out[f"{tag}_g"] = q, k, v, g
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            out[f"{tag}_o"] = exact.angular_attention(inp, gamma, causal=causal)
        dq, dk, dvv = exact.angular_attention_vjp(inp, gamma, g, causal=causal)
        out[f"{tag}_dq"], out[f"{tag}_dk"], out[f"{tag}_dv"] = dq, dk, dvv
        out[f"{tag}_kmat"] = exact.angular_kernel_matrix(q[:40], k[:30], gamma)

    # collision identity: the reference's report for a seeded generator
    for P in (1, 3):
        rep = theory.collision_identity_check(P, 20000, np.random.default_rng(7 + P))
        out[f"coll_P{P}"] = np.array([[r.angle, r.p_hat, r.p_exact, r.std_err, r.z_score, float(r.passed)]
                                      for r in rep.rows])

    # acceptance criteria 4 and 5 at their quick sizes (ra/acceptance.py:224-278): the sweep errors
    def unit(r, n, d):
        x = r.standard_normal((n, d))
        return x / np.linalg.norm(x, axis=1, keepdims=True)

    r = np.random.default_rng(11)
    inp4 = ra.AttnInputs(unit(r, 128, 16), unit(r, 128, 16), unit(r, 128, 16))
    out["crit4_errors"] = theory.variance_sweep(inp4, hyperplanes=2, beta=256.0, l_grid=[4, 16, 64, 256], n_seeds=8,
                                                base_seed=100).errors
    r = np.random.default_rng(13)
    inp5 = ra.AttnInputs(unit(r, 64, 16), unit(r, 64, 16), unit(r, 64, 16))
    out["crit5_errors"] = theory.bias_sweep(inp5, hyperplanes=2, tables=512, beta_grid=[2, 4, 8, 16, 32], n_seeds=4,
                                            base_seed=300, check_monotone=False).errors
    ref5 = exact.angular_attention(inp5, gamma=2)
    gaps = []
    for s_ in range(2):
        c = ra.SketchConfig(hyperplanes=2, tables=512, beta=1e3, seed=400 + s_)
        gaps.append([theory.output_rms_error(ra.race_attention(inp5, c).o, ref5),
                     theory.output_rms_error(theory.hard_race_attention(inp5, c).o, ref5)])
    out["crit5_soft_hard"] = np.array(gaps)

    # bench harness CSV schema (ra/bench.py:37-141, 294-324)
    from race_attention.bench import BenchRecord, demo_kernel_heatmap, heatmap_csv_text, records_to_csv

    recs = [BenchRecord("race", 4096, 128, 4, 2, 2, 1, 8.0, True, "forward_backward", 0.123456789, 1234, 0, "ok",
                        threads=8),
            BenchRecord("angular_exact", 65536, 128, 4, None, None, None, None, False, "forward", None, 99, 3,
                        "time_guard")]
    out["csv"] = np.array(records_to_csv(recs))
    out["csv_ext"] = np.array(records_to_csv(recs, extended=True))
    out["heatmap"] = np.array(heatmap_csv_text(*demo_kernel_heatmap([1, 2, 8], 9)))

    np.savez_compressed(os.path.join(HERE, "golden_aux.npz"), **out)
    print(f"wrote {len(out)} arrays to golden_aux.npz")


if __name__ == "__main__":
    main()
