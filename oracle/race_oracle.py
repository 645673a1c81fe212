"""CPU oracle for the RACE attention hot path (TEST INFRASTRUCTURE ONLY).

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import it.  The shipped path
(``paper_2510_04008_b200``) must never route through it.

It is a numpy restatement of the reference package
``/root/reference/pkg/src/race_attention`` (abbreviated ``ra/`` below):
forward (``ra/forward.py:77-164``) and vector-Jacobian product
(``ra/backward.py:53-235``), non-causal and causal, including the row
normalisation (``ra/core.py:114-139``) and the degenerate-denominator rule
(``ra/forward.py:157-163``).

Pinning: ``tests/golden/make_golden.py`` runs the *real* reference (importable
in the build container) on a deterministic instance grid and commits the
inputs, hyperplanes and outputs as ``tests/golden/*.npz``.  ``tests/test_oracle.py``
checks this restatement against every fixture (1e-10 relative, the reference's
own ORACLE_TOL, ``ra/acceptance.py:36``), so parity is pinned to the reference.

Formulation.  All tables are handled at once through the concatenated feature
map: for T = M*L tables with R = 2**P corners each, the
per-row feature vector phi(x) has F = T*R entries ordered table-major in the
reference's (m, l) task order (``ra/forward.py:128``).  Then

    S = phi(K)^T [V | 1]                  (F x (dv+1)),   num|den = phi(Q) S / T

which is algebraically identical to the per-table loop + in-order sum
(``ra/forward.py:136-144``); float64 accumulation as in the reference.
"""

from __future__ import annotations

import numpy as np

# ra/core.py:14-19
ZERO_ROW_EPS = 1e-12
DEGENERATE_DEN_EPS = 1e-30
# ra/sketch.py:19 -- above this many bits the corner matrix is not built
EXPLICIT_CORNER_LIMIT = 10


# --------------------------------------------------------------------------
# hyperplanes (ra/core.py:93-111, ra/forward.py:54-57)
# --------------------------------------------------------------------------
def table_hyperplanes(seed: int, ensemble: int, table: int, p: int, d: int) -> np.ndarray:
    """W for one (m, l) slot: SeedSequence(seed, spawn_key=(m, l)) -> N(0,1) (P, d) f64."""
    ss = np.random.SeedSequence(entropy=int(seed) & 0xFFFFFFFFFFFFFFFF,
                                spawn_key=(ensemble, table))
    return np.random.default_rng(ss).standard_normal((p, d))


def stacked_hyperplanes(seed: int, p: int, tables: int, ensembles: int, d: int) -> np.ndarray:
    """All tables in task order (m-major, then l): shape (T, P, d) float64 (ra/forward.py:128)."""
    return np.stack([table_hyperplanes(seed, m, l, p, d)
                     for m in range(ensembles) for l in range(tables)])


# --------------------------------------------------------------------------
# row normalisation (ra/core.py:114-139)
# --------------------------------------------------------------------------
def unit_rows(x: np.ndarray) -> np.ndarray:
    """x / ||x|| per row; rows with norm < 1e-12 pass through (ra/core.py:114-123)."""
    nrm = np.sqrt(np.einsum("ij,ij->i", x, x))[:, None]
    return x / np.where(nrm < ZERO_ROW_EPS, x.dtype.type(1), nrm)


def unit_rows_vjp(x: np.ndarray, g: np.ndarray) -> np.ndarray:
    """Sphere-tangent pull-back g -> (g - (g.xhat) xhat)/||x|| (ra/core.py:126-139)."""
    nrm = np.sqrt(np.einsum("ij,ij->i", x, x))[:, None]
    tiny = nrm < ZERO_ROW_EPS
    s = np.where(tiny, 1.0, nrm)
    xh = x / s
    out = (g - np.einsum("ij,ij->i", g, xh)[:, None] * xh) / s
    return np.where(tiny, g, out)


# --------------------------------------------------------------------------
# soft features (ra/sketch.py:52-129)
# --------------------------------------------------------------------------
def corner_signs(p: int) -> np.ndarray:
    """(2**p, p) matrix, entry (r, t) = +1 if bit t of r is 0 else -1 (ra/sketch.py:52-74)."""
    r = np.arange(1 << p)[:, None]
    t = np.arange(p)[None, :]
    return np.where((r >> t) & 1, -1.0, 1.0)


def _logistic(z):
    e = np.exp(-np.abs(z))
    return np.where(z >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def table_features(x: np.ndarray, w: np.ndarray, beta: float) -> tuple[np.ndarray, np.ndarray]:
    """phi (n, 2**p) and u = tanh(x w^T) (n, p) for one table.

    p <= 10: max-shifted softmax over corner logits beta*u.c_r (ra/sketch.py:111-118).
    p > 10: product of per-bit logistic factors (ra/sketch.py:120-129).
    """
    u = np.tanh(x @ w.T.astype(x.dtype, copy=False))
    p = w.shape[0]
    if p <= EXPLICIT_CORNER_LIMIT:
        lg = beta * (u @ corner_signs(p).T.astype(x.dtype, copy=False))
        lg = np.exp(lg - lg.max(axis=1, keepdims=True))
        return lg / lg.sum(axis=1, keepdims=True), u
    pos = _logistic(2.0 * beta * u)
    neg = _logistic(-2.0 * beta * u)
    phi = np.ones((x.shape[0], 1), dtype=x.dtype)
    for t in range(p):
        phi = np.hstack([phi * pos[:, t:t + 1], phi * neg[:, t:t + 1]])
    return phi, u


def features(x: np.ndarray, w_stack: np.ndarray, beta: float) -> np.ndarray:
    """Concatenated phi(x) (n, T*2**P), tables in task order."""
    return np.hstack([table_features(x, w, beta)[0] for w in w_stack])


def table_features_vjp(x, w, beta, dphi):
    """Pull a cotangent on one table's phi back to x (ra/backward.py:53-90)."""
    phi, u = table_features(x, w.astype(x.dtype, copy=False), beta)
    p = w.shape[0]
    if p <= EXPLICIT_CORNER_LIMIT:
        c = corner_signs(p).astype(x.dtype, copy=False)
        dl = phi * (dphi - np.sum(dphi * phi, axis=1, keepdims=True))
        du = beta * (dl @ c)
    else:
        # factored: phi_r = prod_t sigma(2 beta u_t c_rt) -> d phi_r/d u_t = 2 beta c_rt phi_r (1 - sigma_t)
        z = 2.0 * beta * u
        pos = _logistic(z)
        c = corner_signs(p)
        du = np.empty_like(u)
        for t in range(p):
            s = np.where(c[:, t] > 0, 1.0 - pos[:, t:t + 1], pos[:, t:t + 1])
            du[:, t] = 2.0 * beta * np.sum(dphi * phi * c[None, :, t] * s, axis=1)
    return (du * (1.0 - u * u)) @ w.astype(x.dtype, copy=False)


# --------------------------------------------------------------------------
# forward (ra/forward.py:77-164)
# --------------------------------------------------------------------------
def _prep(q, k, normalize):
    # ra/forward.py:47-51
    return (unit_rows(q), unit_rows(k)) if normalize else (q, k)


def key_state(k, v, w_stack, beta, normalize=True, block=65536):
    """(A [F], B [F, dv]) = sum over the rows of phi(k)^T [1 | v] in float64: the causal block
    carry of ra/forward.py:105-120 after these rows.  Seeding num_den / vjp with it (``carry=``)
    checks the tail of a long sequence without re-running its head on the CPU."""
    w_c = w_stack.astype(np.float64)
    f = w_stack.shape[0] << w_stack.shape[1]
    ca, cb = np.zeros(f), np.zeros((f, v.shape[1]))
    for lo in range(0, k.shape[0], block):
        kb = k[lo:lo + block].astype(np.float64)
        pk = features(unit_rows(kb) if normalize else kb, w_c, beta)
        ca += pk.sum(axis=0)
        cb += pk.T @ v[lo:lo + block].astype(np.float64)
    return ca, cb


def num_den(q, k, v, w_stack, beta, causal, block=4096, carry=None):
    """Averaged numerator (n, dv) and denominator (n,) in float64 (ra/forward.py:124-144).

    q, k are already prepared (normalised).  Non-causal: S = phi(K)^T[V|1]
    accumulated over row blocks (ra/forward.py:84-87), then phi(Q) S
    (ra/forward.py:93-96).  Causal: running block carry with an inclusive
    cumulative sum inside the block (ra/forward.py:100-121), starting from
    ``carry`` = (A, B) of the rows before q (key_state; default zero).
    """
    n, dv = q.shape[0], v.shape[1]
    t_tot = w_stack.shape[0]
    w_c = w_stack.astype(q.dtype, copy=False)
    num = np.empty((n, dv), dtype=np.float64)
    den = np.empty(n, dtype=np.float64)
    if not causal:
        f = t_tot << w_stack.shape[1]
        s_a = np.zeros(f)
        s_b = np.zeros((f, dv))
        for lo in range(0, n, block):
            pk = features(k[lo:lo + block], w_c, beta)
            s_a += pk.sum(axis=0, dtype=np.float64)
            s_b += pk.T @ v[lo:lo + block]
        a_c, b_c = s_a.astype(q.dtype), s_b.astype(q.dtype)
        for lo in range(0, n, block):
            pq = features(q[lo:lo + block], w_c, beta)
            num[lo:lo + block] = pq @ b_c
            den[lo:lo + block] = pq @ a_c
    else:
        f = t_tot << w_stack.shape[1]
        carry_a, carry_b = (np.zeros(f), np.zeros((f, dv))) if carry is None else carry
        for lo in range(0, n, block):
            hi = min(lo + block, n)
            pk = features(k[lo:hi], w_c, beta).astype(np.float64)
            pq = features(q[lo:hi], w_c, beta).astype(np.float64)
            vb = v[lo:hi].astype(np.float64)
            cum_a = carry_a + np.cumsum(pk, axis=0)
            cum_b = carry_b + np.cumsum(pk[:, :, None] * vb[:, None, :], axis=0)
            num[lo:hi] = np.einsum("tf,tfd->td", pq, cum_b)
            den[lo:hi] = np.einsum("tf,tf->t", pq, cum_a)
            carry_a, carry_b = cum_a[-1], cum_b[-1]
    return num / t_tot, den / t_tot


def forward(q, k, v, w_stack, beta, causal=False, normalize=True, block=4096, carry=None):
    """(o, den, degenerate_rows) as race_attention returns them (ra/forward.py:147-164)."""
    qp, kp = _prep(q, k, normalize)
    num, den = num_den(qp, kp, v, w_stack, beta, causal, block, carry)
    deg = den <= DEGENERATE_DEN_EPS
    o = np.zeros_like(num)
    np.divide(num, den[:, None], out=o, where=~deg[:, None])
    return o.astype(q.dtype, copy=False), den, tuple(np.nonzero(deg)[0].tolist())


# --------------------------------------------------------------------------
# backward (ra/backward.py:93-235)
# --------------------------------------------------------------------------
def _split_tables(x, t_tot):
    return np.split(x, t_tot, axis=1)


def _feature_grad(x, w_stack, beta, dphi):
    """Sum over tables of the per-table feature VJP (ra/backward.py:219-226)."""
    out = np.zeros(x.shape, dtype=np.float64)
    for w, g in zip(w_stack, _split_tables(dphi, w_stack.shape[0])):
        out += table_features_vjp(x, w, beta, g.astype(x.dtype, copy=False))
    return out


def vjp(q, k, v, w_stack, beta, d_out, causal=False, normalize=True, block=4096, carry=None):
    """(dq, dk, dv) as race_attention_vjp returns them (ra/backward.py:184-235).

    Causal ``carry`` = key_state of earlier rows: the rows given are then the TAIL of a longer
    sequence (nothing follows them, so the reverse scan's suffix carry starts at zero)."""
    qp, kp = _prep(q, k, normalize)
    num, den = num_den(qp, kp, v, w_stack, beta, causal, block, carry)
    t_tot = w_stack.shape[0]
    live = den > DEGENERATE_DEN_EPS
    sden = np.where(live, den, 1.0)
    out = np.where(live[:, None], num / sden[:, None], 0.0)
    # ra/backward.py:201-209 (cotangents of the averaged num / den, scaled by 1/T)
    dn = (np.where(live[:, None], d_out / sden[:, None], 0.0) / t_tot).astype(q.dtype, copy=False)
    dd = (np.where(live, -np.sum(d_out * out, axis=1) / sden, 0.0) / t_tot).astype(q.dtype, copy=False)
    w_c = w_stack.astype(q.dtype, copy=False)
    n, dv = q.shape[0], v.shape[1]
    f = t_tot << w_stack.shape[1]
    gq = np.zeros(q.shape)
    gk = np.zeros(k.shape)
    gv = np.zeros(v.shape)
    if not causal:
        # ra/backward.py:93-129
        s_a = np.zeros(f)
        s_b = np.zeros((f, dv))
        for lo in range(0, n, block):
            pk = features(kp[lo:lo + block], w_c, beta)
            s_a += pk.sum(axis=0, dtype=np.float64)
            s_b += pk.T @ v[lo:lo + block]
        a_c, b_c = s_a.astype(q.dtype), s_b.astype(q.dtype)
        ds_a = np.zeros(f)
        ds_b = np.zeros((f, dv))
        for lo in range(0, n, block):
            sl = slice(lo, lo + block)
            pq = features(qp[sl], w_c, beta)
            dphi = dn[sl] @ b_c.T + dd[sl][:, None] * a_c[None, :]
            gq[sl] = _feature_grad(qp[sl], w_c, beta, dphi)
            ds_b += pq.T @ dn[sl]
            ds_a += pq.T @ dd[sl]
        dsa_c, dsb_c = ds_a.astype(q.dtype), ds_b.astype(q.dtype)
        for lo in range(0, n, block):
            sl = slice(lo, lo + block)
            pk = features(kp[sl], w_c, beta)
            dphi = v[sl] @ dsb_c.T + dsa_c[None, :]
            gk[sl] = _feature_grad(kp[sl], w_c, beta, dphi)
            gv[sl] = pk @ dsb_c
    else:
        # ra/backward.py:132-181: forward carries, then a reverse suffix scan
        bounds = [(lo, min(lo + block, n)) for lo in range(0, n, block)]
        carries = []
        ca, cb = (np.zeros(f), np.zeros((f, dv))) if carry is None else (carry[0].copy(), carry[1].copy())
        for lo, hi in bounds:
            carries.append((ca.copy(), cb.copy()))
            pk = features(kp[lo:hi], w_c, beta).astype(np.float64)
            ca = ca + pk.sum(axis=0)
            cb = cb + pk.T @ v[lo:hi].astype(np.float64)
        sa = np.zeros(f)
        sb = np.zeros((f, dv))
        for idx in range(len(bounds) - 1, -1, -1):
            lo, hi = bounds[idx]
            a_in, b_in = carries[idx]
            pk = features(kp[lo:hi], w_c, beta).astype(np.float64)
            pq = features(qp[lo:hi], w_c, beta).astype(np.float64)
            vb = v[lo:hi].astype(np.float64)
            dnb, ddb = dn[lo:hi], dd[lo:hi]
            cum_a = a_in + np.cumsum(pk, axis=0)
            cum_b = b_in + np.cumsum(pk[:, :, None] * vb[:, None, :], axis=0)
            dphi_q = np.einsum("td,tfd->tf", dnb, cum_b) + ddb[:, None] * cum_a
            gq[lo:hi] = _feature_grad(qp[lo:hi], w_c, beta, dphi_q.astype(q.dtype))
            dca = pq * ddb[:, None]
            dcb = pq[:, :, None] * dnb[:, None, :]
            suf_a = np.cumsum(dca[::-1], axis=0)[::-1] + sa
            suf_b = np.cumsum(dcb[::-1], axis=0)[::-1] + sb
            dphi_k = suf_a + np.einsum("tfd,td->tf", suf_b, vb)
            gk[lo:hi] = _feature_grad(kp[lo:hi], w_c, beta, dphi_k.astype(k.dtype))
            gv[lo:hi] = np.einsum("tf,tfd->td", pk, suf_b)
            sa = sa + dca.sum(axis=0)
            sb = sb + dcb.sum(axis=0)
    if normalize:
        gq = unit_rows_vjp(q.astype(np.float64), gq)
        gk = unit_rows_vjp(k.astype(np.float64), gk)
    return gq.astype(q.dtype), gk.astype(k.dtype), gv.astype(v.dtype)


# --------------------------------------------------------------------------
# helpers used by the tests / CPU baseline
# --------------------------------------------------------------------------
def rel_err(a, b) -> float:
    """max|a-b| / max|b| (ra/acceptance.py:89-91)."""
    b = np.asarray(b, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), 1e-30)


def head_inputs(seed: int, n: int, d: int, heads: int, dtype=np.float32):
    """Synthetic Q, K, V, dO per head in the order of ra/bench.py:161-169."""
    rng = np.random.default_rng(np.random.SeedSequence(seed & 0xFFFFFFFFFFFFFFFF, spawn_key=(n,)))
    out = []
    for _ in range(heads):
        q = rng.standard_normal((n, d)).astype(dtype)
        k = rng.standard_normal((n, d)).astype(dtype)
        v = rng.standard_normal((n, d)).astype(dtype)
        g = rng.standard_normal((n, d)).astype(dtype)
        out.append((q, k, v, g))
    return out
