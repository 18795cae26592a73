"""Directional derivatives of the oracle step (NEXT-4) — TEST INFRASTRUCTURE.

The derivative of one step along a tangent (dq, da) is defined as
    J·v = lim_{ε→0} (step(x + εv) − step(x − εv)) / 2ε
and evaluated here by that central difference in fp64 (PAPER.md:5, :38, :195-203
"differentiable"; SPEC.md:91-136 checks gradients against central differences the
same way).  Away from the step's kinks (contact activation, clamps, friction-cone
regime changes, the ±π wrap of the angles) the truncation error is O(ε²) and the
rounding error O(1e-16/ε).  `kink` flags envs whose ± evaluations differ in a
contact's activity or whose two step sizes disagree: there the derivative is a
convention (R35), not a limit, and parity is not checked.
"""
from __future__ import annotations

import numpy as np

FIELDS = ("pos", "rot", "vel", "ang")


def _axpy(qp, s, dq):
    return {k: np.asarray(qp[k], dtype=np.float64) + s * np.asarray(dq[k], dtype=np.float64) for k in FIELDS}


def jvp_fd(o, qp, action, dq, da, eps=1e-6, threads=1):
    """Central difference of Oracle `o`'s step along (dq, da); returns (J·v, kink)."""
    A = o.act_dim
    a = None if A == 0 else np.asarray(action, dtype=np.float64)
    dav = None if A == 0 else np.asarray(da, dtype=np.float64)

    def f(s):
        out, ex = o.step(_axpy(qp, s, dq), None if A == 0 else a + s * dav, threads=threads)
        return out, ex

    def cd(e):
        p, exp_ = f(e)
        m, exm = f(-e)
        return {k: (p[k] - m[k]) / (2 * e) for k in FIELDS}, exp_, exm

    j1, exp_, exm = cd(eps)
    j2, _, _ = cd(eps * 4)
    n = qp["pos"].shape[0]
    kink = np.zeros(n, dtype=bool)
    if o.n_slots:
        kink |= np.any(exp_["contact_active"] != exm["contact_active"], axis=1)
    kink |= exp_["ambiguous"] | exm["ambiguous"]
    for k in FIELDS:
        d = np.abs(j1[k] - j2[k]).reshape(n, -1).max(1)
        scale = 1.0 + np.abs(j1[k]).reshape(n, -1).max(1)
        kink |= d > 1e-5 * scale
    return j1, kink


def jacobian_fd(o, qp, action, eps=1e-6, threads=1):
    """∂Q_out/∂(Q_in, a) per env by central differences, [n, 13B, 13B + A]: rows and
    columns ordered pos | rot | vel | ang (each [B][w] flattened) then actions.
    Also returns the per-env kink flag (OR over columns)."""
    n, B, A = qp["pos"].shape[0], o.n_bodies, o.act_dim
    widths = {"pos": 3, "rot": 4, "vel": 3, "ang": 3}
    K = 13 * B + A
    J = np.zeros((n, 13 * B, K))
    kink = np.zeros(n, dtype=bool)
    zero = {k: np.zeros_like(np.asarray(qp[k], dtype=np.float64)) for k in FIELDS}
    col = 0
    for k in FIELDS:
        for b in range(B):
            for c in range(widths[k]):
                dq = {f: v.copy() for f, v in zero.items()}
                dq[k][:, b, c] = 1.0
                j, kk = jvp_fd(o, qp, action, dq, None if A == 0 else np.zeros((n, A)), eps, threads)
                J[:, :, col] = np.concatenate([j[f].reshape(n, -1) for f in FIELDS], 1)
                kink |= kk
                col += 1
    for i in range(A):
        da = np.zeros((n, A))
        da[:, i] = 1.0
        j, kk = jvp_fd(o, qp, action, zero, da, eps, threads)
        J[:, :, col] = np.concatenate([j[f].reshape(n, -1) for f in FIELDS], 1)
        kink |= kk
        col += 1
    return J, kink


def vjp_fd(o, qp, action, g_out, eps=1e-6, threads=1):
    """Cotangent of one step: (g_in, g_action) = Jᵀ·g_out per env (J from jacobian_fd)."""
    n, B, A = qp["pos"].shape[0], o.n_bodies, o.act_dim
    J, kink = jacobian_fd(o, qp, action, eps, threads)
    g = np.concatenate([np.asarray(g_out[f], dtype=np.float64).reshape(n, -1) for f in FIELDS], 1)
    gin = np.einsum("nok,no->nk", J, g)
    out, o_ = {}, 0
    for f, w in zip(FIELDS, (3, 4, 3, 3)):
        out[f] = gin[:, o_:o_ + B * w].reshape(n, B, w)
        o_ += B * w
    return out, (gin[:, o_:] if A else None), kink
