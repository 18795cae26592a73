"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
1, 2, 3") and the brax_reset semantics (TEST INFRASTRUCTURE).

Oracle-side copy: the CUDA reset kernel implements the same counter-based
generator independently (the task's "each side implements the same
counter-based generator").  Pinned by the Random123 known-answer vectors in
tests/golden/philox4x32_10_kat.txt.

reset (SURVEY §8(c).1 brax_reset; SPEC.md:352-360 reset noise):
  qp = default_qp broadcast to n envs; then for every non-static body b,
  v += M_pos ⊙ σ_v·u(env, b, 0) and ω += M_rot ⊙ σ_ω·u(env, b, 1), where
  u(e, b, f)_k = (x_k >> 8)·2⁻²⁴·2 − 1 for the first three 32-bit outputs x_k of
  Philox4x32-10 with key = (seed mod 2³², seed >> 32), counter = (e, b, f, 0).
Env auto-reset (NEXT-1): the k-th reset of env e draws from counter
(e, b, f, k), so k = 0 is brax_reset itself; e is the env's global index.
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def _round(ctr, key):
    p0 = M0 * ctr[0]
    p1 = M1 * ctr[2]
    hi0, lo0 = (p0 >> 32) & MASK, p0 & MASK
    hi1, lo1 = (p1 >> 32) & MASK, p1 & MASK
    return [hi1 ^ ctr[1] ^ key[0], lo1, hi0 ^ ctr[3] ^ key[1], lo0]


def philox4x32_10(ctr, key):
    """ctr: 4 uint32, key: 2 uint32 -> 4 uint32 (10 rounds, key bumped between rounds)."""
    ctr = [int(c) & MASK for c in ctr]
    key = [int(k) & MASK for k in key]
    for r in range(10):
        if r:
            key = [(key[0] + W0) & MASK, (key[1] + W1) & MASK]
        ctr = _round(ctr, key)
    return ctr


def uniform_pm1(x: int) -> float:
    """u = (x >> 8)·2⁻²⁴·2 − 1 ∈ [−1, 1)."""
    return ((x >> 8) * 2.0 ** -24) * 2.0 - 1.0


def reset_qp(sys, dqp, n: int, seed: int, vel_noise: float, ang_noise: float, *, env_ids=None, episode=None):
    """default_qp + noise for n envs; env_ids [n] global env indices (default 0..n-1),
    episode [n] reset counts (default 0)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    key = (seed & MASK, seed >> 32)
    B = len(sys.bodies)
    env_ids = np.arange(n) if env_ids is None else np.asarray(env_ids)
    episode = np.zeros(n, dtype=np.int64) if episode is None else np.asarray(episode)
    out = {k: np.broadcast_to(v, (n,) + v.shape).copy() for k, v in dqp.items()}
    for e in range(n):
        for b, body in enumerate(sys.bodies):
            if body.is_static:
                continue
            xv = philox4x32_10((int(env_ids[e]), b, 0, int(episode[e])), key)
            xw = philox4x32_10((int(env_ids[e]), b, 1, int(episode[e])), key)
            for k in range(3):
                out["vel"][e, b, k] += (1.0 - body.frozen_pos[k]) * vel_noise * uniform_pm1(xv[k])
                out["ang"][e, b, k] += (1.0 - body.frozen_rot[k]) * ang_noise * uniform_pm1(xw[k])
    assert out["pos"].shape == (n, B, 3)
    return out


ACT_TAG = 0x41435431  # "ACT1"


def random_actions(n: int, act_dim: int, n_steps: int, seed: int, env_offset: int = 0, step0: int = 0):
    """NEXT-2 on-device random actions (include/brax_b200.h brax_random_actions):
    a[t, i, k] = u(x_(k mod 4)), x = Philox4x32-10(key = seed, counter =
    (env_offset + i, step0 + t, k // 4, ACT_TAG)); returns [n_steps, n, act_dim] fp64
    (every value is exactly representable in fp32)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    key = (seed & MASK, seed >> 32)
    out = np.zeros((n_steps, n, act_dim))
    for t in range(n_steps):
        for i in range(n):
            for g in range((act_dim + 3) // 4):
                x = philox4x32_10(((env_offset + i) & MASK, (step0 + t) & MASK, g, ACT_TAG), key)
                for j in range(4):
                    if 4 * g + j < act_dim:
                        out[t, i, 4 * g + j] = uniform_pm1(x[j])
    return out
