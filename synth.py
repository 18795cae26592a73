"""Seeded synthetic input generators shared by tests/, bench.py and smoke().

Holds none of the method's arithmetic: only random numbers (NumPy PCG64) with
the shapes and distributions of the paper's workloads:
random actions U(−1, 1) per (step, env, dof) — "random actions" of the
benchmark envs — and the uniform velocity kicks used to diversify states.
Both the oracle and the CUDA path receive exactly these arrays (cast to fp32).
"""
from __future__ import annotations

import numpy as np


def actions(seed: int, T: int, n: int, act_dim: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """[T, n, act_dim] fp32, iid U(lo, hi)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(lo, hi, size=(T, n, act_dim)).astype(np.float32)


def velocity_kicks(seed: int, n: int, n_bodies: int, vel: float, ang: float):
    """Additive velocity / angular-velocity kicks [n, B, 3] each, U(−vel, vel), U(−ang, ang), fp64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.uniform(-vel, vel, size=(n, n_bodies, 3)),
            rng.uniform(-ang, ang, size=(n, n_bodies, 3)))


def sample_envs(seed: int, n: int, k: int) -> np.ndarray:
    """k distinct env indices out of n, sorted (for sampled full-size parity)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.sort(rng.choice(n, size=min(k, n), replace=False))


def to_f32(qp):
    return {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in qp.items()}
