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


def chain_text(n_links: int, substeps: int = 4) -> str:
    """Scene text of a free snake of n_links capsules jointed end to end over a
    ground plane, each joint actuated (the maximum-size parity cases: B = n_links + 1,
    J = A = n_links − 1, C = 2·n_links capsule-end slots)."""
    lines = ["dt: 0.02", f"substeps: {substeps}", "gravity { z: -9.8 }", "friction: 0.8",
             'bodies { name: "Ground" frozen { all: true } colliders { plane {} } }']
    for i in range(n_links):
        lines.append(f'bodies {{ name: "L{i}" mass: 1 inertia {{ x: 0.1 y: 0.1 z: 0.1 }} '
                     f'colliders {{ rotation {{ y: 90 }} capsule {{ radius: 0.05 length: 0.3 }} }} }}')
    for i in range(1, n_links):
        lines.append(f'joints {{ name: "J{i}" parent: "L{i - 1}" child: "L{i}" stiffness: 2000 angular_damping: 2 '
                     f'parent_offset {{ x: 0.15 }} child_offset {{ x: -0.15 }} rotation {{ z: 90 }} '
                     f'angle_limit {{ min: -60 max: 60 }} }}')
        lines.append(f'actuators {{ name: "J{i}" joint: "J{i}" strength: 5 torque {{}} }}')
    for i in range(n_links):
        lines.append(f'collide_include {{ first: "L{i}" second: "Ground" }}')
    lines.append('defaults { qps { name: "L0" pos { z: 0.3 } } }')
    return "\n".join(lines)
