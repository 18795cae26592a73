"""fp64 CPU oracle of the Brax physics step (arXiv 2106.13281, Alg. 1).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import, call, link or execute
anything under oracle/.  The product path (paper_2106_13281_b200) never does,
and this package never imports the product path.

Pieces:
  textproto.py   protobuf-text parser (App. A format)
  system.py      schema, validation, contact-slot table (R19), default_qp, lint
  philox.py      Philox4x32-10 counter-based generator + brax_reset semantics
  brax_oracle.cpp the step itself (fp64 scalar C++, plus an op-counting twin)
  env.py         the NEXT-1 env epilogue: observation, reward, done, auto-reset,
                 goal tasks (R30-R36)
  diff.py        central finite differences of the step and of rollouts (NEXT-4 checks)

Parity unpinned: whole-scene trajectories of ant/humanoid/halfcheetah/grasp/
fetch have no closed form; they are pinned only by the invariants in
tests/test_oracle_pins.py (SURVEY §8(c).3 last row).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

from .system import (ANGLE, TORQUE, CyclicJointGraph, ParseError, System,  # noqa: F401
                     ValidationError, default_qp, parse_system, stability_lint)
from .philox import philox4x32_10, reset_qp  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "brax_oracle.cpp")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the C++ oracle with g++ (plain -O2, no fast-math, fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class _OBody(C.Structure):
    _fields_ = [("mass", C.c_double), ("inertia", C.c_double * 3), ("mpos", C.c_double * 3),
                ("mrot", C.c_double * 3), ("is_static", C.c_int32), ("rot_frozen", C.c_int32)]


class _OJoint(C.Structure):
    _fields_ = [("parent", C.c_int32), ("child", C.c_int32), ("dof", C.c_int32), ("act_kind", C.c_int32),
                ("act_offset", C.c_int32), ("pad_", C.c_int32),
                ("o_p", C.c_double * 3), ("o_c", C.c_double * 3), ("jp", C.c_double * 4), ("jc", C.c_double * 4),
                ("k", C.c_double), ("c_l", C.c_double), ("c_a", C.c_double), ("k_l", C.c_double),
                ("k_a", C.c_double), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("act_strength", C.c_double)]


class _OCollider(C.Structure):
    _fields_ = [("body", C.c_int32), ("kind", C.c_int32), ("end", C.c_int32), ("pad_", C.c_int32),
                ("pos", C.c_double * 3), ("rot", C.c_double * 4), ("radius", C.c_double),
                ("length", C.c_double), ("halfsize", C.c_double * 3)]


class _OSlot(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("pair", "type", "a", "b", "col_a", "col_b", "point", "pad_")]


class _OSys(C.Structure):
    _fields_ = [("nb", C.c_int32), ("nj", C.c_int32), ("ncol", C.c_int32), ("ns", C.c_int32),
                ("act_dim", C.c_int32), ("substeps", C.c_int32), ("dt", C.c_double),
                ("gravity", C.c_double * 3), ("mu", C.c_double), ("e", C.c_double), ("beta", C.c_double),
                ("bodies", C.POINTER(_OBody)), ("joints", C.POINTER(_OJoint)),
                ("colliders", C.POINTER(_OCollider)), ("slots", C.POINTER(_OSlot))]


class _OOpts(C.Structure):
    _fields_ = [("combine_sum", C.c_int32), ("pad_", C.c_int32), ("amb_d", C.c_double),
                ("amb_jn", C.c_double), ("amb_par", C.c_double), ("amb_angle", C.c_double)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            dp = C.POINTER(C.c_double)
            lib.oracle_step.argtypes = [C.POINTER(_OSys), C.POINTER(_OOpts), C.c_int64, C.c_int64, dp, dp, dp, dp,
                                        dp, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), dp,
                                        dp]
            lib.oracle_step.restype = C.c_int
            lib.oracle_step_f32.argtypes = lib.oracle_step.argtypes
            lib.oracle_step_f32.restype = C.c_int
            lib.oracle_count_ops.argtypes = [C.POINTER(_OSys), C.POINTER(_OOpts), C.c_int64, C.c_int64, dp, dp, dp,
                                             dp, dp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
            lib.oracle_count_ops.restype = C.c_int
            lib.oracle_count_ops_lean.argtypes = lib.oracle_count_ops.argtypes
            lib.oracle_count_ops_lean.restype = C.c_int
            lib.oracle_slot_geometry.argtypes = [C.POINTER(_OSys), C.c_int32, dp, dp, dp, dp, dp]
            lib.oracle_slot_geometry.restype = C.c_int
            _lib = lib
    return _lib


_KIND = {"sphere": 0, "capsule": 1, "box": 2, "plane": 3}


class Oracle:
    """A parsed scene bound to the C++ oracle step."""

    def __init__(self, text_or_system, *, combine_sum: bool = False, amb_d: float = 1e-5,
                 amb_jn: float = 1e-5, amb_par: float = 1e-6, amb_angle: float = 1e-4):
        self.sys = text_or_system if isinstance(text_or_system, System) else parse_system(text_or_system)
        s = self.sys
        self._bodies = (_OBody * max(1, len(s.bodies)))()
        for i, b in enumerate(s.bodies):
            ob = self._bodies[i]
            ob.mass = b.mass
            ob.inertia[:] = list(b.inertia)
            ob.mpos[:] = list(1.0 - b.frozen_pos)
            ob.mrot[:] = list(1.0 - b.frozen_rot)
            ob.is_static = int(b.is_static)
            ob.rot_frozen = int(np.all(b.frozen_rot == 1))
        self._joints = (_OJoint * max(1, len(s.joints)))()
        act_of = {a.joint: a for a in s.actuators}
        for i, j in enumerate(s.joints):
            oj = self._joints[i]
            oj.parent, oj.child, oj.dof = j.parent, j.child, j.dof
            oj.o_p[:] = list(j.parent_offset)
            oj.o_c[:] = list(j.child_offset)
            oj.jp[:] = list(j.rotation)
            # J_c = conj(reference_rotation) ⊗ rotation
            from .system import qconj, qmul
            oj.jc[:] = list(qmul(qconj(j.reference_rotation), j.rotation))
            oj.k, oj.c_l, oj.c_a = j.stiffness, j.spring_damping, j.angular_damping
            oj.k_l, oj.k_a = j.limit_stiffness, j.angular_stiffness
            lo = np.zeros(3)
            hi = np.zeros(3)
            lo[: j.dof] = j.limits[:, 0]
            hi[: j.dof] = j.limits[:, 1]
            oj.lo[:] = list(lo)
            oj.hi[:] = list(hi)
            a = act_of.get(i)
            oj.act_kind = -1 if a is None else a.kind
            oj.act_offset = 0 if a is None else a.act_offset
            oj.act_strength = 0.0 if a is None else a.strength
        self._cols = (_OCollider * max(1, len(s.colliders)))()
        for i, c in enumerate(s.colliders):
            oc = self._cols[i]
            oc.body, oc.kind, oc.end = c.body, _KIND[c.kind], c.end
            oc.pos[:] = list(c.pos)
            oc.rot[:] = list(c.rot)
            oc.radius, oc.length = c.radius, c.length
            oc.halfsize[:] = list(c.halfsize)
        self._slots = (_OSlot * max(1, len(s.slots)))()
        for i, sl in enumerate(s.slots):
            o = self._slots[i]
            o.pair, o.type, o.a, o.b, o.col_a, o.col_b, o.point = sl
        self._sys = _OSys(nb=len(s.bodies), nj=len(s.joints), ncol=len(s.colliders), ns=len(s.slots),
                          act_dim=s.act_dim, substeps=s.substeps, dt=s.dt, mu=s.friction, e=s.elasticity,
                          beta=s.baumgarte)
        self._sys.gravity[:] = list(s.gravity)
        self._sys.bodies = self._bodies
        self._sys.joints = self._joints
        self._sys.colliders = self._cols
        self._sys.slots = self._slots
        self._opts = _OOpts(combine_sum=int(combine_sum), amb_d=amb_d, amb_jn=amb_jn, amb_par=amb_par,
                            amb_angle=amb_angle)

    # ------------------------------------------------------------------
    @property
    def n_bodies(self):
        return len(self.sys.bodies)

    @property
    def act_dim(self):
        return self.sys.act_dim

    @property
    def n_slots(self):
        return len(self.sys.slots)

    def default_qp(self):
        return default_qp(self.sys)

    def batch_default_qp(self, n):
        d = self.default_qp()
        return {k: np.broadcast_to(v, (n,) + v.shape).copy() for k, v in d.items()}

    def step(self, qp, action=None, *, threads: int = 1, fp32: bool = False, contact_dv: bool = False,
             contact_dp: bool = False):
        """One Brax step (substeps × Alg. 1) on a batch; returns (qp_out, extras).

        qp: dict of arrays pos [n,B,3], rot [n,B,4], vel [n,B,3], ang [n,B,3]
        (any float dtype; promoted to fp64).  action: [n, act_dim] or None.
        extras: contact_active [n,C] u8, status [n] u32, ambiguous [n] bool, and with
        contact_dv=True "contact_dv" [n,B,6]: the last substep's collision-integrator
        velocity change (Δv, Δω) per body; with contact_dp=True "contact_dp" [n,B,6]: that
        change summed over the step's substeps (brax_step_extras.contact_dp).
        fp32=True runs the same code in fp32 arithmetic: a diagnostic of the fp32
        rounding floor of the method, never a parity reference."""
        lib = _load()
        out = {k: np.ascontiguousarray(qp[k], dtype=np.float64).copy() for k in ("pos", "rot", "vel", "ang")}
        n = out["pos"].shape[0]
        B = self.n_bodies
        assert out["pos"].shape == (n, B, 3) and out["rot"].shape == (n, B, 4)
        A = self.act_dim
        if A:
            act = np.ascontiguousarray(action, dtype=np.float64).reshape(n, A)
        else:
            act = np.zeros((n, 1))
        ca = np.zeros((n, self.n_slots), dtype=np.uint8)
        status = np.zeros(n, dtype=np.uint32)
        amb = np.zeros(n, dtype=np.uint8)
        dp = C.POINTER(C.c_double)
        ca_ptr = ca.ctypes.data_as(C.POINTER(C.c_uint8)) if self.n_slots else None
        cdv = np.zeros((n, B, 6)) if contact_dv else None
        cdp = np.zeros((n, B, 6)) if contact_dp else None

        def run(e0, e1):
            fn = lib.oracle_step_f32 if fp32 else lib.oracle_step
            rc = fn(C.byref(self._sys), C.byref(self._opts), e0, e1,
                                 out["pos"].ctypes.data_as(dp), out["rot"].ctypes.data_as(dp),
                                 out["vel"].ctypes.data_as(dp), out["ang"].ctypes.data_as(dp),
                                 act.ctypes.data_as(dp), ca_ptr,
                                 status.ctypes.data_as(C.POINTER(C.c_uint32)),
                                 amb.ctypes.data_as(C.POINTER(C.c_uint8)),
                                 cdv.ctypes.data_as(dp) if cdv is not None else None,
                                 cdp.ctypes.data_as(dp) if cdp is not None else None)
            assert rc == 0

        if threads <= 1 or n < 2 * threads:
            run(0, n)
        else:  # ctypes releases the GIL: envs are partitioned across host threads
            bounds = np.linspace(0, n, threads + 1).astype(int)
            ths = [threading.Thread(target=run, args=(int(bounds[t]), int(bounds[t + 1])))
                   for t in range(threads)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
        ex = {"contact_active": ca, "status": status, "ambiguous": amb.astype(bool)}
        if cdv is not None:
            ex["contact_dv"] = cdv
        if cdp is not None:
            ex["contact_dp"] = cdp
        return out, ex

    def rollout(self, qp, actions, *, threads: int = 1):
        """Apply step T times; actions [T, n, A] (or None).  Returns the final qp and
        the per-env OR of the ambiguity flags and status bits over the run."""
        amb = None
        status = None
        T = len(actions) if actions is not None else 0
        for t in range(T):
            qp, ex = self.step(qp, actions[t], threads=threads)
            amb = ex["ambiguous"] if amb is None else (amb | ex["ambiguous"])
            status = ex["status"] if status is None else (status | ex["status"])
        return qp, {"ambiguous": amb, "status": status}

    def count_ops(self, qp, action=None, *, lean: bool = False):
        """Algorithmic (flops, mufu) summed over the batch for one step.
        lean=True: the second convention — operations made exactly neutral by the scene
        (unit masks, isotropic inertia, zero damping, zero collider offsets / identity
        collider rotations) are not counted."""
        lib = _load()
        out = {k: np.ascontiguousarray(qp[k], dtype=np.float64).copy() for k in ("pos", "rot", "vel", "ang")}
        n = out["pos"].shape[0]
        A = self.act_dim
        act = np.ascontiguousarray(action, dtype=np.float64).reshape(n, A) if A else np.zeros((n, 1))
        fl = C.c_uint64()
        mu = C.c_uint64()
        dp = C.POINTER(C.c_double)
        fn = lib.oracle_count_ops_lean if lean else lib.oracle_count_ops
        rc = fn(C.byref(self._sys), C.byref(self._opts), 0, n,
                                  out["pos"].ctypes.data_as(dp), out["rot"].ctypes.data_as(dp),
                                  out["vel"].ctypes.data_as(dp), out["ang"].ctypes.data_as(dp),
                                  act.ctypes.data_as(dp), C.byref(fl), C.byref(mu))
        assert rc == 0
        return int(fl.value), int(mu.value)

    def slot_geometry(self, slot, pos, rot):
        """Narrowphase (d, n, pt, near_parallel) of one slot for one env's [B,3]/[B,4] pose."""
        lib = _load()
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        rot = np.ascontiguousarray(rot, dtype=np.float64)
        d = C.c_double()
        n = np.zeros(3)
        pt = np.zeros(3)
        dp = C.POINTER(C.c_double)
        par = lib.oracle_slot_geometry(C.byref(self._sys), slot, pos.ctypes.data_as(dp), rot.ctypes.data_as(dp),
                                       C.byref(d), n.ctypes.data_as(dp), pt.ctypes.data_as(dp))
        return d.value, n, pt, bool(par)

    def reset(self, n, seed, vel_noise=0.0, ang_noise=0.0):
        return reset_qp(self.sys, self.default_qp(), n, seed, vel_noise, ang_noise)


def load_scene(name: str) -> str:
    """Scene text from scenes/<name>.bxc (repo root)."""
    path = os.path.join(os.path.dirname(_HERE), "scenes", f"{name}.bxc")
    with open(path) as f:
        return f.read()
