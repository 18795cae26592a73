"""B200-native batched Brax physics step (arXiv 2106.13281, §3 Alg. 1).

Thin ctypes binding over the C ABI in include/brax_b200.h (library
paper_2106_13281_b200/_lib/libbrax_b200.so, sm_100a).  Argument marshalling
only: every step of the physics runs in the library's CUDA kernels.  There is
no CPU fallback — importing fails loudly if the library is missing, and system
creation fails loudly without a CUDA device.

PyTorch is used for device memory and streams only:

    import torch, paper_2106_13281_b200 as bx
    sys = bx.System(open("scenes/ant.bxc").read())
    qp = sys.alloc_qp(8192)                     # dict of fp32 cuda tensors
    sys.reset(qp, seed=0, vel_noise=0.1, ang_noise=0.1)
    sys.step(qp, action, qp)                    # in-place is allowed
"""
from __future__ import annotations

import ctypes as C
import os

__all__ = [
    "BraxError", "System", "brax_config_parse", "brax_config_destroy", "brax_config_counts",
    "brax_config_slot_table", "brax_config_default_qp", "brax_system_create", "brax_system_destroy",
    "brax_system_get_info", "brax_system_slot_table", "brax_default_qp", "brax_reset", "brax_step",
    "brax_step_ex", "brax_rollout", "brax_qp", "brax_step_extras", "brax_system_info", "LIB_PATH", "lib",
    "brax_env_io", "brax_system_task_info", "brax_env_step", "brax_env_reset", "brax_env_observe",
    "brax_random_actions", "brax_rollout_random", "brax_env_step_random", "brax_step_jvp",
    "brax_step_vjp", "brax_config_from_desc", "brax_system_tune", "brax_config_desc", "brax_body_desc",
    "brax_joint_desc", "brax_actuator_desc", "brax_collider_desc", "brax_body_pair",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libbrax_b200.so")
# experiments only (A/B timing of two builds in one process tree): BRAX_LIB_PATH points at
# another in-tree build of the same library
LIB_PATH = os.environ.get("BRAX_LIB_PATH", LIB_PATH)
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2106_13281_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")
lib = C.CDLL(LIB_PATH)

STATUS = ["BRAX_OK", "BRAX_E_INVALID_ARGUMENT", "BRAX_E_PARSE", "BRAX_E_VALIDATION",
          "BRAX_E_CYCLIC_JOINT_GRAPH", "BRAX_E_UNSUPPORTED_PAIR", "BRAX_E_MISALIGNED", "BRAX_E_CUDA",
          "BRAX_E_OUT_OF_MEMORY"]


class BraxError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        self.detail = detail
        super().__init__(f"{self.name}: {detail}")


class brax_qp(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("rot", C.c_void_p), ("vel", C.c_void_p), ("ang", C.c_void_p)]


class brax_step_extras(C.Structure):
    _fields_ = [("status", C.c_void_p), ("contact_active", C.c_void_p), ("contact_dp", C.c_void_p)]


# programmatic config descriptors (brax_config_from_desc)
class brax_body_desc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("mass", C.c_double), ("inertia", C.c_double * 3),
                ("frozen_pos", C.c_double * 3), ("frozen_rot", C.c_double * 3), ("init_pos", C.c_double * 3),
                ("init_rot", C.c_double * 4)]


class brax_joint_desc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("parent", C.c_int32), ("child", C.c_int32),
                ("parent_offset", C.c_double * 3), ("child_offset", C.c_double * 3), ("rotation", C.c_double * 4),
                ("reference_rotation", C.c_double * 4), ("dof", C.c_int32), ("limit_lo", C.c_double * 3),
                ("limit_hi", C.c_double * 3), ("stiffness", C.c_double), ("spring_damping", C.c_double),
                ("angular_damping", C.c_double), ("limit_stiffness", C.c_double),
                ("angular_stiffness", C.c_double)]


class brax_actuator_desc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("joint", C.c_int32), ("kind", C.c_int32), ("strength", C.c_double)]


class brax_collider_desc(C.Structure):
    _fields_ = [("body", C.c_int32), ("shape", C.c_int32), ("pos", C.c_double * 3), ("rot", C.c_double * 4),
                ("radius", C.c_double), ("length", C.c_double), ("halfsize", C.c_double * 3),
                ("capsule_end", C.c_int32)]


class brax_body_pair(C.Structure):
    _fields_ = [("first", C.c_int32), ("second", C.c_int32)]


class brax_config_desc(C.Structure):
    _fields_ = [("dt", C.c_double), ("substeps", C.c_int32), ("gravity", C.c_double * 3),
                ("friction", C.c_double), ("elasticity", C.c_double), ("baumgarte_erp", C.c_double),
                ("n_bodies", C.c_int32), ("n_joints", C.c_int32), ("n_actuators", C.c_int32),
                ("n_colliders", C.c_int32), ("n_pairs", C.c_int32),
                ("bodies", C.POINTER(brax_body_desc)), ("joints", C.POINTER(brax_joint_desc)),
                ("actuators", C.POINTER(brax_actuator_desc)), ("colliders", C.POINTER(brax_collider_desc)),
                ("pairs", C.POINTER(brax_body_pair))]


class brax_env_io(C.Structure):
    _fields_ = [("obs", C.c_void_p), ("reward", C.c_void_p), ("done", C.c_void_p), ("steps", C.c_void_p),
                ("episode", C.c_void_p), ("seed", C.c_uint64), ("env_offset", C.c_int64)]


class brax_random_actions(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("env_offset", C.c_int64), ("step0", C.c_int64)]


class brax_system_info(C.Structure):
    _fields_ = [("n_bodies", C.c_int32), ("n_dynamic", C.c_int32), ("n_joints", C.c_int32),
                ("act_dim", C.c_int32), ("n_contact_slots", C.c_int32), ("substeps", C.c_int32),
                ("dt", C.c_float), ("warps_per_block", C.c_int32), ("n_lint_warnings", C.c_int32),
                ("smem_bytes", C.c_int32)]


_P = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_SIGS = {
    "brax_config_parse": ([C.c_char_p, C.c_size_t, C.POINTER(_P)], C.c_int),
    "brax_config_destroy": ([_P], None),
    "brax_config_from_desc": ([C.POINTER(brax_config_desc), C.POINTER(_P)], C.c_int),
    "brax_system_tune": ([_P, brax_qp, _P, C.c_int64, _P], C.c_int),
    "brax_config_counts": ([_P, _i32p, _i32p, _i32p, _i32p], C.c_int),
    "brax_config_slot_table": ([_P, _i32p], C.c_int),
    "brax_config_default_qp": ([_P, _P, _P], C.c_int),
    "brax_system_create": ([_P, C.c_int, C.POINTER(_P)], C.c_int),
    "brax_system_destroy": ([_P], None),
    "brax_system_get_info": ([_P, C.POINTER(brax_system_info)], C.c_int),
    "brax_system_slot_table": ([_P, _i32p], C.c_int),
    "brax_system_lint_warning": ([_P, C.c_int32], C.c_char_p),
    "brax_system_set_tracing": ([_P, C.c_int], C.c_int),
    "brax_system_phase_cycles": ([_P, C.POINTER(C.c_uint64)], C.c_int),
    "brax_system_set_autotune": ([_P, C.c_int], C.c_int),
    "brax_system_launch_config": ([_P, C.c_int64, C.POINTER(C.c_int32)], C.c_int),
    "brax_default_qp": ([_P, _P, _P, _P, _P], C.c_int),
    "brax_reset": ([_P, brax_qp, C.c_int64, C.c_uint64, C.c_float, C.c_float, _P], C.c_int),
    "brax_step": ([_P, brax_qp, _P, brax_qp, C.c_int64, _P], C.c_int),
    "brax_step_ex": ([_P, brax_qp, _P, brax_qp, C.c_int64, C.POINTER(brax_step_extras), _P], C.c_int),
    "brax_rollout": ([_P, brax_qp, _P, C.c_int64, brax_qp, C.c_int64, C.POINTER(brax_step_extras), _P], C.c_int),
    "brax_system_task_info": ([_P, _i32p], C.c_int),
    "brax_step_jvp": ([_P, brax_qp, _P, brax_qp, _P, brax_qp, brax_qp, C.c_int64, _P], C.c_int),
    "brax_step_vjp": ([_P, brax_qp, _P, brax_qp, brax_qp, _P, C.c_int64, _P], C.c_int),
    "brax_rollout_random": ([_P, brax_qp, C.c_int64, brax_qp, C.c_int64, C.POINTER(brax_random_actions),
                             C.POINTER(brax_step_extras), _P], C.c_int),
    "brax_env_step_random": ([_P, brax_qp, C.c_int64, brax_qp, C.c_int64, C.POINTER(brax_random_actions),
                              C.POINTER(brax_env_io), _P], C.c_int),
    "brax_env_step": ([_P, brax_qp, _P, C.c_int64, brax_qp, C.c_int64, C.POINTER(brax_env_io), _P], C.c_int),
    "brax_env_reset": ([_P, brax_qp, C.c_int64, C.POINTER(brax_env_io), _P], C.c_int),
    "brax_env_observe": ([_P, brax_qp, C.c_int64, _P, _P], C.c_int),
    "brax_status_string": ([C.c_int], C.c_char_p),
    "brax_last_error_detail": ([], C.c_char_p),
    "brax_abi_version": ([], C.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _check(status: int):
    if status != 0:
        raise BraxError(status, lib.brax_last_error_detail().decode())


# ---------------------------------------------------------------- same-name wrappers
def brax_config_parse(text: str) -> int:
    out = _P()
    raw = text.encode()
    _check(lib.brax_config_parse(raw, len(raw), C.byref(out)))
    return out.value


def brax_config_destroy(cfg: int) -> None:
    lib.brax_config_destroy(cfg)


def brax_config_from_desc(desc: "brax_config_desc") -> int:
    """desc: a filled brax_config_desc (its arrays must stay alive during the call)."""
    out = _P()
    _check(lib.brax_config_from_desc(C.byref(desc), C.byref(out)))
    return out.value


def brax_system_tune(sys: int, qp_in, action, n_envs: int, stream=None) -> None:
    _check(lib.brax_system_tune(sys, _qp(qp_in), None if action is None else action.data_ptr(), n_envs,
                                _stream(stream)))


def brax_config_counts(cfg: int):
    v = [C.c_int32() for _ in range(4)]
    _check(lib.brax_config_counts(cfg, *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)  # (n_bodies, n_joints, act_dim, n_slots)


def brax_config_slot_table(cfg: int):
    import numpy as np
    n_slots = brax_config_counts(cfg)[3]
    out = np.zeros((n_slots, 7), dtype=np.int32)
    _check(lib.brax_config_slot_table(cfg, out.ctypes.data_as(_i32p)))
    return out


def brax_config_default_qp(cfg: int):
    import numpy as np
    B = brax_config_counts(cfg)[0]
    pos = np.zeros((B, 3))
    rot = np.zeros((B, 4))
    _check(lib.brax_config_default_qp(cfg, pos.ctypes.data, rot.ctypes.data))
    return pos, rot


def brax_system_create(cfg: int, cuda_device: int = 0) -> int:
    out = _P()
    _check(lib.brax_system_create(cfg, cuda_device, C.byref(out)))
    return out.value


def brax_system_destroy(sys: int) -> None:
    lib.brax_system_destroy(sys)


def brax_system_get_info(sys: int) -> brax_system_info:
    info = brax_system_info()
    _check(lib.brax_system_get_info(sys, C.byref(info)))
    return info


def brax_system_slot_table(sys: int):
    import numpy as np
    info = brax_system_get_info(sys)
    out = np.zeros((info.n_contact_slots, 7), dtype=np.int32)
    _check(lib.brax_system_slot_table(sys, out.ctypes.data_as(_i32p)))
    return out


def brax_default_qp(sys: int):
    import numpy as np
    B = brax_system_get_info(sys).n_bodies
    arrs = {"pos": np.zeros((B, 3), np.float32), "rot": np.zeros((B, 4), np.float32),
            "vel": np.zeros((B, 3), np.float32), "ang": np.zeros((B, 3), np.float32)}
    _check(lib.brax_default_qp(sys, *[arrs[k].ctypes.data for k in ("pos", "rot", "vel", "ang")]))
    return arrs


def _qp(q) -> brax_qp:
    return brax_qp(*(int(q[k].data_ptr()) for k in ("pos", "rot", "vel", "ang")))


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def brax_reset(sys: int, qp_out, n_envs: int, seed: int, vel_noise: float = 0.0, ang_noise: float = 0.0,
               stream=None) -> None:
    _check(lib.brax_reset(sys, _qp(qp_out), n_envs, seed & 0xFFFFFFFFFFFFFFFF, vel_noise, ang_noise,
                          _stream(stream)))


def brax_step(sys: int, qp_in, action, qp_out, n_envs: int, stream=None) -> None:
    _check(lib.brax_step(sys, _qp(qp_in), None if action is None else action.data_ptr(), _qp(qp_out), n_envs,
                         _stream(stream)))


def _extras(status, contact_active, contact_dp=None):
    if status is None and contact_active is None and contact_dp is None:
        return None
    return brax_step_extras(None if status is None else status.data_ptr(),
                            None if contact_active is None else contact_active.data_ptr(),
                            None if contact_dp is None else contact_dp.data_ptr())


def brax_step_ex(sys: int, qp_in, action, qp_out, n_envs: int, status=None, contact_active=None,
                 stream=None, contact_dp=None) -> None:
    x = _extras(status, contact_active, contact_dp)
    _check(lib.brax_step_ex(sys, _qp(qp_in), None if action is None else action.data_ptr(), _qp(qp_out), n_envs,
                            None if x is None else C.byref(x), _stream(stream)))


def brax_rollout(sys: int, qp_in, actions, n_steps: int, qp_out, n_envs: int, status=None, contact_active=None,
                 stream=None, contact_dp=None) -> None:
    x = _extras(status, contact_active, contact_dp)
    _check(lib.brax_rollout(sys, _qp(qp_in), None if actions is None else actions.data_ptr(), n_steps,
                            _qp(qp_out), n_envs, None if x is None else C.byref(x), _stream(stream)))


def _ptr(t):
    return None if t is None else int(t.data_ptr())


def _env_io(obs, reward, done, steps, episode, seed, env_offset):
    return brax_env_io(_ptr(obs), _ptr(reward), _ptr(done), _ptr(steps), _ptr(episode),
                       int(seed) & 0xFFFFFFFFFFFFFFFF, int(env_offset))


def brax_rollout_random(sys: int, qp_in, n_steps: int, qp_out, n_envs: int, seed: int, env_offset: int = 0,
                        step0: int = 0, status=None, contact_active=None, stream=None) -> None:
    ra = brax_random_actions(int(seed) & 0xFFFFFFFFFFFFFFFF, int(env_offset), int(step0))
    x = _extras(status, contact_active)
    _check(lib.brax_rollout_random(sys, _qp(qp_in), n_steps, _qp(qp_out), n_envs, C.byref(ra),
                                   None if x is None else C.byref(x), _stream(stream)))


def brax_env_step_random(sys: int, qp_in, n_steps: int, qp_out, n_envs: int, obs, reward, done, steps, episode,
                         seed: int = 0, env_offset: int = 0, act_seed: int = 0, step0: int = 0,
                         stream=None) -> None:
    io = _env_io(obs, reward, done, steps, episode, seed, env_offset)
    ra = brax_random_actions(int(act_seed) & 0xFFFFFFFFFFFFFFFF, int(env_offset), int(step0))
    _check(lib.brax_env_step_random(sys, _qp(qp_in), n_steps, _qp(qp_out), n_envs, C.byref(ra), C.byref(io),
                                    _stream(stream)))


def _qp_or_null(q) -> brax_qp:
    if q is None:
        return brax_qp(None, None, None, None)
    return brax_qp(*(_ptr(q.get(k)) for k in ("pos", "rot", "vel", "ang")))


def brax_step_jvp(sys: int, qp_in, action, dqp_in, daction, qp_out, dqp_out, n_envs: int, stream=None) -> None:
    _check(lib.brax_step_jvp(sys, _qp(qp_in), _ptr(action), _qp_or_null(dqp_in), _ptr(daction), _qp(qp_out),
                             _qp(dqp_out), n_envs, _stream(stream)))


def brax_step_vjp(sys: int, qp_in, action, g_out, g_in, g_action, n_envs: int, stream=None) -> None:
    _check(lib.brax_step_vjp(sys, _qp(qp_in), _ptr(action), _qp_or_null(g_out), _qp(g_in), _ptr(g_action), n_envs,
                             _stream(stream)))


def brax_system_task_info(sys: int):
    out = (C.c_int32 * 4)()
    _check(lib.brax_system_task_info(sys, out))
    return dict(zip(("has_task", "obs_dim", "episode_length", "torso"), (int(x) for x in out)))


def brax_env_step(sys: int, qp_in, actions, n_steps: int, qp_out, n_envs: int, obs, reward, done, steps, episode,
                  seed: int = 0, env_offset: int = 0, stream=None) -> None:
    io = _env_io(obs, reward, done, steps, episode, seed, env_offset)
    _check(lib.brax_env_step(sys, _qp(qp_in), _ptr(actions), n_steps, _qp(qp_out), n_envs, C.byref(io),
                             _stream(stream)))


def brax_env_reset(sys: int, qp_out, n_envs: int, obs, steps, episode, seed: int = 0, env_offset: int = 0,
                   stream=None) -> None:
    io = _env_io(obs, None, None, steps, episode, seed, env_offset)
    _check(lib.brax_env_reset(sys, _qp(qp_out), n_envs, C.byref(io), _stream(stream)))


def brax_env_observe(sys: int, qp, n_envs: int, obs, stream=None) -> None:
    _check(lib.brax_env_observe(sys, _qp(qp), n_envs, _ptr(obs), _stream(stream)))


# ---------------------------------------------------------------- convenience object
class System:
    """A config parsed and turned into a device-resident system (owns both handles)."""

    def __init__(self, text: str = None, device: int = 0, *, desc: "brax_config_desc" = None):
        if (text is None) == (desc is None):
            raise ValueError("give exactly one of text or desc")
        self._cfg = brax_config_parse(text) if text is not None else brax_config_from_desc(desc)
        try:
            self._sys = brax_system_create(self._cfg, device)
        except Exception:
            brax_config_destroy(self._cfg)
            self._cfg = None
            raise
        self.device = device
        self.info = brax_system_get_info(self._sys)

    def __del__(self):
        try:
            if getattr(self, "_sys", None):
                brax_system_destroy(self._sys)
            if getattr(self, "_cfg", None):
                brax_config_destroy(self._cfg)
        except Exception:  # noqa: BLE001 — interpreter shutdown: the library may already be gone
            pass
        self._sys = self._cfg = None

    handle = property(lambda self: self._sys)
    n_bodies = property(lambda self: self.info.n_bodies)
    act_dim = property(lambda self: self.info.act_dim)
    n_slots = property(lambda self: self.info.n_contact_slots)
    substeps = property(lambda self: self.info.substeps)

    def lint(self):
        return [lib.brax_system_lint_warning(self._sys, i).decode() for i in range(self.info.n_lint_warnings)]

    def set_tracing(self, enable: bool = True):
        _check(lib.brax_system_set_tracing(self._sys, int(enable)))

    def set_autotune(self, enable: bool = True):
        _check(lib.brax_system_set_autotune(self._sys, int(enable)))

    def launch_config(self, n_envs: int):
        """dict(G, V, E, warps, regs, tuned, fixed_gather) of the next step launch of n_envs envs
        (see brax_system_launch_config)."""
        out = (C.c_int32 * 6)()
        _check(lib.brax_system_launch_config(self._sys, int(n_envs), out))
        d = dict(zip(("G", "V", "E", "warps", "regs"), (int(x) for x in out[:5])))
        d["tuned"], d["fixed_gather"], d["lean"] = int(out[5]) & 1, (int(out[5]) >> 1) & 1, (int(out[5]) >> 2) & 1
        return d

    def phase_cycles(self):
        """(prologue, joints+contacts, integrators, epilogue) SM cycles summed over blocks since the last call."""
        out = (C.c_uint64 * 4)()
        _check(lib.brax_system_phase_cycles(self._sys, out))
        return tuple(int(x) for x in out)

    def slot_table(self):
        return brax_system_slot_table(self._sys)

    def default_qp(self):
        return brax_default_qp(self._sys)

    def alloc_qp(self, n: int):
        import torch
        dev = torch.device("cuda", self.device)
        B = self.n_bodies
        return {"pos": torch.empty((n, B, 3), device=dev), "rot": torch.empty((n, B, 4), device=dev),
                "vel": torch.empty((n, B, 3), device=dev), "ang": torch.empty((n, B, 3), device=dev)}

    def reset(self, qp, seed: int = 0, vel_noise: float = 0.0, ang_noise: float = 0.0, stream=None):
        brax_reset(self._sys, qp, qp["pos"].shape[0], seed, vel_noise, ang_noise, stream)
        return qp

    def step(self, qp_in, action, qp_out=None, *, status=None, contact_active=None, contact_dp=None, stream=None):
        qp_out = qp_in if qp_out is None else qp_out
        n = qp_in["pos"].shape[0]
        if status is None and contact_active is None and contact_dp is None:
            brax_step(self._sys, qp_in, action, qp_out, n, stream)
        else:
            brax_step_ex(self._sys, qp_in, action, qp_out, n, status, contact_active, stream, contact_dp)
        return qp_out

    def tune(self, qp_in, action, *, stream=None):
        """brax_system_tune for qp_in's batch size (synchronises; not graph-capturable)."""
        brax_system_tune(self._sys, qp_in, action, qp_in["pos"].shape[0], stream)

    # ---- NEXT-1 env epilogue (needs a `task` block) ----
    def task_info(self):
        return brax_system_task_info(self._sys)

    def env_state(self, n: int):
        """Device buffers for an env batch: qp, steps [n] int32, episode [n] int32 (uint32 bits)."""
        import torch
        dev = torch.device("cuda", self.device)
        return {"qp": self.alloc_qp(n), "steps": torch.zeros(n, dtype=torch.int32, device=dev),
                "episode": torch.zeros(n, dtype=torch.int32, device=dev)}

    def env_reset(self, state, seed: int = 0, env_offset: int = 0, stream=None):
        """Episode-0 reset of state (env_state dict) in place; returns obs [n, obs_dim]."""
        import torch
        n = state["steps"].shape[0]
        obs = torch.empty((n, self.task_info()["obs_dim"]), device=state["steps"].device)
        brax_env_reset(self._sys, state["qp"], n, obs, state["steps"], state["episode"], seed, env_offset, stream)
        return obs

    def env_step(self, state, actions, seed: int = 0, env_offset: int = 0, stream=None):
        """actions [n, A] (one step) or [T, n, A]; advances state in place and returns
        dict(obs [T, n, obs_dim], reward [T, n], done [T, n] uint8) (T = 1 for one step)."""
        import torch
        n = state["steps"].shape[0]
        if actions is not None and actions.dim() == 2:
            actions = actions.unsqueeze(0)
        T = 1 if actions is None else actions.shape[0]
        dev = state["steps"].device
        out = {"obs": torch.empty((T, n, self.task_info()["obs_dim"]), device=dev),
               "reward": torch.empty((T, n), device=dev), "done": torch.empty((T, n), dtype=torch.uint8, device=dev)}
        brax_env_step(self._sys, state["qp"], actions, T, state["qp"], n, out["obs"], out["reward"], out["done"],
                      state["steps"], state["episode"], seed, env_offset, stream)
        return out

    def rollout_random(self, qp_in, n_steps: int, qp_out=None, *, seed: int = 0, env_offset: int = 0,
                       step0: int = 0, status=None, contact_active=None, stream=None):
        """n_steps steps in one launch with on-device random actions (NEXT-2)."""
        qp_out = qp_in if qp_out is None else qp_out
        brax_rollout_random(self._sys, qp_in, n_steps, qp_out, qp_in["pos"].shape[0], seed, env_offset, step0,
                            status, contact_active, stream)
        return qp_out

    # ---- NEXT-4 differentiable step (forward mode) ----
    def step_jvp(self, qp_in, action, dqp_in, daction=None, *, stream=None):
        """One step and its directional derivative: returns (qp_out, dqp_out)."""
        n = qp_in["pos"].shape[0]
        out, dout = self.alloc_qp(n), self.alloc_qp(n)
        brax_step_jvp(self._sys, qp_in, action, dqp_in, daction, out, dout, n, stream)
        return out, dout

    def step_vjp(self, qp_in, action, g_out, *, stream=None):
        """Cotangent of one step: returns (g_in qp dict, g_action [n, A] or None)."""
        import torch
        n = qp_in["pos"].shape[0]
        g_in = self.alloc_qp(n)
        g_a = torch.empty((n, self.act_dim), device=qp_in["pos"].device) if self.act_dim else None
        brax_step_vjp(self._sys, qp_in, action, g_out, g_in, g_a, n, stream)
        return g_in, g_a

    def rollout_vjp(self, qp0, actions, g_final, *, stream=None):
        """Reverse mode through a T-step rollout (APG's "gradient of the loss through a
        short trajectory"): forward T brax_step calls keeping every
        state on the device, then T brax_step_vjp calls backwards.  actions [T, n, A];
        g_final: cotangent of the final QP.  Returns (g_qp0, g_actions [T, n, A])."""
        import torch
        T = actions.shape[0] if actions is not None else 0
        states = [qp0]
        for t in range(T):
            nxt = self.alloc_qp(qp0["pos"].shape[0])
            self.step(states[-1], actions[t], nxt, stream=stream)
            states.append(nxt)
        g = g_final
        g_a = torch.zeros_like(actions) if (actions is not None and self.act_dim) else None
        for t in reversed(range(T)):
            g, ga = self.step_vjp(states[t], actions[t], g, stream=stream)
            if g_a is not None:
                g_a[t] = ga
        return g, g_a

    def step_jacobian(self, qp_in, action, *, stream=None):
        """∂Q_out/∂(Q_in, a) per env, [n, 13B, 13B + A] (rows and columns ordered
        pos | rot | vel | ang (env-major, body-major) then actions), one JVP launch
        per input coordinate."""
        import torch
        n, B, A = qp_in["pos"].shape[0], self.n_bodies, self.act_dim
        widths = {"pos": 3, "rot": 4, "vel": 3, "ang": 3}
        K = 13 * B + A
        jac = torch.empty((n, 13 * B, K), device=qp_in["pos"].device)
        zeros = {k: torch.zeros_like(v) for k, v in qp_in.items()}
        dz_a = torch.zeros_like(action) if A else None
        col = 0
        for k in ("pos", "rot", "vel", "ang"):
            for b in range(B):
                for c in range(widths[k]):
                    d = dict(zeros)
                    d[k] = torch.zeros_like(qp_in[k])
                    d[k][:, b, c] = 1.0
                    _, dout = self.step_jvp(qp_in, action, d, dz_a, stream=stream)
                    jac[:, :, col] = torch.cat([dout[f].reshape(n, -1) for f in ("pos", "rot", "vel", "ang")], 1)
                    col += 1
        for j in range(A):
            da = torch.zeros_like(action)
            da[:, j] = 1.0
            _, dout = self.step_jvp(qp_in, action, zeros, da, stream=stream)
            jac[:, :, col] = torch.cat([dout[f].reshape(n, -1) for f in ("pos", "rot", "vel", "ang")], 1)
            col += 1
        return jac

    def env_observe(self, qp, stream=None):
        import torch
        n = qp["pos"].shape[0]
        obs = torch.empty((n, self.task_info()["obs_dim"]), device=qp["pos"].device)
        brax_env_observe(self._sys, qp, n, obs, stream)
        return obs

    def rollout(self, qp_in, actions, qp_out=None, *, n_steps=None, status=None, contact_active=None,
                contact_dp=None, stream=None):
        qp_out = qp_in if qp_out is None else qp_out
        n = qp_in["pos"].shape[0]
        T = n_steps if n_steps is not None else actions.shape[0]
        brax_rollout(self._sys, qp_in, actions, T, qp_out, n, status, contact_active, stream, contact_dp)
        return qp_out
