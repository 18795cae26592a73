"""Oracle-side scene schema, validation, contact-slot table and default_qp
(TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package).

Everything here is fp64 numpy written straight from the paper and from the
readings of SURVEY.md §8(c) (listed in DESIGN.md).  It shares no code with
the library's C++ builder (paper_2106_13281_b200/csrc/system.cpp).

Citations: PAPER.md line numbers, section in parentheses.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .textproto import ParseError, parse_text

__all__ = [
    "ValidationError", "ParseError", "Body", "Collider", "Joint", "Actuator",
    "System", "parse_system", "euler_deg_to_quat", "SLOT_TYPES",
]

# Contact-slot type codes.  These integer values are part of the C-ABI
# contract documented in include/brax_b200.h (brax_slot_type); the oracle
# restates them here rather than importing anything from the library.
SPHERE_PLANE, CAPSULE_PLANE, BOX_PLANE, SPHERE_SPHERE, SPHERE_CAPSULE, CAPSULE_CAPSULE = range(6)
SLOT_TYPES = {
    "sphere_plane": SPHERE_PLANE, "capsule_plane": CAPSULE_PLANE, "box_plane": BOX_PLANE,
    "sphere_sphere": SPHERE_SPHERE, "sphere_capsule": SPHERE_CAPSULE,
    "capsule_capsule": CAPSULE_CAPSULE,
}
TORQUE, ANGLE = 0, 1


class ValidationError(ValueError):
    def __init__(self, path: str, msg: str):
        super().__init__(f"{path}: {msg}")
        self.path, self.msg = path, msg


class CyclicJointGraph(ValidationError):
    pass


# --------------------------------------------------------------------------
# quaternion helpers (w, x, y, z), Hamilton product — oracle's own copy
# --------------------------------------------------------------------------
def qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    ])


def qconj(q):
    return np.array([q[0], -q[1], -q[2], -q[3]])


def qrotate(q, v):
    """rotate(q, v) = v + w·t + u×t, u = (x,y,z), t = 2u×v."""
    u = np.asarray(q[1:4], dtype=float)
    t = 2.0 * np.cross(u, v)
    return np.asarray(v, dtype=float) + q[0] * t + np.cross(u, t)


def euler_deg_to_quat(deg):
    """E(θ) = qx(θ0) ⊗ qy(θ1) ⊗ qz(θ2): intrinsic X-Y-Z, the same convention
    whose angles the joint transformation extracts.  Degrees, as
    App. A's angle fields."""
    a = [math.radians(float(d)) for d in deg]
    qx = np.array([math.cos(a[0] / 2), math.sin(a[0] / 2), 0.0, 0.0])
    qy = np.array([math.cos(a[1] / 2), 0.0, math.sin(a[1] / 2), 0.0])
    qz = np.array([math.cos(a[2] / 2), 0.0, 0.0, math.sin(a[2] / 2)])
    return qmul(qmul(qx, qy), qz)


def euler_rad_to_quat(rad):
    return euler_deg_to_quat([math.degrees(r) for r in rad])


# --------------------------------------------------------------------------
# schema
# --------------------------------------------------------------------------
@dataclass
class Collider:
    body: int
    kind: str                       # sphere | capsule | box | plane
    pos: np.ndarray                 # local offset o_col
    rot: np.ndarray                 # local rotation r_col (quat)
    radius: float = 0.0
    length: float = 0.0
    end: int = 0                    # capsule end selector (R17): 0 both, +1, -1
    halfsize: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class Body:
    name: str
    mass: float
    inertia: np.ndarray
    frozen_pos: np.ndarray          # 1.0 = frozen axis (App. A `frozen`)
    frozen_rot: np.ndarray
    colliders: list
    init_pos: np.ndarray
    init_rot: np.ndarray

    @property
    def is_static(self) -> bool:
        return bool(np.all(self.frozen_pos == 1) and np.all(self.frozen_rot == 1))


@dataclass
class Joint:
    name: str
    parent: int
    child: int
    stiffness: float
    spring_damping: float
    angular_damping: float
    limit_stiffness: float
    angular_stiffness: float
    parent_offset: np.ndarray
    child_offset: np.ndarray
    rotation: np.ndarray            # quat J
    reference_rotation: np.ndarray  # quat Rf
    limits: np.ndarray              # [dof, 2] radians

    @property
    def dof(self) -> int:
        return int(self.limits.shape[0])


@dataclass
class Actuator:
    name: str
    joint: int
    strength: float
    kind: int                       # TORQUE | ANGLE
    act_offset: int = 0


@dataclass
class Goal:
    """Goal-directed task (grasp / fetch; R36): bring
    `obj` within `radius` of the frozen marker body `target`; the marker is then
    placed again."""
    obj: int
    target: int
    radius: float
    bonus: float
    range: np.ndarray               # marker placement half-extents around its default position


@dataclass
class Task:
    """Locomotion env epilogue (NEXT-1; R30-R35)."""
    torso: int
    forward: np.ndarray             # reward direction (world)
    survive_reward: float
    ctrl_cost: float
    healthy_z: tuple | None         # (min, max) torso height; outside -> done
    episode_length: int
    contact_obs: bool               # append clipped per-body contact Δv, Δω
    reset_vel_noise: float
    reset_ang_noise: float
    goal: Goal | None = None


@dataclass
class System:
    dt: float
    substeps: int
    gravity: np.ndarray
    friction: float
    elasticity: float
    baumgarte: float
    bodies: list
    joints: list
    actuators: list
    colliders: list                 # flat, global collider index order
    pairs: list                     # (colA, colB, type) after orientation
    slots: list                     # (pair, type, bodyA, bodyB, colA, colB, point)
    task: Task | None = None

    @property
    def act_dim(self) -> int:
        return sum(self.joints[a.joint].dof for a in self.actuators)

    @property
    def n_bodies(self) -> int:
        return len(self.bodies)

    @property
    def n_joint_dofs(self) -> int:
        return sum(j.dof for j in self.joints)

    @property
    def obs_dim(self) -> int:
        """torso z, quat (5) | joint angles (Σdof) | torso v, ω (6) | joint rates (Σdof) |
        goal (9, R36) | contacts (6B)."""
        if self.task is None:
            return 0
        return (11 + 2 * self.n_joint_dofs + (9 if self.task.goal is not None else 0)
                + (6 * len(self.bodies) if self.task.contact_obs else 0))

    def slot_table(self) -> np.ndarray:
        """Integer contact-slot table [C, 7] (pair, type, bodyA, bodyB, colA, colB, point)."""
        return np.array(self.slots, dtype=np.int32).reshape(-1, 7)

    def default_qp(self):
        return default_qp(self)

    def lint(self):
        return stability_lint(self)


def _vec3(node, path, default=(0.0, 0.0, 0.0)):
    v = list(default)
    for name, val, line, col in node:
        if name not in ("x", "y", "z") or not isinstance(val, float):
            raise ValidationError(f"{path}.{name}", "expected x/y/z numbers")
        v["xyz".index(name)] = val
    return np.array(v, dtype=float)


def _fields(node, path, allowed):
    seen = {}
    for name, val, line, col in node:
        if name not in allowed:
            raise ValidationError(f"{path}.{name}", "unknown field")
        seen.setdefault(name, []).append(val)
    return seen


def _one(seen, key, path, kind, default=None):
    vals = seen.get(key)
    if not vals:
        return default
    if len(vals) > 1:
        raise ValidationError(f"{path}.{key}", "field given more than once")
    v = vals[0]
    if kind == "num" and not isinstance(v, float):
        raise ValidationError(f"{path}.{key}", "expected a number")
    if kind == "str" and not isinstance(v, str):
        raise ValidationError(f"{path}.{key}", "expected a string")
    if kind == "msg" and not isinstance(v, list):
        raise ValidationError(f"{path}.{key}", "expected a { } block")
    return v


def parse_system(text: str) -> System:
    """Parse + validate a scene (App. A format)."""
    root = parse_text(text)
    top = _fields(root, "config", {
        "dt", "substeps", "gravity", "friction", "elasticity", "baumgarte_erp",
        "bodies", "joints", "actuators", "collide_include", "defaults", "task"})
    dt = _one(top, "dt", "config", "num", 0.01)
    substeps = _one(top, "substeps", "config", "num", 1.0)
    if not dt > 0:
        raise ValidationError("config.dt", "must be > 0")
    if substeps != int(substeps) or substeps < 1:
        raise ValidationError("config.substeps", "must be a positive integer")
    g = _one(top, "gravity", "config", "msg", [])
    gravity = _vec3(g, "config.gravity")
    friction = _one(top, "friction", "config", "num", 1.0)
    elasticity = _one(top, "elasticity", "config", "num", 0.0)
    beta = _one(top, "baumgarte_erp", "config", "num", 0.2)
    if friction < 0:
        raise ValidationError("config.friction", "must be >= 0")
    if not 0 <= elasticity <= 1:
        raise ValidationError("config.elasticity", "must be in [0, 1]")
    if not 0 < beta <= 1:
        raise ValidationError("config.baumgarte_erp", "must be in (0, 1]")

    bodies, colliders = [], []
    names = {}
    for bi, bnode in enumerate(top.get("bodies", [])):
        path = f"bodies[{bi}]"
        if not isinstance(bnode, list):
            raise ValidationError(path, "expected a { } block")
        bf = _fields(bnode, path, {"name", "mass", "inertia", "frozen", "colliders"})
        name = _one(bf, "name", path, "str")
        if name is None:
            raise ValidationError(f"{path}.name", "required")
        if name in names:
            raise ValidationError(f"{path}.name", f"duplicate body name {name!r}")
        names[name] = bi
        mass = _one(bf, "mass", path, "num", 1.0)
        if not mass > 0:
            raise ValidationError(f"{path}.mass", "must be > 0")
        inertia = _vec3(_one(bf, "inertia", path, "msg", []), f"{path}.inertia", (1.0, 1.0, 1.0))
        if not np.all(inertia > 0):
            raise ValidationError(f"{path}.inertia", "must be > 0")
        fpos = np.zeros(3)
        frot = np.zeros(3)
        fz = _one(bf, "frozen", path, "msg", None)
        if fz is not None:
            ff = _fields(fz, f"{path}.frozen", {"position", "rotation", "all"})
            if _one(ff, "all", f"{path}.frozen", None, False) is True:
                fpos[:] = 1
                frot[:] = 1
            fpos = np.maximum(fpos, _vec3(_one(ff, "position", f"{path}.frozen", "msg", []), f"{path}.frozen.position"))
            frot = np.maximum(frot, _vec3(_one(ff, "rotation", f"{path}.frozen", "msg", []), f"{path}.frozen.rotation"))
            if not (np.all(np.isin(fpos, (0, 1))) and np.all(np.isin(frot, (0, 1)))):
                raise ValidationError(f"{path}.frozen", "axis flags must be 0 or 1")
        cols = []
        for ci, cnode in enumerate(bf.get("colliders", [])):
            cpath = f"{path}.colliders[{ci}]"
            cf = _fields(cnode, cpath, {"position", "rotation", "sphere", "capsule", "box", "plane"})
            shapes = [k for k in ("sphere", "capsule", "box", "plane") if k in cf]
            if len(shapes) != 1:
                raise ValidationError(cpath, "exactly one of sphere/capsule/box/plane required")
            kind = shapes[0]
            c = Collider(body=bi, kind=kind,
                         pos=_vec3(_one(cf, "position", cpath, "msg", []), f"{cpath}.position"),
                         rot=euler_deg_to_quat(_vec3(_one(cf, "rotation", cpath, "msg", []), f"{cpath}.rotation")))
            shp = _one(cf, kind, cpath, "msg")
            spath = f"{cpath}.{kind}"
            if kind == "sphere":
                sf = _fields(shp, spath, {"radius"})
                c.radius = _one(sf, "radius", spath, "num", 0.0)
                if not c.radius > 0:
                    raise ValidationError(f"{spath}.radius", "must be > 0")
            elif kind == "capsule":
                sf = _fields(shp, spath, {"radius", "length", "end"})
                c.radius = _one(sf, "radius", spath, "num", 0.0)
                c.length = _one(sf, "length", spath, "num", 0.0)
                end = _one(sf, "end", spath, "num", 0.0)
                if not c.radius > 0:
                    raise ValidationError(f"{spath}.radius", "must be > 0")
                if not c.length >= 2 * c.radius:
                    raise ValidationError(f"{spath}.length", "must be >= 2*radius")
                if end not in (0.0, 1.0, -1.0):
                    raise ValidationError(f"{spath}.end", "must be -1, 0 or 1")
                c.end = int(end)
            elif kind == "box":
                sf = _fields(shp, spath, {"halfsize"})
                c.halfsize = _vec3(_one(sf, "halfsize", spath, "msg", []), f"{spath}.halfsize")
                if not np.all(c.halfsize > 0):
                    raise ValidationError(f"{spath}.halfsize", "must be > 0")
            else:
                _fields(shp, spath, set())
            cols.append(c)
            colliders.append(c)
        bodies.append(Body(name=name, mass=mass, inertia=inertia, frozen_pos=fpos,
                           frozen_rot=frot, colliders=cols,
                           init_pos=np.zeros(3), init_rot=np.array([1.0, 0, 0, 0])))
    if not bodies:
        raise ValidationError("config.bodies", "no bodies")

    for di, dnode in enumerate(top.get("defaults", [])):
        dpath = f"defaults[{di}]"
        df = _fields(dnode, dpath, {"qps"})
        for qi, qnode in enumerate(df.get("qps", [])):
            qpath = f"{dpath}.qps[{qi}]"
            qf = _fields(qnode, qpath, {"name", "pos", "rot"})
            nm = _one(qf, "name", qpath, "str")
            if nm not in names:
                raise ValidationError(f"{qpath}.name", f"unknown body {nm!r}")
            b = bodies[names[nm]]
            b.init_pos = _vec3(_one(qf, "pos", qpath, "msg", []), f"{qpath}.pos")
            b.init_rot = euler_deg_to_quat(_vec3(_one(qf, "rot", qpath, "msg", []), f"{qpath}.rot"))

    joints, jnames = [], {}
    for ji, jnode in enumerate(top.get("joints", [])):
        path = f"joints[{ji}]"
        jf = _fields(jnode, path, {
            "name", "parent", "child", "stiffness", "spring_damping", "angular_damping",
            "limit_stiffness", "angular_stiffness", "parent_offset", "child_offset",
            "rotation", "reference_rotation", "angle_limit"})
        name = _one(jf, "name", path, "str")
        if name is None:
            raise ValidationError(f"{path}.name", "required")
        if name in jnames:
            raise ValidationError(f"{path}.name", f"duplicate joint name {name!r}")
        jnames[name] = ji
        pn = _one(jf, "parent", path, "str")
        cn = _one(jf, "child", path, "str")
        if pn not in names:
            raise ValidationError(f"{path}.parent", f"unknown body {pn!r}")
        if cn not in names:
            raise ValidationError(f"{path}.child", f"unknown body {cn!r}")
        if pn == cn:
            raise ValidationError(f"{path}.child", "parent and child must differ")
        k = _one(jf, "stiffness", path, "num", 0.0)
        if not k > 0:
            raise ValidationError(f"{path}.stiffness", "must be > 0")
        lims = []
        for li, lnode in enumerate(jf.get("angle_limit", [])):
            lpath = f"{path}.angle_limit[{li}]"
            lf = _fields(lnode, lpath, {"min", "max"})
            lo = _one(lf, "min", lpath, "num", 0.0)
            hi = _one(lf, "max", lpath, "num", 0.0)
            if lo > hi:
                raise ValidationError(lpath, "min > max")
            if lo < -180 or hi > 180:
                raise ValidationError(lpath, "limits must lie in [-180, 180] degrees (R9)")
            lims.append((math.radians(lo), math.radians(hi)))
        if len(lims) > 3:
            raise ValidationError(f"{path}.angle_limit", "at most 3 (dof <= 3)")
        joints.append(Joint(
            name=name, parent=names[pn], child=names[cn], stiffness=k,
            spring_damping=_one(jf, "spring_damping", path, "num", 0.0),
            angular_damping=_one(jf, "angular_damping", path, "num", 0.0),
            limit_stiffness=_one(jf, "limit_stiffness", path, "num", k),
            angular_stiffness=_one(jf, "angular_stiffness", path, "num", k),
            parent_offset=_vec3(_one(jf, "parent_offset", path, "msg", []), f"{path}.parent_offset"),
            child_offset=_vec3(_one(jf, "child_offset", path, "msg", []), f"{path}.child_offset"),
            rotation=euler_deg_to_quat(_vec3(_one(jf, "rotation", path, "msg", []), f"{path}.rotation")),
            reference_rotation=euler_deg_to_quat(_vec3(_one(jf, "reference_rotation", path, "msg", []), f"{path}.reference_rotation")),
            limits=np.array(lims, dtype=float).reshape(-1, 2)))
        for fld in ("spring_damping", "angular_damping", "limit_stiffness", "angular_stiffness"):
            if getattr(joints[-1], fld) < 0:
                raise ValidationError(f"{path}.{fld}", "must be >= 0")

    # joint graph must be a forest: each body is the child of at most one joint, no cycles
    parent_of = {}
    for ji, j in enumerate(joints):
        if j.child in parent_of:
            raise ValidationError(f"joints[{ji}].child", "body is already the child of another joint")
        parent_of[j.child] = j.parent
    for b in range(len(bodies)):
        seen, x = set(), b
        while x in parent_of:
            if x in seen:
                raise CyclicJointGraph(f"bodies[{b}]", "cyclic joint graph")
            seen.add(x)
            x = parent_of[x]

    actuators = []
    used_joints = set()
    off = 0
    for ai, anode in enumerate(top.get("actuators", [])):
        path = f"actuators[{ai}]"
        af = _fields(anode, path, {"name", "joint", "strength", "torque", "angle"})
        jn = _one(af, "joint", path, "str")
        if jn not in jnames:
            raise ValidationError(f"{path}.joint", f"unknown joint {jn!r}")
        kinds = [k for k in ("torque", "angle") if k in af]
        if len(kinds) != 1:
            raise ValidationError(path, "exactly one of torque/angle required")
        ji = jnames[jn]
        if ji in used_joints:
            raise ValidationError(f"{path}.joint", "joint already has an actuator")
        if joints[ji].dof == 0:
            raise ValidationError(f"{path}.joint", "actuated joint must have dof >= 1")
        used_joints.add(ji)
        actuators.append(Actuator(name=_one(af, "name", path, "str", ""), joint=ji,
                                  strength=_one(af, "strength", path, "num", 0.0),
                                  kind=TORQUE if kinds[0] == "torque" else ANGLE,
                                  act_offset=off))
        off += joints[ji].dof

    pairs = _enumerate_pairs(top, bodies, colliders, names, joints)
    slots = []
    for pi, (ca, cb, ptype) in enumerate(pairs):
        A, B = colliders[ca], colliders[cb]
        if ptype == CAPSULE_PLANE:
            pts = [0, 1] if A.end == 0 else [0 if A.end == 1 else 1]
        elif ptype == BOX_PLANE:
            pts = list(range(8))
        else:
            pts = [0]
        for p in pts:
            slots.append((pi, ptype, A.body, B.body, ca, cb, p))
    if len(slots) > 255:
        raise ValidationError("config", "more than 255 contact slots")

    task = _parse_task(_one(top, "task", "config", "msg", None), bodies, names, colliders)
    return System(dt=dt, substeps=int(substeps), gravity=gravity, friction=friction,
                  elasticity=elasticity, baumgarte=beta, bodies=bodies, joints=joints,
                  actuators=actuators, colliders=colliders, pairs=pairs, slots=slots, task=task)


def _parse_goal(node, bodies, names, colliders, path):
    """goal { object target radius bonus range { x y z } } (R36)."""
    gf = _fields(node, path, {"object", "target", "radius", "bonus", "range"})
    ix = {}
    for key in ("object", "target"):
        nm = _one(gf, key, path, "str")
        if nm is None:
            raise ValidationError(f"{path}.{key}", "required")
        if nm not in names:
            raise ValidationError(f"{path}.{key}", f"unknown body '{nm}'")
        ix[key] = names[nm]
    if bodies[ix["object"]].is_static:
        raise ValidationError(f"{path}.object", "must not be a static body")
    if not bodies[ix["target"]].is_static:
        raise ValidationError(f"{path}.target", "must be a frozen { all: true } marker body")
    if any(c.body == ix["target"] for c in colliders):
        raise ValidationError(f"{path}.target", "must have no colliders")
    radius = _one(gf, "radius", path, "num", None)
    if radius is None or not radius > 0:
        raise ValidationError(f"{path}.radius", "must be > 0")
    rng = _vec3(_one(gf, "range", path, "msg", []), f"{path}.range")
    if np.any(rng < 0):
        raise ValidationError(f"{path}.range", "must be >= 0")
    return Goal(obj=ix["object"], target=ix["target"], radius=radius, bonus=_one(gf, "bonus", path, "num", 0.0),
                range=rng)


def _parse_task(node, bodies, names, colliders):
    """task { torso forward survive_reward ctrl_cost healthy_z episode_length contact_obs reset_noise goal }."""
    if node is None:
        return None
    path = "config.task"
    tf = _fields(node, path, {"torso", "forward", "survive_reward", "ctrl_cost", "healthy_z", "episode_length",
                              "contact_obs", "reset_noise", "goal"})
    tn = _one(tf, "torso", path, "str")
    if tn is None:
        raise ValidationError(f"{path}.torso", "required")
    if tn not in names:
        raise ValidationError(f"{path}.torso", f"unknown body '{tn}'")
    torso = names[tn]
    if bodies[torso].is_static:
        raise ValidationError(f"{path}.torso", "must not be a static body")
    fwd = _vec3(_one(tf, "forward", path, "msg", [("x", 1.0, 0, 0)]), f"{path}.forward")
    if not np.any(fwd != 0):
        raise ValidationError(f"{path}.forward", "must be nonzero")
    ctrl = _one(tf, "ctrl_cost", path, "num", 0.5)
    if ctrl < 0:
        raise ValidationError(f"{path}.ctrl_cost", "must be >= 0")
    hz = _one(tf, "healthy_z", path, "msg", None)
    healthy = None
    if hz is not None:
        hf = _fields(hz, f"{path}.healthy_z", {"min", "max"})
        lo = _one(hf, "min", f"{path}.healthy_z", "num", None)
        hi = _one(hf, "max", f"{path}.healthy_z", "num", None)
        if lo is None or hi is None or not lo < hi:
            raise ValidationError(f"{path}.healthy_z", "needs min < max")
        healthy = (lo, hi)
    L = _one(tf, "episode_length", path, "num", 1000.0)
    if L != int(L) or L < 1:
        raise ValidationError(f"{path}.episode_length", "must be a positive integer")
    co = _one(tf, "contact_obs", path, None, False)
    if co not in (True, False):
        raise ValidationError(f"{path}.contact_obs", "expected true or false")
    rn = _one(tf, "reset_noise", path, "msg", [])
    rf = _fields(rn, f"{path}.reset_noise", {"vel", "ang"})
    sv = _one(rf, "vel", f"{path}.reset_noise", "num", 0.1)
    sw = _one(rf, "ang", f"{path}.reset_noise", "num", 0.1)
    if sv < 0 or sw < 0:
        raise ValidationError(f"{path}.reset_noise", "must be >= 0")
    gn = _one(tf, "goal", path, "msg", None)
    goal = None if gn is None else _parse_goal(gn, bodies, names, colliders, f"{path}.goal")
    return Task(torso=torso, forward=fwd, survive_reward=_one(tf, "survive_reward", path, "num", 1.0),
                ctrl_cost=ctrl, healthy_z=healthy, episode_length=int(L), contact_obs=bool(co),
                reset_vel_noise=sv, reset_ang_noise=sw, goal=goal)


def _orient(colliders, i, j):
    """Pair orientation and type: plane is always B; sphere is A
    vs capsule; same-shape pairs put the lower collider index in A."""
    ki, kj = colliders[i].kind, colliders[j].kind
    order = {"sphere": 0, "capsule": 1, "box": 2, "plane": 3}
    if order[ki] > order[kj] or (order[ki] == order[kj] and i > j):
        i, j, ki, kj = j, i, kj, ki
    table = {("sphere", "plane"): SPHERE_PLANE, ("capsule", "plane"): CAPSULE_PLANE,
             ("box", "plane"): BOX_PLANE, ("sphere", "sphere"): SPHERE_SPHERE,
             ("sphere", "capsule"): SPHERE_CAPSULE, ("capsule", "capsule"): CAPSULE_CAPSULE}
    t = table.get((ki, kj))
    return i, j, t


def _enumerate_pairs(top, bodies, colliders, names, joints):
    """Naive pairwise collision (§6.2) as a static pair list (R19)."""
    includes = top.get("collide_include", [])
    cand = []
    if includes:
        for ii, inode in enumerate(includes):
            path = f"collide_include[{ii}]"
            f = _fields(inode, path, {"first", "second"})
            a = _one(f, "first", path, "str")
            b = _one(f, "second", path, "str")
            for nm, key in ((a, "first"), (b, "second")):
                if nm not in names:
                    raise ValidationError(f"{path}.{key}", f"unknown body {nm!r}")
            ba, bb = names[a], names[b]
            if ba == bb:
                raise ValidationError(path, "a body cannot collide with itself")
            if bodies[ba].is_static and bodies[bb].is_static:
                raise ValidationError(path, "static-static pair")
            ca = [k for k, c in enumerate(colliders) if c.body == ba]
            cb = [k for k, c in enumerate(colliders) if c.body == bb]
            for i in ca:
                for j in cb:
                    cand.append((i, j, path))
    else:
        jointed = {(j.parent, j.child) for j in joints} | {(j.child, j.parent) for j in joints}
        for i in range(len(colliders)):
            for j in range(i + 1, len(colliders)):
                bi, bj = colliders[i].body, colliders[j].body
                if bi == bj or (bi, bj) in jointed:
                    continue
                if bodies[bi].is_static and bodies[bj].is_static:
                    continue
                cand.append((i, j, f"colliders[{i}]x[{j}]"))
    pairs = []
    for i, j, path in cand:
        a, b, t = _orient(colliders, i, j)
        if t is None:
            raise ValidationError(path, f"unsupported collider pair {colliders[a].kind}-{colliders[b].kind}")
        pairs.append((a, b, t))
    return pairs


# --------------------------------------------------------------------------
# default_qp ("places each body in a valid joint configuration")
# --------------------------------------------------------------------------
def default_qp(sys: System):
    """Roots at their defaults; then joints in config order, repeated until every
    child is placed (a BFS over the forest).  Child rotation
    q_c = q_p ⊗ J ⊗ E(θ⁰) ⊗ conj(J) ⊗ Rf with θ⁰_i = clamp(0, lo_i, hi_i) for the
    free axes, so that the joint-frame relative rotation equals E(θ⁰); child
    position x_c = x_p + rotate(q_p, o_p) − rotate(q_c, o_c) makes the anchors
    coincide (SURVEY §8(c).1 default_qp)."""
    B = len(sys.bodies)
    pos = np.zeros((B, 3))
    rot = np.zeros((B, 4))
    placed = [False] * B
    children = {j.child for j in sys.joints}
    for b, body in enumerate(sys.bodies):
        if b not in children:
            pos[b] = body.init_pos
            rot[b] = body.init_rot
            placed[b] = True
    progress = True
    while progress:
        progress = False
        for j in sys.joints:
            if placed[j.parent] and not placed[j.child]:
                theta0 = np.zeros(3)
                for i in range(j.dof):
                    theta0[i] = min(max(0.0, j.limits[i, 0]), j.limits[i, 1])
                E = euler_rad_to_quat(theta0)
                qp_ = rot[j.parent]
                qc = qmul(qmul(qmul(qmul(qp_, j.rotation), E), qconj(j.rotation)), j.reference_rotation)
                rot[j.child] = qc
                pos[j.child] = pos[j.parent] + qrotate(qp_, j.parent_offset) - qrotate(qc, j.child_offset)
                placed[j.child] = True
                progress = True
    assert all(placed)
    return {"pos": pos, "rot": rot, "vel": np.zeros((B, 3)), "ang": np.zeros((B, 3))}


def stability_lint(sys: System):
    """Create-time stability lint: warn if k·w·h² ≥ 3.6 or c_l·w·h ≥ 1.8,
    w = Σ_X not static (1/m_X + |o_X|²/min I_X) over the joint's two bodies."""
    h = sys.dt / sys.substeps
    out = []
    for ji, j in enumerate(sys.joints):
        w = 0.0
        for b, o in ((j.parent, j.parent_offset), (j.child, j.child_offset)):
            body = sys.bodies[b]
            if not body.is_static:
                w += 1.0 / body.mass + float(np.dot(o, o)) / float(np.min(body.inertia))
        if j.stiffness * w * h * h >= 3.6:
            out.append(f"joints[{ji}]: stiffness*w*h^2 = {j.stiffness * w * h * h:.3g} >= 3.6")
        if j.spring_damping * w * h >= 1.8:
            out.append(f"joints[{ji}]: spring_damping*w*h = {j.spring_damping * w * h:.3g} >= 1.8")
    return out
