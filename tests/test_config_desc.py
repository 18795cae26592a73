"""Programmatic system construction through the C ABI (brax_config_from_desc):
"users can define systems in text, or they can define systems programmatically"
(§4.1; the App. A Python listing).  A config
built from descriptors must equal the text parse of the same scene: integer
tables bit-exact, default_qp equal.  CPU only (host-side library calls); the GPU
check that both step identically is in test_gpu_parity.py."""
import ctypes as C
import math
import re

import numpy as np
import pytest

import oracle
import paper_2106_13281_b200 as bx

SCENES = ["ball", "appA", "pendulum", "chain2", "ant", "humanoid", "halfcheetah", "grasp", "fetch", "coverage"]
_KIND = {"sphere": 0, "capsule": 1, "box": 2, "plane": 3}


def desc_from_system(s, text):
    """brax_config_desc of an oracle-parsed scene (the oracle's own parser is the
    independent reading of the text); returns (desc, keepalive)."""
    keep = []
    bodies = (bx.brax_body_desc * len(s.bodies))()
    for i, b in enumerate(s.bodies):
        nm = b.name.encode()
        keep.append(nm)
        bodies[i] = bx.brax_body_desc(nm, b.mass, (C.c_double * 3)(*b.inertia), (C.c_double * 3)(*b.frozen_pos),
                                      (C.c_double * 3)(*b.frozen_rot), (C.c_double * 3)(*b.init_pos),
                                      (C.c_double * 4)(*b.init_rot))
    joints = (bx.brax_joint_desc * max(1, len(s.joints)))()
    for i, j in enumerate(s.joints):
        nm = j.name.encode()
        keep.append(nm)
        lo = [0.0] * 3
        hi = [0.0] * 3
        for k in range(j.dof):
            lo[k], hi[k] = float(j.limits[k, 0]), float(j.limits[k, 1])
        joints[i] = bx.brax_joint_desc(nm, j.parent, j.child, (C.c_double * 3)(*j.parent_offset),
                                       (C.c_double * 3)(*j.child_offset), (C.c_double * 4)(*j.rotation),
                                       (C.c_double * 4)(*j.reference_rotation), j.dof, (C.c_double * 3)(*lo),
                                       (C.c_double * 3)(*hi), j.stiffness, j.spring_damping, j.angular_damping,
                                       j.limit_stiffness, j.angular_stiffness)
    acts = (bx.brax_actuator_desc * max(1, len(s.actuators)))()
    for i, a in enumerate(s.actuators):
        nm = a.name.encode()
        keep.append(nm)
        acts[i] = bx.brax_actuator_desc(nm, a.joint, a.kind, a.strength)
    cols = (bx.brax_collider_desc * max(1, len(s.colliders)))()
    # descriptors listed with the bodies in reverse order (in-body order kept): the library
    # restores the text format's global order (body order, stable within a body)
    by_body = {}
    for i in range(len(s.colliders)):
        by_body.setdefault(s.colliders[i].body, []).append(i)
    flat = [i for b in sorted(by_body, reverse=True) for i in by_body[b]]  # bodies reversed, in-body order kept
    for slot, i in enumerate(flat):
        c = s.colliders[i]
        cols[slot] = bx.brax_collider_desc(c.body, _KIND[c.kind],
                                           (C.c_double * 3)(*c.pos), (C.c_double * 4)(*c.rot), c.radius, c.length,
                                           (C.c_double * 3)(*c.halfsize), c.end)
    names = {b.name: i for i, b in enumerate(s.bodies)}
    inc = re.findall(r'collide_include\s*\{\s*first:\s*"([^"]+)"\s*second:\s*"([^"]+)"\s*\}', text)
    pairs = (bx.brax_body_pair * max(1, len(inc)))()
    for i, (a, b) in enumerate(inc):
        pairs[i] = bx.brax_body_pair(names[a], names[b])
    keep += [bodies, joints, acts, cols, pairs]
    d = bx.brax_config_desc(s.dt, s.substeps, (C.c_double * 3)(*s.gravity), s.friction, s.elasticity, s.baumgarte,
                            len(s.bodies), len(s.joints), len(s.actuators), len(s.colliders), len(inc),
                            bodies, joints, acts, cols, pairs if inc else None)
    return d, keep


@pytest.mark.parametrize("scene", SCENES)
def test_desc_equals_text_parse(scene):
    text = oracle.load_scene(scene)
    s = oracle.system.parse_system(text)
    d, keep = desc_from_system(s, text)
    a = bx.brax_config_from_desc(d)
    b = bx.brax_config_parse(text)
    try:
        assert bx.brax_config_counts(a) == bx.brax_config_counts(b)
        assert np.array_equal(bx.brax_config_slot_table(a), bx.brax_config_slot_table(b))
        pa, ra = bx.brax_config_default_qp(a)
        pb, rb = bx.brax_config_default_qp(b)
        assert np.array_equal(pa, pb) and np.array_equal(ra, rb)
    finally:
        bx.brax_config_destroy(a)
        bx.brax_config_destroy(b)
    del keep


def app_a_desc():
    """The paper's programmatic App. A listing, field by field: dt .01,
    gravity z −9.8; Parent frozen in all six axes, mass 1, inertia 1; Child mass 1,
    inertia 1; Joint Parent→Child, stiffness 10000, child_offset z 1, one angle limit.
    The listing's limit (180, 180) is read as the text's (−180, 180) (R10)."""
    I3 = (C.c_double * 3)(1, 1, 1)
    ident = (C.c_double * 4)(1, 0, 0, 0)
    z3 = (C.c_double * 3)(0, 0, 0)
    bodies = (bx.brax_body_desc * 2)(
        bx.brax_body_desc(b"Parent", 1.0, I3, (C.c_double * 3)(1, 1, 1), (C.c_double * 3)(1, 1, 1), z3, ident),
        bx.brax_body_desc(b"Child", 1.0, I3, z3, z3, z3, ident))
    joints = (bx.brax_joint_desc * 1)(
        bx.brax_joint_desc(b"Joint", 0, 1, z3, (C.c_double * 3)(0, 0, 1), ident, ident, 1,
                           (C.c_double * 3)(-math.pi, 0, 0), (C.c_double * 3)(math.pi, 0, 0), 10000.0, 0.0, 0.0,
                           -1.0, -1.0))
    d = bx.brax_config_desc(0.01, 1, (C.c_double * 3)(0, 0, -9.8), 1.0, 0.0, 0.2, 2, 1, 0, 0, 0,
                            bodies, joints, None, None, None)
    return d, (bodies, joints)


def test_app_a_programmatic_listing():
    """App. A built programmatically equals App. A parsed from text: same
    counts, same (empty) slot table, default_qp child at (0, 0, −1)."""
    d, keep = app_a_desc()
    a = bx.brax_config_from_desc(d)
    b = bx.brax_config_parse(oracle.load_scene("appA"))
    try:
        assert bx.brax_config_counts(a) == bx.brax_config_counts(b) == (2, 1, 0, 0)
        pa, ra = bx.brax_config_default_qp(a)
        pb, rb = bx.brax_config_default_qp(b)
        assert np.array_equal(pa, pb) and np.array_equal(ra, rb)
        assert np.allclose(pa[1], [0, 0, -1], atol=1e-15)
    finally:
        bx.brax_config_destroy(a)
        bx.brax_config_destroy(b)
    del keep


@pytest.mark.parametrize("field,value,status,detail", [
    ("stiffness", 0.0, "BRAX_E_VALIDATION", "joints[0].stiffness"),
    ("parent", 7, "BRAX_E_VALIDATION", "joints[0].parent"),
    ("rotation", (2.0, 0, 0, 0), "BRAX_E_VALIDATION", "joints[0].rotation"),
    ("dof", 4, "BRAX_E_VALIDATION", "joints[0].dof"),
])
def test_desc_validation_errors(field, value, status, detail):
    d, keep = app_a_desc()
    j = d.joints[0]
    if field == "rotation":
        j.rotation = (C.c_double * 4)(*value)
    else:
        setattr(j, field, value)
    with pytest.raises(bx.BraxError) as e:
        bx.brax_config_from_desc(d)
    assert e.value.name == status and detail in e.value.detail
    del keep


def test_desc_cycle_and_unsupported_pair():
    d, keep = app_a_desc()
    joints = (bx.brax_joint_desc * 2)(d.joints[0], d.joints[0])
    joints[1].parent, joints[1].child = 1, 0
    joints[1].name = b"Back"
    d.joints, d.n_joints = joints, 2
    d.bodies[0].frozen_pos = (C.c_double * 3)(0, 0, 0)
    with pytest.raises(bx.BraxError) as e:
        bx.brax_config_from_desc(d)
    assert e.value.name in ("BRAX_E_CYCLIC_JOINT_GRAPH", "BRAX_E_VALIDATION")
    d2, keep2 = app_a_desc()
    ident = (C.c_double * 4)(1, 0, 0, 0)
    z3 = (C.c_double * 3)(0, 0, 0)
    cols = (bx.brax_collider_desc * 2)(bx.brax_collider_desc(0, 2, z3, ident, 0, 0, (C.c_double * 3)(1, 1, 1), 0),
                                       bx.brax_collider_desc(1, 2, z3, ident, 0, 0, (C.c_double * 3)(1, 1, 1), 0))
    d2.colliders, d2.n_colliders = cols, 2
    d2.joints, d2.n_joints = None, 0
    with pytest.raises(bx.BraxError) as e:
        bx.brax_config_from_desc(d2)
    assert e.value.name == "BRAX_E_UNSUPPORTED_PAIR"
    del keep, keep2
