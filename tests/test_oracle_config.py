"""Oracle-side scene parsing, validation, slot enumeration and default_qp pins
(App. A golden PAPER.md:324-347).  CPU only."""
import itertools
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from oracle.system import ParseError, ValidationError, CyclicJointGraph, parse_system

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_app_a_golden():
    s = parse_system(oracle.load_scene("appA"))
    gold = {}
    with open(os.path.join(GOLD, "appA_parse.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, *v = line.split()
                gold[k] = v
    num = lambda k: np.array([float(x) for x in gold[k]])
    assert s.dt == num("dt")[0] and s.substeps == int(num("substeps")[0])
    assert np.array_equal(s.gravity, num("gravity"))
    assert len(s.bodies) == int(num("n_bodies")[0])
    for b in range(2):
        assert s.bodies[b].name == gold[f"body{b}.name"][0]
        assert s.bodies[b].mass == num(f"body{b}.mass")[0]
        assert np.array_equal(s.bodies[b].inertia, num(f"body{b}.inertia"))
    assert np.array_equal(s.bodies[0].frozen_pos, num("body0.frozen_pos"))
    assert np.array_equal(s.bodies[0].frozen_rot, num("body0.frozen_rot"))
    assert s.bodies[0].is_static and not s.bodies[1].is_static
    j = s.joints[0]
    assert (j.parent, j.child) == (int(num("joint0.parent")[0]), int(num("joint0.child")[0]))
    assert j.stiffness == num("joint0.stiffness")[0]
    assert np.array_equal(j.child_offset, num("joint0.child_offset"))
    assert np.array_equal(j.parent_offset, num("joint0.parent_offset"))
    assert np.allclose(np.degrees(j.limits[0]), num("joint0.limits_deg"))
    assert j.dof == 1
    dq = s.default_qp()
    assert np.allclose(dq["pos"][1], num("default_qp.pos1"), atol=1e-15)


@pytest.mark.parametrize("text,line,col", [
    ("dt: 0.01\nbodies { name: \"A\" ", 2, 20),
    ("dt 0.01", 1, 4),
    ("bodies { name: \"A\" } }", 1, 22),
    ("dt: @", 1, 5),
])
def test_parse_errors_have_positions(text, line, col):
    with pytest.raises(ParseError) as e:
        parse_system(text)
    assert (e.value.line, e.value.col) == (line, col)


@pytest.mark.parametrize("text,path", [
    ("", "config.bodies"),
    ('bodies { name: "A" mass: 0 }', "bodies[0].mass"),
    ('bodies { name: "A" } bodies { name: "A" }', "bodies[1].name"),
    ('bodies { name: "A" } joints { name: "J" parent: "A" child: "Ghost" stiffness: 1 }', "joints[0].child"),
    ('bodies { name: "A" } bodies { name: "B" } joints { name: "J" parent: "A" child: "B" stiffness: 1 '
     'angle_limit { min: 10 max: -10 } }', "joints[0].angle_limit[0]"),
    ('bodies { name: "A" colliders { box { halfsize { x: 1 y: 1 z: 1 } } } } '
     'bodies { name: "B" colliders { capsule { radius: 0.1 length: 1 } } }', "colliders[0]x[1]"),
    ('bodies { name: "A" wings: 2 }', "bodies[0].wings"),
])
def test_validation_errors_name_the_path(text, path):
    with pytest.raises(ValidationError) as e:
        parse_system(text)
    assert e.value.path == path


def test_cyclic_joint_graph():
    txt = ('bodies { name: "A" } bodies { name: "B" } bodies { name: "C" }\n'
           'joints { name: "1" parent: "A" child: "B" stiffness: 1 }\n'
           'joints { name: "2" parent: "B" child: "C" stiffness: 1 }\n'
           'joints { name: "3" parent: "C" child: "A" stiffness: 1 }')
    with pytest.raises(CyclicJointGraph):
        parse_system(txt)


def _brute_pairs(sys):
    """Brute-force R19 default rule: every collider pair (i < j) on different,
    non-jointed, not-both-static bodies; orientation plane → B, sphere → A vs
    capsule, lower index → A for same shapes."""
    rank = {"sphere": 0, "capsule": 1, "box": 2, "plane": 3}
    jointed = set()
    for j in sys.joints:
        jointed |= {(j.parent, j.child), (j.child, j.parent)}
    out = []
    cols = sys.colliders
    for i, j in itertools.combinations(range(len(cols)), 2):
        bi, bj = cols[i].body, cols[j].body
        if bi == bj or (bi, bj) in jointed or (sys.bodies[bi].is_static and sys.bodies[bj].is_static):
            continue
        a, b = (i, j) if (rank[cols[i].kind], i) <= (rank[cols[j].kind], j) else (j, i)
        out.append((a, b))
    return out


def test_slot_table_default_rule_brute_force():
    txt = """
bodies { name: "G" frozen { all: true } colliders { plane {} } }
bodies { name: "S" colliders { sphere { radius: 0.1 } } }
bodies { name: "C" colliders { capsule { radius: 0.1 length: 0.5 } } colliders { sphere { radius: 0.05 } } }
bodies { name: "K" colliders { capsule { radius: 0.1 length: 0.5 end: -1 } } }
bodies { name: "F" frozen { all: true } colliders { sphere { radius: 0.2 } } }
joints { name: "j" parent: "S" child: "K" stiffness: 10 }
"""
    s = parse_system(txt)
    pairs = [(a, b) for a, b, t in s.pairs]
    assert pairs == _brute_pairs(s)
    npts = {0: 1, 1: 2, 2: 8, 3: 1, 4: 1, 5: 1}
    tab = s.slot_table()
    total = 0
    for pi, (a, b, t) in enumerate(s.pairs):
        k = npts[t]
        if t == 1 and s.colliders[a].end != 0:
            k = 1
        rows = tab[tab[:, 0] == pi]
        assert len(rows) == k and np.all(rows[:, 1] == t)
        assert list(rows[:, 6]) == ([1] if (t == 1 and s.colliders[a].end == -1) else list(range(k)))
        total += k
    assert total == len(tab)
    assert list(tab[:, 0]) == sorted(tab[:, 0])  # slot id = prefix sum over pairs


def test_slot_table_box_corners():
    txt = """
bodies { name: "G" frozen { all: true } colliders { plane {} } }
bodies { name: "X" colliders { box { halfsize { x: 0.1 y: 0.2 z: 0.3 } } } }
bodies { name: "S" colliders { sphere { radius: 0.1 } } }
collide_include { first: "G" second: "X" }
collide_include { first: "S" second: "G" }
"""
    tab = parse_system(txt).slot_table()
    assert tab.tolist() == [[0, 2, 1, 0, 1, 0, k, ] for k in range(8)] + [[1, 0, 2, 0, 2, 0, 0]]


def test_slot_table_include_order():
    s = parse_system(oracle.load_scene("ant"))
    tab = s.slot_table()
    assert len(tab) == 9
    assert list(tab[:, 1]) == [0] + [1] * 8           # torso sphere–plane, then capsule ends
    assert list(tab[:, 6]) == [0] + [0, 1] * 4
    assert np.all(tab[:, 3] == 0)                      # plane (ground) is always B


@pytest.mark.parametrize("scene", ["appA", "chain2", "ant", "humanoid", "halfcheetah", "grasp", "fetch"])
def test_default_qp_valid_joint_configuration(scene):
    """Anchors coincide and the joint-frame relative rotation equals E(θ⁰) — checked
    with scipy's rotation algebra (independent of the oracle's quaternion code)."""
    s = parse_system(oracle.load_scene(scene))
    dq = s.default_qp()
    R = lambda q: Rotation.from_quat([q[1], q[2], q[3], q[0]])
    for j in s.joints:
        rp, rc = R(dq["rot"][j.parent]), R(dq["rot"][j.child])
        ap = dq["pos"][j.parent] + rp.apply(j.parent_offset)
        ac = dq["pos"][j.child] + rc.apply(j.child_offset)
        assert np.linalg.norm(ap - ac) < 1e-12
        Jp = R(j.rotation)
        Jc = R(j.reference_rotation).inv() * R(j.rotation)
        rel = (rp * Jp).inv() * (rc * Jc)
        th = rel.as_euler("XYZ")
        th0 = np.zeros(3)
        for i in range(j.dof):
            th0[i] = min(max(0.0, j.limits[i, 0]), j.limits[i, 1])
        assert np.allclose(th, th0, atol=1e-12)


def test_default_qp_chain():
    """Three-link chain with offsets z = 1: (0,0,0), (0,0,−1), (0,0,−2)."""
    s = parse_system(oracle.load_scene("chain2"))
    assert np.allclose(s.default_qp()["pos"], [[0, 0, 0], [0, 0, -1], [0, 0, -2]], atol=1e-15)


def test_euler_convention_matches_scipy():
    rng = np.random.default_rng(0)
    for _ in range(20):
        d = rng.uniform(-170, 170, 3)
        q = oracle.system.euler_deg_to_quat(d)
        ref = Rotation.from_euler("XYZ", d, degrees=True).as_quat()  # x y z w
        ref = np.array([ref[3], ref[0], ref[1], ref[2]])
        assert np.allclose(q, ref, atol=1e-14) or np.allclose(q, -ref, atol=1e-14)


def test_stability_lint():
    txt = ('bodies { name: "P" frozen { all: true } } bodies { name: "C" }\n'
           'joints { name: "J" parent: "P" child: "C" stiffness: 1e6 child_offset { z: 1 } }')
    assert parse_system(txt).lint()
    for sc in ("ant", "humanoid", "halfcheetah", "grasp", "fetch", "pendulum", "chain2"):
        assert parse_system(oracle.load_scene(sc)).lint() == []


def test_table1_action_dims():
    """Act dims of Table 1."""
    dims = {"halfcheetah": 7, "ant": 8, "humanoid": 17, "grasp": 19, "fetch": 10}
    for sc, a in dims.items():
        assert parse_system(oracle.load_scene(sc)).act_dim == a
