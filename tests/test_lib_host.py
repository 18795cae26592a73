"""Host-side checks of the C-ABI library (no GPU): it loads, exports every
symbol include/brax_b200.h declares, and its independent C++ parser / slot
enumerator / default_qp agree with the oracle's (integer tables bit-exact)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2106_13281_b200 as bx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENES = ["ball", "appA", "pendulum", "chain2", "ant", "humanoid", "halfcheetah", "grasp", "fetch", "coverage"]


def declared_functions():
    with open(os.path.join(ROOT, "include", "brax_b200.h")) as f:
        txt = f.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(brax_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(bx.lib, n), n
        assert ctypes.cast(getattr(bx.lib, n), ctypes.c_void_p).value


def test_abi_version_and_status_strings():
    assert bx.lib.brax_abi_version() == 1
    assert bx.lib.brax_status_string(0) == b"BRAX_OK"
    assert bx.lib.brax_status_string(7) == b"BRAX_E_CUDA"


@pytest.mark.parametrize("scene", SCENES)
def test_tables_match_oracle(scene):
    text = oracle.load_scene(scene)
    o = oracle.Oracle(text)
    cfg = bx.brax_config_parse(text)
    try:
        B, J, A, C = bx.brax_config_counts(cfg)
        assert (B, J, A, C) == (o.n_bodies, len(o.sys.joints), o.act_dim, o.n_slots)
        assert np.array_equal(bx.brax_config_slot_table(cfg), o.sys.slot_table())  # bit-exact
        pos, rot = bx.brax_config_default_qp(cfg)
        d = o.default_qp()
        assert np.max(np.abs(pos - d["pos"])) < 1e-12
        assert np.max(np.abs(rot - d["rot"])) < 1e-12
    finally:
        bx.brax_config_destroy(cfg)


@pytest.mark.parametrize("text", [
    "dt: 0.01\nbodies { name: \"A\" ",
    "dt 0.01",
    "bodies { name: \"A\" } }",
    "dt: @",
])
def test_parse_errors_agree_with_oracle(text):
    with pytest.raises(oracle.ParseError) as oe:
        oracle.parse_system(text)
    with pytest.raises(bx.BraxError) as le:
        bx.brax_config_parse(text)
    assert le.value.name == "BRAX_E_PARSE"
    assert le.value.detail.startswith(f"{oe.value.line}:{oe.value.col}:")


@pytest.mark.parametrize("text,status", [
    ("", "BRAX_E_VALIDATION"),
    ('bodies { name: "A" mass: 0 }', "BRAX_E_VALIDATION"),
    ('bodies { name: "A" } joints { name: "J" parent: "A" child: "Ghost" stiffness: 1 }', "BRAX_E_VALIDATION"),
    ('bodies { name: "A" colliders { box { halfsize { x: 1 y: 1 z: 1 } } } } '
     'bodies { name: "B" colliders { capsule { radius: 0.1 length: 1 } } }', "BRAX_E_UNSUPPORTED_PAIR"),
    ('bodies { name: "A" } bodies { name: "B" } bodies { name: "C" }\n'
     'joints { name: "1" parent: "A" child: "B" stiffness: 1 }\n'
     'joints { name: "2" parent: "B" child: "C" stiffness: 1 }\n'
     'joints { name: "3" parent: "C" child: "A" stiffness: 1 }', "BRAX_E_CYCLIC_JOINT_GRAPH"),
])
def test_validation_errors(text, status):
    with pytest.raises(oracle.ValidationError) as oe:
        oracle.parse_system(text)
    with pytest.raises(bx.BraxError) as le:
        bx.brax_config_parse(text)
    assert le.value.name == status
    assert le.value.detail.startswith(oe.value.path + ":")


GOAL_BASE = ('bodies { name: "Ball" colliders { sphere { radius: 0.1 } } } '
             'bodies { name: "T" frozen { all: true } } bodies { name: "W" } ')


@pytest.mark.parametrize("goal", [
    'goal { object: "Ball" target: "W" radius: 0.1 }',
    'goal { object: "T" target: "T" radius: 0.1 }',
    'goal { object: "Ball" target: "Ghost" radius: 0.1 }',
    'goal { object: "Ball" target: "T" }',
    'goal { object: "Ball" target: "T" radius: -1 }',
    'goal { object: "Ball" target: "T" radius: 0.1 range { y: -0.5 } }',
    'goal { target: "T" radius: 0.1 }',
    'goal { object: "Ball" target: "T" radius: 0.1 size: 1 }',
])
def test_goal_validation_errors_agree_with_oracle(goal):
    """The goal block (R36) is checked identically by both parsers (same field path)."""
    text = GOAL_BASE + 'task { torso: "Ball" ' + goal + " }"
    with pytest.raises(oracle.ValidationError) as oe:
        oracle.parse_system(text)
    with pytest.raises(bx.BraxError) as le:
        bx.brax_config_parse(text)
    assert le.value.name == "BRAX_E_VALIDATION"
    assert le.value.detail.startswith(oe.value.path + ":"), (le.value.detail, oe.value.path)


def test_goal_marker_with_collider_rejected_by_both():
    text = ('bodies { name: "Ball" } bodies { name: "T" frozen { all: true } colliders { sphere { radius: 1 } } } '
            'task { torso: "Ball" goal { object: "Ball" target: "T" radius: 0.1 } }')
    with pytest.raises(oracle.ValidationError, match="collider"):
        oracle.parse_system(text)
    with pytest.raises(bx.BraxError, match="collider"):
        bx.brax_config_parse(text)


def test_random_scenes_tables_match_oracle():
    """Randomly generated small scenes: both builders produce identical integer tables."""
    rng = np.random.default_rng(0)
    shapes = ["sphere { radius: 0.1 }", "capsule { radius: 0.1 length: 0.5 }",
              "capsule { radius: 0.1 length: 0.5 end: 1 }", "plane {}"]
    for trial in range(30):
        nb = int(rng.integers(2, 6))
        lines = []
        for b in range(nb):
            frozen = "frozen { all: true }" if rng.random() < 0.3 else ""
            cols = " ".join(f"colliders {{ {shapes[int(rng.integers(0, 4))]} }}"
                            for _ in range(int(rng.integers(0, 3))))
            lines.append(f'bodies {{ name: "b{b}" {frozen} {cols} }}')
        text = "\n".join(lines)
        try:
            o = oracle.Oracle(text)
        except oracle.ValidationError:
            with pytest.raises(bx.BraxError):
                bx.brax_config_parse(text)
            continue
        cfg = bx.brax_config_parse(text)
        try:
            assert np.array_equal(bx.brax_config_slot_table(cfg), o.sys.slot_table())
        finally:
            bx.brax_config_destroy(cfg)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = bx.brax_config_parse(oracle.load_scene("ant"))
    try:
        with pytest.raises(bx.BraxError) as e:
            bx.brax_system_create(cfg, 0)
        assert e.value.name == "BRAX_E_CUDA"
    finally:
        bx.brax_config_destroy(cfg)
