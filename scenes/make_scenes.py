"""Writes the synthetic benchmark scenes (ant, humanoid, halfcheetah, grasp, fetch).

Scene-authoring tool only: string formatting of offsets, no physics.  The
paper gives only obs/act dims and prose for these envs (PAPER.md:109-135,
Table 1; App. E :497-511); the body/joint/collider definitions it cites
([antdef]) are not in the paper, so these are synthetic
stand-ins with the structure SURVEY.md §8(d) M3-M5 states (body/joint/dof/
contact-slot counts).  Constants marked † there are proposals; each scene is
checked for 1000-step random-action stability by tests/test_scenes.py.

Run:  python scenes/make_scenes.py   (rewrites scenes/*.bxc for these five)
"""
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def f(x):
    s = f"{x:.7f}".rstrip("0").rstrip(".")
    return "0" if s in ("-0", "") else s


def vec(name, v):
    parts = [f"{a}: {f(c)}" for a, c in zip("xyz", v) if abs(c) > 0]
    return f"{name} {{ {' '.join(parts)} }}" if parts else ""


def ant():
    out = ["# M3 ant (SURVEY §8(d)): ground + torso sphere + 4 x (thigh, shin) capsules;",
           "# 8 hinge joints (hips about the vertical, knees about the horizontal),",
           "# 8 TORQUE actuators; pairs torso-ground and 4 shins-ground (C = 1 + 4*2 = 9).",
           "dt: 0.05", "substeps: 10", "gravity { z: -9.8 }", "friction: 1", "elasticity: 0",
           "baumgarte_erp: 0.2",
           'bodies { name: "Ground" frozen { all: true } colliders { plane {} } }',
           'bodies { name: "Torso" mass: 10 inertia { x: 1 y: 1 z: 1 }',
           '  colliders { sphere { radius: 0.25 } } }']
    joints, acts, incl = [], [], ['collide_include { first: "Torso" second: "Ground" }']
    for i, phi in enumerate((45, 135, 225, 315)):
        u = (math.cos(math.radians(phi)), math.sin(math.radians(phi)), 0.0)
        rot = f"rotation {{ x: -90 y: {90 - phi} }}"
        out.append(f'bodies {{ name: "Thigh{i}" mass: 1 inertia {{ x: 1 y: 1 z: 1 }}')
        out.append(f"  colliders {{ {rot} capsule {{ radius: 0.08 length: 0.56 }} }} }}")
        out.append(f'bodies {{ name: "Shin{i}" mass: 1 inertia {{ x: 1 y: 1 z: 1 }}')
        out.append(f"  colliders {{ {rot} capsule {{ radius: 0.08 length: 0.66 }} }} }}")
        joints.append(
            f'joints {{ name: "Hip{i}" parent: "Torso" child: "Thigh{i}" stiffness: 5000 angular_damping: 35\n'
            f"  {vec('parent_offset', [0.25 * c for c in u])} {vec('child_offset', [-0.2 * c for c in u])}\n"
            f"  rotation {{ y: -90 }} angle_limit {{ min: -30 max: 30 }} }}")
        joints.append(
            f'joints {{ name: "Knee{i}" parent: "Thigh{i}" child: "Shin{i}" stiffness: 5000 angular_damping: 35\n'
            f"  {vec('parent_offset', [0.2 * c for c in u])} {vec('child_offset', [-0.25 * c for c in u])}\n"
            f"  rotation {{ z: {phi + 90} }} angle_limit {{ min: 30 max: 70 }} }}")
        acts.append(f'actuators {{ name: "Hip{i}" joint: "Hip{i}" strength: 350 torque {{}} }}')
        acts.append(f'actuators {{ name: "Knee{i}" joint: "Knee{i}" strength: 350 torque {{}} }}')
        incl.append(f'collide_include {{ first: "Shin{i}" second: "Ground" }}')
    out += joints + acts + incl
    out.append('defaults { qps { name: "Torso" pos { z: 0.35 } } }')
    return "\n".join(out) + "\n"


def humanoid():
    # 11 dynamic bodies, 10 joints with dof 2,1,3,3,1,1,2,2,1,1 = 17 (Table 1)
    Y = "rotation { x: 90 }"  # capsule axis along world y
    bodies = [  # name, mass, capsule radius, length, collider rotation
        ("Torso", 8, 0.07, 0.42, Y), ("Lwaist", 2, 0.06, 0.34, Y), ("Pelvis", 5, 0.09, 0.36, Y),
        ("RThigh", 4, 0.06, 0.46, ""), ("RShin", 3, 0.05, 0.5, ""),
        ("LThigh", 4, 0.06, 0.46, ""), ("LShin", 3, 0.05, 0.5, ""),
        ("RUpperArm", 1.5, 0.04, 0.36, ""), ("RLowerArm", 1, 0.031, 0.3, ""),
        ("LUpperArm", 1.5, 0.04, 0.36, ""), ("LLowerArm", 1, 0.031, 0.3, ""),
    ]
    # name, parent, child, parent_offset, child_offset, rotation, limits (deg), strength
    joints = [
        ("Abdomen", "Torso", "Lwaist", (0, 0, -0.12), (0, 0, 0.06), "", [(-45, 45), (-75, 30)], 150),
        ("AbdomenX", "Lwaist", "Pelvis", (0, 0, -0.06), (0, 0, 0.06), "", [(-35, 35)], 150),
        ("RHip", "Pelvis", "RThigh", (0, -0.1, -0.04), (0, 0, 0.2), "", [(-110, 20), (-30, 10), (-60, 35)], 150),
        ("LHip", "Pelvis", "LThigh", (0, 0.1, -0.04), (0, 0, 0.2), "", [(-110, 20), (-10, 30), (-35, 60)], 150),
        ("RKnee", "RThigh", "RShin", (0, 0, -0.2), (0, 0, 0.2), "rotation { z: 90 }", [(-160, -2)], 150),
        ("LKnee", "LThigh", "LShin", (0, 0, -0.2), (0, 0, 0.2), "rotation { z: 90 }", [(-160, -2)], 150),
        ("RShoulder", "Torso", "RUpperArm", (0, -0.2, 0.05), (0, 0, 0.14), "", [(-85, 60), (-85, 60)], 50),
        ("LShoulder", "Torso", "LUpperArm", (0, 0.2, 0.05), (0, 0, 0.14), "", [(-60, 85), (-60, 85)], 50),
        ("RElbow", "RUpperArm", "RLowerArm", (0, 0, -0.14), (0, 0, 0.12), "rotation { z: 90 }", [(-90, 50)], 50),
        ("LElbow", "LUpperArm", "LLowerArm", (0, 0, -0.14), (0, 0, 0.12), "rotation { z: 90 }", [(-90, 50)], 50),
    ]
    out = ["# M4a humanoid (SURVEY §8(d)): 11 capsule bodies, 10 joints, 17 actuated dofs,",
           "# all 11 capsules vs ground, both ends (C = 22).",
           "dt: 0.015", "substeps: 8", "gravity { z: -9.8 }", "friction: 1", "elasticity: 0",
           "baumgarte_erp: 0.2",
           'bodies { name: "Ground" frozen { all: true } colliders { plane {} } }']
    for name, m, r, L, rot in bodies:
        out.append(f'bodies {{ name: "{name}" mass: {f(m)} inertia {{ x: 1 y: 1 z: 1 }}')
        out.append(f"  colliders {{ {rot} capsule {{ radius: {f(r)} length: {f(L)} }} }} }}")
    for name, p, c, po, co, rot, lims, s in joints:
        lim = " ".join(f"angle_limit {{ min: {lo} max: {hi} }}" for lo, hi in lims)
        out.append(f'joints {{ name: "{name}" parent: "{p}" child: "{c}" stiffness: 5000 angular_damping: 20\n'
                   f"  {vec('parent_offset', po)} {vec('child_offset', co)} {rot}\n  {lim} }}")
    for name, *_rest in joints:
        s = _rest[-1]
        out.append(f'actuators {{ name: "{name}" joint: "{name}" strength: {s} torque {{}} }}')
    for name, *_ in bodies:
        out.append(f'collide_include {{ first: "{name}" second: "Ground" }}')
    out.append('defaults { qps { name: "Torso" pos { z: 1.2 } } }')
    return "\n".join(out) + "\n"


def halfcheetah():
    # torso + 7 links, 7 hinges (Table 1); planar via frozen masks (App. E.1, :499)
    X = "rotation { y: 90 }"  # capsule axis along world x
    frz = "frozen { position { y: 1 } rotation { x: 1 z: 1 } }"
    links = [  # name, parent, parent_offset, half length, limits, strength
        ("BThigh", "Torso", (-0.5, 0, 0), 0.145, (-30, 60), 120),
        ("BShin", "BThigh", None, 0.15, (-45, 45), 90),
        ("BFoot", "BShin", None, 0.094, (-23, 45), 60),
        ("FThigh", "Torso", (0.5, 0, 0), 0.133, (-57, 40), 120),
        ("FShin", "FThigh", None, 0.106, (-69, 50), 60),
        ("FFoot", "FShin", None, 0.07, (-29, 29), 30),
    ]
    out = ["# M4b halfcheetah (SURVEY §8(d)): planar torso + 7 links (incl. head), 7 hinges,",
           "# frozen pos y / rot x,z on every body; 8 capsules vs ground, both ends (C = 16).",
           "dt: 0.05", "substeps: 10", "gravity { z: -9.8 }", "friction: 1", "elasticity: 0",
           "baumgarte_erp: 0.2",
           'bodies { name: "Ground" frozen { all: true } colliders { plane {} } }',
           f'bodies {{ name: "Torso" mass: 6 inertia {{ x: 1 y: 1 z: 1 }} {frz}',
           f"  colliders {{ {X} capsule {{ radius: 0.046 length: 1.092 }} }} }}",
           f'bodies {{ name: "Head" mass: 1 inertia {{ x: 0.5 y: 0.5 z: 0.5 }} {frz}',
           f"  colliders {{ {X} capsule {{ radius: 0.046 length: 0.3 }} }} }}"]
    half = {}
    for name, p, po, hl, lim, s in links:
        half[name] = hl
        out.append(f'bodies {{ name: "{name}" mass: 1 inertia {{ x: 0.5 y: 0.5 z: 0.5 }} {frz}')
        out.append(f"  colliders {{ capsule {{ radius: 0.046 length: {f(2 * hl + 0.092)} }} }} }}")
    joints, acts = [], []
    for name, p, po, hl, lim, s in links:
        if po is None:
            po = (0, 0, -half[p])
        joints.append(f'joints {{ name: "{name}" parent: "{p}" child: "{name}" stiffness: 5000 angular_damping: 10\n'
                      f"  {vec('parent_offset', po)} {vec('child_offset', (0, 0, hl))} rotation {{ z: 90 }}\n"
                      f"  angle_limit {{ min: {lim[0]} max: {lim[1]} }} }}")
        acts.append(f'actuators {{ name: "{name}" joint: "{name}" strength: {s} torque {{}} }}')
    joints.append('joints { name: "Neck" parent: "Torso" child: "Head" stiffness: 5000 angular_damping: 10\n'
                  "  parent_offset { x: 0.6 z: 0.1 } child_offset { x: -0.1 } rotation { z: 90 }\n"
                  "  angle_limit { min: -20 max: 20 } }")
    acts.append('actuators { name: "Neck" joint: "Neck" strength: 30 torque {} }')
    out += joints + acts
    for name in ["Torso", "Head"] + [lk[0] for lk in links]:
        out.append(f'collide_include {{ first: "{name}" second: "Ground" }}')
    out.append('defaults { qps { name: "Torso" pos { z: 0.85 } } }')
    return "\n".join(out) + "\n"


def grasp():
    # frozen base + 3-dof wrist + 4 fingers x (2-dof knuckle, 1, 1) = 19 dofs (Table 1)
    out = ["# M5a grasp (SURVEY §8(d)): a 4-fingered claw over a ball (PAPER.md:132).",
           "# Contacts: 12 finger capsules-ball (sphere-capsule), 6 fingertip pairs",
           "# (capsule-capsule), ball-ground, 4 fingertips-ground (both ends): C = 27.",
           "dt: 0.02", "substeps: 4", "gravity { z: -9.8 }", "friction: 1", "elasticity: 0",
           "baumgarte_erp: 0.2",
           'bodies { name: "Ground" frozen { all: true } colliders { plane {} } }',
           'bodies { name: "Base" mass: 1 inertia { x: 1 y: 1 z: 1 } frozen { all: true } }',
           'bodies { name: "Palm" mass: 1 inertia { x: 0.2 y: 0.2 z: 0.2 } }',
           'bodies { name: "Ball" mass: 0.5 inertia { x: 0.01 y: 0.01 z: 0.01 }',
           "  colliders { sphere { radius: 0.1 } } }"]
    links = (("Prox", 0.12, 0.02), ("Mid", 0.1, 0.02), ("Dist", 0.08, 0.02))
    joints = ['joints { name: "Wrist" parent: "Base" child: "Palm" stiffness: 1000 angular_damping: 5\n'
              "  parent_offset { z: -0.05 } child_offset { z: 0.05 }\n"
              "  angle_limit { min: -30 max: 30 } angle_limit { min: -30 max: 30 } angle_limit { min: -30 max: 30 } }"]
    acts = ['actuators { name: "Wrist" joint: "Wrist" strength: 10 torque {} }']
    incl = []
    for i, phi in enumerate((45, 135, 225, 315)):
        u = (math.cos(math.radians(phi)), math.sin(math.radians(phi)))
        prev = "Palm"
        prev_len = None
        for k, (nm, L, r) in enumerate(links):
            body = f"{nm}{i}"
            out.append(f'bodies {{ name: "{body}" mass: 0.2 inertia {{ x: 0.1 y: 0.1 z: 0.1 }}')
            out.append(f"  colliders {{ capsule {{ radius: {r} length: {f(L + 2 * r)} }} }} }}")
            po = (0.09 * u[0], 0.09 * u[1], -0.05) if k == 0 else (0, 0, -prev_len / 2)
            lim = ("angle_limit { min: -30 max: 60 } angle_limit { min: -15 max: 15 }" if k == 0
                   else "angle_limit { min: 0 max: 80 }")
            joints.append(f'joints {{ name: "{body}" parent: "{prev}" child: "{body}" stiffness: 1000 angular_damping: 5\n'
                          f"  {vec('parent_offset', po)} {vec('child_offset', (0, 0, L / 2))} rotation {{ z: {phi + 90} }}\n"
                          f"  {lim} }}")
            acts.append(f'actuators {{ name: "{body}" joint: "{body}" strength: 5 torque {{}} }}')
            incl.append(f'collide_include {{ first: "Ball" second: "{body}" }}')
            prev, prev_len = body, L
    for i in range(4):
        for j in range(i + 1, 4):
            incl.append(f'collide_include {{ first: "Dist{i}" second: "Dist{j}" }}')
    incl.append('collide_include { first: "Ball" second: "Ground" }')
    for i in range(4):
        incl.append(f'collide_include {{ first: "Dist{i}" second: "Ground" }}')
    out += joints + acts + incl
    out.append('defaults { qps { name: "Base" pos { z: 0.6 } } qps { name: "Ball" pos { z: 0.098775 } } }')
    return "\n".join(out) + "\n"


def fetch():
    # box torso + 4 legs x 2 hinges + 2-dof head = 10 actuated dofs (Table 1)
    out = ["# M5b fetch (SURVEY §8(d)): boxy dog-like quadruped (PAPER.md:135) + a frozen,",
           "# non-colliding target marker.  Contacts: box-plane 8 corners + 4 shins-ground x 2.",
           "dt: 0.02", "substeps: 4", "gravity { z: -9.8 }", "friction: 1", "elasticity: 0",
           "baumgarte_erp: 0.2",
           'bodies { name: "Ground" frozen { all: true } colliders { plane {} } }',
           'bodies { name: "Torso" mass: 5 inertia { x: 1 y: 1 z: 1 }',
           "  colliders { box { halfsize { x: 0.3 y: 0.15 z: 0.1 } } } }",
           'bodies { name: "Head" mass: 0.5 inertia { x: 1 y: 1 z: 1 }',
           "  colliders { rotation { y: 90 } capsule { radius: 0.05 length: 0.2 } } }",
           'bodies { name: "Target" mass: 1 inertia { x: 1 y: 1 z: 1 } frozen { all: true } }']
    joints = ['joints { name: "Neck" parent: "Torso" child: "Head" stiffness: 5000 angular_damping: 10\n'
              "  parent_offset { x: 0.35 z: 0.1 } child_offset { x: -0.05 }\n"
              "  angle_limit { min: -30 max: 30 } angle_limit { min: -20 max: 20 } }"]
    acts = ['actuators { name: "Neck" joint: "Neck" strength: 10 torque {} }']
    incl = ['collide_include { first: "Torso" second: "Ground" }']
    for i, (sx, sy) in enumerate(((1, 1), (1, -1), (-1, 1), (-1, -1))):
        out.append(f'bodies {{ name: "Thigh{i}" mass: 0.5 inertia {{ x: 1 y: 1 z: 1 }}')
        out.append("  colliders { capsule { radius: 0.04 length: 0.28 } } }")
        out.append(f'bodies {{ name: "Shin{i}" mass: 0.5 inertia {{ x: 1 y: 1 z: 1 }}')
        out.append("  colliders { capsule { radius: 0.04 length: 0.28 } } }")
        joints.append(f'joints {{ name: "Hip{i}" parent: "Torso" child: "Thigh{i}" stiffness: 5000 angular_damping: 10\n'
                      f"  {vec('parent_offset', (0.25 * sx, 0.12 * sy, -0.1))} child_offset {{ z: 0.1 }} rotation {{ z: 90 }}\n"
                      "  angle_limit { min: -45 max: 45 } }")
        joints.append(f'joints {{ name: "Knee{i}" parent: "Thigh{i}" child: "Shin{i}" stiffness: 5000 angular_damping: 10\n'
                      "  parent_offset { z: -0.1 } child_offset { z: 0.1 } rotation { z: 90 }\n"
                      "  angle_limit { min: -60 max: 0 } }")
        acts.append(f'actuators {{ name: "Hip{i}" joint: "Hip{i}" strength: 30 torque {{}} }}')
        acts.append(f'actuators {{ name: "Knee{i}" joint: "Knee{i}" strength: 30 torque {{}} }}')
        incl.append(f'collide_include {{ first: "Shin{i}" second: "Ground" }}')
    out += joints + acts + incl
    out.append('defaults { qps { name: "Torso" pos { z: 0.55 } } qps { name: "Target" pos { x: 5 z: 0.5 } } }')
    return "\n".join(out) + "\n"


# env epilogue blocks (NEXT-1; R30-R34)
TASKS = {
    "ant": """# Env epilogue (NEXT-1; PAPER.md:505 "Brax's reward function ignores the contact
# cost"; SPEC.md:366 ant reward and done): 87 observations (Table 1).
task {
  torso: "Torso"
  forward { x: 1 }
  survive_reward: 1
  ctrl_cost: 0.5
  healthy_z { min: 0.2 max: 1.0 }
  episode_length: 1000
  contact_obs: true
  reset_noise { vel: 0.1 ang: 0.1 }
}
""",
    "humanoid": """# Env epilogue (NEXT-1; PAPER.md:509: control cost 0.01, done when the torso
# leaves [0.6, 2.1]).  Observation layout of DESIGN.md R32 (117 values; Table 1's
# 299 uses MuJoCo-specific features the paper does not define).
task {
  torso: "Torso"
  forward { x: 1 }
  survive_reward: 1
  ctrl_cost: 0.01
  healthy_z { min: 0.6 max: 2.1 }
  episode_length: 1000
  contact_obs: true
  reset_noise { vel: 0.1 ang: 0.1 }
}
""",
    "halfcheetah": """# Env epilogue (NEXT-1; SPEC.md:366: forward velocity − 0.1·‖a‖², no survive
# bonus, no height-based done): 25 observations (Table 1).
task {
  torso: "Torso"
  forward { x: 1 }
  survive_reward: 0
  ctrl_cost: 0.1
  episode_length: 1000
  contact_obs: false
  reset_noise { vel: 0.1 ang: 0.1 }
}
""",
}


if __name__ == "__main__":
    for name, fn in (("ant", ant), ("humanoid", humanoid), ("halfcheetah", halfcheetah),
                     ("grasp", grasp), ("fetch", fetch)):
        with open(os.path.join(HERE, f"{name}.bxc"), "w") as fh:
            fh.write(fn() + TASKS.get(name, ""))
        print("wrote", name)
