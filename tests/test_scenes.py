"""The synthetic benchmark scenes: structure as specified
and 1000-step random-action stability in the oracle (no status bit)."""
import numpy as np
import pytest

import oracle
import synth

STRUCT = {  # scene: (B, J, A, C, substeps)
    "ball": (2, 0, 0, 1, 1), "pendulum": (2, 1, 1, 0, 1), "chain2": (3, 2, 2, 0, 2),
    "ant": (10, 8, 8, 9, 10), "humanoid": (12, 10, 17, 22, 8), "halfcheetah": (9, 7, 7, 16, 10),
    "grasp": (17, 13, 19, 27, 4), "fetch": (12, 9, 10, 16, 4), "coverage": (7, 3, 6, 16, 5),
}


@pytest.mark.parametrize("name", list(STRUCT))
def test_structure(name):
    o = oracle.Oracle(oracle.load_scene(name))
    assert (o.n_bodies, len(o.sys.joints), o.act_dim, o.n_slots, o.sys.substeps) == STRUCT[name]
    assert o.sys.lint() == []


@pytest.mark.parametrize("name", list(STRUCT))
def test_1000_step_random_action_stability(name):
    o = oracle.Oracle(oracle.load_scene(name))
    n = 8
    qp = o.reset(n, 0, 0.1, 0.1)
    acts = synth.actions(1, 1000, n, o.act_dim)
    status = np.zeros(n, np.uint32)
    for t in range(1000):
        qp, ex = o.step(qp, acts[t], threads=4)
        status |= ex["status"]
    assert np.all(status == 0)
    for k in qp:
        assert np.all(np.isfinite(qp[k]))
    assert np.max(np.abs(qp["vel"])) < 100 and np.max(np.abs(qp["ang"])) < 200


@pytest.mark.parametrize("links", [24, 60])
def test_generated_chain_is_stable(links):
    """The maximum-size parity scenes (synth.chain_text): valid, lint-free, and
    100 random-action steps without a status bit in the oracle."""
    o = oracle.Oracle(synth.chain_text(links))
    assert (o.n_bodies, len(o.sys.joints), o.act_dim, o.n_slots) == (links + 1, links - 1, links - 1, 2 * links)
    assert o.sys.lint() == []
    n = 4
    qp = o.reset(n, 0, 0.1, 0.1)
    acts = synth.actions(1, 100, n, o.act_dim)
    status = np.zeros(n, np.uint32)
    for t in range(100):
        qp, ex = o.step(qp, acts[t], threads=4)
        status |= ex["status"]
    assert np.all(status == 0)
