"""Memory-safety and race evidence without compute-sanitizer (closed on this GPU pool,
DESIGN.md §5 "Checks"): guard regions around every device buffer the step kernels
write must stay bit-identical (out-of-bounds writes, ragged last blocks, every
entry point), and repeated launches must give identical bits (a shared-memory race
between the phases would show as run-to-run differences).  SURVEY §5."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
import paper_2106_13281_b200 as bx  # noqa: E402

GUARD = 64  # floats (256 B, a multiple of 16 B: the arrays stay 16-byte aligned)
SENTINEL = np.float32(-12345.678)


class Guarded:
    """A device tensor of `shape` inside a larger buffer whose margins hold a sentinel."""

    def __init__(self, shape, dtype=torch.float32):
        n = int(np.prod(shape))
        self.buf = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
        if dtype == torch.float32:
            self.buf.fill_(float(SENTINEL))
        else:
            self.buf.fill_(0x5A)
        self.t = self.buf[GUARD:GUARD + n].view(*shape)
        self.before = self.buf.clone()

    def margins_intact(self):
        m = torch.cat([self.buf[:GUARD], self.buf[-GUARD:]])
        ref = torch.cat([self.before[:GUARD], self.before[-GUARD:]])
        return bool(torch.equal(m, ref))


def guarded_qp(s, n, init=None):
    B = s.n_bodies
    g = {k: Guarded((n, B, w)) for k, w in (("pos", 3), ("rot", 4), ("vel", 3), ("ang", 3))}
    if init is not None:
        for k in g:
            g[k].t.copy_(init[k])
    return g


def views(g):
    return {k: v.t for k, v in g.items()}


@pytest.mark.parametrize("name,n", [("ant", 1), ("ant", 17), ("ant", 95), ("ant", 257), ("grasp", 33),
                                    ("coverage", 49), ("chain60", 33)])
def test_no_write_outside_the_buffers(name, n):
    text = synth.chain_text(60) if name == "chain60" else oracle.load_scene(name)
    s = bx.System(text)
    o = oracle.Oracle(text)
    qp0 = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
           for k, v in o.reset(n, 5, 0.1, 0.1).items()}
    A = s.act_dim
    act = Guarded((3, n, max(A, 1)))
    act.t.copy_(torch.from_numpy(synth.actions(6, 3, n, max(A, 1))))
    act.before = act.buf.clone()
    out = guarded_qp(s, n)
    status = Guarded((n,), torch.int32)
    ca = Guarded((n, max(1, s.n_slots)), torch.uint8)
    cdp = Guarded((n, s.n_bodies, 6))
    a0 = act.t[0] if A else None
    s.step(qp0, a0, views(out), status=status.t, contact_active=ca.t if s.n_slots else None, contact_dp=cdp.t)
    plans = ("1,1", "2,1", "4,1", "1,2", "2,2", "4,2")
    try:
        for plan in plans:
            for lean in ("0", "1"):
                os.environ.update({"BRAX_PLAN": plan, "BRAX_LEAN": lean, "BRAX_FIXED_GATHER": lean})
                s.step(qp0, a0, views(out), status=status.t)
    finally:
        for k in ("BRAX_PLAN", "BRAX_LEAN", "BRAX_FIXED_GATHER"):
            os.environ.pop(k, None)
    roll = guarded_qp(s, n, qp0)
    s.rollout(views(roll), act.t if A else None, n_steps=3)
    if s.task_info()["has_task"]:
        st = s.env_state(n)
        s.env_reset(st, seed=2)
        s.env_step(st, act.t[0] if A else None, seed=2)
    if name != "chain60":  # the JVP / VJP kernels reject the 60-link chain (too large)
        dq = {k: torch.full_like(v, 1e-3) for k, v in qp0.items()}
        jo, jd = guarded_qp(s, n), guarded_qp(s, n)
        bx.brax_step_jvp(s.handle, qp0, a0, dq, None, views(jo), views(jd), n)
        gi = guarded_qp(s, n)
        ga = Guarded((n, max(A, 1)))
        g = {k: torch.ones_like(v) for k, v in qp0.items()}
        bx.brax_step_vjp(s.handle, qp0, a0, g, views(gi), ga.t if A else None, n)
        guards = [*jo.values(), *jd.values(), *gi.values(), ga]
    else:
        guards = []
    torch.cuda.synchronize()
    for x in [*out.values(), *roll.values(), status, ca, cdp, act, *guards]:
        assert x.margins_intact()


@pytest.mark.parametrize("name", ["ant", "humanoid", "halfcheetah"])
def test_repeated_launches_are_bit_identical(name):
    """20 launches of the same input, tuned plan and both kernels: identical bits every time."""
    o = oracle.Oracle(oracle.load_scene(name))
    s = bx.System(oracle.load_scene(name))
    n = 4096
    q = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda() for k, v in o.reset(n, 9, 0.1, 0.1).items()}
    act = torch.from_numpy(synth.actions(10, 1, n, o.act_dim)[0]).cuda()
    s.tune(q, act)
    ref = s.alloc_qp(n)
    s.step(q, act, ref)
    for rep in range(20):
        out = s.alloc_qp(n)
        s.step(q, act, out)
        torch.cuda.synchronize()
        for k in ref:
            assert torch.equal(out[k], ref[k]), (rep, k)
