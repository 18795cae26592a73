"""NEXT-3 on the GPU: the Fig. 5 "astronaut" protocol —
momentum conserved to fp32 rounding under random actuation (equal-and-opposite
joint/actuator impulses, R4/R5), energy drift shrinking as the substep length h
halves (SPEC.md:568-576 monotone-drift criterion)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import astronaut  # noqa: E402


def test_astronaut_protocol():
    res = astronaut.run(seeds=64, substeps_list=(2, 4, 8, 16))
    for r in res:
        # momenta are exact invariants of the discrete map (isotropic inertia, no
        # damping/gravity/contacts): only fp32 rounding remains (|P| ~ 1, |L| ~ 1)
        assert r["linear_momentum_drift"] < 1e-3, r
        assert r["angular_momentum_drift"] < 1e-3, r
    e = [r["energy_drift"] for r in res]
    assert all(e[i + 1] < e[i] for i in range(len(e) - 1)), e   # monotone in h
    assert e[-1] < 0.5 * e[0], e
