"""bench.py end to end on the GPU (short run): the JSON line carries every key the
driver contract asks for, with consistent values (the rate equals envs / step
time, the roofline fraction equals achieved / peak, the clocks were sampled)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "40", "--warmup", "3",
                        "--no-cpu-baseline", "--e2e-steps", "12"],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 40 and d["warmup"] == 3 and d["higher_is_better"] is True
    n = d["config"]["envs_per_gpu"]
    assert abs(d["value"] - n / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    roof = d["roofline"]
    assert roof["bound"] in ("alu", "hbm", "tensor")
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) <= 1e-9
    assert 0.0 < roof["frac"] < 1.0
    e2e = d["e2e"]
    assert 0 < e2e["value"] < d["value"] and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 40
    assert "exactly 40 brax_step launches" in d["config"]["launch"]
    assert d["clocks"]["samples"] >= 10 and d["clocks"]["sm_max_mhz"] > 0
    assert 0.0 < roof["frac_lean"] < roof["frac"]
    assert d["config"]["comm"]["nranks"] == 1
    for sc in ("humanoid", "halfcheetah", "grasp", "fetch"):
        line = d["scenes"][sc]
        assert line["value"] > 0 and 0.0 < line["frac"] < 1.0 and line["blowups"] == 0, (sc, line)
    assert d["blowups"] == 0
    big = d["large_batch"]
    assert big["envs_per_gpu"] == 65536 and big["blowups"] == 0 and 0.0 < big["frac"] < 1.0
    roll = d["rollout"]
    assert roll["value"] > 0 and roll["blowups"] == 0 and 0.0 < roll["frac"] < 1.0
    if d.get("vjp"):
        assert d["vjp"]["value"] > 0 and d["vjp"]["over_step"] > 1.0
