"""Mapping/size sweep of the step kernel: env-steps/s and achieved FP32 TFLOP/s
for (scene, n_envs, warps_per_block) combinations.  In-place stepping of one
batch (L2-resident for small N: a kernel-characterisation sweep, not the bench).

    python tools/sweep.py --scenes ant --envs 8192,65536 --warps 9,17 [--steps 200]
"""
import argparse
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--scenes", default="ant")
p.add_argument("--envs", default="8192")
p.add_argument("--warps", default="0", help="0 = library default")
p.add_argument("--steps", type=int, default=200)
p.add_argument("--rollout", type=int, default=0, help="steps per launch via brax_rollout (0 = brax_step)")
p.add_argument("--substeps", type=int, default=0, help="override the scene's substeps (staging-cost study)")
p.add_argument("--groups", default="0", help="plans 'G:V' (lane groups, envs per lane) or G; 0 = library heuristic")
a = p.parse_args()
with open(os.path.join(ROOT, "profiles", "algorithmic_counts.json")) as f:
    counts = json.load(f)["scenes"]
for scene in a.scenes.split(","):
    text = open(os.path.join(ROOT, "scenes", f"{scene}.bxc")).read()
    if a.substeps:
        import re
        text = re.sub(r"^substeps: *\d+", f"substeps: {a.substeps}", text, flags=re.M)
    for w in [int(x) for x in a.warps.split(",")]:
        if w:
            os.environ["BRAX_WARPS_PER_BLOCK"] = str(w)
        else:
            os.environ.pop("BRAX_WARPS_PER_BLOCK", None)
        s = bx.System(text)
        for n, G in [(int(x), g) for x in a.envs.split(",") for g in a.groups.split(",")]:
            if G != "0":
                os.environ["BRAX_PLAN"] = G.replace(":", ",") if ":" in G else f"{G},1"
            else:
                os.environ.pop("BRAX_PLAN", None)
            qp = s.alloc_qp(n)
            s.reset(qp, 0, 0.1, 0.1)
            T = a.steps
            acts = torch.from_numpy(synth.actions(1, T, n, s.act_dim)).cuda() if s.act_dim else None
            for t in range(min(T, 20)):  # tune on a state of the trajectory (contact activity matters)
                s.step(qp, acts[t] if acts is not None else None, qp)
            if G == "0":
                s.tune(qp, acts[0] if acts is not None else None)
            def run():  # noqa: E306
                if a.rollout:
                    for t0 in range(0, T, a.rollout):
                        s.rollout(qp, acts[t0:t0 + a.rollout] if acts is not None else None, qp,
                                  n_steps=min(a.rollout, T - t0))
                else:
                    for t in range(T):
                        s.step(qp, acts[t] if acts is not None else None, qp)
            run()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()  # replay: kernel time, not Python launch overhead
            with torch.cuda.graph(graph):
                run()
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            rate = n * T / (ms / 1e3)
            # the count is per env-step at the scene's own substeps; per-substep work is the same,
            # so an overridden substep count scales it
            S0 = int(re.search(r"^substeps: *(\d+)", open(os.path.join(ROOT, "scenes", f"{scene}.bxc")).read(),
                               flags=re.M).group(1))
            tf = rate * counts[scene]["flops_per_env_step"] * s.substeps / S0 / 1e12
            print(json.dumps({"scene": scene, "substeps": s.substeps, "envs": n, "G": G, "cfg": s.launch_config(n), "rollout": a.rollout,
                              "us_per_step": 1e3 * ms / T, "env_steps_per_s": rate, "tflops": tf,
                              "frac_fp32_1965": tf / 74.45}), flush=True)
