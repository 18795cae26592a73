"""Benchmark of the batched Brax physics step on B200 (BASELINE.json metric:
env-steps/sec, ant, 8192 envs/GPU, at 1/2/4/8 GPUs; roofline fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--scene ant] [--envs 8192]
    torchrun --nproc-per-node N bench.py --gpus N ...   (what `python bench.py --gpus N` starts itself)
    python bench.py --impl reference ...                 (the fp64 oracle on host cores)

One "step" = one brax_step launch advancing every env of this rank's batch by
one env-step (`substeps` × Alg. 1).  Envs are sharded across
ranks (weak scaling: 8192 envs per GPU); there is no data-path collective — one
all-reduce of ≤ 32 B of statistics after the timed region (SURVEY §8(e),
paper_2106_13281_b200/dist.py, gloo-tested through `--dist-selftest`).

Timed region: exactly K brax_step launches captured in ONE CUDA graph (any K),
replayed once untimed, then replayed once between CUDA events on the launch
stream, with a barrier and a device synchronize on both sides; value = all
ranks' env-steps ÷ the max over ranks of that time.  L2 hygiene: the K launches
cycle over R independent env batches whose QP buffers together exceed the
126 MB L2, so every launch reads its inputs from HBM.  The launch configuration
is measured before (brax_system_tune), never inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_ENVS = {"ant": 8192, "humanoid": 4096, "halfcheetah": 4096, "grasp": 2048, "fetch": 2048,
                "pendulum": 1024, "chain2": 1024, "ball": 1}
OTHER_SCENES = ("humanoid", "halfcheetah", "grasp", "fetch")  # BASELINE.json configs[3], [4] at their sizes
L2_BYTES = 126 * 1024 * 1024


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=50)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--scene", default="ant")
    p.add_argument("--envs", type=int, default=None, help="envs per GPU")
    p.add_argument("--no-env", action="store_true", help="skip the brax_env_step (NEXT-1) measurement")
    p.add_argument("--no-rollout", action="store_true", help="skip the fused-rollout (NEXT-2) measurement")
    p.add_argument("--no-vjp", action="store_true", help="skip the brax_step_vjp (NEXT-4) measurement")
    p.add_argument("--no-scenes", action="store_true", help="skip the other scenes' lines")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=200)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--soak-seconds", type=float, default=0.3,
                   help="untimed graph replays right before the timed one (clock sampling under load)")
    p.add_argument("--dist-selftest", action="store_true",
                   help="CPU check of the rank launch + statistics all-reduce (gloo), no GPU work")
    return p.parse_args(argv)


def _dist():
    """paper_2106_13281_b200/dist.py by path: the rank plumbing without importing the
    package (whose import loads the CUDA library; the reference arm must not)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("brax_b200_dist",
                                                  os.path.join(ROOT, "paper_2106_13281_b200", "dist.py"))
    if spec.name in sys.modules:
        return sys.modules[spec.name]
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    return mod


def metric_for(scene, n):
    return f"env-steps/sec ({scene}, {n} envs/GPU)"


def load_counts(scene):
    with open(os.path.join(ROOT, "profiles", "algorithmic_counts.json")) as f:
        return json.load(f)["scenes"][scene]


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks (NVML, during the load window)
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """Samples the SM clock and throttle reasons every ~2 ms while active."""

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 — clocks are reported as unavailable
            self.nv = None

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()
            self._sample()  # one more right at the end of the window

    def report(self, window):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "window": window}
        names = [v for k, v in REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_min_mhz": float(np.min(self.samples)),
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples), "window": window}


# ------------------------------------------------------------------ oracle legs (host cores)
def oracle_rate(scene, n, seconds, max_steps=None, seed=0, threads=None):
    """fp64 oracle, envs partitioned over `threads` host threads (default: all cores);
    returns (env-steps/s, threads, steps, elapsed s)."""
    import oracle
    import synth
    cores = threads or len(os.sched_getaffinity(0))
    o = oracle.Oracle(oracle.load_scene(scene))
    qp = o.reset(n, seed, 0.1, 0.1)
    acts = synth.actions(seed + 1, 64, n, o.act_dim)
    done, t0 = 0, time.perf_counter()
    while True:
        qp, _ = o.step(qp, acts[done % 64], threads=cores)
        done += 1
        el = time.perf_counter() - t0
        if (max_steps is not None and done >= max_steps) or (max_steps is None and el >= seconds):
            break
    return n * done / el, cores, done, el


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return  # under torchrun only rank 0 runs and prints
    n = args.envs or DEFAULT_ENVS[args.scene]
    sample = min(n, 1024)
    # warmup W steps, then exactly K timed steps, each a bounded sample of the workload
    oracle_rate(args.scene, sample, 0, max_steps=max(1, args.warmup))
    rate, cores, steps, el = oracle_rate(args.scene, sample, 0, max_steps=args.steps)
    line = {"impl": "reference", "metric": metric_for(args.scene, n), "value": rate, "unit": "env-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.scene} random actions; each step = {sample} of the {n} envs/GPU",
                       "envs_per_gpu": n},
            "cpu_baseline": {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} {args.scene} envs x {steps} steps (fp64 oracle, "
                                       f"{cores} host threads)"},
            "e2e": {"value": rate, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ rank plumbing self-test (CPU, gloo)
def run_dist_selftest(args):
    """The rank launch and statistics path bench.py's B200 arm runs (dist.init_ranks,
    dist.barrier, dist.allreduce_stats), on gloo with synthetic per-rank numbers."""
    bd = _dist()
    r = bd.init_ranks("gloo")
    bd.barrier(r)
    steps, blow, _, ms = bd.allreduce_stats(float(100 * (r.rank + 1)), float(r.rank), 10.0 + r.rank)
    bd.barrier(r)
    if r.rank == 0:
        print(json.dumps({"selftest": "dist", "n_gpus": r.world, "nranks": r.nranks, "backend": r.backend,
                          "env_steps": steps, "blowups": blow, "ms_max": ms}), flush=True)
    bd.finalize(r)


# ------------------------------------------------------------------ B200 arm
class Workload:
    """One scene at one batch size on this rank: R rotating env batches (> L2 together),
    their actions, the tuned launch configuration, and a CUDA graph of exactly K steps."""

    def __init__(self, bx, synth, torch, scene, n, rank, stream):
        with open(os.path.join(ROOT, "scenes", f"{scene}.bxc")) as f:
            self.system = bx.System(f.read(), device=torch.cuda.current_device())
        s = self.system
        self.scene, self.n, self.stream, self.torch = scene, n, stream, torch
        B, A = s.n_bodies, s.act_dim
        self.qp_bytes = n * B * 13 * 4
        self.R = min(64, max(2, int(np.ceil(1.5 * L2_BYTES / max(1, 2 * self.qp_bytes + n * A * 4)))))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.sets = []
        with torch.cuda.stream(stream):
            for r in range(self.R):  # rank-distinct seeds: env ids are global (weak scaling)
                qp = s.alloc_qp(n)
                s.reset(qp, seed=1000 * rank + r, vel_noise=0.1, ang_noise=0.1, stream=stream)
                self.sets.append(qp)
            self.acts = torch.from_numpy(synth.actions(17 + rank, self.R, n, A)).to(dev) if A else None
        stream.synchronize()
        self.graph = None
        self.tuned = False

    def tune(self):
        """The launch configuration, measured outside any timed region on a state of the
        workload's own trajectory (after warm-up: contact activity decides between plans)."""
        self.system.tune(self.sets[0], self.act(0), stream=self.stream)
        self.tuned = True

    def act(self, i):
        return self.acts[i % self.R] if self.acts is not None else None

    def launch(self, i):
        r = i % self.R
        self.system.step(self.sets[r], self.act(r), self.sets[r], stream=self.stream)

    def warmup(self, W):
        with self.torch.cuda.stream(self.stream):
            for i in range(W):
                self.launch(i)
                if i == min(W, 2 * self.R) - 1 and not self.tuned:
                    self.stream.synchronize()
                    self.tune()
        self.stream.synchronize()
        if not self.tuned:
            self.tune()

    def capture(self, K):
        torch = self.torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            for i in range(K):
                self.launch(i)
        self.stream.synchronize()
        with torch.cuda.stream(self.stream):  # CUDAGraph.replay launches on the current stream
            self.graph.replay()  # untimed: upload + first execution
        self.stream.synchronize()

    def timed_replay(self, ranks, bd, soak_s=0.0, sampler=None):
        """Soak (untimed replays, clocks sampled), then ONE timed replay: barrier + sync on
        both sides, CUDA events on the launch stream; returns this rank's ms."""
        torch = self.torch
        with torch.cuda.stream(self.stream):  # CUDAGraph.replay launches on the current stream
            if soak_s > 0:
                t0 = time.perf_counter()
                while time.perf_counter() - t0 < soak_s:
                    self.graph.replay()
                    self.stream.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            bd.barrier(ranks)
            torch.cuda.synchronize()
            ev0.record(self.stream)
            self.graph.replay()
            ev1.record(self.stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        bd.barrier(ranks)
        return ev0.elapsed_time(ev1)

    def blowups(self):
        torch = self.torch
        status = torch.zeros(self.n, dtype=torch.int32, device=self.sets[0]["pos"].device)
        probe = self.system.alloc_qp(self.n)
        self.system.step(self.sets[0], self.act(0), probe, status=status, stream=self.stream)
        self.stream.synchronize()
        return int((status != 0).sum())


def roofline(counts, n, launch_s, peaks, peak_src, clocks):
    """Algorithmic flops (or bytes) per launch ÷ the launch's duration, against the FP32
    (or HBM) peak; both flop conventions of profiles/algorithmic_counts.json."""
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tflops = 148 * 128 * 2 * f_max * 1e6 / 1e12
    flops = counts["flops_per_env_step"] * n
    bytes_ = counts["bytes_per_env_step"] * n
    intensity = counts["flops_per_env_step"] / counts["bytes_per_env_step"]
    balance = peak_tflops * 1e12 / (float(peaks["hbm_gbs"]) * 1e9)
    if intensity >= balance:
        ach = flops / launch_s / 1e12
        out = {"bound": "alu", "achieved": ach, "peak": peak_tflops, "unit": "TFLOP/s", "frac": ach / peak_tflops,
               "peak_source": f"148 SM x 128 FP32 lanes x 2 x {f_max:.0f} MHz (sm_max_mhz, {peak_src})",
               "algorithmic_flops_per_launch": flops, "launch_us": launch_s * 1e6,
               "hbm_frac": bytes_ / launch_s / (float(peaks["hbm_gbs"]) * 1e9)}
        if "flops_per_env_step_lean" in counts:
            lean = counts["flops_per_env_step_lean"] * n / launch_s / 1e12
            out["achieved_lean"] = lean
            out["frac_lean"] = lean / peak_tflops
            out["conventions"] = ("frac: oracle op counter, every operation of SURVEY 8(c).1 "
                                  f"({counts['flops_per_env_step']:.0f} flop/env-step); frac_lean: operations an "
                                  "exactly neutral scene value makes not counted "
                                  f"({counts['flops_per_env_step_lean']:.0f} flop/env-step)")
        if clocks.get("sm_mhz"):
            out["frac_at_run_clock"] = ach / (148 * 128 * 2 * clocks["sm_mhz"] * 1e6 / 1e12)
        return out
    ach = bytes_ / launch_s / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
            "frac": ach / float(peaks["hbm_gbs"]), "peak_source": f"hbm_gbs ({peak_src})",
            "algorithmic_bytes_per_launch": bytes_, "launch_us": launch_s * 1e6}


def run_b200(args):
    import torch

    import paper_2106_13281_b200 as bx
    import synth
    bd = _dist()

    ranks = bd.init_ranks("nccl")
    rank, world = ranks.rank, ranks.world
    dev = torch.device("cuda", ranks.local)
    n = args.envs or DEFAULT_ENVS[args.scene]
    K, W = args.steps, args.warmup
    stream = torch.cuda.Stream(device=dev)
    wl = Workload(bx, synth, torch, args.scene, n, rank, stream)
    system = wl.system
    B, A = system.n_bodies, system.act_dim
    wl.warmup(W)
    wl.capture(K)
    with ClockSampler(ranks.local) as clk:
        ms = wl.timed_replay(ranks, bd, soak_s=args.soak_seconds)
    clocks = clk.report(f"{args.soak_seconds:.2f} s of untimed replays of the timed graph, then the timed replay")
    blowups = wl.blowups()
    total_env_steps, total_blowups, _, ms_max = bd.allreduce_stats(float(n * K), float(blowups), ms, device=dev)
    value = total_env_steps / (ms_max / 1e3)

    # ---- e2e through the public API with host buffers: every step copies its inputs (qp +
    # action) from pinned host memory, steps, and copies the resulting qp back.  A
    # three-stage pipeline over NB independent env batches: one stream per stage
    # (H2D copy | brax_step | D2H copy) chained by events, so step i's upload, step
    # i-1's kernel and step i-2's download run at once on the two copy engines and the
    # SMs.  Timed on the device from a start event every stage stream waits on to the
    # last download's completion.
    NB = 6
    sizes = [n * B * 3, n * B * 4, n * B * 3, n * B * 3]
    nq = sum(sizes)

    def views(flat):
        out, o = {}, 0
        for k, sz, w in zip(("pos", "rot", "vel", "ang"), sizes, (3, 4, 3, 3)):
            out[k] = flat[o:o + sz].view(n, B, w)
            o += sz
        return out, (flat[o:o + n * A].view(n, A) if A else None)

    host_in, host_out, dflat = [], [], []
    for r in range(NB):
        h = torch.empty(nq + n * A, dtype=torch.float32).pin_memory()
        hq, ha = views(h)
        for k in hq:
            hq[k].copy_(wl.sets[r % wl.R][k].cpu())
        if A:
            ha.copy_(wl.act(r).cpu())
        host_in.append(h)
        host_out.append(torch.empty(nq, dtype=torch.float32).pin_memory())
        dflat.append(torch.empty(nq + n * A, dtype=torch.float32, device=dev))
    dviews = [views(f) for f in dflat]
    s_in, s_k, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_k = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]
    used = [False] * NB
    Ke = max(NB, min(args.e2e_steps, K))

    def e2e_step(i):
        j = i % NB
        if used[j]:
            s_in.wait_event(ev_out[j])  # batch j's buffer is free once its last result left
        with torch.cuda.stream(s_in):
            dflat[j].copy_(host_in[j], non_blocking=True)
            ev_in[j].record(s_in)
        s_k.wait_event(ev_in[j])
        dq, da = dviews[j]
        system.step(dq, da, dq, stream=s_k)
        ev_k[j].record(s_k)
        s_out.wait_event(ev_k[j])
        with torch.cuda.stream(s_out):
            host_out[j].copy_(dflat[j][:nq], non_blocking=True)
            ev_out[j].record(s_out)
        used[j] = True

    for i in range(2 * NB):
        e2e_step(i)
    torch.cuda.synchronize()
    bd.barrier(ranks)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for st in (s_in, s_k, s_out):
        st.wait_event(e0)
    for i in range(Ke):
        e2e_step(i)
    stream.wait_stream(s_out)
    e1.record(stream)
    e1.synchronize()
    e_ms = bd.allreduce_max(e0.elapsed_time(e1), device=dev)
    e2e = {"value": n * world * Ke / (e_ms / 1e3), "unit": "env-steps/s",
           "h2d_bytes_per_step": int(wl.qp_bytes + n * A * 4), "d2h_bytes_per_step": int(wl.qp_bytes),
           "steps": Ke, "batches": NB,
           "path": "pinned host -> one cudaMemcpyAsync (qp + actions) -> brax_step -> one cudaMemcpyAsync (qp) "
                   f"-> pinned host, every step; three-stage stream pipeline (upload | step | download) over "
                   f"{NB} independent batches"}

    # ---- the other benchmark scenes at their BASELINE sizes (configs[3], [4]), same protocol
    scene_lines = None
    if not args.no_scenes and args.scene == "ant" and args.envs is None:
        scene_lines = {}
        for sc in OTHER_SCENES:
            m = DEFAULT_ENVS[sc]
            w2 = Workload(bx, synth, torch, sc, m, rank, stream)
            w2.warmup(max(3, min(W, 20)))
            w2.capture(K)
            ms2 = bd.allreduce_max(w2.timed_replay(ranks, bd), device=dev)
            c2 = load_counts(sc)
            peaks, peak_src = load_peaks()
            rf = roofline(c2, m, (ms2 / 1e3) / K, peaks, peak_src, {})
            scene_lines[sc] = {"metric": metric_for(sc, m), "value": m * world * K / (ms2 / 1e3),
                               "unit": "env-steps/s", "ms_per_step": ms2 / K, "envs_per_gpu": m,
                               "substeps": w2.system.substeps, "frac": rf["frac"], "frac_lean": rf.get("frac_lean"),
                               "kernel_config": w2.system.launch_config(m), "blowups": w2.blowups(),
                               "l2": f"{w2.R} rotating batches"}
            del w2
            torch.cuda.empty_cache()

    # ---- the M6 N-sweep's large end: the same scene at 65536 envs per GPU,
    # same protocol, a graph of min(K, 200) launches
    large_line = None
    if not args.no_scenes and args.envs is None:
        m, Kl = 65536, max(1, min(K, 200))
        w3 = Workload(bx, synth, torch, args.scene, m, rank, stream)
        w3.warmup(max(3, min(W, 20)))
        w3.capture(Kl)
        ms3 = bd.allreduce_max(w3.timed_replay(ranks, bd), device=dev)
        peaks, peak_src = load_peaks()
        rf = roofline(load_counts(args.scene), m, (ms3 / 1e3) / Kl, peaks, peak_src, {})
        large_line = {"envs_per_gpu": m, "value": m * world * Kl / (ms3 / 1e3), "unit": "env-steps/s",
                      "ms_per_step": ms3 / Kl, "steps": Kl, "frac": rf["frac"], "frac_lean": rf.get("frac_lean"),
                      "kernel_config": w3.system.launch_config(m), "blowups": w3.blowups(),
                      "l2": f"{w3.R} rotating batches"}
        del w3
        torch.cuda.empty_cache()

    # ---- NEXT-1: the same workload through brax_env_step (reward, done, auto-reset and
    # observations fused into the step), when the scene has a task block
    env_line = None
    tinfo = system.task_info()
    if tinfo["has_task"] and not args.no_env:
        od = tinfo["obs_dim"]
        R = wl.R
        with torch.cuda.stream(stream):
            est = [{"steps": torch.zeros(n, dtype=torch.int32, device=dev),
                    "episode": torch.zeros(n, dtype=torch.int32, device=dev),
                    "obs": torch.empty((n, od), device=dev), "reward": torch.empty(n, device=dev),
                    "done": torch.empty(n, dtype=torch.uint8, device=dev)} for _ in range(R)]

            def env_launch(i):
                r, st = i % R, est[i % R]
                bx.brax_env_step(system.handle, wl.sets[r], wl.act(r), 1, wl.sets[r], n, st["obs"], st["reward"],
                                 st["done"], st["steps"], st["episode"], seed=rank + 1, env_offset=rank * n,
                                 stream=stream)
            for i in range(R):
                env_launch(i)
        stream.synchronize()
        Kv = max(R, min(K, 200))
        egraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(egraph, stream=stream):
            for i in range(Kv):
                env_launch(i)
        with torch.cuda.stream(stream):
            egraph.replay()
            stream.synchronize()
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x0.record(stream)
            egraph.replay()
            x1.record(stream)
        x1.synchronize()
        env_ms = bd.allreduce_max(x0.elapsed_time(x1), device=dev)
        env_line = {"value": n * world * Kv / (env_ms / 1e3), "unit": "env-steps/s", "ms_per_step": env_ms / Kv,
                    "steps": Kv, "obs_dim": od,
                    "api": "brax_env_step: physics + reward/done/auto-reset/observation epilogue, one launch"}

    # ---- NEXT-2: T steps of the same workload in ONE launch (brax_rollout_random: the QP
    # stays in shared memory for all T·S substeps, actions drawn in the kernel), on a copy
    # of one batch; device-timed like the step
    roll_line = None
    if not args.no_rollout:
        Tr, reps = 100, 3
        with torch.cuda.stream(stream):
            rq = {k: v.clone() for k, v in wl.sets[0].items()}
            system.rollout_random(rq, Tr, seed=rank + 5, env_offset=rank * n, stream=stream)
            stream.synchronize()
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record(stream)
            for j in range(reps):
                system.rollout_random(rq, Tr, seed=rank + 5, env_offset=rank * n, step0=(j + 1) * Tr, stream=stream)
            r1.record(stream)
            r1.synchronize()
        r_ms = bd.allreduce_max(r0.elapsed_time(r1), device=dev)
        bad = int((~torch.isfinite(rq["pos"]).all(dim=(1, 2))).sum().item())
        rrf = roofline(load_counts(args.scene), n, (r_ms / 1e3) / (reps * Tr), *load_peaks(), clocks)
        roll_line = {"value": n * world * reps * Tr / (r_ms / 1e3), "unit": "env-steps/s",
                     "ms_per_step": r_ms / (reps * Tr), "steps_per_launch": Tr, "launches": reps,
                     "frac": rrf["frac"], "frac_lean": rrf.get("frac_lean"), "blowups": bad,
                     "api": "brax_rollout_random: T steps in one launch, actions from the in-kernel Philox stream"}
        del rq

    # ---- NEXT-4: reverse mode of the same step (brax_step_vjp: g_in = Jᵀ·g_out and
    # g_action, one launch) on one batch of the workload; device-timed like the step
    vjp_line = None
    if not args.no_vjp:
        gen = torch.Generator(device="cpu").manual_seed(7)
        g_out = {k: torch.randn(v.shape, generator=gen).to(dev) for k, v in wl.sets[0].items()}
        with torch.cuda.stream(stream):
            for _ in range(2):
                system.step_vjp(wl.sets[0], wl.act(0), g_out, stream=stream)
            stream.synchronize()
            Kv = 20
            v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            v0.record(stream)
            for _ in range(Kv):
                system.step_vjp(wl.sets[0], wl.act(0), g_out, stream=stream)
            v1.record(stream)
            v1.synchronize()
        v_ms = bd.allreduce_max(v0.elapsed_time(v1), device=dev)
        vjp_line = {"value": n * world * Kv / (v_ms / 1e3), "unit": "env-steps/s", "ms_per_step": v_ms / Kv,
                    "steps": Kv, "over_step": (v_ms / Kv) / (ms_max / K),
                    "api": "brax_step_vjp: Jᵀ·g of one step (QP and action cotangents), one launch"}

    bd.barrier(ranks)
    if rank != 0:
        bd.finalize(ranks)
        return

    counts = load_counts(args.scene)
    peaks, peak_src = load_peaks()
    launch_s = (ms / 1e3) / K  # this rank's average launch duration (events on the launch stream)
    roof = roofline(counts, n, launch_s, peaks, peak_src, clocks)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    roof["traffic"] = None
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(args.scene, {})
        if tr.get("envs") == n and tr.get("bytes_per_launch"):
            roof["traffic"] = tr["bytes_per_launch"]
            roof["traffic_source"] = tr.get("source")

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        m = min(n, 2048)
        rate, cores, steps, el = oracle_rate(args.scene, m, args.cpu_seconds)
        rate1, _, steps1, el1 = oracle_rate(args.scene, min(m, 256), args.cpu_seconds / 2, threads=1)
        cpu = {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
               "sample": f"{m} {args.scene} envs x {steps} steps, fp64 oracle, {cores} host threads, {el:.1f} s",
               "single_thread": {"value": rate1, "cores": 1,
                                 "sample": f"{min(m, 256)} envs x {steps1} steps, 1 thread, {el1:.1f} s"}}

    line = {
        "metric": metric_for(args.scene, n), "value": value, "unit": "env-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.scene}, {n} envs/GPU, random actions U(-1,1), "
                               f"{system.substeps} substeps/step",
                   "envs_per_gpu": n, "global_envs": n * world, "parallelism": f"env-shard x{world}",
                   "l2": f"inputs larger than L2: {wl.R} rotating batches x {2 * wl.qp_bytes / 1e6:.1f} MB "
                         f"(> 126 MB L2)",
                   "launch": f"one CUDA graph of exactly {K} brax_step launches, replayed once untimed, "
                             f"then timed; consecutive launches overlap, ordered per env granule "
                             f"(DESIGN.md §5 'Launch overlap')",
                   "kernel_config": system.launch_config(n),
                   "comm": {"backend": ranks.backend, "nranks": ranks.nranks}},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K, "clocks": clocks,
        "scenes": scene_lines, "large_batch": large_line, "env_epilogue": env_line, "rollout": roll_line,
        "vjp": vjp_line,
        "blowups": total_blowups, "substeps_per_s": value * system.substeps,
    }
    print(json.dumps(line), flush=True)
    bd.finalize(ranks)


def main():
    args = parse()
    rc = _dist().launch_or_check(args.gpus, os.path.abspath(__file__), sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    if args.dist_selftest:
        run_dist_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
