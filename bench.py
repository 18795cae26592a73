"""Benchmark of the batched Brax physics step on B200 (BASELINE.json metric:
env-steps/sec, ant, 8192 envs/GPU, at 1/2/4/8 GPUs; roofline fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--scene ant] [--envs 8192]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)
    python bench.py --impl reference ...                        (the fp64 oracle on host cores)

One "step" = one brax_step launch advancing every env of this rank's batch by
one env-step (`substeps` × Alg. 1).  Envs are sharded across ranks (weak
scaling: 8192 envs per GPU); there is no data-path collective — one NCCL
all-reduce of ≤ 64 B of statistics after the timed region.

L2 hygiene: the timed loop cycles over R independent env batches whose QP
buffers together exceed the 126 MB L2 (R × 4.26 MB for ant), so every step
reads its inputs from HBM.  Actions are pre-generated on device outside the
timed region.  Timing: CUDA events on the launch stream, barrier + synchronize
on both sides, max over ranks.
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
METRIC = "env-steps/sec (ant, 8192 envs/GPU)"
L2_BYTES = 126 * 1024 * 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=4000)
    p.add_argument("--warmup", type=int, default=50)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--scene", default="ant")
    p.add_argument("--envs", type=int, default=None, help="envs per GPU")
    p.add_argument("--no-graph", action="store_true", help="launch each step from Python instead of a CUDA graph")
    p.add_argument("--no-env", action="store_true", help="skip the brax_env_step (NEXT-1) measurement")
    p.add_argument("--no-vjp", action="store_true", help="skip the brax_step_vjp (NEXT-4) measurement")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=200)
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def metric_for(scene, n):
    return METRIC if (scene == "ant" and n == 8192) else f"env-steps/sec ({scene}, {n} envs/GPU)"


def load_counts(scene):
    path = os.path.join(ROOT, "profiles", "algorithmic_counts.json")
    with open(path) as f:
        return json.load(f)["scenes"][scene]


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks (NVML, during the timed region)
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
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

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
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

    def report(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [v for k, v in REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ oracle legs (host cores)
def oracle_rate(scene, n, seconds, max_steps=None, seed=0):
    """fp64 oracle, envs partitioned over all host cores; returns (env-steps/s, cores, steps, n)."""
    import oracle
    import synth
    cores = len(os.sched_getaffinity(0))
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
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
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


# ------------------------------------------------------------------ B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2106_13281_b200 as bx
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = args.envs or DEFAULT_ENVS[args.scene]
    with open(os.path.join(ROOT, "scenes", f"{args.scene}.bxc")) as f:
        text = f.read()
    system = bx.System(text, device=local)
    B, A = system.n_bodies, system.act_dim
    qp_bytes = n * B * 13 * 4
    R = max(2, int(np.ceil(1.5 * L2_BYTES / max(1, 2 * qp_bytes + n * A * 4))))
    R = min(R, 64)
    stream = torch.cuda.Stream(device=dev)
    # R independent batches (rank-distinct seeds: env ids are global, weak scaling)
    sets = []
    with torch.cuda.stream(stream):
        for r in range(R):
            qp = system.alloc_qp(n)
            system.reset(qp, seed=1000 * rank + r, vel_noise=0.1, ang_noise=0.1, stream=stream)
            sets.append(qp)
        G = R  # one graph = one step of each of the R batches
        acts = torch.from_numpy(synth.actions(17 + rank, G, n, A)).to(dev) if A else None

    def one_round():
        for r in range(R):
            system.step(sets[r], acts[r] if A else None, sets[r], stream=stream)

    # warmup W steps (untimed), then capture the round as a graph
    with torch.cuda.stream(stream):
        for w in range(args.warmup):
            r = w % R
            system.step(sets[r], acts[r] if A else None, sets[r], stream=stream)
    stream.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            one_round()
        stream.synchronize()
    K = args.steps
    full, rem = divmod(K, R)

    def timed_loop():
        with torch.cuda.stream(stream):
            for _ in range(full):
                if graph is not None:
                    graph.replay()
                else:
                    one_round()
            for r in range(rem):
                system.step(sets[r], acts[r] if A else None, sets[r], stream=stream)

    # one untimed pass of the timed loop body (graph upload etc.)
    with torch.cuda.stream(stream):
        if graph is not None:
            graph.replay()
    stream.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record(stream)
        timed_loop()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)

    # health of the result (no blow-ups) and the statistics all-reduce
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    probe = system.alloc_qp(n)
    system.step(sets[0], acts[0] if A else None, probe, status=status, stream=stream)
    stream.synchronize()
    blowups = int((status != 0).sum())
    stats = torch.tensor([float(n * K), float(blowups), ms], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats[2:3].clone()
        dist.all_reduce(stats[:2], op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        stats[2] = mx[0]
    total_env_steps, total_blowups, ms_max = float(stats[0]), int(stats[1]), float(stats[2])
    value = total_env_steps / (ms_max / 1e3)

    # e2e through the public API with host buffers: every step copies its inputs (qp +
    # action) from pinned host memory, steps, and copies the resulting qp back.  A
    # three-stage pipeline over NB independent env batches: one stream per stage
    # (H2D copy | brax_step | D2H copy) chained by events, so step i's upload, step
    # i-1's kernel and step i-2's download run at once on the two copy engines and the
    # SMs (tools/experiments/e2e_pipe.py: +7 % over round-robin streams; PCIe-bound).
    # Timed on the device from a start event every stage stream waits on to the last
    # download's completion.
    e2e = None
    if rank == 0 or world > 1:
        NB = 6
        # one contiguous buffer per batch: pos | rot | vel | ang | actions (the brax_qp
        # members point into it), so each direction is a single copy per step
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
                hq[k].copy_(sets[r % R][k].cpu())
            if A:
                ha.copy_(acts[r % R].cpu())
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
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in (s_in, s_k, s_out):
            st.wait_event(e0)
        for i in range(Ke):
            e2e_step(i)
        stream.wait_stream(s_out)
        e1.record(stream)
        e1.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": n * world * Ke / (float(e_ms[0]) / 1e3), "unit": "env-steps/s",
               "h2d_bytes_per_step": int(qp_bytes + n * A * 4), "d2h_bytes_per_step": int(qp_bytes),
               "steps": Ke, "batches": NB,
               "path": "pinned host -> one cudaMemcpyAsync (qp + actions) -> brax_step -> one cudaMemcpyAsync (qp) "
                       f"-> pinned host, every step; three-stage stream pipeline (upload | step | download) over "
                       f"{NB} independent batches"}

    # NEXT-1: the same workload through brax_env_step (reward, done, auto-reset and
    # observations fused into the step), when the scene has a task block
    env_line = None
    tinfo = system.task_info()
    if tinfo["has_task"] and not args.no_env:
        od = tinfo["obs_dim"]
        with torch.cuda.stream(stream):
            est = []
            for r in range(R):
                st = {"steps": torch.zeros(n, dtype=torch.int32, device=dev),
                      "episode": torch.zeros(n, dtype=torch.int32, device=dev),
                      "obs": torch.empty((n, od), device=dev), "reward": torch.empty(n, device=dev),
                      "done": torch.empty(n, dtype=torch.uint8, device=dev)}
                est.append(st)

            def env_round():
                for r in range(R):
                    st = est[r]
                    bx.brax_env_step(system.handle, sets[r], acts[r] if A else None, 1, sets[r], n, st["obs"],
                                     st["reward"], st["done"], st["steps"], st["episode"], seed=rank + 1,
                                     env_offset=rank * n, stream=stream)
            for _ in range(3):
                env_round()
        stream.synchronize()
        egraph = None
        if not args.no_graph:
            egraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(egraph, stream=stream):
                env_round()
            stream.synchronize()
        Kr = max(1, full)
        with torch.cuda.stream(stream):
            (egraph.replay() if egraph is not None else env_round())
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(Kr):
                egraph.replay() if egraph is not None else env_round()
            e1.record(stream)
            e1.synchronize()
        env_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(env_ms, op=dist.ReduceOp.MAX)
        steps_env = Kr * R
        env_line = {"value": n * world * steps_env / (float(env_ms[0]) / 1e3), "unit": "env-steps/s",
                    "ms_per_step": float(env_ms[0]) / steps_env, "steps": steps_env, "obs_dim": od,
                    "api": "brax_env_step: physics + reward/done/auto-reset/observation epilogue, one launch"}

    # NEXT-4: reverse mode of the same step (brax_step_vjp: g_in = Jᵀ·g_out and g_action,
    # one launch) on one batch of the workload; device-timed like the step
    vjp_line = None
    if not args.no_vjp:
        gen = torch.Generator(device="cpu").manual_seed(7)
        g_out = {k: torch.randn(v.shape, generator=gen).to(dev) for k, v in sets[0].items()}
        a0 = acts[0] if A else None
        with torch.cuda.stream(stream):
            for _ in range(2):
                system.step_vjp(sets[0], a0, g_out, stream=stream)
            stream.synchronize()
            Kv = 20
            v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            v0.record(stream)
            for _ in range(Kv):
                system.step_vjp(sets[0], a0, g_out, stream=stream)
            v1.record(stream)
            v1.synchronize()
        v_ms = torch.tensor([v0.elapsed_time(v1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(v_ms, op=dist.ReduceOp.MAX)
        vjp_line = {"value": n * world * Kv / (float(v_ms[0]) / 1e3), "unit": "env-steps/s",
                    "ms_per_step": float(v_ms[0]) / Kv, "steps": Kv,
                    "over_step": (float(v_ms[0]) / Kv) / (ms_max / K),
                    "api": "brax_step_vjp: Jᵀ·g of one step (QP and action cotangents), one launch"}

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return

    # roofline of the step kernel (the only kernel in the timed region)
    counts = load_counts(args.scene)
    peaks, peak_src = load_peaks()
    per_launch_s = (ms / 1e3) / K  # this rank's average launch duration (events on the launch stream)
    flops_launch = counts["flops_per_env_step"] * n
    bytes_launch = counts["bytes_per_env_step"] * n
    clocks = clk.report()
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tflops = 148 * 128 * 2 * f_max * 1e6 / 1e12
    achieved_tflops = flops_launch / per_launch_s / 1e12
    intensity = counts["flops_per_env_step"] / counts["bytes_per_env_step"]
    balance = peak_tflops * 1e12 / (float(peaks["hbm_gbs"]) * 1e9)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        tr = tj.get(args.scene, {})
        if tr.get("envs") == n and tr.get("bytes_per_launch"):
            traffic = tr["bytes_per_launch"]
    if intensity >= balance:
        roof = {"bound": "alu", "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": achieved_tflops / peak_tflops, "traffic": traffic,
                "peak_source": f"148 SM x 128 FP32 lanes x 2 x {f_max:.0f} MHz (sm_max_mhz, {peak_src})",
                "peak_at_run_clock": (148 * 128 * 2 * clocks["sm_mhz"] * 1e6 / 1e12) if clocks["sm_mhz"] else None,
                "algorithmic_flops_per_launch": flops_launch, "launch_us": per_launch_s * 1e6,
                "hbm_frac": bytes_launch / per_launch_s / (float(peaks["hbm_gbs"]) * 1e9)}
    else:
        ach = bytes_launch / per_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                "frac": ach / float(peaks["hbm_gbs"]), "traffic": traffic,
                "peak_source": f"hbm_gbs ({peak_src})", "algorithmic_bytes_per_launch": bytes_launch,
                "launch_us": per_launch_s * 1e6}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, cores, steps, el = oracle_rate(args.scene, min(n, 2048), args.cpu_seconds)
        cpu = {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
               "sample": f"{min(n, 2048)} {args.scene} envs x {steps} steps, fp64 oracle, {cores} host threads, "
                         f"{el:.1f} s"}

    line = {
        "metric": metric_for(args.scene, n), "value": value, "unit": "env-steps/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.scene}, {n} envs/GPU, random actions U(-1,1), "
                               f"{system.substeps} substeps/step",
                   "envs_per_gpu": n, "global_envs": n * world, "parallelism": f"env-shard x{world}",
                   "l2": f"inputs larger than L2: {R} rotating batches x {2 * qp_bytes / 1e6:.1f} MB "
                         f"(> 126 MB L2)",
                   "launch": "CUDA graph of brax_step launches" if graph is not None else "eager launches",
                   "kernel_config": system.launch_config(n)},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K, "clocks": clocks,
        "env_epilogue": env_line, "vjp": vjp_line,
        "blowups": total_blowups, "substeps_per_s": value * system.substeps,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
