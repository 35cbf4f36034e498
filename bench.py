#!/usr/bin/env python
"""Benchmark: batched contact manifolds/sec (BASELINE.json metric).

One step = generate_manifold over the whole env batch of config B (box-box,
65,536 envs per GPU, 304 contacts/env) through the C ABI with poses resident
in HBM ("value"), and the same through the host-buffer C-ABI call with the
H2D pose copy and the D2H per-env mean contact distance inside the timed
region ("e2e"). Multi-GPU: one process per GPU (torchrun), contiguous env
shards, no collective on the data path (weak scaling: 65,536 envs per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic work per manifold (counted on the reference
# formulation with an op-counting scalar: 733,352 arith + 29,811 transcendental).
W_FLOP_PER_ENV = 763_163.0
BYTES_PER_ENV = 48.0 + 304 * 32.0  # FP32 poses-equivalent in + fixed-layout contacts out


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-env", type=int, default=65536, help="envs per GPU (weak scaling)")
    ap.add_argument("--cpu-sample", type=int, default=16384, help="envs in the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="box-box", choices=["box-box", "mixed", "drop", "drop-fwd", "demo"],
                    help="box-box = config B (headline); mixed = config C (4 x 65,536 envs of "
                         "primitive families vs a convex mesh); drop = config D (all 10 body pairs "
                         "of a 5-body scene, 32,768 envs, forward + 12-tangent pose JVP); drop-fwd = "
                         "config D forward only; demo = batched DemoSim steps of a 3-box scene")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def wait_first(self, busy, timeout=3.0):
        """Keep the GPU loaded (busy()) until nvidia-smi has produced its first
        sample, so the samples that follow fall inside the timed region."""
        import torch

        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            busy()
            torch.cuda.synchronize()

    def mark(self):
        """Samples before this point are dropped when later ones exist."""
        self.n_pre = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        lines = self.lines[getattr(self, "n_pre", 0):] or self.lines
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def cpu_reference_run(sample: int, reps: int = 1):
    """The reference's own bench_manifold (oracle/_ref, unmodified reference
    sources) on this host's cores; falls back to the C oracle port."""
    from paper_2602_20304_b200 import workloads as W

    ws = W.box_box(sample)
    cores = os.cpu_count() or 1
    try:
        from oracle import Ref
        if not Ref.available():
            raise FileNotFoundError("oracle/_ref not built")
        from paper_2602_20304_b200.scene import SmoothingConfig
        meshes = [Ref.Mesh.box(b.mesh.box_half) for b in ws.bodies]
        rs = [Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk) for m, b in zip(meshes, ws.bodies)]
        med, _ = Ref.bench_manifold(rs[0], rs[1], ws.bodies[0].pose, ws.bodies[1].pose, sample, "ours",
                                    SmoothingConfig(), seed=0, reps=reps, workers=cores)
        return dict(value=sample / med, unit="manifolds/s", cores=cores, kind="reference",
                    sample=f"bench_manifold (src/batch.cpp:184-228) box-box, {sample} envs, {reps} rep(s), "
                           f"{cores} worker threads, -O3 build of the unmodified reference")
    except Exception as e:  # noqa: BLE001
        from oracle import Oracle
        from paper_2602_20304_b200 import api
        meshes = [api.surface_from_spec(b).mesh for b in ws.bodies]
        s = [Oracle.Surface(m.vertices, m.edges, b.sdf, b.vertex_topk, b.edge_topk)
             for m, b in zip(meshes, ws.bodies)]
        p1, p2 = ws.poses(sample)
        t = time.perf_counter()
        Oracle.manifold_batch(s[0], s[1], p1, p2, None, threads=cores, want_meta=False)
        dt = time.perf_counter() - t
        return dict(value=sample / dt, unit="manifolds/s", cores=cores, kind="port",
                    sample=f"C oracle port, box-box {sample} envs, {cores} threads ({e})")


def run_reference_arm(args, rank):
    if rank != 0:
        return
    # the reference's own bench_manifold protocol: time_run(reps, warmups = min(3, reps))
    reps = max(1, min(args.steps, 5))
    cb = cpu_reference_run(args.cpu_sample, reps=reps)
    line = {
        "impl": "reference", "metric": "contact manifolds/sec (box-box, 65,536 envs)",
        "value": cb["value"], "unit": "manifolds/s", "n_gpus": args.gpus, "steps": reps,
        "warmup": min(3, reps), "ms_per_step": 1e3 * args.cpu_sample / cb["value"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "box-box (config B), sampled on the host CPU", "n_env": args.cpu_sample,
                   "contacts_per_env": 304},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "manifolds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_secondary(args, dev, rank, world):
    """Configs C and D: device-resident throughput of the same path on the
    mixed-primitive buckets / the all-pairs multi-body scene."""
    import torch
    import torch.distributed as dist

    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    cfg = SmoothingConfig()
    if args.workload == "mixed":
        n = 65536 if args.n_env == 65536 else args.n_env
        calls = []
        for kind in W.MIXED_KINDS:
            ws = W.mixed_bucket(kind, n)
            s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
            p1, p2 = ws.poses(n)
            calls.append((s1, s2, torch.as_tensor(p1, device=dev), torch.as_tensor(p2, device=dev), {}))
        units = n * len(calls)

        def step():
            for s1, s2, p1, p2, out in calls:
                api.generate_manifold_batch(s1, s2, p1, p2, cfg, out=out)
        metric, unit, cfgd = "contact manifolds/sec (mixed primitives vs convex mesh, 4 x %d envs)" % n, \
            "manifolds/s", {"workload": "mixed (config C): rounded box / cylinder / ellipsoid / capsule vs "
                            "convex mesh plate, soft top-K 16/16 vertices 8/8 edges, 160 contacts/env",
                            "n_env_total": units}
    elif args.workload == "demo":
        n = 32768 if args.n_env == 65536 else args.n_env
        sc = W.demo_scene(n)
        bodies = [api.surface_from_spec(b) for b in sc.bodies]
        demo = api.DemoBatch(bodies, np.ones(len(bodies)), is_static=sc.is_static(), cfg=cfg, poses=sc.poses(n),
                             n_env=n, device=dev)
        units = n

        def step():
            demo.step(1e-3)
        metric, unit, cfgd = "env steps/sec (DemoSim::step: all-pairs manifolds + penalty forces + SE(3) Euler, " \
            "%d envs)" % n, "env-steps/s", {
                "workload": "demo: 3 SQ boxes released over a static box_planes ground, 6 pairs x 48 contacts, "
                            "dt 1 ms", "n_env": n, "pairs_per_env": 6}
    else:
        n = 32768 if args.n_env == 65536 else args.n_env
        sc = W.drop_scene(n)
        bodies = [api.surface_from_spec(b) for b in sc.bodies]
        P = torch.as_tensor(sc.poses(n), device=dev)
        outs = None
        pairs = api.scene_pairs(len(bodies), sc.is_static())
        units = n * len(pairs)

        jvp = args.workload == "drop"
        fn = api.generate_manifold_scene_jvp_batch if jvp else api.generate_manifold_scene_batch

        def step():
            nonlocal outs
            outs = fn(bodies, P, cfg, is_static=sc.is_static(), outs=outs)
        what = "forward + 12-tangent pose JVP" if jvp else "forward only"
        metric, unit, cfgd = "pair manifolds/sec, %s (5-body drop scene, all %d pairs, %d envs)" % (
            what, len(pairs), n), "manifolds/s", {
                "workload": "drop (config D): 4 stacked SQ boxes over a static box_planes ground, edge_topk 4, "
                            "48 contacts/pair, %s" % what, "n_env": n, "pairs_per_env": len(pairs)}
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s)
    for _ in range(args.steps):
        step()
    t1.record(s)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if rank == 0:
        print(json.dumps({"metric": metric, "value": units / (ms * 1e-3), "unit": unit, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f64 (FP32 outputs)", "data": "synthetic", "config": cfgd}), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2602_20304_b200 import abi, api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig
    from paper_2602_20304_b200.sharding import shard_range

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.workload != "box-box":
        run_secondary(args, dev, rank, world)
        return

    n_local = args.n_env
    n_total = n_local * world
    ws = W.box_box(n_total)
    lo, hi = shard_range(n_total, rank, world)
    p1_all, p2_all = ws.poses(n_total)  # global env order, then sliced (bitwise shard-independent)
    p1 = p1_all
    p2 = np.ascontiguousarray(p2_all[lo:hi])
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    cfg = SmoothingConfig()
    P1 = torch.as_tensor(p1, device=dev)
    P2 = torch.as_tensor(p2, device=dev)
    L = api.layout(s1, s2, cfg)
    out = {}
    stream = torch.cuda.current_stream()

    def step():
        api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=out)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident value ----------------------------------------------------
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.wait_first(step)
    clocks.mark()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for a, b in ev:
        a.record(stream)
        step()
        b.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    total_ms = max_over_ranks(t0.elapsed_time(t1))
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    ms_per_step = total_ms / args.steps
    value = n_total / (ms_per_step * 1e-3)

    # ---- end-to-end through the host-buffer C-ABI call --------------------------
    h1 = torch.as_tensor(p1).pin_memory().numpy()
    h2 = torch.as_tensor(p2).pin_memory().numpy()
    mean_h = torch.empty(hi - lo, dtype=torch.float32).pin_memory().numpy()

    def e2e_step():
        api.generate_manifold_batch_host(s1, s2, h1, h2, cfg, mean_out=mean_h, stream=stream)

    for _ in range(max(3, args.warmup)):
        e2e_step()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    e2e_value = n_total / (e2e_ms * 1e-3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the manifold kernel ----------------------------
    # Primary, as SURVEY §8(d) defines it: the reference formulation's algorithmic
    # flops per env (763,163) x envs / kernel time, against the CUDA-core FP32
    # peak (no dense contraction: tensor cores unused). Secondary: the FP64 pipe
    # the kernel actually runs on, with its ncu-executed FP64 flops per env.
    lib = abi.load()
    import ctypes as C
    f64 = C.c_double()
    f32 = C.c_double()
    lib.cmgb_probe_fma_tflops.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.c_void_p]
    lib.cmgb_probe_fma_tflops(1, 4096, C.byref(f64), stream.cuda_stream)
    lib.cmgb_probe_fma_tflops(0, 8192, C.byref(f32), stream.cuda_stream)
    achieved = W_FLOP_PER_ENV * n_local / (kernel_ms * 1e-3) / 1e12
    peaks = measured_peaks()

    def prof_json(name):
        path = os.path.join(ROOT, "profiles", name)
        try:
            return json.load(open(path))
        except (OSError, ValueError):
            return {}

    tr = prof_json("manifold_dram_bytes.json").get("dram_bytes_per_launch_per_env")
    traffic = tr * n_local if tr else None
    ops = prof_json("manifold_fp64_ops.json")
    x64 = ops.get("fp64_flop_per_env")
    f64_achieved = x64 * n_local / (kernel_ms * 1e-3) / 1e12 if x64 else None
    hbm_gbs = BYTES_PER_ENV * n_local / (kernel_ms * 1e-3) / 1e9
    roof = {
        "bound": "fp32", "achieved": achieved, "peak": f32.value, "unit": "TFLOP/s",
        "frac": achieved / f32.value if f32.value else None, "traffic": traffic,
        "peak_source": "measured live on this GPU: FFMA-chain microbenchmark (cmgb_probe_fma_tflops); "
                       "MEASURED_PEAKS.json has no FP32/FP64 CUDA-core figure",
        "work_per_env_flop": W_FLOP_PER_ENV,
        "work_note": "algorithmic flops of the reference formulation (SURVEY §8(d), CUDA-core bound, tensor "
                     "cores unused); traffic = ncu dram read+write bytes per launch (profiles/)",
        "fp64_pipe": {"executed_flop_per_env": x64, "achieved": f64_achieved, "peak": f64.value,
                      "unit": "TFLOP/s", "frac": f64_achieved / f64.value if (f64_achieved and f64.value) else None,
                      "ncu_pipe_active_pct": ops.get("ncu_fp64_pipe_active_pct"),
                      "note": "the kernel computes in FP64 (DESIGN.md §4); executed DFMA x2 + DMUL + DADD per "
                              "env from ncu (profiles/manifold_fp64_ops.json); peak = live DFMA microbenchmark"},
        "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks.get("hbm_gbs"),
                "frac": hbm_gbs / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None},
        "kernel_ms": kernel_ms,
    }
    cb = None if args.no_cpu_baseline else cpu_reference_run(args.cpu_sample, reps=3)
    line = {
        "metric": "contact manifolds/sec (box-box, 65,536 envs)",
        "value": value, "unit": "manifolds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (FP32 outputs)", "data": "synthetic",
        "config": {"workload": "box-box (config B): quad cube half 0.5 + SQ eps 0.1, M=12, 304 contacts/env",
                   "n_env_per_gpu": n_local, "n_env_total": n_total, "contacts_per_env": L["n_contacts"],
                   "variant": "ours (default SmoothingConfig)", "parallelism": f"env-shard x{world}",
                   "l2": "per-step working set 6.3 MB poses in + 637 MB contacts out > 126 MB L2"},
        "e2e": {"value": e2e_value, "unit": "manifolds/s",
                "h2d_bytes_per_step": int(h1.nbytes + h2.nbytes) * world,
                "d2h_bytes_per_step": int(mean_h.nbytes) * world,
                "path": "cmgb_manifold_batch_host (pinned host poses -> H2D -> kernel -> D2H mean distance)"},
        "gpu_launches": 3 * args.steps,  # per step: frames_kernel (both bodies) + vs_kernel + manifold_kernel
        "roofline": roof,
        "cpu_baseline": cb,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
