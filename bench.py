#!/usr/bin/env python
"""Benchmark: batched contact manifolds/sec (BASELINE.json metric).

One step = generate_manifold over the whole env batch through the C ABI
("value": poses resident in HBM), and the same through the host-buffer call
with the H2D pose copy and a D2H of the step's result inside the timed region
("e2e"). Workloads (one JSON line each):

  box-box   config B (default): quad cube + SQ eps 0.1 per body, 304 contacts/env,
            65,536 envs on 1 GPU; under torchrun (N > 1) config E: 1,048,576
            envs in total, contiguous shards (strong scaling; --n-total / --n-env
            override). --eps picks another superquadric boxiness.
  mixed     config C: 4 buckets x 65,536 envs (rounded box / cylinder /
            ellipsoid / capsule vs a convex mesh), soft top-K active.
  drop      config D: 5-body drop scene, all 10 pairs, 32,768 envs, forward +
            12-tangent pose Jacobians;  drop-fwd: the same, forward only.
  ee | vf   the witness batches of run_ee_batch / run_vf_batch (K6), 4 M pairs.
  demo      batched DemoSim::step (3-box scene).

Every line carries roofline (algorithmic work per unit counted by the
reference itself: profiles/work_per_unit.json, tools/count_work.py),
cpu_baseline (the compiled reference on this host's cores, N = 1, rank 0) and
e2e. Timing mirrors time_run (src/batch.cpp:100-120): per-step device events,
median and population std beside the contract's mean.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload box-box|mixed|drop|drop-fwd|ee|vf|demo]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = ["box-box", "mixed", "drop", "drop-fwd", "ee", "vf", "demo"]
CONFIG_E_ENVS = 1_048_576


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="box-box", choices=WORKLOADS)
    ap.add_argument("--n-env", type=int, default=None,
                    help="envs per GPU (weak scaling); default: config size")
    ap.add_argument("--n-total", type=int, default=None,
                    help="envs over all GPUs (strong scaling); default 1,048,576 (config E) under torchrun")
    ap.add_argument("--eps", type=float, default=None, help="box-box: superquadric eps1 = eps2 (default 0.1)")
    ap.add_argument("--variant", default="ours", help="ours | ours_ns | ours_ne | ours_ne_s (config_for_variant)")
    ap.add_argument("--compact-thr", type=float, default=0.01,
                    help="box-box: activity threshold of the compaction extra (added-cost measurement)")
    ap.add_argument("--cpu-sample", type=int, default=None, help="units in the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the full-manifold e2e and compaction legs")
    return ap.parse_args()


# ----------------------------------------------------------------------------------------
# measurement plumbing
# ----------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.n_pre = 0

    def start(self, busy):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None
            return
        # keep the GPU loaded until the first sample exists, so the rest fall inside the timed region
        import torch
        t0 = time.time()
        while not self.lines and time.time() - t0 < 3.0:
            busy()
            torch.cuda.synchronize()
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
        lines = self.lines[self.n_pre:] or self.lines
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


class Ctx:
    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.args = args
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local_rank)
        self.dev = torch.device("cuda", self.local_rank)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
        self.stream = torch.cuda.current_stream()
        from paper_2602_20304_b200 import abi
        self.lib = abi.load()
        self.lib.cmgb_kernel_launches.restype = C.c_uint64
        self.lib.cmgb_kernel_launches.argtypes = []
        self.lib.cmgb_probe_fma_tflops.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.c_void_p]

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def launches(self):
        return int(self.lib.cmgb_kernel_launches())


def timed(ctx, step, steps, warmup, clocks=False):
    """W untimed warm-ups, then exactly K steps bracketed by barrier +
    synchronize, each step between CUDA events on the launching stream.
    Returns dict(total_ms = max over ranks, per-step median / std / mean,
    launches per step, clocks)."""
    import torch

    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize()
    cs = ClockSampler(ctx.local_rank) if clocks else None
    if cs:
        cs.start(step)
    ctx.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches()
    t0.record(ctx.stream)
    for a, b in ev:
        a.record(ctx.stream)
        step()
        b.record(ctx.stream)
    t1.record(ctx.stream)
    l1 = ctx.launches()
    torch.cuda.synchronize()
    ctx.barrier()
    clk = cs.stop() if cs else None
    per = np.array([a.elapsed_time(b) for a, b in ev])
    total = ctx.max_over_ranks(t0.elapsed_time(t1))
    return {"total_ms": total, "ms_per_step": total / steps, "median_ms": float(np.median(per)),
            "std_ms": float(per.std()), "mean_ms": float(per.mean()), "launches_per_step": (l1 - l0) / steps,
            "clocks": clk}


def work_per_unit(name):
    try:
        with open(os.path.join(ROOT, "profiles", "work_per_unit.json")) as f:
            return json.load(f)["units"][name]["W"]
    except (OSError, ValueError, KeyError):
        return None


def prof_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def measured_peaks():
    return prof_json("../MEASURED_PEAKS.json")


def fp_peaks(ctx):
    import torch
    f32, f64 = C.c_double(), C.c_double()
    ctx.lib.cmgb_probe_fma_tflops(0, 8192, C.byref(f32), ctx.stream.cuda_stream)
    ctx.lib.cmgb_probe_fma_tflops(1, 4096, C.byref(f64), ctx.stream.cuda_stream)
    props = torch.cuda.get_device_properties(ctx.dev)
    mhz = measured_peaks().get("sm_max_mhz") or 1965.0
    nominal = props.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12
    return f32.value, f64.value, nominal


def compute_roofline(ctx, W, units_local, kernel_ms, extra=None):
    """FP32 CUDA-core roofline (no dense contraction, tensor
    cores unused): W algorithmic flop per unit (the reference formulation,
    counted by the reference) x units / device time of the step's kernels."""
    f32, f64, nominal = fp_peaks(ctx)
    achieved = W * units_local / (kernel_ms * 1e-3) / 1e12 if W else None
    roof = {"bound": "fp32", "achieved": achieved, "peak": f32, "unit": "TFLOP/s",
            "frac": achieved / f32 if (achieved and f32) else None,
            "frac_of_nominal": achieved / nominal if achieved else None, "nominal_peak": nominal,
            "peak_source": "measured live on this GPU: FFMA-chain microbenchmark (cmgb_probe_fma_tflops); "
                           "MEASURED_PEAKS.json has no FP32 CUDA-core figure. nominal_peak = SMs x 128 x 2 x "
                           "max SM clock",
            "work_per_unit_flop": W, "work_source": "profiles/work_per_unit.json (tools/count_work.py: the "
                                                    "reference's generate_manifold<T> with a counting scalar)",
            "kernel_ms": kernel_ms, "fp64_dfma_peak": f64}
    if extra:
        roof.update(extra)
    return roof


def hbm_roofline(bytes_per_unit, units_local, kernel_ms, traffic=None):
    peak = measured_peaks().get("hbm_gbs") or 6546.2
    achieved = bytes_per_unit * units_local / (kernel_ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "bytes_per_unit": bytes_per_unit, "kernel_ms": kernel_ms,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"}


def line(ctx, metric, unit, t, units_total, config, dtype, **extra):
    args = ctx.args
    out = {"metric": metric, "value": units_total / (t["ms_per_step"] * 1e-3), "unit": unit,
           "n_gpus": ctx.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t["ms_per_step"],
           "higher_is_better": True, "scaling": extra.pop("scaling", "weak"), "vs_baseline": None,
           "dtype": dtype, "data": "synthetic", "config": config,
           "timing": {"median_ms": t["median_ms"], "std_ms": t["std_ms"], "mean_ms": t["mean_ms"],
                      "protocol": "per-step CUDA events (time_run: median + population std); value = "
                                  "units / (max-over-ranks total / K)"},
           "gpu_launches": int(round(t["launches_per_step"] * args.steps)),
           "gpu_launches_per_step": t["launches_per_step"],
           "clocks": t["clocks"]}
    out.update(extra)
    return out


# ----------------------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference compiled from source)
# ----------------------------------------------------------------------------------------
def ref_surface(b):
    from oracle import Ref
    m = Ref.Mesh.box(b.mesh.box_half, b.mesh.subdivisions, b.mesh.quad_edges) if b.mesh.box_half is not None \
        else Ref.Mesh.parse_obj(b.mesh.obj_text)
    return Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk)


def cpu_reference(workload, args, sample, reps):
    """The reference's own implementation of the workload on all host cores:
    (units/s, median_s, std_s, description)."""
    from oracle import Ref
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    if not Ref.available():
        raise FileNotFoundError("oracle/_ref/libcmgref.so not built")
    cores = os.cpu_count() or 1
    cfg = SmoothingConfig()
    if workload == "box-box":
        ws = W.box_box(sample) if args.eps is None else W.box_box_eps(args.eps, sample)
        s = [ref_surface(b) for b in ws.bodies]
        med, sd = Ref.bench_manifold(s[0], s[1], ws.bodies[0].pose, ws.bodies[1].pose, sample, args.variant, cfg,
                                     seed=0, reps=reps, workers=cores)
        return sample / med, med, sd, cores, (f"bench_manifold (src/batch.cpp:184-228), {ws.name}, {sample} envs, "
                                              f"variant {args.variant}, time_run median of {reps} rep(s) after "
                                              f"{min(3, reps)} warm-up(s), {cores} worker threads")
    if workload == "mixed":
        tot = 0.0
        sds = []
        for kind in W.MIXED_KINDS:
            ws = W.mixed_bucket(kind, sample)
            s = [ref_surface(b) for b in ws.bodies]
            med, sd = Ref.bench_manifold(s[0], s[1], ws.bodies[0].pose, ws.bodies[1].pose, sample, args.variant,
                                         cfg, seed=0, reps=reps, workers=cores)
            tot += med
            sds.append(sd)
        units = sample * len(W.MIXED_KINDS)
        return units / tot, tot, float(np.sqrt(np.sum(np.square(sds)))), cores, (
            f"bench_manifold per config-C bucket (4 x {sample} envs), summed medians of {reps} rep(s), "
            f"{cores} worker threads")
    if workload in ("drop", "drop-fwd"):
        sc = W.drop_scene(sample)
        bodies = [ref_surface(b) for b in sc.bodies]
        pairs = np.array([(i, j) for i in range(len(bodies)) for j in range(i + 1, len(bodies))
                          if not (sc.bodies[i].is_static and sc.bodies[j].is_static)], np.int32)
        jvp = workload == "drop"
        med, sd, _ = Ref.scene_bench(bodies, pairs, sc.poses(sample), cfg, jvp=jvp, reps=reps, warmups=1,
                                     workers=cores)
        units = sample * len(pairs)
        what = "generate_manifold<Dual12> (seed_pose_tangents; main.cpp:202-205)" if jvp else \
            "generate_manifold<double>"
        return units / med, med, sd, cores, (f"every pair of the drop scene ({len(pairs)} pairs x {sample} envs) "
                                             f"through the reference's {what}, std::thread chunks, time_run "
                                             f"median of {reps} rep(s), {cores} threads")
    if workload in ("ee", "vf"):
        med, sd = Ref.bench_witness(workload, sample, args.variant, seed=0, reps=reps, workers=cores)
        return sample / med, med, sd, cores, (f"bench_witness (src/batch.cpp:152-182) kind {workload}, {sample} "
                                              f"pairs, variant {args.variant}, make_random_{workload}_pairs seed 0, "
                                              f"time_run median of {reps} rep(s), {cores} worker threads")
    raise ValueError(f"no CPU reference for workload {workload}")


def cpu_baseline(ctx, workload, unit, sample):
    if ctx.args.no_cpu_baseline or ctx.rank != 0 or ctx.world != 1:
        return None
    try:
        v, med, sd, cores, desc = cpu_reference(workload, ctx.args, sample, reps=2)
        return {"value": v, "unit": unit, "cores": cores, "kind": "reference", "sample": desc,
                "median_s": med, "std_s": sd}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": unit, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {e}"}


DEFAULT_SAMPLE = {"box-box": 65536, "mixed": 16384, "drop": 1024, "drop-fwd": 8192, "ee": 4_194_304,
                  "vf": 4_194_304}
UNITS = {"box-box": "manifolds/s", "mixed": "manifolds/s", "drop": "manifolds/s", "drop-fwd": "manifolds/s",
         "ee": "pairs/s", "vf": "pairs/s", "demo": "env-steps/s"}


def run_reference_arm(args):
    """`--impl reference`: the reference's own CPU implementation of the
    workload (oracle/_ref, compiled from /root/reference's unmodified sources)
    on all host cores, same metric / unit / config; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = args.workload
    if wl == "demo":
        print(json.dumps({"impl": "reference", "unavailable": "no CPU reference timing harness for the demo "
                                                              "integrator workload"}), flush=True)
        return
    sample = args.cpu_sample or DEFAULT_SAMPLE[wl]
    reps = max(1, min(args.steps, 5))
    v, med, sd, cores, desc = cpu_reference(wl, args, sample, reps)
    unit = UNITS[wl]
    out = {"impl": "reference", "metric": METRICS[wl](args, args.gpus), "value": v, "unit": unit,
           "n_gpus": args.gpus, "steps": reps, "warmup": min(3, reps), "ms_per_step": med * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{wl} on the host CPU (the reference's own code path)", "sample_units": sample,
                      "eps": args.eps, "variant": args.variant},
           "timing": {"median_ms": med * 1e3, "std_ms": sd * 1e3,
                      "protocol": "the reference's time_run (src/batch.cpp:100-120)"},
           "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "reference", "sample": desc},
           "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


METRICS = {
    "box-box": lambda a, n: "contact manifolds/sec (box-box, 65,536 envs)" if n == 1 and not a.eps else
    f"contact manifolds/sec (box-box{'' if not a.eps else f' eps {a.eps:g}'}, config {'E' if n > 1 else 'B'})",
    "mixed": lambda a, n: "contact manifolds/sec (mixed primitives vs convex mesh, 262,144 envs)",
    "drop": lambda a, n: "pair manifolds/sec, forward + 12-tangent pose JVP (drop scene, 10 pairs, 32,768 envs)",
    "drop-fwd": lambda a, n: "pair manifolds/sec, forward only (drop scene, 10 pairs, 32,768 envs)",
    "ee": lambda a, n: "E-E witness pairs/sec (run_ee_batch, 4,194,304 pairs)",
    "vf": lambda a, n: "V-F witness pairs/sec (run_vf_batch, 4,194,304 pairs)",
    "demo": lambda a, n: "env steps/sec (DemoSim::step, 3-box scene, 32,768 envs)",
}


# ----------------------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------------------
def bench_box_box(ctx):
    import torch

    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig
    from paper_2602_20304_b200.sharding import shard_range

    a = ctx.args
    if a.n_env is not None:
        n_total, scaling = a.n_env * ctx.world, "weak"
    elif a.n_total is not None:
        n_total, scaling = a.n_total, "strong"
    else:
        n_total, scaling = (65536, "weak") if ctx.world == 1 else (CONFIG_E_ENVS, "strong")
    ws = W.box_box(n_total) if a.eps is None else W.box_box_eps(a.eps, n_total)
    lo, hi = shard_range(n_total, ctx.rank, ctx.world)
    n_local = hi - lo
    p1, p2_all = ws.poses(n_total)  # global env order, then sliced: shards equal the 1-GPU result bitwise
    p2 = np.ascontiguousarray(p2_all[lo:hi])
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    cfg = SmoothingConfig().for_variant(a.variant)
    P1 = torch.as_tensor(p1, device=ctx.dev)
    P2 = torch.as_tensor(p2, device=ctx.dev)
    L = api.layout(s1, s2, cfg)
    out = {}

    def step():
        api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=out)

    t = timed(ctx, step, a.steps, a.warmup, clocks=True)

    # e2e: host-buffer C-ABI call, pinned host poses H2D + per-env mean distance D2H
    # (bench_manifold keeps exactly that per env: sums[i], batch.cpp:212)
    h1 = torch.as_tensor(p1).pin_memory().numpy()
    h2 = torch.as_tensor(p2).pin_memory().numpy()
    mean_h = torch.empty(n_local, dtype=torch.float32).pin_memory().numpy()

    def e2e_step():
        api.generate_manifold_batch_host(s1, s2, h1, h2, cfg, mean_out=mean_h, stream=ctx.stream)

    te = timed(ctx, e2e_step, a.steps, a.warmup)
    extras = {}
    if not a.no_extras:
        # e2e with the WHOLE fixed-layout manifold returned to the host (what
        # generate_manifold returns by value; 9,728 B/env box-box): D2H-bound
        contacts_h = torch.empty((n_local, L["n_contacts"], 8), dtype=torch.float32).pin_memory().numpy()

        def e2e_full():
            api.generate_manifold_batch_host(s1, s2, h1, h2, cfg, mean_out=mean_h, contacts_out=contacts_h,
                                             stream=ctx.stream)

        kf = max(3, min(a.steps, 20))
        tf = timed(ctx, e2e_full, kf, 2)
        extras["e2e_full_manifold"] = {
            "value": n_total / (tf["ms_per_step"] * 1e-3), "unit": "manifolds/s", "steps": kf,
            "h2d_bytes_per_step": int(h1.nbytes + h2.nbytes) * ctx.world,
            "d2h_bytes_per_step": int(mean_h.nbytes + contacts_h.nbytes) * ctx.world,
            "path": "cmgb_manifold_batch_host with contacts_host: the whole fixed layout back to pinned host "
                    "memory, pipelined in env chunks (D2H overlaps the next chunk's kernels)",
            "d2h_gbs": contacts_h.nbytes / (tf["median_ms"] * 1e-3) / 1e9}
        del contacts_h
        # compaction extra: its added cost on top of the step, (a) fused: the
        # kernels emit per-env activity masks / counts beside the fixed layout
        # and a scan + gather kernel reads only the kept contacts; (b) the
        # standalone one-pass compaction of an existing fixed layout
        comp = {}
        outm = {}

        def step_fused():
            api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=outm, active_threshold=a.compact_thr)
            api.compact_contacts(outm["contacts"], mask=outm["active_mask"], count=outm["active_count"], out=comp)

        def step_standalone():
            step()
            api.compact_contacts(out["contacts"], a.compact_thr, out=comp)

        tcf = timed(ctx, step_fused, a.steps, a.warmup)
        total_kept = int(comp["total"].item())
        tcs = timed(ctx, step_standalone, a.steps, a.warmup)
        n_c = n_local * L["n_contacts"]
        added_f = tcf["median_ms"] - t["median_ms"]
        added_s = tcs["median_ms"] - t["median_ms"]
        # e2e of the active contacts only (what a consumer of the manifold keeps):
        # pinned poses H2D, the step with activity masks, the compaction, then the
        # kept rows + per-env offsets D2H (the total is read first to size the copy)
        hP2 = torch.as_tensor(p2).pin_memory()
        P2d = torch.empty_like(P2)
        kept_h = torch.empty((n_c, 8), dtype=torch.float32).pin_memory()
        off_h = torch.empty((n_local + 1,), dtype=torch.int64).pin_memory()
        oute, compe = {}, {}
        d2h = [0]

        def e2e_active():
            P2d.copy_(hP2, non_blocking=True)
            api.generate_manifold_batch(s1, s2, P1, P2d, cfg, out=oute, active_threshold=a.compact_thr)
            api.compact_contacts(oute["contacts"], mask=oute["active_mask"], count=oute["active_count"], out=compe)
            tot = int(compe["total"].item())
            kept_h[:tot].copy_(compe["contacts"][:tot], non_blocking=True)
            off_h.copy_(compe["env_offset"], non_blocking=True)
            ctx.stream.synchronize()
            d2h[0] = tot * 32 + off_h.numel() * 8 + 8

        ta = timed(ctx, e2e_active, max(3, min(a.steps, 20)), 2)
        extras["e2e_active_contacts"] = {
            "value": n_total / (ta["ms_per_step"] * 1e-3), "unit": "manifolds/s",
            "h2d_bytes_per_step": int(hP2.numel() * 8) * ctx.world, "d2h_bytes_per_step": d2h[0] * ctx.world,
            "activity_threshold": a.compact_thr,
            "path": "api.generate_manifold_batch(active_threshold) + api.compact_contacts (masked): pinned poses "
                    "H2D, kept contacts (activity > threshold, fixed-layout order) + per-env offsets D2H"}
        del kept_h
        extras["compaction"] = {
            "activity_threshold": a.compact_thr, "kept": total_kept, "kept_fraction": total_kept / n_c,
            "fused": {"added_ms_per_step": added_f, "added_fraction": added_f / t["median_ms"],
                      "value_with_compaction": n_total / (tcf["ms_per_step"] * 1e-3),
                      "launches_per_step": tcf["launches_per_step"],
                      "path": "manifold kernels emit activity masks + counts (active_threshold); "
                              "cmgb_compact_masked scans the counts and copies only the kept contacts"},
            "standalone": {"added_ms_per_step": added_s, "added_fraction": added_s / t["median_ms"],
                           "hbm_gbs": (n_c * 32 + total_kept * 36) / (added_s * 1e-3) / 1e9 if added_s > 0 else None,
                           "path": "cmgb_compact_contacts: one pass over the fixed layout (ballots, look-back scan)"},
            "note": "median per-step device time with compaction minus the step alone"}

    if ctx.world > 1:
        # the optional end-of-run result gather (NCCL over NVLink), timed apart
        # from the hot path: every rank's per-env mean distances to every rank
        from paper_2602_20304_b200.sharding import gather_shards
        md = out["mean_dist"]
        g = {}

        def gather():
            g["all"] = gather_shards(md, n_total, ctx.rank, ctx.world)

        tg = timed(ctx, gather, max(3, min(a.steps, 20)), 2)
        extras["gather"] = {"what": "all-gather of the per-env mean contact distance (4 B/env)",
                            "bytes": 4 * n_total, "median_ms": tg["median_ms"],
                            "note": "not part of value: the hot path has no collective"}

    W_env = work_per_unit("box-box" if a.eps is None else f"box-box-eps{a.eps:g}") or work_per_unit("box-box")
    tr = prof_json("manifold_dram_bytes.json").get("dram_bytes_per_launch_per_env")
    ops = prof_json("manifold_fp64_ops.json")
    x64 = ops.get("fp64_flop_per_env")
    kernel_ms = t["median_ms"]
    f64_ach = x64 * n_local / (kernel_ms * 1e-3) / 1e12 if x64 else None
    bytes_env = 48.0 + L["n_contacts"] * 32.0
    hbm = bytes_env * n_local / (kernel_ms * 1e-3) / 1e9
    peaks = measured_peaks()
    roof = compute_roofline(ctx, W_env, n_local, kernel_ms, {
        "traffic": tr * n_local if (tr and a.eps is None) else None,
        "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per step (profiles/"
                          "manifold_dram_bytes.json)",
        "fp64_pipe": {"executed_flop_per_env": x64, "achieved": f64_ach,
                      "ncu_pipe_active_pct": ops.get("ncu_fp64_pipe_active_pct"),
                      "note": "the kernel computes in FP64 (DESIGN.md §4): executed DFMA x2 + DMUL + DADD per env "
                              "from ncu (profiles/manifold_fp64_ops.json) against the live DFMA peak"},
        "hbm": {"algorithmic_bytes_per_env": bytes_env, "achieved_gbs": hbm, "peak_gbs": peaks.get("hbm_gbs"),
                "frac": hbm / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None}})
    if roof.get("fp64_pipe") and f64_ach:
        roof["fp64_pipe"]["frac"] = f64_ach / roof["fp64_dfma_peak"]
    cb = cpu_baseline(ctx, "box-box", "manifolds/s", a.cpu_sample or n_local)
    return line(ctx, METRICS["box-box"](a, ctx.world), "manifolds/s", t, n_total,
                {"workload": ws.notes + (" (config B)" if ctx.world == 1 and a.eps is None else
                                         (" (config E)" if a.eps is None else "")),
                 "n_env_total": n_total, "n_env_per_gpu": n_local, "contacts_per_env": L["n_contacts"],
                 "variant": a.variant, "parallelism": f"env-shard x{ctx.world}",
                 "l2": f"per-step working set {(p2.nbytes + bytes_env * n_local) / 1e6:.0f} MB > 126 MB L2"},
                "f64 (FP32 outputs)", scaling=scaling,
                e2e={"value": n_total / (te["ms_per_step"] * 1e-3), "unit": "manifolds/s",
                     "h2d_bytes_per_step": int(h1.nbytes + h2.nbytes) * ctx.world,
                     "d2h_bytes_per_step": int(mean_h.nbytes) * ctx.world,
                     "median_ms": te["median_ms"], "std_ms": te["std_ms"],
                     "path": "cmgb_manifold_batch_host (pinned host poses -> H2D -> kernels -> D2H of the per-env "
                             "mean contact distance, bench_manifold's per-env result)"},
                roofline=roof, cpu_baseline=cb, **extras)


def bench_mixed(ctx):
    import torch

    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    a = ctx.args
    n = a.n_env or 65536
    cfg = SmoothingConfig()
    calls = []
    for kind in W.MIXED_KINDS:
        ws = W.mixed_bucket(kind, n)
        s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
        p1, p2 = ws.poses(n)
        calls.append(dict(s1=s1, s2=s2, P1=torch.as_tensor(p1, device=ctx.dev), P2=torch.as_tensor(p2, device=ctx.dev),
                          h1=torch.as_tensor(p1).pin_memory().numpy(), h2=torch.as_tensor(p2).pin_memory().numpy(),
                          mean=torch.empty(n, dtype=torch.float32).pin_memory().numpy(), out={},
                          C=api.layout(s1, s2, cfg)["n_contacts"]))
    units = n * len(calls) * ctx.world

    def step():
        for c in calls:
            api.generate_manifold_batch(c["s1"], c["s2"], c["P1"], c["P2"], cfg, out=c["out"])

    def e2e_step():
        for c in calls:
            api.generate_manifold_batch_host(c["s1"], c["s2"], c["h1"], c["h2"], cfg, mean_out=c["mean"],
                                             stream=ctx.stream)

    t = timed(ctx, step, a.steps, a.warmup, clocks=True)
    te = timed(ctx, e2e_step, a.steps, a.warmup)
    roof = compute_roofline(ctx, work_per_unit("mixed"), n * len(calls), t["median_ms"], {
        "traffic": None, "per_bucket_W": {k: work_per_unit(f"mixed-{k}") for k in W.MIXED_KINDS}})
    cb = cpu_baseline(ctx, "mixed", "manifolds/s", a.cpu_sample or DEFAULT_SAMPLE["mixed"])
    h2d = sum(c["h1"].nbytes + c["h2"].nbytes for c in calls)
    return line(ctx, METRICS["mixed"](a, ctx.world), "manifolds/s", t, units,
                {"workload": "mixed (config C): rounded box / cylinder / ellipsoid / capsule vs convex mesh plate, "
                             "soft top-K 16/16 vertices 8/8 edges, 160 contacts/env",
                 "n_env_total": units, "buckets": len(calls), "n_env_per_bucket": n,
                 "parallelism": f"env-shard x{ctx.world}"},
                "f64 (FP32 outputs)",
                e2e={"value": units / (te["ms_per_step"] * 1e-3), "unit": "manifolds/s",
                     "h2d_bytes_per_step": h2d * ctx.world, "d2h_bytes_per_step": 4 * n * len(calls) * ctx.world,
                     "path": "cmgb_manifold_batch_host per bucket (pinned poses H2D, per-env mean D2H)"},
                roofline=roof, cpu_baseline=cb)


def bench_drop(ctx, jvp):
    import torch

    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    a = ctx.args
    n = a.n_env or 32768
    cfg = SmoothingConfig()
    sc = W.drop_scene(n)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    poses = sc.poses(n)
    P = torch.as_tensor(poses, device=ctx.dev)
    pairs = api.scene_pairs(len(bodies), sc.is_static())
    units_local = n * len(pairs)
    fn = api.generate_manifold_scene_jvp_batch if jvp else api.generate_manifold_scene_batch
    outs = [dict() for _ in range(len(pairs))]

    def step():
        fn(bodies, P, cfg, is_static=sc.is_static(), outs=outs)

    t = timed(ctx, step, a.steps, a.warmup, clocks=True)
    # e2e through the public Python API: pinned host poses -> H2D, all pairs, D2H of
    # every pair's per-env mean distance (+ its 12 pose tangents with the JVP)
    hP = torch.as_tensor(poses).pin_memory()
    Pd = torch.empty_like(P)
    # contiguous pinned destinations: a strided host destination would make torch
    # stage each copy through a pageable temporary and synchronise
    mean_h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in pairs]
    grad_h = [torch.empty((n, 12), dtype=torch.float32).pin_memory() for _ in pairs] if jvp else []

    mean_all = torch.empty((len(pairs), n), dtype=torch.float32).pin_memory().numpy()
    hPn = hP.numpy()

    def e2e_step():
        if not jvp:  # the host-buffer C-ABI scene call (pipelined upload, means back)
            api.generate_manifold_scene_batch_host(bodies, hPn, cfg, is_static=sc.is_static(), mean_out=mean_all,
                                                   stream=ctx.stream)
            return
        Pd.copy_(hP, non_blocking=True)
        r = fn(bodies, Pd, cfg, is_static=sc.is_static(), outs=outs)
        for q, o in enumerate(r):
            mean_h[q].copy_(o["mean_dist"], non_blocking=True)
            grad_h[q].copy_(o["mean_dist_grad"], non_blocking=True)
        ctx.stream.synchronize()

    te = timed(ctx, e2e_step, a.steps, a.warmup)
    wname = "drop" if jvp else "drop-fwd"
    roof = compute_roofline(ctx, work_per_unit(wname), units_local, t["median_ms"], {
        "traffic": None,
        "work_note": "W of the reference formulation: generate_manifold<Dual<12>> per pair (every operation "
                     "carries 12 tangents) for the JVP workload" if jvp else "generate_manifold<double> per pair"})
    ops = prof_json("jvp_fp64_ops.json") if jvp else {}
    if jvp and ops.get("fp64_flop_per_unit") and roof.get("fp64_dfma_peak"):
        # The reference's Dual<12> count (every scalar carries 12 tangents) is ~10x the work this
        # kernel's Jacobian compression performs, so a fraction against it says nothing about the
        # kernel: the primary roofline is the FP64 pipe with the executed FP64 work (ncu).
        ach = ops["fp64_flop_per_unit"] * units_local / (t["median_ms"] * 1e-3) / 1e12
        ref_view = {k: roof[k] for k in ("achieved", "peak", "frac", "frac_of_nominal", "nominal_peak",
                                         "work_per_unit_flop", "work_source", "work_note", "peak_source")}
        ref_view["bound"] = "fp32"
        roof = {"bound": "fp64", "achieved": ach, "peak": roof["fp64_dfma_peak"], "unit": "TFLOP/s",
                "frac": ach / roof["fp64_dfma_peak"], "traffic": None, "kernel_ms": t["median_ms"],
                "work_per_unit_flop": ops["fp64_flop_per_unit"],
                "work_source": "executed DFMA x2 + DMUL + DADD per pair manifold (ncu metric pass, "
                               "profiles/jvp_fp64_ops.json)",
                "ncu_fp64_pipe_active_pct": ops.get("ncu_fp64_pipe_active_pct_mean"),
                "peak_source": "measured live on this GPU: DFMA-chain microbenchmark (cmgb_probe_fma_tflops)",
                "reference_formulation": ref_view}
    cb = cpu_baseline(ctx, wname, "manifolds/s", a.cpu_sample or DEFAULT_SAMPLE[wname])
    what = "forward + 12-tangent pose JVP" if jvp else "forward only"
    return line(ctx, METRICS[wname](a, ctx.world), "manifolds/s", t, units_local * ctx.world,
                {"workload": f"drop (config D): 4 stacked SQ boxes over a static box_planes ground, edge_topk 4, "
                             f"48 contacts/pair, {what}", "n_env": n * ctx.world, "pairs_per_env": len(pairs),
                 "parallelism": f"env-shard x{ctx.world}"},
                "f64 (FP32 outputs and tangents)",
                e2e={"value": units_local * ctx.world / (te["ms_per_step"] * 1e-3), "unit": "manifolds/s",
                     "h2d_bytes_per_step": int(hP.numel() * 8) * ctx.world,
                     "d2h_bytes_per_step": int(sum(r.numel() * 4 for r in mean_h + grad_h)) * ctx.world,
                     "path": ("api.generate_manifold_scene_jvp_batch: pinned [n_env, 5, 6] poses H2D, every pair's "
                              "per-env mean distance + its 12 pose tangents D2H") if jvp else
                             ("api.generate_manifold_scene_batch_host (cmgb_manifold_scene_batch_host): pinned "
                              "[n_env, 5, 6] host poses in, every pair's per-env mean distance out")},
                roofline=roof, cpu_baseline=cb)


def bench_witness(ctx, kind):
    import torch

    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    a = ctx.args
    n = a.n_env or 4_194_304
    cfg = SmoothingConfig().for_variant(a.variant)
    pairs = W.mt19937_64_uniform(0, 12 * n, 0.0, 1.0).reshape(n, 12)  # make_random_*_pairs(n, seed 0)
    D = torch.as_tensor(pairs, device=ctx.dev)
    fn = api.run_ee_batch if kind == "ee" else api.run_vf_batch
    width = 6 if kind == "ee" else 3

    def step():
        fn(D, cfg)

    t = timed(ctx, step, a.steps, a.warmup, clocks=True)
    # e2e through the reference-facing host-buffer call (run_ee_batch /
    # run_vf_batch: host problem set in, doubles out), pinned buffers
    hp = torch.as_tensor(pairs).pin_memory().numpy()
    oh = torch.empty((n, width), dtype=torch.float64).pin_memory().numpy()
    fn_host = api.run_ee_batch_host if kind == "ee" else api.run_vf_batch_host

    def e2e_step():
        fn_host(hp, cfg, out=oh, stream=ctx.stream)

    te = timed(ctx, e2e_step, max(3, min(a.steps, 20)), 2)
    bytes_pair = 96 + 4 * width  # FP64 pair in (as the reference stores it) + FP32 witness points out
    tr = prof_json(f"witness_{kind}_dram_bytes.json").get("dram_bytes_per_pair")
    roof = hbm_roofline(bytes_pair, n, t["median_ms"], tr * n if tr else None)
    cb = cpu_baseline(ctx, kind, "pairs/s", a.cpu_sample or n)
    return line(ctx, METRICS[kind](a, ctx.world), "pairs/s", t, n * ctx.world,
                {"workload": f"{kind} witness batch (K6): make_random_{kind}_pairs(n, seed 0), variant {a.variant}",
                 "n_pairs": n * ctx.world, "parallelism": f"pair-shard x{ctx.world}"},
                "f64 in (FP32 out)",
                e2e={"value": n * ctx.world / (te["ms_per_step"] * 1e-3), "unit": "pairs/s",
                     "h2d_bytes_per_step": int(hp.nbytes) * ctx.world,
                     "d2h_bytes_per_step": int(oh.nbytes) * ctx.world,
                     "path": f"api.run_{kind}_batch_host (cmgb_{kind}_witness_batch_host, the reference's "
                             f"run_{kind}_batch signature): pinned FP64 pairs in, FP64 witness points out"
                             f"{' (FP64 solver)' if kind == 'ee' else ' (FP32 solver, widened on the device)'}, "
                             "pipelined over 8 pair chunks on two streams (PCIe-bound)"},
                roofline=roof, cpu_baseline=cb)


def bench_demo(ctx):
    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    a = ctx.args
    n = a.n_env or 32768
    sc = W.demo_scene(n)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    demo = api.DemoBatch(bodies, np.ones(len(bodies)), is_static=sc.is_static(), cfg=SmoothingConfig(),
                         poses=sc.poses(n), n_env=n, device=ctx.dev)

    def step():
        demo.step(1e-3)

    t = timed(ctx, step, a.steps, a.warmup, clocks=True)
    return line(ctx, METRICS["demo"](a, ctx.world), "env-steps/s", t, n * ctx.world,
                {"workload": "demo: 3 SQ boxes released over a static box_planes ground, 6 pairs x 48 contacts, "
                             "dt 1 ms", "n_env": n * ctx.world, "pairs_per_env": 6},
                "f64 (FP32 contacts)", roofline=None, cpu_baseline=None, e2e=None)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    ctx = Ctx(args)
    wl = args.workload
    if wl == "box-box":
        out = bench_box_box(ctx)
    elif wl == "mixed":
        out = bench_mixed(ctx)
    elif wl in ("drop", "drop-fwd"):
        out = bench_drop(ctx, wl == "drop")
    elif wl in ("ee", "vf"):
        out = bench_witness(ctx, wl)
    else:
        out = bench_demo(ctx)
    if ctx.rank == 0:
        print(json.dumps(out), flush=True)
    if ctx.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
