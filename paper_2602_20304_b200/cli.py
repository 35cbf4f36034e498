"""Command-line front end with the reference tool's commands, options and
outputs (proj/tools/main.cpp), every computation on the GPU path:

    python -m paper_2602_20304_b200 manifold    --scene S --out F [--json] [smoothing flags]
    python -m paper_2602_20304_b200 sweep-edges --out F [--samples N]
    python -m paper_2602_20304_b200 bench       --kind ee|vf|manifold --out F [--batch ..] [--variants ..]
    python -m paper_2602_20304_b200 gradcheck   --scene S [--tol T] [smoothing flags]
    python -m paper_2602_20304_b200 sim         --scene S --out F [--duration D] [--dt DT] [smoothing flags]

Exit codes and stdout lines follow main.cpp:124-254."""
from __future__ import annotations

import argparse
import math
import sys

import numpy as np

from . import abi, api, scene_io
from . import workloads as W
from .scene import PenaltyParams, SmoothingConfig

_TAUS = ("clip", "min", "comp", "sign", "pen", "nn", "clash", "cont", "topk-verts", "topk-edges", "normal", "union")


def _add_smoothing_flags(p):
    """SmoothingFlags::attach (main.cpp:28-43)."""
    for t in _TAUS:
        p.add_argument(f"--tau-{t}", type=float, default=None, help=f"override tau_{t.replace('-', '_')}")
    p.add_argument("--lambda", dest="lam", type=float, default=-1.0, help="QP regularization weight")
    p.add_argument("--mode", default="", help="contact mode: full | no-ee | one-sided")
    p.add_argument("--sphere-trace-iters", type=int, default=-1, help="witness projection iterations (0 disables)")
    p.add_argument("--no-sphere-trace", action="store_true", help="disable witness projection")
    p.add_argument("--containment", action="store_true", help="enable the containment safeguard factors")
    p.add_argument("--hard-ops", action="store_true", help="use exact (non-smooth) operators")


def _apply_flags(a, cfg: SmoothingConfig) -> SmoothingConfig:
    """SmoothingFlags::apply (main.cpp:45-78)."""
    for t in _TAUS:
        v = getattr(a, f"tau_{t.replace('-', '_')}")
        if v is not None:
            setattr(cfg, f"tau_{t.replace('-', '_')}", v)
    if a.lam > 0.0:
        cfg.lambda_ = a.lam
    if a.mode:
        modes = {"full": abi.MODE_FULL, "no-ee": abi.MODE_NO_EE, "one-sided": abi.MODE_ONE_SIDED}
        if a.mode not in modes:
            raise ValueError("--mode must be full, no-ee or one-sided")
        cfg.mode = modes[a.mode]
    if a.sphere_trace_iters >= 0:
        cfg.sphere_trace_iters = a.sphere_trace_iters
        cfg.sphere_trace = a.sphere_trace_iters > 0
    if a.no_sphere_trace:
        cfg.sphere_trace = False
    if a.containment:
        cfg.containment_safeguard = True
    if a.hard_ops:
        cfg.hard_ops = True
    api.validate_config(cfg)
    return cfg


def _rebuild(body, vertex_topk=None, edge_topk=None):
    vk = body.vertex_topk if vertex_topk is None else vertex_topk
    ek = body.edge_topk if edge_topk is None else edge_topk
    if (vk, ek) != (body.vertex_topk, body.edge_topk):
        body.surface = api.Surface(body.surface.mesh, body.sdf, vk, ek)
        body.vertex_topk, body.edge_topk = vk, ek


def _two(csv, what):
    parts = csv.split(",")
    if len(parts) != 2:
        raise ValueError(f"{what} expects 'K1,K2'")
    return int(parts[0]), int(parts[1])


def cmd_manifold(a) -> int:
    sc = scene_io.load_scene(a.scene)
    if len(sc.bodies) != 2:
        print("manifold: scene must contain exactly two bodies", file=sys.stderr)
        return 1
    cfg = _apply_flags(a, sc.smoothing)
    if a.topk_verts:
        k1, k2 = _two(a.topk_verts, "--topk-verts")
        _rebuild(sc.bodies[0], vertex_topk=k1)
        _rebuild(sc.bodies[1], vertex_topk=k2)
    if a.topk_edges:
        k1, k2 = _two(a.topk_edges, "--topk-edges")
        _rebuild(sc.bodies[0], edge_topk=k1)
        _rebuild(sc.bodies[1], edge_topk=k2)
    for b in sc.bodies:
        for w in b.surface.build_warnings:
            print(f"warning [{b.name}]: {w}", file=sys.stderr)
    b0, b1 = sc.bodies
    m = api.generate_manifold(b0.surface, b1.surface, b0.pose, b1.pose, cfg)
    with open(a.out, "w") as f:
        if a.json:
            f.write(scene_io.manifold_to_json(m["contacts"], m["meta"], m["layout"]) + "\n")
        else:
            scene_io.write_manifold_csv(f, m["contacts"], m["meta"])
    print(f"wrote {len(m['contacts'])} contacts to {a.out}")
    return 0


def cmd_sweep(a) -> int:
    ns, l2, sm = (api.rotating_edge_sweep(v, a.samples) for v in (0, 1, 2))
    with open(a.out, "w") as f:
        scene_io.write_sweep_csv(f, ns, l2, sm)
    jump = lambda s: float(np.linalg.norm(np.diff(s[:, 1:4], axis=0), axis=1).max())  # noqa: E731
    print(f"max adjacent-sample jump: no-smoothing {jump(ns):g}, smooth {jump(sm):g}")
    return 0


def _time_device(fn, reps, warm):
    """time_run (batch.cpp:104-120) on the device: median / std of CUDA-event
    times of `reps` runs after `warm` warm-ups."""
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts)), float(np.std(ts))


def cmd_bench(a) -> int:
    import torch

    batches = [int(x) for x in a.batch.split(",") if x]
    if not batches:
        raise ValueError("--batch needs at least one size")
    variants = [v for v in a.variants.split(",") if v]
    records = []
    if a.kind == "manifold":
        if not a.scene:
            print("bench: kind manifold needs --scene", file=sys.stderr)
            return 1
        sc = scene_io.load_scene(a.scene)
        if len(sc.bodies) < 2:
            raise ValueError("manifold benchmark needs a two-body scene")
        b0, b1 = sc.bodies[0], sc.bodies[1]
        for n in batches:
            # bench_manifold's poses (batch.cpp:196-203): body 1 fixed, body 2 jittered
            j = W.mt19937_64_uniform(a.seed, 6 * n, -0.05, 0.05).reshape(n, 6)
            p1 = torch.as_tensor(b0.pose.reshape(1, 6), device="cuda")
            p2 = torch.as_tensor(b1.pose[None, :] + j, device="cuda")
            for v in variants:
                cfg = sc.smoothing.for_variant(v)
                out = {}
                med, sd = _time_device(lambda: api.generate_manifold_batch(b0.surface, b1.surface, p1, p2, cfg,
                                                                           out=out), a.repetitions,
                                       min(3, a.repetitions))
                records.append(dict(kind="manifold", variant=v, batch=n, repetitions=a.repetitions, median_s=med,
                                    std_s=sd, throughput_qps=n / max(med, 1e-12)))
    elif a.kind in ("ee", "vf"):
        for n in batches:
            # make_random_ee/vf_pairs (batch.cpp:44-50): U[0,1) from mt19937_64(seed)
            pairs = torch.as_tensor(W.mt19937_64_uniform(a.seed, 12 * n, 0.0, 1.0).reshape(n, 12), device="cuda")
            for v in variants:
                cfg = SmoothingConfig().for_variant(v)
                fn = (lambda: api.run_ee_batch(pairs, cfg)) if a.kind == "ee" else (lambda: api.run_vf_batch(pairs, cfg))
                med, sd = _time_device(fn, a.repetitions, 3)
                records.append(dict(kind=a.kind, variant=v, batch=n, repetitions=a.repetitions, median_s=med,
                                    std_s=sd, throughput_qps=n / max(med, 1e-12)))
    else:
        raise ValueError("bench kind must be ee or vf")
    with open(a.out, "w") as f:
        scene_io.write_bench_csv(f, records)
    for r in records:
        print(f"{r['kind']}/{r['variant']} batch {r['batch']}: median {r['median_s']:g} s, "
              f"{r['throughput_qps']:g} q/s")
    return 0


def cmd_gradcheck(a) -> int:
    """cmd_gradcheck (main.cpp:190-235): the GPU pose Jacobian of
    mean_contact_distance vs central differences (h = 1e-6) of the same FP64
    mean, all 25 evaluations in one batch."""
    import torch

    sc = scene_io.load_scene(a.scene)
    if len(sc.bodies) != 2:
        print("gradcheck: scene must contain exactly two bodies", file=sys.stderr)
        return 1
    cfg = _apply_flags(a, sc.smoothing)
    b0, b1 = sc.bodies
    h = 1e-6
    P1 = np.repeat(b0.pose[None], 25, axis=0)
    P2 = np.repeat(b1.pose[None], 25, axis=0)
    for k in range(12):
        (P1 if k < 6 else P2)[1 + 2 * k, k % 6] += h
        (P1 if k < 6 else P2)[2 + 2 * k, k % 6] -= h
    r = api.generate_manifold_jvp_batch(b0.surface, b1.surface, torch.as_tensor(P1, device="cuda"),
                                        torch.as_tensor(P2, device="cuda"), cfg, want_f64_mean=True)
    torch.cuda.synchronize()
    mean = r["mean_dist_f64"].cpu().numpy()
    fwd = r["mean_dist_grad_f64"][0].cpu().numpy()
    fd = np.array([(mean[1 + 2 * k] - mean[2 + 2 * k]) / (2 * h) for k in range(12)])
    max_rel = 0.0
    print("dir  forward        finite-diff")
    for k in range(12):
        rel = abs(fwd[k] - fd[k]) / max(1e-7, abs(fd[k]))
        max_rel = max(max_rel, rel)
        print(f"{k:3d}  {fwd[k]:+.8e} {fd[k]:+.8e}")
    print(f"max relative error: {max_rel:g} (tolerance {a.tol:g})")
    return 0 if max_rel < a.tol else 1


def cmd_sim(a) -> int:
    """cmd_sim (main.cpp:237-254) + run_demosim_csv (demosim.cpp:157-186) on the
    batched GPU integrator (one env)."""
    if not (0.0 < a.dt <= 0.01):
        print("sim: dt must lie in (0, 0.01]", file=sys.stderr)
        return 1
    sc = scene_io.load_scene(a.scene)
    cfg = _apply_flags(a, sc.smoothing)
    sim = api.DemoBatch([b.surface for b in sc.bodies], [b.mass for b in sc.bodies],
                        inertia=[b.inertia_diag for b in sc.bodies], is_static=[b.is_static for b in sc.bodies],
                        cfg=cfg, params=PenaltyParams(), poses=np.array([b.pose for b in sc.bodies]), n_env=1)
    steps = int(math.floor(a.duration / a.dt + 0.5))  # std::llround (half away from zero)
    with open(a.out, "w") as f:
        f.write("time")
        for b in sc.bodies:
            f.write("".join(f",{b.name}_{c}" for c in ("tx", "ty", "tz", "rx", "ry", "rz", "vx", "vy", "vz",
                                                       "wx", "wy", "wz")))
        f.write("\n")
        for s in range(steps + 1):
            if s % 10 == 0:
                P = sim.poses[0].cpu().numpy()
                V = sim.velocities[0].cpu().numpy()
                row = [sim.time] + [x for i in range(len(sc.bodies)) for x in list(P[i]) + list(V[i])]
                f.write(",".join(scene_io._g17(x) for x in row) + "\n")
            if s < steps:
                sim.step(a.dt)
                if int(sim.ok[0].item()) == 0:
                    print("sim: state became non-finite (instability)", file=sys.stderr)
                    return 1
    print(f"simulated {a.duration:g} s -> {a.out}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2602_20304_b200",
                                 description="smooth differentiable contact manifolds (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("manifold", help="generate and dump a contact manifold")
    p.add_argument("--scene", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--json", action="store_true", help="emit JSON instead of CSV")
    p.add_argument("--topk-verts", default="", help="override vertex budgets 'N1,N2'")
    p.add_argument("--topk-edges", default="", help="override edge budgets 'M1,M2'")
    _add_smoothing_flags(p)
    p = sub.add_parser("sweep-edges", help="rotating-edge witness sweep")
    p.add_argument("--out", required=True)
    p.add_argument("--samples", type=int, default=10000)
    p = sub.add_parser("bench", help="witness / manifold throughput benchmark")
    p.add_argument("--kind", default="ee", help="ee | vf | manifold")
    p.add_argument("--batch", default="1000", help="comma-separated batch sizes")
    p.add_argument("--variants", default="ours,ours_ns", help="comma-separated variant list")
    p.add_argument("--scene", default="")
    p.add_argument("--out", required=True)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--repetitions", type=int, default=10)
    p.add_argument("--workers", type=int, default=1, help="accepted for compatibility (GPU path)")
    p = sub.add_parser("gradcheck", help="forward-mode vs finite-difference Jacobian")
    p.add_argument("--scene", required=True)
    p.add_argument("--tol", type=float, default=1e-3)
    _add_smoothing_flags(p)
    p = sub.add_parser("sim", help="penalty-force demo simulation")
    p.add_argument("--scene", required=True)
    p.add_argument("--duration", type=float, default=2.0)
    p.add_argument("--dt", type=float, default=1e-3)
    p.add_argument("--out", required=True)
    _add_smoothing_flags(p)
    a = ap.parse_args(argv)
    try:
        return {"manifold": cmd_manifold, "sweep-edges": cmd_sweep, "bench": cmd_bench,
                "gradcheck": cmd_gradcheck, "sim": cmd_sim}[a.cmd](a)
    except (ValueError, OSError, abi.CmgbError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
