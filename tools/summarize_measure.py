#!/usr/bin/env python
"""Turn one tools/final_measure_r02.sh run (gpurun_out/<tag>_*) into the
committed evidence under profiles/ (developer tool):

  profiles/<round>_bench_<workload>.json   the bench lines
  profiles/<round>_launches.csv            ncu launch list of the default bench command (+ kernel shares)
  profiles/<round>_ncu_<kernel>.txt        full-capture summaries (metrics, stalls, hot lines, SASS mix)
  profiles/manifold_fp64_ops.json          executed FP64 work per env  -> bench.py roofline.fp64_pipe
  profiles/manifold_dram_bytes.json        DRAM bytes per step per env -> bench.py roofline.traffic
  profiles/witness_{ee,vf}_dram_bytes.json DRAM bytes per pair         -> bench.py roofline.traffic (K6)

python tools/summarize_measure.py <tag> <round>   e.g. r02m r02
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def ncu_csv(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    return [dict(zip(h, r)) for r in rows[1:]]


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    n_env = 65536
    # bench lines
    for f in sorted(os.listdir(G)):
        if f.startswith(f"{tag}_bench") and f.endswith(".json"):
            lines = [ln for ln in open(os.path.join(G, f)) if ln.strip().startswith("{")]
            if lines:
                dst = os.path.join(P, f.replace(tag, rnd, 1))
                open(dst, "w").write(lines[-1])
                print("wrote", dst)
    # launch list: kernel shares of the default bench command
    rows = ncu_csv(os.path.join(G, f"{tag}_launches.csv"))
    shutil.copy(os.path.join(G, f"{tag}_launches.csv"), os.path.join(P, f"{rnd}_launches.csv"))
    tot = collections.Counter()
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            tot[name] += float(r["Metric Value"])
    s = sum(tot.values())
    share = {k: round(100 * v / s, 2) for k, v in tot.most_common()}
    json.dump({"command": "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras",
               "kernel_time_share_pct": share}, open(os.path.join(P, f"{rnd}_launch_shares.json"), "w"), indent=1)
    print("launch shares", share)
    # FP64 work and DRAM traffic of the box-box step (vs_kernel + manifold_kernel, one launch each)
    rows = ncu_csv(os.path.join(G, f"{tag}_fp64.csv"))
    per = collections.defaultdict(dict)
    for r in rows:
        per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    dfma = sum(v.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) for v in per.values())
    dmul = sum(v.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) for v in per.values())
    dadd = sum(v.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0) for v in per.values())
    rd = sum(v.get("dram__bytes_read.sum", 0) for v in per.values())
    wr = sum(v.get("dram__bytes_write.sum", 0) for v in per.values())
    pipe = [v.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") for k, v in per.items()
            if "manifold_kernel" in k[1]]
    kns = {("manifold_kernel" if "manifold_kernel" in k[1] else "vs_kernel"): v.get("gpu__time_duration.sum")
           for k, v in per.items()}
    json.dump({"kernels": "manifold_kernel<3,3,0,1> + vs_kernel<3,3> (box-box, 65,536 envs), ncu --metrics pass "
                          f"(tools/final_measure_r02.sh, {rnd})",
               "dfma_per_env": dfma / n_env, "dmul_per_env": dmul / n_env, "dadd_per_env": dadd / n_env,
               "fp64_flop_per_env": (2 * dfma + dmul + dadd) / n_env, "fp64_inst_per_env": (dfma + dmul + dadd) / n_env,
               "ncu_fp64_pipe_active_pct": pipe[0] if pipe else None, "kernel_ns": kns,
               "note": "executed FP64 arithmetic of this kernel's analytic formulation (DFMA = 2 flop); the "
                       "reference formulation's algorithmic count is 763,164 flop/env (profiles/work_per_unit.json)"},
              open(os.path.join(P, "manifold_fp64_ops.json"), "w"), indent=1)
    json.dump({"kernels": "manifold_kernel<3,3,0,1> + vs_kernel<3,3> (box-box, 65,536 envs)",
               "dram_bytes_read_per_launch": rd, "dram_bytes_write_per_launch": wr,
               "dram_bytes_per_launch_per_env": (rd + wr) / n_env, "algorithmic_bytes_per_env": 9776,
               "source": f"ncu --metrics pass (tools/final_measure_r02.sh, {rnd})"},
              open(os.path.join(P, "manifold_dram_bytes.json"), "w"), indent=1)
    # FP64 work of the JVP kernels (config D: one step = 10 pair launches of 32,768 envs)
    jp = os.path.join(G, f"{tag}_jvp_fp64.csv")
    if os.path.exists(jp):
        per = collections.defaultdict(dict)
        for r in ncu_csv(jp):
            per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        units = 10 * 32768
        dfma = sum(v.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) for v in per.values())
        dmul = sum(v.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) for v in per.values())
        dadd = sum(v.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0) for v in per.values())
        pipe = [v.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") for v in per.values()]
        json.dump({"kernels": f"manifold_jvp_kernel, the 10 pair launches of one config D step (32,768 envs), "
                              f"ncu --metrics pass (tools/final_measure_r02.sh, {rnd})",
                   "fp64_flop_per_unit": (2 * dfma + dmul + dadd) / units, "dfma_per_unit": dfma / units,
                   "dmul_per_unit": dmul / units, "dadd_per_unit": dadd / units,
                   "ncu_fp64_pipe_active_pct_mean": sum(pipe) / len(pipe) if pipe else None,
                   "kernel_ns_sum": sum(v.get("gpu__time_duration.sum", 0) for v in per.values()),
                   "unit": "pair manifold (one env of one body pair) with its 12 pose tangents"},
                  open(os.path.join(P, "jvp_fp64_ops.json"), "w"), indent=1)
        print("wrote jvp_fp64_ops.json")
    for kind in ("ee", "vf"):
        rows = ncu_csv(os.path.join(G, f"{tag}_{kind}_dram.csv"))
        m = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
        n = 4194304
        json.dump({"kernel": f"witness_kernel ({kind}, soft, {n} FP64 pairs)",
                   "dram_bytes_per_pair": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / n,
                   "algorithmic_bytes_per_pair": 96 + (24 if kind == "ee" else 12), "kernel_ns": m["gpu__time_duration.sum"],
                   "source": f"ncu --metrics pass (tools/final_measure_r02.sh, {rnd})"},
                  open(os.path.join(P, f"witness_{kind}_dram_bytes.json"), "w"), indent=1)
    # full-capture summaries
    for name in ("manifold", "mixed", "jvp", "ee", "compact"):
        rep = os.path.join(G, f"{tag}_{name}.ncu-rep")
        txt = os.path.join(G, f"{tag}_ncu_{name}.txt")
        if not os.path.exists(rep):
            if os.path.exists(txt):  # summarised on the GPU box (final_measure_r02.sh)
                shutil.copy(txt, os.path.join(P, f"{rnd}_ncu_{name}.txt"))
                print("wrote", os.path.join(P, f"{rnd}_ncu_{name}.txt"))
            continue
        a = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "30"],
                           capture_output=True, text=True).stdout
        b = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_mix.py"), rep, "25"],
                           capture_output=True, text=True).stdout
        dst = os.path.join(P, f"{rnd}_ncu_{name}.txt")
        open(dst, "w").write(a + "\n--- executed SASS mix ---\n" + b)
        print("wrote", dst)


if __name__ == "__main__":
    main()
