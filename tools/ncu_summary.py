"""Summarise an ncu report: key metrics, stall reasons, and the source lines
with the most instructions / stall samples (developer tool)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, vals = raw[0], raw[2]
d = dict(zip(h, vals))
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
for k, v in zip(h, vals):
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            if float(v) > 0.1:
                print(f"  stall {k.split('stalled_')[1].split('_per')[0]:24s} {float(v):.2f}")
        except ValueError:
            pass
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
agg = collections.defaultdict(lambda: [0, 0, ""])
cur = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] != "":
        cur = (f, int(r[0]))
        agg[cur][2] = r[1][:80]
        continue
    for j, col in ((0, ie), (1, ss)):
        try:
            agg[cur][j] += int(r[col])
        except (ValueError, IndexError):
            pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
byf = collections.defaultdict(lambda: [0, 0])
for (f, _), v in agg.items():
    byf[f][0] += v[0]
    byf[f][1] += v[1]
print("per file (instr %, stall %):", {f: (round(100 * a / ti, 1), round(100 * b / ts, 1)) for f, (a, b) in byf.items()})
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:14s}:{k[1]:4d} instr {100 * v[0] / ti:5.1f}% stall {100 * v[1] / ts:5.1f}% | {v[2]}")
