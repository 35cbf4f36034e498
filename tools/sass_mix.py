"""Executed-instruction mix of one kernel in an ncu report, by SASS opcode
(developer tool): python tools/sass_mix.py <report.ncu-rep> [top]."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    t = r[1].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    try:
        mix[op.split(".")[0]] += int(r[ie])
    except ValueError:
        pass
tot = sum(mix.values())
print(f"total warp instructions {tot}")
for op, n in mix.most_common(top):
    print(f"{op:12s} {n:14d} {100 * n / tot:6.2f} %")
