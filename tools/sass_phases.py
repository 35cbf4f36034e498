"""Executed warp instructions of one kernel in an ncu report, split into the
segments between its barriers (BAR.SYNC) in address order -- the manifold
kernel's phases A..H (developer tool; out-of-line blocks the compiler moves to
the end of the function land in the last segment):
python tools/sass_phases.py <report.ncu-rep> [top opcodes per segment]."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 6
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
ia = hdr.index("Address") if "Address" in hdr else 0
segs = [collections.Counter()]
addr0 = [None]
for r in rows[2:]:
    if len(r) <= ie:
        continue
    t = r[1].strip().split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).rstrip(";")
    try:
        n = int(r[ie])
    except ValueError:
        n = 0
    if addr0[-1] is None:
        addr0[-1] = r[ia]
    segs[-1][op.split(".")[0]] += n
    if op.startswith("BAR.SYNC"):
        segs.append(collections.Counter())
        addr0.append(None)
tot = sum(sum(s.values()) for s in segs) or 1
for k, (s, a) in enumerate(zip(segs, addr0)):
    n = sum(s.values())
    if n == 0:
        continue
    mix = ", ".join(f"{op} {100 * c / n:.0f}%" for op, c in s.most_common(top))
    print(f"seg {k:2d} @{a}: {n:12d} instr {100 * n / tot:5.1f}%  [{mix}]")
print(f"total {tot}")
