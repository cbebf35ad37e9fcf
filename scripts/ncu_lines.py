"""Per-source-line totals (instructions executed, stall samples) of one kernel in an ncu
report, from the sass,cuda source view.  usage: python scripts/ncu_lines.py REP [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot = {}
cur = None
for r in rows:
    if len(r) < len(hdr) or r[0] == "Line No":
        continue
    if r[0]:  # a cuda source line row
        cur = (int(r[0]), r[1].strip()[:90])
    if r[2] and cur:
        t = tot.setdefault(cur, [0, 0])
        try:
            t[0] += int(r[ie] or 0)
            t[1] += int(r[ss] or 0)
        except ValueError:
            pass
I = sum(v[0] for v in tot.values()) or 1
S = sum(v[1] for v in tot.values()) or 1
for (ln, src), (i, s) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {100 * i / I:5.1f}% inst {100 * s / S:5.1f}% stall  {src}")
