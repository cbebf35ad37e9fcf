"""Summarise an `ncu --metrics gpu__time_duration.sum` launch list: per kernel + grid,
count / mean / share of total device time.  usage: python scripts/summarize_launches.py CSV"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr, data = rows[0], rows[1:]
ik, ig, iv = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    agg.setdefault((r[ik].split("(")[0].replace("void ", ""), r[ig]), []).append(v)
total = sum(sum(v) for v in agg.values())
print(f"{'kernel':45s} {'grid':>16s} {'n':>4s} {'mean_us':>10s} {'share':>7s}")
for (k, g), v in agg.items():
    print(f"{k:45s} {g:>16s} {len(v):4d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / total:7.1%}")
