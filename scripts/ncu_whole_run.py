"""Whole-run DRAM evidence for one coh_elem_eval call: per-kernel-name sums of
gpu__time_duration, dram__bytes_read and dram__bytes_write from an ncu --metrics launch
list (serialised, cold-cache replays) of scripts/bench_elem.py --reps 1, which makes two
identical coh_elem_eval calls (a counting pass, then the timed one); the second half of
the launches is the measured call.
usage: python scripts/ncu_whole_run.py LAUNCHES.csv [alg_bytes]"""
import collections
import csv
import json
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ix = {h: j for j, h in enumerate(hdr)}
    per = {}
    for r in data:
        k = int(r[ix["ID"]])
        per.setdefault(k, {"name": r[ix["Kernel Name"]].split("(")[0]})[r[ix["Metric Name"]]] = float(
            r[ix["Metric Value"]].replace(",", ""))
    ids = sorted(per)
    timed = ids[len(ids) // 2:]
    agg = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    for k in timed:
        d, a = per[k], agg[per[k]["name"]]
        a["launches"] += 1
        a["ms"] += d.get("gpu__time_duration.sum", 0) / 1e6
        a["dram_read"] += d.get("dram__bytes_read.sum", 0)
        a["dram_write"] += d.get("dram__bytes_write.sum", 0)
    tot = {"launches": len(timed), "ms": sum(a["ms"] for a in agg.values()),
           "dram_read": sum(a["dram_read"] for a in agg.values()), "dram_write": sum(a["dram_write"] for a in agg.values())}
    out = {"kernels": dict(agg), "total": tot}
    if len(sys.argv) > 2:
        alg = float(sys.argv[2])
        out["alg_bytes"] = alg
        out["physical_over_algorithmic"] = (tot["dram_read"] + tot["dram_write"]) / alg
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
