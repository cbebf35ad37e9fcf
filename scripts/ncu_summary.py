"""Extract the judged metrics of one ncu --set full capture into profiles/.
usage: python scripts/ncu_summary.py REP.ncu-rep OUT_PREFIX [traces_per_launch] [kernel-substring]"""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    traces = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    d[k] = float(v)
                except ValueError:
                    d[k] = v
                d[k + ".unit"] = units[i]
        # the per-SM average is all the raw page has for the whole data pipe: x SMs
        ka, kn = "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg", "device__attribute_multiprocessor_count"
        if ka in hdr and kn in hdr and "l1tex__data_pipe_lsu_wavefronts.sum" not in hdr:
            try:
                d["l1tex__data_pipe_lsu_wavefronts.sum"] = float(vals[hdr.index(ka)].replace(",", "")) * \
                    float(vals[hdr.index(kn)].replace(",", ""))
                d["l1tex__data_pipe_lsu_wavefronts.sum.unit"] = "wavefront (per-SM avg x SMs)"
            except ValueError:
                pass
        kernels.append(d)
    pick = sys.argv[4] if len(sys.argv) > 4 else ""
    k = next(kk for kk in kernels if pick in kk["kernel"])
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
    dram = k["dram__bytes_read.sum"] * scale.get(k["dram__bytes_read.sum.unit"], 1) + \
        k["dram__bytes_write.sum"] * scale.get(k["dram__bytes_write.sum.unit"], 1)
    summary = {"source": rep, "kernel": k["kernel"], "dram_bytes_per_launch": dram, "traces_per_launch": traces,
               "metrics": {kk: v for kk, v in k.items() if not kk.endswith(".unit") and kk != "kernel"}}
    with open(prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu --set full: {k['kernel']}\n\nsource: `{rep}`\n\n| metric | value | unit |\n|---|---|---|\n")
        for kk in KEYS:
            if kk in k:
                f.write(f"| {kk} | {k[kk]} | {k.get(kk + '.unit', '')} |\n")
        f.write(f"\nDRAM bytes per launch (read+write): {dram:.0f}\n")
    print(json.dumps(summary["metrics"], indent=0)[:2000])


if __name__ == "__main__":
    main()
