#!/usr/bin/env python
"""Benchmark of the batched access-mode-calculus evaluator (BASELINE.json metric).

One step = one pass of the hot path over one batch: trace_eval over this rank's traces
(BASELINE config 2 per GPU: 1M traces x 64 arrays x 256 calls, whole-array validity)
+ the counter reduction, + for N>1 the NCCL allreduce of the counter vector (config 4).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  See DESIGN.md §6 for every field.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "component-call transitions/sec at 1/2/4/8 B200; bitmap GB/s vs HBM peak"
N_ARRAYS, N_CALLS, ADV, FUEL, SEED = 64, 256, 1, 10000, 1
TRACES_PER_GPU = 1 << 20
WORKLOAD = "C2/C4: 1M traces x 64 arrays x 256 whole-array component calls per GPU (BASELINE configs[1], sharded by trace id for N>1)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--traces", type=int, default=TRACES_PER_GPU, help="traces per GPU")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=3.0, help="wall seconds of the CPU baseline sample")
    ap.add_argument("--bitmap-buffers", type=int, default=256, help="C3 buffers per GPU (0 = skip)")
    ap.add_argument("--bitmap-log2-cells", type=int, default=24)
    ap.add_argument("--bitmap-calls", type=int, default=8)
    ap.add_argument("--container-log2-floats", type=int, default=28, help="C5 vector size (0 = skip)")
    ap.add_argument("--container-calls", type=int, default=64)
    ap.add_argument("--sweep-seeds", type=int, default=100000, help="acceptance-sweep seeds (0 = skip)")
    ap.add_argument("--overlap-views", type=int, default=1 << 20, help="overlap registry views (0 = skip)")
    ap.add_argument("--overlap-blocks", type=int, default=1 << 20)
    ap.add_argument("--c4-traces", type=int, default=1 << 26, help="C4 total traces, split over the ranks (0 = skip)")
    ap.add_argument("--checker-programs", type=int, default=20000, help="batched checker programs (0 = skip)")
    ap.add_argument("--blocks-traces", type=int, default=1 << 20, help="multi-mode block traces (0 = skip)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        loaded = [r for r in self.rows if r[2].isdigit() and int(r[2]) > 0] or self.rows
        sm = [float(r[0]) for r in loaded if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in loaded if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in loaded for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(loaded)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_issue(n_traces, kernel_ms, sm_mhz, sms):
    """The binding roofline of k_trace_eval (instruction issue: "INT pipe
    is the expected binder"): warp instructions per launch from the committed ncu capture
    (scaled to this launch's traces) over the measured kernel time, against the issue peak
    of one warp instruction per clock per SM sub-partition (4 per SM) at the sampled clock."""
    p = os.path.join(ROOT, "profiles", "ncu_trace_eval.json")
    if not os.path.exists(p) or not kernel_ms or not sm_mhz:
        return None
    with open(p) as f:
        d = json.load(f)
    inst = d.get("metrics", {}).get("smsp__inst_executed.sum")
    if not inst or not d.get("traces_per_launch"):
        return None
    inst = inst * n_traces / d["traces_per_launch"]
    achieved = inst / (kernel_ms / 1e3)
    peak = 4.0 * sms * sm_mhz * 1e6
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp inst/s", "frac": achieved / peak,
            "inst_per_launch": inst, "source": "profiles/ncu_trace_eval.json smsp__inst_executed.sum, "
                                              "peak = 4 x SMs x sampled SM clock"}


def ncu_l1_pipe(n_traces, kernel_ms, sm_mhz, sms):
    """The shared-memory / L1 data pipe of k_trace_eval (3 LDS/STS per call + the record
    loads): wavefronts per launch from the committed ncu capture (scaled to this launch's
    traces) over the measured kernel time, against one wavefront per clock per SM."""
    p = os.path.join(ROOT, "profiles", "ncu_trace_eval.json")
    if not os.path.exists(p) or not kernel_ms or not sm_mhz:
        return None
    with open(p) as f:
        d = json.load(f)
    wf = d.get("metrics", {}).get("l1tex__data_pipe_lsu_wavefronts.sum")
    if not wf or not d.get("traces_per_launch"):
        return None
    wf = wf * n_traces / d["traces_per_launch"]
    achieved = wf / (kernel_ms / 1e3)
    peak = 1.0 * sms * sm_mhz * 1e6
    return {"bound": "l1_data_pipe", "achieved": achieved, "peak": peak, "unit": "wavefronts/s", "frac": achieved / peak,
            "wavefronts_per_launch": wf, "source": "profiles/ncu_trace_eval.json l1tex__data_pipe_lsu_wavefronts.sum, "
                                                   "peak = 1 x SMs x sampled SM clock"}


def ncu_traffic():
    """dram bytes per trace_eval launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_trace_eval.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("traces_per_launch")
    return None, None


# ------------------------------------------------------------------- CPU baselines
def cpu_eval_fn():
    """(kind, fn) for the CPU baseline: the reference compiled in place (oracle/_ref) if it
    shipped, else the C restatement (oracle/_build).  Test infrastructure, timed only."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as orc

    if orc.have_ref():
        return "reference", lambda recs, n, threads: orc.ref_eval(recs, n, N_CALLS, N_ARRAYS, FUEL, threads=threads, mode=1)
    return "port", lambda recs, n, threads: orc.orc_eval(recs, n, N_CALLS, N_ARRAYS, FUEL)


def evaluated_calls(res):
    st = res["status"]
    return int(res["calls_done"].astype(np.int64).sum() + (st != 0).sum())


def cpu_sample(seconds, threads, trace0=0):
    """Time the CPU evaluator on a bounded sample of the same workload (trace ids from
    trace0), sized to ~`seconds` of wall time on `threads` host threads.  The records come
    from the oracle's own generator (orc_gen_records, the same splitmix64 stream as the
    device generator), so this leg never loads the product library."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as orc

    kind, fn = cpu_eval_fn()
    cores = threads if kind == "reference" else 1
    n = 64 if kind == "reference" else 2048
    while True:
        recs = orc.orc_gen(SEED, trace0, n, N_CALLS, N_ARRAYS, ADV)
        t0 = time.perf_counter()
        res, _ = fn(recs, n, cores)
        dt = time.perf_counter() - t0
        if dt >= 0.25 * seconds or n >= (1 << 22):
            if dt < seconds and n < (1 << 22):
                n = int(n * seconds / max(dt, 1e-3))
                recs = orc.orc_gen(SEED, trace0, n, N_CALLS, N_ARRAYS, ADV)
                t0 = time.perf_counter()
                res, _ = fn(recs, n, cores)
                dt = time.perf_counter() - t0
            calls = evaluated_calls(res)
            return {"value": calls / dt, "unit": "calls/s", "cores": cores, "kind": kind,
                    "sample": f"{n} traces (ids {trace0}..{trace0 + n - 1}) of the same workload, {dt:.2f} s wall",
                    "traces": n, "seconds": dt, "calls": calls}
        n *= 4


def bench_config(world, traces_per_gpu):
    """The `config` object of both arms (identical by construction)."""
    return {"workload": WORKLOAD, "traces_per_gpu": traces_per_gpu, "arrays": N_ARRAYS, "calls": N_CALLS,
            "adv_per1024": ADV, "fuel": FUEL, "parallelism": f"dp{world} (trace-id shards)",
            "l2": "inputs larger than L2 (records 512 MiB per GPU), no flush"}


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation of the path (oracle/_ref: the unmodified
    reference headers, cohere::run_annotated per trace, on all host threads; the C
    restatement if the reference did not ship).  Nothing from the product package is
    imported or loaded here: records come from the oracle's generator."""
    if rank != 0:
        return  # rank 0 alone runs the reference arm
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as orc

    threads = os.cpu_count() or 1
    kind, fn = cpu_eval_fn()
    cores = threads if kind == "reference" else 1
    # one calibration, then every step evaluates a fixed-size sample of fresh trace ids,
    # sized so warmup + steps finish within ~2 minutes
    per_step = max(0.05, min(5.0, 110.0 / max(1, args.steps + args.warmup)))
    cal = cpu_sample(min(per_step, 1.0), threads, trace0=1 << 40)
    n_step = max(cores, int(cal["traces"] * per_step / max(cal["seconds"], 1e-3)))
    t_calls, t_sec = 0, 0.0
    for k in range(args.warmup + args.steps):
        recs = orc.orc_gen(SEED, (1 << 30) + k * n_step, n_step, N_CALLS, N_ARRAYS, ADV)
        t0 = time.perf_counter()
        res, _ = fn(recs, n_step, cores)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            t_calls += evaluated_calls(res)
            t_sec += dt
    value = t_calls / t_sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "calls/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_sec / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
        "data": "synthetic (counter-based splitmix64 call records, seed 1)",
        "config": bench_config(world, args.traces),
        "cpu_baseline": {"value": value, "unit": "calls/s", "cores": cores, "kind": kind,
                         "sample": f"per step: {n_step} traces of the same workload (fresh trace ids per step), "
                                   f"cohere::run_annotated on {cores} host threads"},
        "e2e": {"value": value, "unit": "calls/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- bitmaps (C3)
RHOS = (("0", 0), ("2^-16", 16), ("2^-8", 8), ("1/2", 1))


def run_bitmap(args, ctx, rank, world):
    """BASELINE config 3 per GPU: B buffers x 2^24 cells, 8 overlapping views each, K calls
    per buffer through the element path (overlap closure, whole-view syncs + transfer-range
    extraction, element range bodies, per-view boundary checks), at each SURVEY §8(d)
    pre-fragmentation level rho in {0, 2^-16, 2^-8, 1/2} (that fraction of the cells starts
    coherent, so the syncs' transfer ranges fragment).  Every transfer range is written on
    the device (runs_cap from a counting pass; none are copied back inside the timing).
    Algorithmic bytes per SURVEY §8(d), 8 B per written range; device time by CUDA events
    inside coh_elem_eval (best of 3); max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1910_11110_b200.elem import Program, elem_eval

    B, n, K = args.bitmap_buffers, 1 << args.bitmap_log2_cells, args.bitmap_calls
    peak, src = peaks()
    per_rho = {}
    for name, k in RHOS:
        progs = [Program.generate(3, rank * B + b, n, 8, K, 64, frag_log2=k) for b in range(B)]
        t0 = time.perf_counter()
        count = elem_eval(ctx, progs, want_planes=False, runs_cap=0, download_runs=False)  # counts the ranges
        wall_ms = 1e3 * (time.perf_counter() - t0)
        res = count["results"]
        cap = max(1, max(int(res[i].n_runs) for i in range(B)))
        best = None
        for _ in range(3):
            out = elem_eval(ctx, progs, want_planes=False, runs_cap=cap, download_runs=False)
            st = out["stats"]
            if best is None or st.device_ms < best[0]:
                best = (st.device_ms, st.alg_bytes, st.stages, st.launches)
        ms, alg, stages, launches = best
        runs = sum(int(res[i].n_runs) for i in range(B))
        if world > 1:
            t = torch.tensor([ms, float(alg), float(runs)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t[0:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t[1:3])
            ms, alg, runs = float(t[0].item()), int(t[1].item()), int(t[2].item())
        gbs = alg / (ms / 1e3) / 1e9
        per_rho[name] = {"value": gbs, "unit": "GB/s", "frac": gbs / peak, "device_ms": ms, "alg_bytes": alg,
                         "runs_written": runs, "runs_cap_per_buffer": cap, "stages": stages, "launches": launches,
                         "host_compile_upload_ms": wall_ms - float(count["stats"].device_ms),
                         "stuck": sum(1 for i in range(B) if res[i].status == 1),
                         "transfers": sum(res[i].transfers for i in range(B)),
                         "transfer_cells": sum(int(res[i].transfer_cells) for i in range(B))}
        del progs, count, out
    head = per_rho["2^-16"]
    return {"metric": "bitmap GB/s (algorithmic bytes / device time), element path C3", "value": head["value"],
            "unit": "GB/s", "frac": head["frac"], "peak": peak, "peak_source": src, "headline_rho": "2^-16",
            "rho": per_rho,
            "config": {"workload": "C3: element-granular bit planes, overlapping views, pre-fragmented", "buffers_per_gpu": B,
                       "cells": n, "views": 8, "calls": K, "adv_per1024": 64,
                       "l2": "1 GiB of planes per GPU > L2, no flush"},
            "cpu_reference": bitmap_cpu_reference(ctx) if rank == 0 and not args.no_cpu_baseline else None}


def bitmap_cpu_reference(ctx):
    """The reference on the C3 workload's shape, bounded (the reference only at
    n <= 2^20): one program of 2^20 cells, 8 views, 8 calls, run through the reference's
    own run_annotated over its std::map store (oracle/_ref, one host thread); its
    algorithmic bytes (the same count as the GPU line's) over its wall time."""
    from paper_1910_11110_b200.elem import Program, elem_eval
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_ffi as o
        if not o.have_ref():
            return {"unavailable": "oracle/_ref not built"}
        p = Program.generate(3, 0, 1 << 20, 8, 8, 64, frag_log2=16)
        alg = int(elem_eval(ctx, [p], want_planes=False, runs_cap=1 << 20, download_runs=False)["stats"].alg_bytes)
        t0 = time.perf_counter()
        rc = o.elem_run("ref", p)[0]
        dt = time.perf_counter() - t0
        return {"value": alg / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference", "seconds": dt,
                "rc": int(rc), "sample": "one program of 2^20 cells, 8 views, 8 calls, rho 2^-16 (seed 3, program 0)"}
    except Exception as ex:  # test infrastructure; its absence is not fatal here
        return {"error": f"{type(ex).__name__}: {ex}"}


def run_bitmap_primitives(args, ctx):
    """SURVEY §8(b) item 2 primitives on C3-sized planes: 256 planes x 2^24 cells (512 MiB
    per plane array, > L2), one range per plane covering a random 60-100% of it.  Each
    primitive timed with CUDA events on the stream (best of 6, the whole API call: range
    prefix, scratch, kernels); algorithmic bytes per SURVEY §8(d): set/clear m/8 written,
    first zero m/8 read, view check 2 x m/8 read, zero runs m/8 read + 8 B per run."""
    import torch

    from paper_1910_11110_b200.bitmap import RANGE_DTYPE

    P, n = args.bitmap_buffers, 1 << args.bitmap_log2_cells
    words = n // 32
    rng = np.random.default_rng(3)
    L = torch.full((P * words,), -1, dtype=torch.int32, device="cuda")
    Rp = torch.zeros(P * words, dtype=torch.int32, device="cuda")
    ranges = np.zeros(P, RANGE_DTYPE)
    ranges["word_off"] = np.arange(P) * words
    ranges["lo"] = rng.integers(0, n // 5, P)
    ranges["hi"] = n - 1 - rng.integers(0, n // 5, P)
    m = int((ranges["hi"].astype(np.int64) - ranges["lo"] + 1).sum())
    d_r = torch.from_numpy(ranges.view(np.uint8).copy()).cuda()
    # fragment R: a sparse pattern of set cells (zero runs of ~2^12 cells)
    frag = np.zeros(P, RANGE_DTYPE)
    frag_r = []
    for k in range(P):
        for c in rng.integers(0, n - 64, 64):
            frag_r.append((k * words, int(c), int(c) + int(rng.integers(0, 64))))
    frag = np.array(frag_r, RANGE_DTYPE)
    d_f = torch.from_numpy(frag.view(np.uint8).copy()).cuda()
    Lb = coh_lib()
    s = torch.cuda.current_stream().cuda_stream
    assert Lb.coh_bitmap_range_set(ctx._h, Rp.data_ptr(), d_f.data_ptr(), len(frag), s) == 0
    first = torch.empty(P, dtype=torch.int32, device="cuda")
    ok = torch.empty(P, dtype=torch.uint8, device="cuda")
    ab = torch.ones(P, dtype=torch.uint8, device="cuda")
    cap = 1 << 22
    rs = torch.empty(cap, dtype=torch.int32, device="cuda")
    re_ = torch.empty(cap, dtype=torch.int32, device="cuda")
    roff = torch.empty(P + 1, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        best = None
        for _ in range(6):
            e0.record()
            rc = fn()
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return best

    peak, src = peaks()
    out = {"metric": "bit-plane primitives GB/s (algorithmic bytes / device time)", "planes": P, "cells": n,
           "cells_in_ranges": m, "peak": peak, "peak_source": src}
    t = timed(lambda: Lb.coh_bitmap_first_zero(ctx._h, L.data_ptr(), d_r.data_ptr(), P, first.data_ptr(), s))
    out["first_zero"] = {"ms": t, "gbs": m / 8 / (t / 1e3) / 1e9}
    t = timed(lambda: Lb.coh_bitmap_view_check(ctx._h, L.data_ptr(), Rp.data_ptr(), d_r.data_ptr(), ab.data_ptr(), P,
                                               ok.data_ptr(), s))
    out["view_check"] = {"ms": t, "gbs": 2 * m / 8 / (t / 1e3) / 1e9}
    t = timed(lambda: Lb.coh_bitmap_extract_zero_runs(ctx._h, Rp.data_ptr(), d_r.data_ptr(), P, rs.data_ptr(),
                                                      re_.data_ptr(), cap, roff.data_ptr(), s))
    runs = int(roff[-1].item())
    out["zero_runs"] = {"ms": t, "runs": runs, "gbs": (m / 8 + 8 * runs) / (t / 1e3) / 1e9,
                        "note": "collect pass reads the plane once; chunks with > 1024 runs re-walk it in the place pass"}
    t = timed(lambda: Lb.coh_bitmap_range_set(ctx._h, L.data_ptr(), d_r.data_ptr(), P, s))
    out["range_set"] = {"ms": t, "gbs": m / 8 / (t / 1e3) / 1e9}
    t = timed(lambda: Lb.coh_bitmap_range_clear(ctx._h, L.data_ptr(), d_r.data_ptr(), P, s))
    out["range_clear"] = {"ms": t, "gbs": m / 8 / (t / 1e3) / 1e9}
    for k in ("first_zero", "view_check", "zero_runs", "range_set", "range_clear"):
        out[k]["frac"] = out[k]["gbs"] / peak
    # run extraction across fragmentation (rho in {0, 2^-16, 2^-8, 1/2} of
    # cells set in the destination plane, independently per cell): the same planes and
    # ranges; output-bound at rho = 1/2 (a run every four cells)
    Pf = P
    sweep = {}
    for name, ands in (("0", None), ("2^-16", 16), ("2^-8", 8), ("1/2", 1)):
        plane = torch.zeros(Pf * words, dtype=torch.int32, device="cuda")
        if ands:
            plane.fill_(-1)
            for _ in range(ands):
                plane &= torch.randint(-(1 << 31), 1 << 31, (Pf * words,), dtype=torch.int32, device="cuda")
        mf = int((ranges["hi"][:Pf].astype(np.int64) - ranges["lo"][:Pf] + 1).sum())
        capf = mf // 3 + 16 if ands == 1 else cap
        rsf = torch.empty(capf, dtype=torch.int32, device="cuda")
        ref_ = torch.empty(capf, dtype=torch.int32, device="cuda")
        t = timed(lambda: Lb.coh_bitmap_extract_zero_runs(ctx._h, plane.data_ptr(), d_r.data_ptr(), Pf, rsf.data_ptr(),
                                                          ref_.data_ptr(), capf, roff.data_ptr(), s))
        runs = int(roff[Pf].item())
        gbs = (mf / 8 + 8 * runs) / (t / 1e3) / 1e9
        sweep[name] = {"ms": t, "runs": runs, "gbs": gbs, "frac": gbs / peak}
        del plane, rsf, ref_
    out["zero_runs_by_fragmentation"] = {"planes": Pf, "cells_in_ranges": mf, "rho": sweep,
                                         "note": "bytes = m/8 read + 8 per run written (SURVEY 8(d))"}
    return out


# ------------------------------------------------------------- container (C5)
def run_container(args, ctx):
    """BASELINE config 5: 4 vectors x 2^28 float32 (1 GiB each), a seeded chain of
    component calls with random modes and sites over built-in trivial CPU / GPU
    components; every copy is a real cudaMemcpyAsync issued by the runtime.  Reports bytes
    moved vs the evaluator's prediction (must be equal) and the achieved link bandwidth
    against a measured pinned-copy peak."""
    from paper_1910_11110_b200.container import Runtime

    n = 1 << args.container_log2_floats
    rt = Runtime(ctx)
    rt.set_async(True)  # CPU components as stream-ordered host functions: copies overlap them
    vecs = [rt.vector(n) for _ in range(4)]
    peaks_gbs = ctx.measure_link(n * 4, 3)  # pinned cudaMemcpyAsync, best of 3, per direction
    rng = np.random.default_rng(5)
    t0 = time.perf_counter()
    for _ in range(args.container_calls):
        k = int(rng.integers(1, 4))
        idx = rng.choice(4, size=k, replace=False)
        site = "gpu" if rng.random() < 0.5 else "cpu"
        rt.call(site, [(vecs[i], ["R", "W", "RW"][int(rng.integers(0, 3))]) for i in idx])
    rt.sync()
    dt = time.perf_counter() - t0
    st = rt.stats()
    pred = rt.predicted()
    moved = st["h2d_bytes"] + st["d2h_bytes"]
    out = {"metric": "container chain: bytes moved == evaluator prediction", "match": int(pred["transfer_bytes"]) == moved,
           "bytes_moved": moved, "bytes_predicted": int(pred["transfer_bytes"]), "copies": st["h2d_copies"] + st["d2h_copies"],
           "syncs_elided": st["syncs_elided"], "calls": st["calls"], "wall_s": dt,
           "link_gbs_achieved": moved / dt / 1e9, "copy_ms": st["copy_ms"],
           "link_gbs_during_copies": moved / (st["copy_ms"] / 1e3) / 1e9 if st["copy_ms"] else None,
           "link_peak_gbs": {"h2d": peaks_gbs[0], "d2h": peaks_gbs[1]},
           "note": "link_gbs_achieved divides by the whole chain's wall time (CPU components are host loops "
                   "over 1 GiB, run as stream-ordered host functions; uploads / downloads on side streams); "
                   "link_gbs_during_copies by the copies' own device time (summed, so overlapping copies count twice)",
           "config": {"workload": "C5: 4 x 1 GiB float32 vectors, seeded chain of CPU/GPU components",
                      "vector_bytes": n * 4, "calls": args.container_calls}}
    rt.close()
    # the same chain with coherence only (component=None: no CPU loop or GPU kernel), so the
    # wall time is the runtime's own: its copies on the two side streams, ordered per vector
    rt = Runtime(ctx)
    rt.set_async(True)
    vecs = [rt.vector(n) for _ in range(4)]
    rng = np.random.default_rng(5)
    t0 = time.perf_counter()
    for _ in range(args.container_calls):
        k = int(rng.integers(1, 4))
        idx = rng.choice(4, size=k, replace=False)
        site = "gpu" if rng.random() < 0.5 else "cpu"
        rt.call(site, [(vecs[i], ["R", "W", "RW"][int(rng.integers(0, 3))]) for i in idx], component=None)
    rt.sync()
    dt2 = time.perf_counter() - t0
    st2 = rt.stats()
    moved2 = st2["h2d_bytes"] + st2["d2h_bytes"]
    out["coherence_only"] = {"match": moved2 == moved and int(rt.predicted()["transfer_bytes"]) == moved2,
                             "bytes_moved": moved2, "wall_s": dt2, "link_gbs_achieved": moved2 / dt2 / 1e9,
                             "note": "same seeded chain, components omitted: the runtime's copy schedule alone"}
    rt.close()
    out["views"] = run_container_views(args, ctx)
    return out


def run_container_views(args, ctx):
    """C5 with pvector views: one mother vector of 2^24 float32 cells, 8 overlapping views,
    a seeded chain of component calls on them (element bodies, closure shadows);
    every transfer range is one cudaMemcpyAsync.  Bytes and copies must equal the element
    evaluator's prediction for the same program (and the stuck call, if any)."""
    from paper_1910_11110_b200 import CohError
    from paper_1910_11110_b200.container import Runtime
    from paper_1910_11110_b200.elem import Program, elem_eval

    # element bodies cost one step per cell and the calculus' fuel is an int32: 2^24
    # cells (64 MiB) x 64 calls stays inside it, so the run completes (status 0 below)
    n = 1 << min(24, args.container_log2_floats)
    prog = Program.generate(21, 0, n, 8, args.container_calls, 16, fuel=(1 << 31) - 1)
    pred = elem_eval(ctx, [prog], want_planes=False, runs_cap=1 << 16)["results"][0]
    rt = Runtime(ctx)
    buf = rt.buffer(n, 4)
    for lo, hi in zip(prog.view_lo, prog.view_hi):
        buf.view(int(lo), int(hi))
    stuck_at = None
    t0 = time.perf_counter()
    for c in range(prog.n_calls):
        try:
            buf.call(prog.calls[c])
        except CohError:
            stuck_at = c
            break
    rt.sync()
    dt = time.perf_counter() - t0
    st = rt.stats()
    moved = st["h2d_bytes"] + st["d2h_bytes"]
    copies = st["h2d_copies"] + st["d2h_copies"]
    rt.close()
    return {"metric": "view chain: bytes moved == evaluator prediction",
            "match": moved == 4 * int(pred.transfer_cells) and copies == int(pred.n_runs) and
            (stuck_at == int(pred.stuck_call) if pred.status == 1 else stuck_at is None),
            "bytes_moved": moved, "bytes_predicted": 4 * int(pred.transfer_cells), "copies": copies,
            "runs_predicted": int(pred.n_runs), "calls_done": int(st["calls"]), "stuck_call": stuck_at,
            "evaluator_status": int(pred.status),
            "vpu_whole_view_bytes": 4 * int(pred.vpu_cells), "wall_s": dt, "copy_ms": st["copy_ms"],
            "link_gbs_during_copies": moved / (st["copy_ms"] / 1e3) / 1e9 if st["copy_ms"] else None,
            "config": {"workload": "C5 views: a 64 MiB float32 mother vector, 8 overlapping views",
                       "cells": n, "calls": prog.n_calls}}


def run_sweep(args, ctx):
    """the acceptance corpus (gen_well_declared programs) swept over
    every schedule of <= 6 opaque decisions, one GPU thread per run; the reference does
    the same sweep single-threaded (criterion 4: 10000 seeds = 85335 runs in ~4.5 s)."""
    from paper_1910_11110_b200.sweep import sweep

    t0 = time.perf_counter()
    _, st = sweep(ctx, 0, args.sweep_seeds, 6, 10000)
    wall = time.perf_counter() - t0
    return {"metric": "acceptance-sweep runs/s", "seeds": args.sweep_seeds, "runs": st["runs"],
            "done": st["done"], "stuck": st["stuck"], "fuel_exhausted": st["fuel_exhausted"],
            "runs_with_violation": st["runs_with_violation"], "device_ms": st["device_ms"],
            "device_runs_per_s": st["nodes"] / (st["device_ms"] / 1e3) if st["device_ms"] else None,
            "wall_s": wall, "wall_runs_per_s": st["runs"] / wall,
            "note": "wall includes host program generation, bytecode compile and frontier management"}


def run_checker(args):
    """the static checker batched over program texts on the host
    threads (coh_cli_batch "check": parse, closure-free check, notes), gen_well_declared
    programs; the reference's own checker (ref_cli "check", one thread) on a sample."""
    from paper_1910_11110_b200.cli import run_cli_batch
    from paper_1910_11110_b200.sweep import gen_program_text

    srcs = [gen_program_text(s) for s in range(args.checker_programs)]
    run_cli_batch("check", srcs[:256])  # warm
    t0 = time.perf_counter()
    res = run_cli_batch("check", srcs)
    dt = time.perf_counter() - t0
    out = {"metric": "batched static checker programs/s (host threads)", "programs": len(srcs),
           "value": len(srcs) / dt, "unit": "programs/s", "threads": os.cpu_count(), "wall_s": dt,
           "with_diagnostics": sum(1 for r in res if r[2] != 0)}
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        import oracle_ffi as o
        if o.have_ref():
            from make_golden_cli import ref_fn
            ref_fn()  # registers ref_cli's signature
            R = o.reference()
            k = min(2000, len(srcs))
            cap = 1 << 16
            ob, eb, code = ctypes.create_string_buffer(cap), ctypes.create_string_buffer(cap), ctypes.c_int()
            agree = True
            t0 = time.perf_counter()
            for i in range(k):
                R.ref_cli(b"check", srcs[i].encode(), 0, 0, 10000, b"", 0, ob, cap, eb, cap, ctypes.byref(code))
                agree = agree and (ob.value.decode(), eb.value.decode(), code.value) == res[i]
            out["cpu_reference"] = {"value": k / (time.perf_counter() - t0), "unit": "programs/s", "cores": 1,
                                    "kind": "reference", "sample": f"first {k} programs", "agree": agree}
    except Exception as ex:  # test infrastructure; its absence is not fatal here
        out["cpu_reference"] = {"error": f"{type(ex).__name__}: {ex}"}
    return out


def run_overlap(args, ctx):
    """the batched overlap registry + closure.  1M views over 4096
    buffers of 2^20 cells (lengths up to 2^12), 1M blocks of 1-4 view modes; registry
    build (CUB sort + max-hi tree) and closure timed with CUDA events on the stream; the
    reference's build_registry + infer_overlap_closure timed on the host for a sample."""
    import torch

    from paper_1910_11110_b200.overlap import Registry, gen_workload_fast

    nv, nb = args.overlap_views, args.overlap_blocks
    views, modes, off = gen_workload_fast(11, 4096, 1 << 20, nv, nb, 4, 1 << 12)
    s = torch.cuda.current_stream()
    d_views = torch.from_numpy(views.view(np.uint8).copy()).cuda()
    d_modes = torch.from_numpy(modes.view(np.uint8).copy()).cuda()
    d_off = torch.from_numpy(off.view(np.int32).copy()).cuda()
    stride = 64
    d_out = torch.empty(nb * stride * 8, dtype=torch.uint8, device="cuda")
    d_cnt = torch.empty(nb, dtype=torch.int32, device="cuda")
    d_st = torch.empty(nb, dtype=torch.int32, device="cuda")
    L = coh_lib()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    best_b = best_c = None
    for it in range(6):  # the first round is a warm-up (lazy module loading, pool growth)
        h = ctypes.c_void_p()
        e[0].record()
        rc = L.coh_registry_build(ctx._h, d_views.data_ptr(), nv, ctypes.byref(h), s.cuda_stream)
        e[1].record()
        assert rc == 0
        e[2].record()
        rc = L.coh_overlap_closure(ctx._h, h, d_modes.data_ptr(), d_off.data_ptr(), nb, d_out.data_ptr(), stride,
                                   d_cnt.data_ptr(), d_st.data_ptr(), s.cuda_stream)
        e[3].record()
        torch.cuda.synchronize()
        assert rc == 0
        L.coh_registry_destroy(h)
        tb, tc = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])
        if it == 0:
            continue
        best_b = tb if best_b is None else min(best_b, tb)
        best_c = tc if best_c is None else min(best_c, tc)
    st = d_st.cpu().numpy()
    cnt = d_cnt.cpu().numpy()
    out = {"metric": "overlap closure blocks/s", "views": nv, "blocks": nb, "modes": int(len(modes)),
           "registry_build_ms": best_b, "closure_ms": best_c, "blocks_per_s": nb / (best_c / 1e3),
           "closed": int((st == -1).sum()), "conflicts": int((st >= 0).sum()), "over_limit": int((st == -2).sum()),
           "inferred_modes": int((cnt[st == -1] - np.diff(off)[st == -1]).sum())}
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_ffi as o
        if o.have_ref():
            # The reference's Declarations add views with a linear duplicate-name scan, so
            # registering 1M views is quadratic: its baseline runs on 64 buffers of the same
            # density (16K views) and that workload's blocks, also checked against the GPU.
            sv, sm, so = gen_workload_fast(12, 64, 1 << 20, nv * 64 // 4096, 5000, 4, 1 << 12)
            R = o.reference()
            sb = len(so) - 1
            o_cnt, o_st = np.zeros(sb, np.uint32), np.zeros(sb, np.int32)
            o_out = np.zeros(sb * stride * 8, np.uint8)
            t0 = time.perf_counter()
            R.ref_overlap_closure(sv.ctypes.data, len(sv), 0, sm.ctypes.data, so.ctypes.data, 0, o_out.ctypes.data,
                                  stride, o_cnt.ctypes.data, o_st.ctypes.data)
            t_build = time.perf_counter() - t0
            t0 = time.perf_counter()
            R.ref_overlap_closure(sv.ctypes.data, len(sv), 0, sm.ctypes.data, so.ctypes.data, sb, o_out.ctypes.data,
                                  stride, o_cnt.ctypes.data, o_st.ctypes.data)
            t_all = time.perf_counter() - t0
            reg = Registry(ctx, sv)
            _, g_cnt, g_st = reg.closure(sm, so, stride=stride)
            reg.close()
            out["cpu_reference"] = {
                "blocks_per_s": sb / max(1e-9, t_all - t_build), "sample": f"{len(sv)} views on 64 buffers, {sb} blocks",
                "build_registry_s": t_build, "cores": 1, "kind": "reference",
                "agree_with_gpu": bool(np.array_equal(g_st, o_st) and np.array_equal(g_cnt[g_st == -1], o_cnt[o_st == -1]))}
    except Exception as ex:  # the reference .so is test infrastructure; its absence is not fatal here
        out["cpu_reference"] = {"error": f"{type(ex).__name__}: {ex}"}
    return out


def run_c4(args, ctx, rank, world, allreduce):
    """BASELINE config 4: 64M traces (C2 format) split over the ranks as contiguous id
    ranges (strong scaling), each shard generated on its own device; device time of the
    evaluation (max over ranks), the NCCL allreduce of the counters, and an order-free
    checksum of every per-trace result (sum over ranks), equal for any rank count."""
    import torch
    import torch.distributed as dist

    import paper_1910_11110_b200 as coh
    from paper_1910_11110_b200 import shard

    total = args.c4_traces
    first, cnt = shard.split_range(rank, world, total)
    s = torch.cuda.current_stream()
    d_rec = torch.empty(coh.records_elems(cnt, N_CALLS), dtype=torch.int16, device="cuda")
    d_res = torch.empty(cnt * 64, dtype=torch.uint8, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    ctx.gen_records(SEED, first, cnt, N_CALLS, N_ARRAYS, ADV, d_rec, s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(s)
        ctx.eval_traces_counted(d_rec, cnt, N_CALLS, N_ARRAYS, FUEL, d_res, d_cnt, None, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    chk = shard.results_checksum(d_res)
    t = torch.tensor([best], dtype=torch.float64, device="cuda")
    c = torch.tensor([chk - (1 << 64) if chk >= 1 << 63 else chk], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        allreduce(d_cnt)
        torch.cuda.synchronize()
        dist.all_reduce(c)
    counters = d_cnt.cpu().numpy().view(np.uint64)[:11]
    ms = float(t.item())
    calls = int(counters[8] + counters[0] + counters[1] + counters[3])
    del d_rec, d_res
    torch.cuda.empty_cache()
    return {"metric": "C4: 64M traces split over the ranks (strong scaling), calls/s", "traces": total,
            "traces_per_rank": cnt, "value": calls / (ms / 1e3), "unit": "calls/s", "ms": ms, "scaling": "strong",
            "checksum": f"{int(c.item()) & ((1 << 64) - 1):016x}",
            "counters": {n: int(v) for n, v in zip(coh.COUNTER_NAMES, counters)},
            "note": "device time of one evaluation (best of 3, max over ranks); records generated on each device"}


def run_blocks(args, ctx):
    """Multi-mode blocks (COH_BATCH_BLOCKS, k_trace_blocks): the C2 shape (1M traces x 256
    calls x 64 arrays, adv 1/1024) with ~30% of the calls continuing their predecessor's
    DeclBlock (coh_gen_records_blocks, device-generated); device time of one evaluation
    (best of 3, CUDA events).  Throughput in records (calls) per second."""
    import torch

    import paper_1910_11110_b200 as coh

    nt, nc, na, cont = args.blocks_traces, N_CALLS, N_ARRAYS, 300
    s = torch.cuda.current_stream()
    d_rec = torch.empty(coh.records_elems(nt, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records_blocks(SEED, 0, nt, nc, na, ADV, cont, d_rec, s.cuda_stream)
    d_res = torch.empty(nt * 64, dtype=torch.uint8, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(4):
        e0.record(s)
        ctx.eval_traces_counted(d_rec, nt, nc, na, FUEL, d_res, d_cnt, None, stream=s.cuda_stream,
                                flags=coh.BATCH_BLOCKS)
        e1.record(s)
        torch.cuda.synchronize()
        best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
    cnt = d_cnt.cpu().numpy().view(np.uint64)
    cont_frac = float((d_rec[: 8 * nt].view(torch.int16) & 1).float().mean().item())
    del d_rec, d_res
    return {"metric": "multi-mode blocks: records/s (COH_BATCH_BLOCKS)", "traces": nt, "calls": nc, "arrays": na,
            "cont_fraction": cont_frac, "ms": best, "value": nt * nc / (best / 1e3), "unit": "records/s",
            "blocks_completed": int(cnt[8]), "stuck_traces": int(cnt[0]), "unsafe_traces": int(cnt[10])}


def run_c1(ctx):
    """BASELINE config 1: one trace of 1000 random calls on one array (seed 0, default
    mix), the latency case.  gpu_us: the evaluation as a CUDA graph replayed between two
    events (device-side latency: graph launch + the kernel, no Python in the window);
    api_us: the same through the Python API call (host dispatch included).  Best of 50.
    One trace on one array takes the block-scan path (k_trace_scan: the calls spread over
    a block and combined by an associative scan of per-call state maps).  cpu_us: the
    reference's run_annotated on the same records (host, best of 5)."""
    import torch

    import paper_1910_11110_b200 as coh

    recs = coh.gen_records_host(0, 0, 1, 1000, 1, ADV)
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.from_numpy(recs.view(np.int16).copy()).cuda()
    d_res = torch.empty(64, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def best_of(fn, k=20):
        best = None
        for _ in range(k):
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e3
            best = t if best is None else min(best, t)
        return best

    api = best_of(lambda: ctx.eval_traces(d_rec, 1, 1000, 1, FUEL, d_res, None, stream=s), 50)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.eval_traces(d_rec, 1, 1000, 1, FUEL, d_res, None, stream=torch.cuda.current_stream().cuda_stream)
    for _ in range(10):  # warm the graph and the clocks
        g.replay()
    torch.cuda.synchronize()
    dev = best_of(g.replay, 50)
    want = torch.empty_like(d_res)
    ctx.eval_traces(d_rec, 1, 1000, 1, FUEL, want, None, stream=s)
    torch.cuda.synchronize()
    assert torch.equal(want, d_res)
    kind, fn = cpu_eval_fn()
    ref = None
    for _ in range(5):
        t0 = time.perf_counter()
        fn(recs, 1, 1)
        t = (time.perf_counter() - t0) * 1e6
        ref = t if ref is None else min(ref, t)
    return {"metric": "C1 latency: one trace of 1000 calls on one array", "gpu_us": dev, "api_us": api,
            "cpu_us": ref, "cpu_kind": kind,
            "note": "block-scan path (one block, calls combined by an associative scan of state maps) vs one CPU thread"}


def coh_lib():
    import paper_1910_11110_b200 as coh

    return coh.lib()


# ---------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_1910_11110_b200 as coh

    # one rank per GPU over NCCL.  COH_BENCH_BACKEND=gloo runs the same multi-rank flow
    # with several ranks sharing GPUs (device = local rank mod device count): a plumbing
    # check on a one-GPU box, never a scaling number.
    backend = os.environ.get("COH_BENCH_BACKEND", "nccl")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if backend == "nccl" and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, found {torch.cuda.device_count()}")
    dev = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    ctx = coh.Context(dev)
    stream = torch.cuda.Stream()
    s = stream.cuda_stream
    from paper_1910_11110_b200 import shard

    # The data-path exchange (the counter allreduce) goes through the library's own NCCL
    # communicator (coh_comm_allreduce_counters); torch.distributed only carries the
    # unique id, the barriers and the max-over-ranks timing.  With COH_BENCH_BACKEND=gloo
    # (ranks sharing one GPU, a plumbing check) NCCL cannot run and torch/gloo sums instead.
    comm = None
    if world > 1 and backend == "nccl":
        box = [coh.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm = coh.Comm.init_rank(ctx, box[0], world, rank)

    def allreduce(d_counters):
        if comm is not None:
            comm.allreduce_counters(d_counters, s)
        else:
            with torch.cuda.stream(stream):
                shard.allreduce_counters(d_counters)

    trace0, N = shard.shard_range(rank, world, args.traces)  # contiguous trace ids, generated on-device
    with torch.cuda.stream(stream):
        d_rec = torch.empty(coh.records_elems(N, N_CALLS), dtype=torch.int16, device="cuda")
        # outputs double-buffered: consecutive steps are launched with COH_BATCH_OVERLAP (a
        # step may begin on the SMs its predecessor's last blocks free), which requires that
        # they do not share outputs
        res2 = [torch.empty(N * 64, dtype=torch.uint8, device="cuda") for _ in range(2)]
        bnd2 = [torch.empty(coh.boundary_words(N_CALLS) * N, dtype=torch.int32, device="cuda") for _ in range(2)]
        cnt2 = [torch.zeros(16, dtype=torch.int64, device="cuda") for _ in range(2)]
    ctx.gen_records(SEED, trace0, N, N_CALLS, N_ARRAYS, ADV, d_rec, s)
    stream.synchronize()

    def step(k, flags=coh.BATCH_OVERLAP, ev0=None, ev1=None):
        if ev0 is not None:
            ev0.record(stream)
        # trace_eval with the counter reduction fused into the kernel epilogue
        ctx.eval_traces_counted(d_rec, N, N_CALLS, N_ARRAYS, FUEL, res2[k & 1], cnt2[k & 1], bnd2[k & 1], stream=s,
                                flags=flags)
        if ev1 is not None:
            ev1.record(stream)
        if world > 1:
            allreduce(cnt2[k & 1])  # the only exchange; exact integer sums

    clocks = ClockSampler(dev)
    clocks.start()
    for k in range(max(3, args.warmup)):
        step(k)
    stream.synchronize()
    counters = cnt2[0].cpu().numpy().astype(np.uint64)  # whole-job counters of one step
    assert np.array_equal(counters, cnt2[1].cpu().numpy().astype(np.uint64))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count
    t_start.record(stream)
    for k in range(args.steps):
        step(k)
    t_end.record(stream)
    stream.synchronize()
    launches = ctx.launch_count - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end)
    ms_local = ms  # this rank's timed region: args.steps launches of k_trace_eval, back to back
    # one launch alone (events on both sides, no overlap), for the kernel's roofline
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for k in range(10):
        step(k, 0, *kev[k])
    stream.synchronize()
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    calls_per_step = int(counters[8] + counters[0] + counters[1] + counters[3])  # all ranks
    value = calls_per_step * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (trace_eval) on this rank: algorithmic bytes per
    # launch = 2 B per evaluated call (records) + 64 B result + 4 B per boundary word
    local_calls = calls_per_step // world
    alg_bytes = 2 * local_calls + N * (64 + 4 * coh.boundary_words(N_CALLS))
    k_ms_iso = statistics.mean(kern_ms)
    # the kernel's average launch duration over the timed region (one launch per step; with
    # COH_BATCH_OVERLAP a launch's tail overlaps the next one's start)
    k_ms = ms_local / args.steps
    peak, peak_src = peaks()
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    achieved_iso = alg_bytes / (k_ms_iso / 1e3) / 1e9
    traffic, traffic_traces = ncu_traffic()
    if traffic is not None and traffic_traces:
        traffic = traffic * N / traffic_traces

    # end-to-end through the public C-ABI host entry point (pinned host buffers,
    # H2D of the step's records + D2H of results and boundary bitmaps inside the region)
    e2e = None
    if args.e2e_steps > 0:
        rec_elems = coh.records_elems(N, N_CALLS)
        L = coh.lib()
        import ctypes as C

        # the records cross the link in the 12-bit packed form (COH_BATCH_PACKED12: 12 B per
        # 8 calls), unpacked on the device per pipeline slice
        pk_bytes = rec_elems // 8 * 12
        p_rec = L.coh_host_alloc(pk_bytes)
        p_res = L.coh_host_alloc(N * 64)
        p_bnd = L.coh_host_alloc(coh.boundary_words(N_CALLS) * N * 4)
        h_rec = np.ctypeslib.as_array((C.c_uint8 * pk_bytes).from_address(p_rec))
        h_res = np.ctypeslib.as_array((C.c_uint8 * (N * 64)).from_address(p_res)).view(coh.RESULT_DTYPE)
        h_bnd = np.ctypeslib.as_array((C.c_uint32 * (coh.boundary_words(N_CALLS) * N)).from_address(p_bnd))
        coh.pack_records12(d_rec.cpu().numpy().view(np.uint16), N, N_CALLS, out=h_rec)
        ctx.eval_traces_host(h_rec, N, N_CALLS, N_ARRAYS, FUEL, results=h_res, boundary=h_bnd,
                             flags=coh.BATCH_PACKED12)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ctx.eval_traces_host(h_rec, N, N_CALLS, N_ARRAYS, FUEL, results=h_res, boundary=h_bnd,
                                 flags=coh.BATCH_PACKED12)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        # e2e results equal the device-resident results
        assert np.array_equal(h_res.view(np.uint8), res2[0].cpu().numpy()), "host entry != device entry"
        e2e = {"value": calls_per_step * args.e2e_steps / dt, "unit": "calls/s",
               "h2d_bytes_per_step": pk_bytes, "d2h_bytes_per_step": N * 64 + coh.boundary_words(N_CALLS) * N * 4,
               "ms_per_step": 1e3 * dt / args.e2e_steps,
               "records": "COH_BATCH_PACKED12 (12 bits per call on the link, unpacked on the device)"}
        for p in (p_rec, p_res, p_bnd):
            L.coh_host_free(p)
    bitmap = run_bitmap(args, ctx, rank, world) if args.bitmap_buffers > 0 else None
    if bitmap is not None and rank == 0:
        bitmap["primitives"] = run_bitmap_primitives(args, ctx)
    clocks.stop()
    sweep_info = run_sweep(args, ctx) if (args.sweep_seeds > 0 and rank == 0) else None
    c1 = run_c1(ctx) if rank == 0 else None
    c4 = run_c4(args, ctx, rank, world, allreduce) if args.c4_traces > 0 else None
    overlap = run_overlap(args, ctx) if (args.overlap_views > 0 and rank == 0) else None
    checker = run_checker(args) if (args.checker_programs > 0 and rank == 0) else None
    blocks = run_blocks(args, ctx) if (args.blocks_traces > 0 and rank == 0) else None
    container = None
    if args.container_log2_floats > 0 and rank == 0:
        try:
            container = run_container(args, ctx)
        except Exception as e:  # keep the contract line even if the host lacks 8 GiB of pinned memory
            container = {"error": f"{type(e).__name__}: {e}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.cpu_seconds, os.cpu_count() or 1)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "calls/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u16",
            "data": "synthetic (counter-based splitmix64 call records generated in HBM, seed 1)",
            "config": bench_config(world, N),
            "transitions_per_s": float(counters[4]) * args.steps / (ms / 1e3),
            "counters_per_step": {n: int(v) for n, v in zip(coh.COUNTER_NAMES, counters[:11])},
            "roofline": {"bound": "hbm", "kernel": "k_trace_eval", "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes, "kernel_ms": k_ms,
                         "kernel_ms_basis": "timed region / launches (one k_trace_eval per step)",
                         "note": "bound in practice by the L1 data pipe (shared-memory wavefronts) together with "
                                 "instruction issue: see `l1_data_pipe`, `issue` and profiles/; `isolated_launch` = "
                                 "the same for one launch with nothing around it (its whole tail exposed)",
                         "isolated_launch": {
                             "kernel_ms": k_ms_iso, "achieved": achieved_iso, "frac": achieved_iso / peak,
                             "issue": ncu_issue(N, k_ms_iso, (clk or {}).get("sm_mhz"),
                                                torch.cuda.get_device_properties(dev).multi_processor_count),
                             "l1_data_pipe": ncu_l1_pipe(N, k_ms_iso, (clk or {}).get("sm_mhz"),
                                                         torch.cuda.get_device_properties(dev).multi_processor_count)},
                         "issue": ncu_issue(N, k_ms, (clk or {}).get("sm_mhz"), torch.cuda.get_device_properties(dev)
                                            .multi_processor_count),
                         "l1_data_pipe": ncu_l1_pipe(N, k_ms, (clk or {}).get("sm_mhz"),
                                                     torch.cuda.get_device_properties(dev).multi_processor_count)},
            "step_launch": "one coh_eval_traces_counted per step with COH_BATCH_OVERLAP: a step may start on the "
                           "SMs its predecessor's last blocks free (programmatic dependent launch); step outputs "
                           "double-buffered; roofline kernel_ms = the timed region per launch (isolated_launch: separate "
                           "non-overlapped launches)",
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
            "bitmap": bitmap, "container": container, "sweep": sweep_info, "c1": c1, "c4": c4, "overlap": overlap,
            "checker": checker, "blocks": blocks,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args):
    """`--gpus N` (N > 1) without a launcher: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1) and exit with its
    status; the driver's own torchrun launch sets WORLD_SIZE and never comes here."""
    import socket

    if os.environ.get("COH_BENCH_BACKEND", "nccl") == "nccl" and args.impl == "ours":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, found {have}")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
