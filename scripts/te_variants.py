"""k_trace_eval A/B timing on the C2 step (1M traces x 256 calls x 64 arrays, adv 1/1024):
one subprocess per (library, env) configuration, device time of the counted launch with
the boundary words written (the bench step), median of 30 after warm-up, plus a parity
check of results + boundary words against the default build's output.

usage: python scripts/te_variants.py [LIB[:ENV=V,...] ...]   (LIB 'default' = lib/libcohere_b200.so)
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    import numpy as np
    import torch

    sys.path.insert(0, ROOT)
    import paper_1910_11110_b200 as coh

    ctx = coh.Context(0)
    s = torch.cuda.current_stream().cuda_stream
    N, NC, NA = 1 << 20, 256, 64
    d_rec = torch.empty(coh.records_elems(N, NC), dtype=torch.int16, device="cuda")
    ctx.gen_records(1, 0, N, NC, NA, 1, d_rec, s)
    d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.empty(coh.boundary_words(NC) * N, dtype=torch.int32, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(40):
        e0.record()
        if os.environ.get("COH_TV_NOCOUNT"):
            ctx.eval_traces(d_rec, N, NC, NA, 10000, d_res, d_bnd, stream=s)
        else:
            ctx.eval_traces_counted(d_rec, N, NC, NA, 10000, d_res, d_cnt, d_bnd, stream=s)
        e1.record()
        torch.cuda.synchronize()
        if i >= 10:
            ts.append(e0.elapsed_time(e1) * 1e3)
    h = hashlib.sha256(d_res.cpu().numpy().tobytes() + d_bnd.cpu().numpy().tobytes()).hexdigest()[:16]
    # back-to-back stream of K launches (the bench's step loop), plain and COH_BATCH_OVERLAP
    # with double-buffered outputs
    res2 = [d_res, torch.empty_like(d_res)]
    bnd2 = [d_bnd, torch.empty_like(d_bnd)]
    cnt2 = [d_cnt, torch.zeros_like(d_cnt)]
    stream_us = {}
    for name, flags in (("plain", 0), ("overlap", coh.BATCH_OVERLAP)):
        for i in range(5):
            ctx.eval_traces_counted(d_rec, N, NC, NA, 10000, res2[i & 1], cnt2[i & 1], bnd2[i & 1], stream=s, flags=flags)
        torch.cuda.synchronize()
        K = 40
        e0.record()
        for i in range(K):
            ctx.eval_traces_counted(d_rec, N, NC, NA, 10000, res2[i & 1], cnt2[i & 1], bnd2[i & 1], stream=s, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        stream_us[name] = e0.elapsed_time(e1) * 1e3 / K
    h2 = hashlib.sha256(res2[1].cpu().numpy().tobytes() + bnd2[1].cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"us_median": float(np.median(ts)), "us_min": float(np.min(ts)), "digest": h,
                      "stream_us_per_launch": stream_us, "digest_overlap": h2,
                      "counters": d_cnt.cpu().tolist()[:11], "counters_overlap": cnt2[1].cpu().tolist()[:11]}))


def main(argv):
    out = []
    for spec in argv or ["default"]:
        lib, _, envs = spec.partition(":")
        env = dict(os.environ)
        if lib != "default":
            env["COH_B200_LIB"] = os.path.join(ROOT, "paper_1910_11110_b200", "lib", "variants", lib)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-400:]})
        d = json.loads(line)
        d["spec"] = spec
        out.append(d)
        print(json.dumps(d), flush=True)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        main(sys.argv[1:])
