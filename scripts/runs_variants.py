"""coh_bitmap_extract_zero_runs A/B timing over the bench's fragmentation sweep (256 planes x
2^24 cells, rho in {0, 2^-16, 2^-8, 1/2}, every run written): one subprocess per
(library, env) configuration, best of 6 device times per rho, a digest of the outputs so
variants can be checked against each other, and the HBM fraction of (m/8 + 8 B per run).

usage: python scripts/runs_variants.py [LIB[:ENV=V,...] ...]   (LIB 'default' = lib/libcohere_b200.so)
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
    from paper_1910_11110_b200._ffi import lib as coh_lib
    from paper_1910_11110_b200.bitmap import RANGE_DTYPE

    ctx = coh.Context(0)
    Lb = coh_lib()
    s = torch.cuda.current_stream().cuda_stream
    P, n = 256, 1 << 24
    words = n // 32
    rng = np.random.default_rng(3)
    ranges = np.zeros(P, RANGE_DTYPE)
    ranges["word_off"] = np.arange(P) * words
    ranges["lo"] = rng.integers(0, n // 5, P)
    ranges["hi"] = n - 1 - rng.integers(0, n // 5, P)
    m = int((ranges["hi"].astype(np.int64) - ranges["lo"] + 1).sum())
    d_r = torch.from_numpy(ranges.view(np.uint8).copy()).cuda()
    roff = torch.empty(P + 1, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6549.1
    out = {}
    for name, ands in (("0", None), ("2^-16", 16), ("2^-8", 8), ("1/2", 1)):
        torch.manual_seed(7)
        plane = torch.zeros(P * words, dtype=torch.int32, device="cuda")
        if ands:
            plane.fill_(-1)
            for _ in range(ands):
                plane &= torch.randint(-(1 << 31), 1 << 31, (P * words,), dtype=torch.int32, device="cuda")
        cap = m // 3 + 16 if ands == 1 else 1 << 22
        rs = torch.empty(cap, dtype=torch.int32, device="cuda")
        re_ = torch.empty(cap, dtype=torch.int32, device="cuda")
        best = None
        for _ in range(6):
            e0.record()
            rc = Lb.coh_bitmap_extract_zero_runs(ctx._h, plane.data_ptr(), d_r.data_ptr(), P, rs.data_ptr(),
                                                 re_.data_ptr(), cap, roff.data_ptr(), s)
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        # 10 calls back to back (host launch work overlaps the previous call's kernels)
        e0.record()
        for _ in range(10):
            Lb.coh_bitmap_extract_zero_runs(ctx._h, plane.data_ptr(), d_r.data_ptr(), P, rs.data_ptr(),
                                            re_.data_ptr(), cap, roff.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        stream_ms = e0.elapsed_time(e1) / 10
        runs = int(roff[P].item())
        k = min(runs, cap)
        h = hashlib.sha256(rs[:k].cpu().numpy().tobytes() + re_[:k].cpu().numpy().tobytes() +
                           roff.cpu().numpy().tobytes()).hexdigest()[:12]
        gbs = (m / 8 + 8 * runs) / (best / 1e3) / 1e9
        out[name] = {"ms": round(best, 4), "stream_ms": round(stream_ms, 4), "runs": runs, "frac": round(gbs / peak, 3), "digest": h}
        del plane, rs, re_
    print(json.dumps(out))


def main(argv):
    for spec in argv or ["default"]:
        lib, _, envs = spec.partition(":")
        env = dict(os.environ)
        if lib != "default":
            env["COH_B200_LIB"] = os.path.join(ROOT, "paper_1910_11110_b200", "lib", "variants", lib)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-600:]})
        print(spec, line, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        main(sys.argv[1:])
