"""C1 latency probe: one trace of 1000 calls on one array through eval_traces (for ncu)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11110_b200 as coh  # noqa: E402

ctx = coh.Context(0)
recs = coh.gen_records_host(0, 0, 1, 1000, 1, 64)
d_rec = torch.from_numpy(recs.view(np.int16).copy()).cuda()
d_res = torch.empty(64, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for path in ("scan", "thread"):
    os.environ["COH_TE_PATH"] = path
    best = None
    for _ in range(20):
        e0.record()
        ctx.eval_traces(d_rec, 1, 1000, 1, 10000, d_res, None, stream=s)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3
        best = t if best is None else min(best, t)
    print(path, "best us", round(best, 2))
