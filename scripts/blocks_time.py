"""k_trace_blocks timing on the bench's multi-mode shape (1M traces x 256 calls x 64 arrays,
adv 1/1024, cont 300/1024): best of 5 device times, digest of results + counters."""
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11110_b200 as coh  # noqa: E402

ctx = coh.Context(0)
nt, nc, na = 1 << 20, 256, 64
s = torch.cuda.current_stream()
d_rec = torch.empty(coh.records_elems(nt, nc), dtype=torch.int16, device="cuda")
ctx.gen_records_blocks(1, 0, nt, nc, na, 1, 300, d_rec, s.cuda_stream)
d_res = torch.empty(nt * 64, dtype=torch.uint8, device="cuda")
d_bnd = torch.empty(coh.boundary_words(nc) * nt, dtype=torch.int32, device="cuda")
d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(6):
    e0.record(s)
    ctx.eval_traces_counted(d_rec, nt, nc, na, 10000, d_res, d_cnt, d_bnd, stream=s.cuda_stream, flags=coh.BATCH_BLOCKS)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
h = hashlib.sha256(d_res.cpu().numpy().tobytes() + d_bnd.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps({"ms_best": min(ts[1:]), "digest": h, "counters": d_cnt.cpu().tolist()[:11]}))
