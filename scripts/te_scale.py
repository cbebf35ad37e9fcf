"""trace_eval device time vs batch size (fixed cost per launch = intercept of the fit)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11110_b200 as coh  # noqa: E402

ctx = coh.Context(0)
s = torch.cuda.current_stream().cuda_stream
nc, na = 256, 64
adv = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = 1 << 24
d_rec = torch.empty(coh.records_elems(N, nc), dtype=torch.int16, device="cuda")
d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
xs, ys = [], []
for n in (1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22, 1 << 23, 1 << 24):
    ctx.gen_records(1, 0, n, nc, na, adv, d_rec, s)
    ts = []
    for _ in range(12):
        e0.record()
        ctx.eval_traces_counted(d_rec, n, nc, na, 10000, d_res, d_cnt, None, stream=s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts[2:]))
    xs.append(n)
    ys.append(t)
    print(f"{n:9d} traces  {t * 1e3:9.1f} us   {t * 1e3 / (n / 2**20):7.1f} us per 1M")
b, a = np.polyfit(np.array(xs[2:]) / 2**20, ys[2:], 1)
print(f"fit: {b * 1e3:.1f} us per 1M traces + {a * 1e3:.1f} us fixed")
