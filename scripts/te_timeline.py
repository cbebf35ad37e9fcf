"""Per-block timeline of one k_trace_eval launch (debug build with COH_TE_TIMELINE)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11110_b200 as coh  # noqa: E402

ctx = coh.Context(0)
s = torch.cuda.current_stream().cuda_stream
nc, na, adv = 256, 64, 1
for N in (1 << 20, 1 << 22):
    d_rec = torch.empty(coh.records_elems(N, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records(1, 0, N, nc, na, adv, d_rec, s)
    d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.zeros(coh.boundary_words(nc) * N, dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        e0.record()
        ctx.eval_traces(d_rec, N, nc, na, 10000, d_res, d_bnd, stream=s)
        e1.record()
        torch.cuda.synchronize()
    tl = d_bnd.cpu().numpy().view(np.uint64)
    nb = 600
    tl = tl[: 3 * nb].reshape(nb, 3).astype(np.int64)
    tl = tl[tl[:, 0] > 0]
    t0 = tl[:, 0].min()
    st, su, en = (tl[:, 0] - t0) / 1e3, (tl[:, 1] - t0) / 1e3, (tl[:, 2] - t0) / 1e3
    print(f"N={N}: event {e0.elapsed_time(e1) * 1e3:.1f} us, blocks {len(tl)}")
    print(f"  start  min/med/max {st.min():.1f} {np.median(st):.1f} {st.max():.1f} us")
    print(f"  setup  dur med/max {np.median(su - st):.1f} {np.max(su - st):.1f} us")
    print(f"  end    min/med/max {en.min():.1f} {np.median(en):.1f} {en.max():.1f} us")
    print(f"  block duration min/med/max {np.min(en - st):.1f} {np.median(en - st):.1f} {np.max(en - st):.1f}")
