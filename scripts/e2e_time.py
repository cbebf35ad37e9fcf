"""End-to-end (host buffers) timing of the C2 step through coh_eval_traces_host with
COH_BATCH_PACKED12 records, as bench.py's e2e: median of 8 after one warm-up."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11110_b200 as coh  # noqa: E402

ctx = coh.Context(0)
N, NC, NA = 1 << 20, 256, 64
d_rec = torch.empty(coh.records_elems(N, NC), dtype=torch.int16, device="cuda")
ctx.gen_records(1, 0, N, NC, NA, 1, d_rec, torch.cuda.current_stream().cuda_stream)
L = coh.lib()
rec_elems = coh.records_elems(N, NC)
pk = rec_elems // 8 * 12
p_rec, p_res, p_bnd = L.coh_host_alloc(pk), L.coh_host_alloc(N * 64), L.coh_host_alloc(coh.boundary_words(NC) * N * 4)
h_rec = np.ctypeslib.as_array((C.c_uint8 * pk).from_address(p_rec))
h_res = np.ctypeslib.as_array((C.c_uint8 * (N * 64)).from_address(p_res)).view(coh.RESULT_DTYPE)
h_bnd = np.ctypeslib.as_array((C.c_uint32 * (coh.boundary_words(NC) * N)).from_address(p_bnd))
coh.pack_records12(d_rec.cpu().numpy().view(np.uint16), N, NC, out=h_rec)
ts = []
for i in range(9):
    t0 = time.perf_counter()
    ctx.eval_traces_host(h_rec, N, NC, NA, 10000, results=h_res, boundary=h_bnd, flags=coh.BATCH_PACKED12)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"slice": os.environ.get("COH_HOST_SLICE", "default"), "ms_median": 1e3 * float(np.median(ts[1:])),
                  "ms_min": 1e3 * min(ts[1:]), "calls_per_s": N * NC / float(np.median(ts[1:]))}))
