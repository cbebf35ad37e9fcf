"""Debug helper: run the golden trace batches through the device kernel and print the
fields of the first mismatching traces (GPU box)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1910_11110_b200 as coh  # noqa: E402
from test_trace_gpu import dev_eval, golden  # noqa: E402

ctx = coh.Context(0)
for name, recs, nt, nc, na, fuel, ab, want, want_b in golden():
    res, bnd = dev_eval(ctx, recs, nt, nc, na, fuel, ab)
    bad = np.nonzero((res.view(np.uint8).reshape(-1, 64) != want.view(np.uint8).reshape(-1, 64)).any(1))[0]
    bb = int((bnd != want_b).sum())
    print(f"{name}: {len(bad)} bad traces of {nt}, {bb} bad boundary words")
    for i in bad[:3]:
        for f in want.dtype.names:
            if not np.array_equal(res[i][f], want[i][f]):
                print(f"   trace {i} {f}: got {res[i][f]} want {want[i][f]}")
        r = recs.reshape(-1)
        calls = [int(r[((c // 8) * nt + i) * 8 + c % 8]) for c in range(min(nc, int(want[i]['stuck_call']) + 1))]
        print("   calls (array,type):", [((x >> 8) & 63, (x >> 2) & 63) for x in calls][-4:])
