"""Zero-run extraction on 256 planes x 2^24 cells at one fragmentation (for ncu)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11110_b200 as coh  # noqa: E402
from paper_1910_11110_b200.bitmap import RANGE_DTYPE, zero_runs  # noqa: E402

ands = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = coh.Context(0)
P, n = 256, 1 << 24
words = n // 32
rng = np.random.default_rng(3)
ranges = np.zeros(P, RANGE_DTYPE)
ranges["word_off"] = np.arange(P) * words
ranges["lo"] = rng.integers(0, n // 5, P)
ranges["hi"] = n - 1 - rng.integers(0, n // 5, P)
plane = torch.full((P * words,), -1, dtype=torch.int32, device="cuda")
for _ in range(ands):
    plane &= torch.randint(-(1 << 31), 1 << 31, (P * words,), dtype=torch.int32, device="cuda")
# argv[2] == "full": room for every run (rho = 1/2 has a run every ~4 cells)
m = int((ranges["hi"].astype(np.int64) - ranges["lo"] + 1).sum())
cap = m // 3 + 16 if len(sys.argv) > 2 and sys.argv[2] == "full" else 1 << 26
for _ in range(2):
    off, st, en = zero_runs(ctx, plane, ranges, cap=cap)
print("runs", int(off[-1]))
