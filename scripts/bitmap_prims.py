"""Run each bit-plane primitive once on the bench's C3-sized planes (for ncu captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1910_11110_b200 as coh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--buffers", type=int, default=256)
a = ap.parse_args()
ctx = coh.Context(0)
sys.argv = [sys.argv[0], "--bitmap-buffers", str(a.buffers)]
args = bench.parse()
print(bench.run_bitmap_primitives(args, ctx))
