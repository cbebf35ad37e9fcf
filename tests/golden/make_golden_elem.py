"""Element-program golden fixtures from the REFERENCE (oracle/_ref, the reference headers
compiled in place): overlap closure, whole-view syncs with their transfer-range deltas,
element bodies, boundary checks.  Run in the build container:
    make -C oracle && python tests/golden/make_golden_elem.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_ffi as o  # noqa: E402
from paper_1910_11110_b200.elem import ElemCall, Program  # noqa: E402

# (prog_id, n_cells, n_views, n_calls, adv_per1024, fuel)
CASES = []
for pid in range(48):
    rng = np.random.default_rng(1000 + pid)
    CASES.append((pid, int(rng.choice([32, 33, 100, 257, 1024, 4096, 16384])), int(rng.integers(1, 9)),
                  int(rng.integers(1, 12)), int(rng.choice([0, 64, 400, 1024])),
                  int(rng.choice([1 << 30, 1 << 30, 60, 700, 20000]))))


def main():
    assert o.have_ref()
    out = {}
    for pid, n, V, K, adv, fuel in CASES:
        p = Program.generate(11, pid, n, V, K, adv, fuel)
        rc, r, L, R, va, b, runs = o.elem_run("ref", p)
        assert rc == 0, (pid, rc)
        key = f"p{pid}"
        out[key + ".params"] = np.array([pid, n, V, K, adv, fuel], np.int64)
        out[key + ".views"] = np.stack([p.view_lo, p.view_hi])
        out[key + ".calls"] = np.frombuffer(bytes(p.calls), np.uint8)[: 32 * K].copy()
        out[key + ".result"] = np.array(r.as_tuple(), np.uint64)
        out[key + ".planes"] = np.stack([L, R])
        out[key + ".view_abs"] = va
        out[key + ".boundary"] = b
        out[key + ".runs"] = runs
    np.savez_compressed(os.path.join(HERE, "elem.npz"), **out)
    print("wrote", len(CASES), "element programs")


if __name__ == "__main__":
    main()
