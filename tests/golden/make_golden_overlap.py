"""Regenerate the overlap registry / closure fixtures from the REFERENCE itself
(oracle/_ref ref_overlap.cpp: OverlapRegistry + infer_overlap_closure of overlap.hpp on the
same records).  Run where /root/reference exists:

    make -C oracle && python tests/golden/make_golden_overlap.py

Output (committed): overlap.npz, per case: views, modes, block offsets, the reference's
closure (modes, counts, status) and query results (hits, counts) for every view.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]

import oracle_ffi as o  # noqa: E402
from paper_1910_11110_b200.overlap import gen_workload  # noqa: E402

# name: (seed, n_buffers, buf_len, n_views, n_blocks, modes_per_block, max_view_len, p_same_site)
CASES = {
    "tiny": (1, 1, 10, 4, 64, 3, None, 0.9),
    "few_long": (2, 3, 64, 24, 500, 4, None, 0.85),
    "many_short": (3, 16, 4096, 3000, 2000, 4, 64, 0.9),
    "conflicts": (4, 2, 32, 40, 800, 6, 16, 0.5),
    "single_cell": (5, 4, 8, 40, 400, 5, 1, 0.8),
}
STRIDE_Q, STRIDE_C = 64, 32


def ref_closure_stride(views, modes, off, stride):
    global STRIDE_C
    old, STRIDE_C = STRIDE_C, stride
    try:
        return ref_closure(views, modes, off)
    finally:
        STRIDE_C = old


def ref_closure(views, modes, off):
    nb = len(off) - 1
    out = np.zeros((nb, STRIDE_C), np.dtype([("var", "<u4"), ("kind", "u1"), ("site", "u1"), ("flags", "u1"), ("pad", "u1")]))
    cnt = np.zeros(nb, np.uint32)
    st = np.zeros(nb, np.int32)
    o.reference().ref_overlap_closure(views.ctypes.data, len(views), 4, modes.ctypes.data, off.ctypes.data, nb,
                                      out.ctypes.data, STRIDE_C, cnt.ctypes.data, st.ctypes.data)
    return out, cnt, st


def ref_query(views, backend):
    n = len(views)
    probes = np.arange(n, dtype=np.uint32)
    hits = np.zeros((n, STRIDE_Q), np.uint32)
    cnt = np.zeros(n, np.uint32)
    o.reference().ref_registry_query(views.ctypes.data, n, probes.ctypes.data, n, hits.ctypes.data, STRIDE_Q,
                                     cnt.ctypes.data, backend)
    return hits, cnt


def main():
    assert o.have_ref()
    arrays = {}
    for name, (seed, nbuf, blen, nv, nb, mpb, mvl, pss) in CASES.items():
        views, modes, off = gen_workload(seed, nbuf, blen, nv, nb, mpb, 4, mvl, pss)
        out, cnt, st = ref_closure(views, modes, off)
        hits, hcnt = ref_query(views, 0)
        hits2, hcnt2 = ref_query(views, 1)
        assert np.array_equal(hits, hits2) and np.array_equal(hcnt, hcnt2)  # both reference backends agree
        for k, v in dict(views=views, modes=modes, off=off, out=out, cnt=cnt, status=st, hits=hits, hcnt=hcnt).items():
            arrays[f"{name}.{k}"] = v
        print(name, "blocks", nb, "closed", int((st == -1).sum()), "conflicts", int((st >= 0).sum()),
              "max hits", int(hcnt.max()), "mean shadows", float((cnt[st == -1] - np.diff(off)[st == -1]).mean()))
    np.savez_compressed(os.path.join(HERE, "overlap.npz"), **arrays)


if __name__ == "__main__":
    main()
