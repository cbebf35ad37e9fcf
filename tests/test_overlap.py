"""Batched overlap registry + closure against the reference's
OverlapRegistry::query (both backends) and infer_overlap_closure: committed fixtures made by
the reference (tests/golden/make_golden_overlap.py) and, where oracle/_ref is present, the
live reference on fresh workloads.  Bit-exact: same hits in name order, same closed mode
lists, the same view named by every OverlapInferenceError."""
import os

import numpy as np
import pytest

import oracle_ffi as o
from paper_1910_11110_b200.overlap import MODE_DTYPE, VIEW_DTYPE, Registry, gen_workload

HERE = os.path.dirname(os.path.abspath(__file__))
Z = np.load(os.path.join(HERE, "golden", "overlap.npz"))
NAMES = sorted({k.split(".")[0] for k in Z.files})


def case(name):
    g = {k.split(".")[1]: Z[k] for k in Z.files if k.startswith(name + ".")}
    g["views"] = g["views"].view(VIEW_DTYPE).reshape(-1)
    g["modes"] = g["modes"].view(MODE_DTYPE).reshape(-1)
    return g


def check_closure(got, want, off=None, stride=None):
    out, cnt, st = got
    w_out, w_cnt, w_st = want
    if off is not None:  # the documented per-block limits: -2 exactly where they are exceeded
        nm = np.diff(off).astype(np.int64)
        over = (w_st == -1) & ((w_cnt > stride) | (w_cnt - nm > 64))
        assert np.array_equal(st == -2, over)
        w_st = np.where(over, -2, w_st)
    assert np.array_equal(st, w_st)
    ok = st == -1
    assert np.array_equal(cnt[ok], w_cnt[ok])
    for b in np.nonzero(ok)[0]:
        assert out[b, : cnt[b]].tobytes() == w_out[b, : cnt[b]].tobytes(), b


def test_fixtures_cover_conflicts_and_shadows():
    seen_conflict = seen_shadow = 0
    for n in NAMES:
        g = case(n)
        seen_conflict += int((g["status"] >= 0).sum())
        seen_shadow += int((g["cnt"] > np.diff(g["off"])).sum())
    assert seen_conflict > 100 and seen_shadow > 1000


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not present")
def test_fixtures_match_live_reference():
    import sys
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden_overlap import ref_closure
    for n in NAMES:
        g = case(n)
        out, cnt, st = ref_closure(g["views"], g["modes"], g["off"])
        assert np.array_equal(st, g["status"]) and np.array_equal(cnt, g["cnt"])


@pytest.mark.gpu
def test_gpu_query_and_closure_match_fixtures(ctx):
    for n in NAMES:
        g = case(n)
        reg = Registry(ctx, g["views"])
        hits, hcnt = reg.query(np.arange(len(g["views"]), dtype=np.uint32), stride=g["hits"].shape[1])
        assert np.array_equal(hcnt, g["hcnt"]), n
        for q in range(len(hcnt)):
            k = min(int(hcnt[q]), hits.shape[1])
            assert np.array_equal(hits[q, :k], g["hits"][q, :k]), (n, q)
        check_closure(reg.closure(g["modes"], g["off"], stride=g["out"].shape[1]), (g["out"], g["cnt"], g["status"]))
        reg.close()


@pytest.mark.gpu
@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not present")
def test_gpu_closure_live_reference_fresh(ctx):
    import sys
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden_overlap import ref_closure_stride
    for seed, shape in enumerate([(8, 256, 600, 3000, 5, 32), (64, 1 << 16, 20000, 20000, 4, 512), (1, 12, 30, 2000, 8, 4)]):
        nbuf, blen, nv, nb, mpb, mvl = shape
        views, modes, off = gen_workload(100 + seed, nbuf, blen, nv, nb, mpb, n_scalars=4, max_view_len=mvl,
                                         p_same_site=0.8)
        reg = Registry(ctx, views)
        check_closure(reg.closure(modes, off, stride=64), ref_closure_stride(views, modes, off, 64), off, 64)
        reg.close()


@pytest.mark.gpu
def test_gpu_limits_and_empty(ctx):
    views = np.zeros(70, VIEW_DTYPE)
    views["lo"], views["hi"], views["name_rank"] = 0, 9, np.arange(70)
    reg = Registry(ctx, views)
    modes = np.zeros(1, MODE_DTYPE)
    modes[0] = (0, 1, 0, 1, 0)  # W on a view overlapping 69 others: more than 64 inferred
    out, cnt, st = reg.closure(modes, np.array([0, 1], np.uint32), stride=128)
    assert st.tolist() == [-2]
    out, cnt, st = reg.closure(modes[:0], np.array([0, 0], np.uint32))
    assert st.tolist() == [-1] and cnt.tolist() == [0]
    reg.close()
    empty = Registry(ctx, views[:0])
    empty.close()
