"""GPU parity tests of the element-granular path (bit planes, whole-view syncs with
transfer-range extraction, element range effects, per-view boundary checks): bit-exact
against the reference's golden fixtures, the C oracle at up to 2^24 cells, and batch
invariance."""
import numpy as np
import pytest

import oracle_ffi as o
from paper_1910_11110_b200.elem import Program, elem_eval
from test_elem_oracle import golden_programs

pytestmark = pytest.mark.gpu


def compare(out, i, want, key, runs_cap=4096):
    r = out["results"][i]
    assert np.array_equal(np.array(r.as_tuple(), np.uint64), want["result"]), (key, r.as_tuple(), want["result"])
    pw = want["planes"].shape[1]
    assert np.array_equal(out["planes"][i][:, :pw], want["planes"]), key
    nv = len(want["view_abs"])
    assert np.array_equal(out["view_abs"][i][:nv], want["view_abs"]), key
    bw = len(want["boundary"])
    assert np.array_equal(out["boundary"][i][:bw], want["boundary"]), key
    m = min(int(r.n_runs), runs_cap)
    assert np.array_equal(out["runs"][i][:m], want["runs"][:m]), key


def test_golden_batch(ctx):
    items = list(golden_programs())
    out = elem_eval(ctx, [p for _, _, p, _ in items])
    for i, (key, params, p, want) in enumerate(items):
        compare(out, i, want, key)


def test_golden_one_by_one(ctx):
    for key, params, p, want in list(golden_programs())[:12]:
        compare(elem_eval(ctx, [p]), 0, want, key)


def oracle_want(p, runs_cap=1 << 16):
    rc, r, L, R, va, b, runs = o.elem_run("orc", p, runs_cap)
    assert rc in (0, -3)
    return {"result": np.array(r.as_tuple(), np.uint64), "planes": np.stack([L, R]), "view_abs": va,
            "boundary": b, "runs": runs}


@pytest.mark.parametrize("n_cells,n_progs,adv", [(1 << 16, 16, 64), (1 << 20, 8, 128), ((1 << 20) + 37, 4, 1024),
                                                 (1 << 24, 2, 64)])
def test_vs_oracle_large(ctx, n_cells, n_progs, adv):
    progs = [Program.generate(5, i, n_cells, 8, 12, adv) for i in range(n_progs)]
    out = elem_eval(ctx, progs, runs_cap=1 << 16)
    for i, p in enumerate(progs):
        compare(out, i, oracle_want(p), f"n={n_cells} prog={i}", runs_cap=1 << 16)


def test_fuel_limited_vs_oracle(ctx):
    progs = [Program.generate(6, i, 5000, 6, 10, 300, fuel=f) for i, f in enumerate([0, 1, 2, 3, 50, 777, 4999, 30000])]
    out = elem_eval(ctx, progs)
    for i, p in enumerate(progs):
        compare(out, i, oracle_want(p), f"fuel prog {i}")


def test_runs_capacity_overflow_counts_everything(ctx):
    p = Program.generate(8, 3, 1 << 16, 8, 16, 1024)
    full = elem_eval(ctx, [p], runs_cap=1 << 16)
    small = elem_eval(ctx, [p], runs_cap=4)
    assert small["results"][0].n_runs == full["results"][0].n_runs
    assert np.array_equal(small["runs"][0][:4], full["runs"][0][:4])


@pytest.mark.parametrize("frag_log2,cap", [(8, 5), (8, 333), (1, 7), (1, 4099)])
def test_runs_capacity_fragmented(ctx, frag_log2, cap):
    """Truncation at runs_cap inside sparse (rho 2^-8) and dense (rho 1/2) steps: the
    written prefix equals the uncapped output, the run count is the full count."""
    p = Program.generate(9, 2, 1 << 18, 8, 8, 64, frag_log2=frag_log2)
    full = elem_eval(ctx, [p], runs_cap=1 << 20)
    small = elem_eval(ctx, [p], runs_cap=cap)
    n = int(full["results"][0].n_runs)
    assert n > cap and int(small["results"][0].n_runs) == n
    assert np.array_equal(small["runs"][0][:cap], full["runs"][0][:cap])


def test_malformed_program_is_construction_error(ctx):
    import paper_1910_11110_b200 as coh

    bad = Program(100, [10], [200], [(0, 0, 0, [])])  # view outside its buffer
    with pytest.raises(coh.CohError) as e:
        elem_eval(ctx, [bad])
    assert e.value.code == 1


def test_reference_sample_element_gpu(ctx):
    # proj/samples/element_gpu.coh + proj/tests/golden/element_gpu.run.txt:
    #   buffer b[10]; view x = b[0:9]; GRW(x) { gw x[3]; }
    #   -> done, 5 steps, b[3] (I,V), every other cell (V,V), x^ (I,V)
    p = Program(10, [0], [9], [(0, 2, 1, [(3, 1, 3, 3)])])
    out = elem_eval(ctx, [p])
    r = out["results"][0]
    assert r.status == 0 and r.steps == 5 and r.transfers == 1
    L, R = out["planes"][0][0][0], out["planes"][0][1][0]
    cells = [("V" if (L >> i) & 1 else "I") + ("V" if (R >> i) & 1 else "I") for i in range(10)]
    assert cells == ["VV"] * 3 + ["IV"] + ["VV"] * 6
    assert out["view_abs"][0][0] == 2  # (I,V)
    assert list(map(list, out["runs"][0][:1])) == [[0, 9]]  # the push copies the whole view once


def test_two_chain_batch_vs_oracle(ctx):
    """A batch of >= 64 programs runs as two concurrent stage chains (each half its own
    plan, with different stage counts): every output still equals the oracle's, and the
    reference goldens repeated past the threshold still match."""
    progs = [Program.generate(9, i, (1 << 14) + 97 * i, 8, 6 + (i % 11), 64 + 8 * (i % 5)) for i in range(96)]
    out = elem_eval(ctx, progs, runs_cap=1 << 14)
    for i, p in enumerate(progs):
        compare(out, i, oracle_want(p, 1 << 14), f"prog {i}", runs_cap=1 << 14)
    items = list(golden_programs()) * 2
    out = elem_eval(ctx, [p for _, _, p, _ in items])
    for i, (key, params, p, want) in enumerate(items):
        compare(out, i, want, key)


def test_too_many_calls_is_construction_error(ctx):
    """ElemOp carries a 16-bit call index: programs over COH_ELEM_MAX_CALLS calls are
    refused with ConstructionError instead of wrapping the boundary/stuck indices."""
    from paper_1910_11110_b200.elem import Program, elem_eval
    from paper_1910_11110_b200 import CohError
    p = Program.generate(5, 0, 1024, 2, 65536, 0)
    with pytest.raises(CohError) as e:
        elem_eval(ctx, [p], want_planes=False)
    assert e.value.code == 1
    ok = Program.generate(5, 0, 1024, 2, 65535, 0, fuel=(1 << 31) - 1)
    elem_eval(ctx, [ok], want_planes=False)


def _want(which, p, runs_cap):
    rc, r, L, R, va, b, runs = o.elem_run(which, p, runs_cap)
    assert rc in (0, -3)
    return {"result": np.array(r.as_tuple(), np.uint64), "planes": np.stack([L, R]), "view_abs": va,
            "boundary": b, "runs": runs}


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n_cells", [1 << 16, 1 << 20])
def test_vs_live_reference_large(ctx, n_cells):
    """coh_elem_eval against the reference itself (rewrite_program + run_annotated over its
    std::map store, oracle/_ref) at 2^16 and 2^20 cells, plain and pre-fragmented starts
    (rho = 2^-8 and 1/2): results, planes, abstract pairs, boundary bits and every
    transfer range."""
    cap = 1 << 20
    progs = [Program.generate(31, i, n_cells, 8, 8, 64, frag_log2=f) for i, f in enumerate([0, 8, 1])]
    out = elem_eval(ctx, progs, runs_cap=cap)
    for i, p in enumerate(progs):
        compare(out, i, _want("ref", p, cap), f"n={n_cells} prog={i}", runs_cap=cap)


@pytest.mark.parametrize("frag_log2", [16, 8, 1])
def test_fragmented_vs_oracle_2p24(ctx, frag_log2):
    """The C3 shape with the SURVEY §8(d) fragmentation levels at 2^24 cells, against the
    C restatement (pinned to the reference above and in the CPU tests)."""
    cap = 1 << 23
    progs = [Program.generate(41, i, 1 << 24, 8, 8, 64, frag_log2=frag_log2) for i in range(2)]
    out = elem_eval(ctx, progs, runs_cap=cap)
    for i, p in enumerate(progs):
        compare(out, i, _want("orc", p, cap), f"rho=2^-{frag_log2} prog={i}", runs_cap=cap)
