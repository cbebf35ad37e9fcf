"""CPU tests of the element-granular oracle (oracle/cohere_oracle.c orc_elem_run) against
golden fixtures produced by the reference (tests/golden/make_golden_elem.py) and, when
oracle/_ref is present, the live reference."""
import os

import numpy as np
import pytest

import oracle_ffi as o
from paper_1910_11110_b200.elem import Program

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "elem.npz")


def golden_programs():
    z = np.load(GOLDEN)
    for key in sorted({k.split(".")[0] for k in z.files}, key=lambda s: int(s[1:])):
        pid, n, V, K, adv, fuel = (int(x) for x in z[key + ".params"])
        views = z[key + ".views"]
        p = Program.from_bytes(n, views[0], views[1], z[key + ".calls"], K, fuel)
        yield key, (pid, n, V, K, adv, fuel), p, {k: z[key + "." + k] for k in
                                                  ("result", "planes", "view_abs", "boundary", "runs")}


def check_same(got, want, key):
    rc, r, L, R, va, b, runs = got
    assert rc == 0, key
    assert np.array_equal(np.array(r.as_tuple(), np.uint64), want["result"]), (key, r.as_tuple(), want["result"])
    assert np.array_equal(np.stack([L, R]), want["planes"]), key
    assert np.array_equal(va, want["view_abs"]), key
    assert np.array_equal(b, want["boundary"]), key
    assert np.array_equal(runs, want["runs"]), key


def test_oracle_matches_reference_goldens():
    n = 0
    for key, params, p, want in golden_programs():
        check_same(o.elem_run("orc", p), want, key)
        n += 1
    assert n == 48


def test_generator_reproduces_golden_programs():
    for key, (pid, n, V, K, adv, fuel), p, want in golden_programs():
        g = Program.generate(11, pid, n, V, K, adv, fuel)
        assert np.array_equal(g.view_lo, p.view_lo) and np.array_equal(g.view_hi, p.view_hi)
        assert bytes(g.calls)[: 32 * K] == bytes(p.calls)[: 32 * K], key


def test_golden_coverage():
    # the fixtures exercise every outcome the path has
    statuses, transfers, runs, viol = set(), 0, 0, 0
    for key, params, p, want in golden_programs():
        r = want["result"]
        statuses.add(int(r[0]))
        transfers += int(r[8])
        runs += int(r[11])
        viol += int(r[7])
    assert statuses >= {0, 1, 2} and transfers > 20 and runs > 20 and viol > 0


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not built")
def test_oracle_vs_live_reference_fresh_programs():
    for pid in range(60):
        rng = np.random.default_rng(pid)
        p = Program.generate(99, pid, int(rng.choice([40, 333, 2048])), int(rng.integers(1, 9)),
                             int(rng.integers(1, 9)), int(rng.choice([0, 200, 1024])),
                             int(rng.choice([1 << 30, 100, 1500])))
        a, b = o.elem_run("ref", p), o.elem_run("orc", p)
        assert a[0] == b[0] == 0
        assert a[1].as_tuple() == b[1].as_tuple(), pid
        for x, y in zip(a[2:], b[2:]):
            assert np.array_equal(x, y), pid


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("frag_log2", [1, 4, 8])
def test_oracle_vs_live_reference_fragmented(frag_log2):
    """Pre-fragmented starts (coh_elem_program.frag_*: 2^-frag_log2 of the cells already
    coherent): the reference run from that store and the oracle agree, and the first
    syncs' transfer ranges are split by the coherent cells."""
    runs = 0
    for pid in range(12):
        rng = np.random.default_rng(1000 + pid)
        p = Program.generate(77, pid, int(rng.choice([333, 4096, 1 << 14])), int(rng.integers(1, 9)),
                             int(rng.integers(2, 9)), int(rng.choice([0, 200])), frag_log2=frag_log2)
        a, b = o.elem_run("ref", p, 1 << 14), o.elem_run("orc", p, 1 << 14)
        assert a[0] == b[0] == 0
        assert a[1].as_tuple() == b[1].as_tuple(), pid
        for x, y in zip(a[2:], b[2:]):
            assert np.array_equal(x, y), pid
        runs += a[1].n_runs
    assert runs > 12 * (1 if frag_log2 == 8 else 4)
