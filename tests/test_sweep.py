"""General block programs + schedule sweeps: the native generator is
pinned to the reference's gen_well_declared text; the GPU sweep reproduces the reference's
all_schedules_run leaves (status, steps, store, boundary bits, schedule cursor) and the
acceptance aggregate (criteria 4/5: 10000 seeds -> 85335 runs, all Done, all boundaries
OK)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_ffi as o
from paper_1910_11110_b200.sweep import gen_program_text, sweep

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_generator_text_digest_matches_reference():
    h = hashlib.sha256()
    for seed in range(10000):
        h.update(gen_program_text(seed).encode())
    with open(os.path.join(GOLDEN, "sweep.json")) as f:
        want = json.load(f)["program_text_sha256_0_9999"]
    assert h.hexdigest() == want


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not built")
def test_generator_text_matches_live_reference_beyond_corpus():
    for seed in list(range(10000, 10500)) + [2**40 + 3, 2**63 - 1]:
        assert gen_program_text(seed) == o.ref_program_text(seed), seed


def _key(lv):
    return np.lexsort((lv["schedule"], lv["sched_len"], lv["seed"]))


def _same_leaves(got, want):
    got, want = got[_key(got)], want[_key(want)]
    assert len(got) == len(want)
    for f in ("seed", "schedule", "sched_len", "status", "blocks_done", "boundary_ok", "steps", "consumed",
              "overflowed", "stuck_key", "stuck_info", "store"):
        bad = np.nonzero(got[f] != want[f])[0]
        assert not len(bad), (f, got[bad[:3]], want[bad[:3]])


@pytest.mark.gpu
def test_gpu_sweep_matches_reference_leaves(ctx):
    z = np.load(os.path.join(GOLDEN, "sweep_leaves.npz"))
    got, st = sweep(ctx, 0, 1000, 6, 10000, leaves_cap=1 << 16)
    _same_leaves(got, z["fuel10000"])
    got, st = sweep(ctx, 0, 300, 6, 25, leaves_cap=1 << 16)
    assert st["fuel_exhausted"] > 0
    _same_leaves(got, z["fuel25"])


@pytest.mark.gpu
def test_gpu_acceptance_criteria_4_and_5(ctx):
    with open(os.path.join(GOLDEN, "sweep.json")) as f:
        want = json.load(f)["acceptance_0_9999"]
    leaves, st = sweep(ctx, 0, 10000, 6, 10000, leaves_cap=1 << 17)
    assert st["runs"] == want["runs"] == 85335
    assert st["done"] == want["done"] and st["stuck"] == 0 and st["fuel_exhausted"] == 0
    assert st["runs_with_violation"] == 0 and st["conflicts"] == 0
    if o.have_ref():
        _same_leaves(leaves, o.ref_sweep_leaves(0, 10000))


@pytest.mark.gpu
@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not shipped")
def test_gpu_sweep_other_limits_vs_live_reference(ctx):
    # fuel cut-offs at several depths exercise FuelExhausted inside blocks and loops
    for fuel in (1, 7, 40):
        got, _ = sweep(ctx, 5000, 200, 6, fuel, leaves_cap=1 << 16)
        _same_leaves(got, o.ref_sweep_leaves(5000, 200, fuel=fuel))
    got, _ = sweep(ctx, 0, 200, 3, 10000, leaves_cap=1 << 16)
    _same_leaves(got, o.ref_sweep_leaves(0, 200, max_dec=3))


@pytest.mark.gpu
def test_acceptance_criterion_1_enumeration(ctx):
    # tests/acceptance.cpp:107-138: 11111 straight-line programs -> 4565 done / 6546 stuck,
    # no fully-invalid state; per-program statuses equal the reference's (tests/golden/enum4.npy)
    from paper_1910_11110_b200.sweep import enum_straight_line
    st, statuses = enum_straight_line(ctx, 4, 16)
    assert (st["programs"], st["done"], st["stuck"], st["fuel_exhausted"], st["unsafe"]) == (11111, 4565, 6546, 0, 0)
    want = np.load(os.path.join(os.path.dirname(__file__), "golden", "enum4.npy"))
    assert np.array_equal(statuses, want)


@pytest.mark.gpu
def test_sweep_rejects_more_than_8_blocks(ctx):
    """SweepOut carries boundary_ok for 8 blocks: larger limits are an argument error."""
    from paper_1910_11110_b200 import CohError
    from paper_1910_11110_b200.sweep import GenLimits, sweep
    with pytest.raises(CohError) as e:
        sweep(ctx, 0, 4, 2, 10000, limits=GenLimits(max_blocks=9))
    assert e.value.code == 6
    sweep(ctx, 0, 4, 2, 10000, limits=GenLimits(max_blocks=8))
