"""TraceMode::Full for whole-array traces (coh_trace_steps, DESIGN §4g'): the device step
log of run_annotated over a trace's blocks equals the reference's own TraceStep lists
(rule, head statement, changed key), single-mode and multi-mode blocks, stuck and fuel
cut-offs."""
import numpy as np
import pytest

import oracle_ffi as o

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("na,nc,adv,cont,fuel", [(4, 64, 200, 0, 10000), (8, 128, 60, 500, 10000),
                                                  (3, 96, 400, 300, 57), (64, 256, 16, 200, 10000)])
def test_step_log_equals_reference(ctx, na, nc, adv, cont, fuel):
    flags = 1 if cont else 0
    n = 0
    for t in range(40):
        recs = o.orc_gen(5 + t, 0, 1, nc, na, adv)[:nc]  # one trace: call-major == call order
        if cont:
            recs = o.add_blocks(recs, 1, nc, cont, t)[:nc]
        got, gs = ctx.trace_steps(recs, nc, na, fuel, flags)
        want, ws = o.ref_trace_steps(recs, nc, na, fuel, flags)
        assert gs == ws, t
        assert np.array_equal(got, want), t
        n += len(got)
    assert n > 500
