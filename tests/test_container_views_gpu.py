"""Views in the live container runtime (pvector<T>): every generated
element program (overlapping views, closure shadows, whole-view syncs, element bodies,
adversarial calls that get stuck) runs call by call through coh_rt_call_view, which
issues real cudaMemcpyAsync copies.  The copies must be exactly the element evaluator's
transfer ranges (same cells, same order, one copy per run, the right direction), and
the stuck call, final planes and abstract pairs must equal coh_elem_eval's."""
import numpy as np
import pytest

from paper_1910_11110_b200 import CohError
from paper_1910_11110_b200.container import Runtime
from paper_1910_11110_b200.elem import Program, elem_eval

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [
    # (seed, n_cells, n_views, n_calls, adv_per1024)
    (11, 1 << 12, 8, 24, 64),
    (12, 1 << 16, 8, 16, 300),
    (13, (1 << 16) + 37, 6, 24, 1024),
    (14, 1000, 16, 40, 128),
    (15, 1 << 20, 8, 12, 16),
]


@pytest.mark.parametrize("case", CASES, ids=[f"s{c[0]}" for c in CASES])
def test_view_copies_equal_evaluator_ranges(ctx, case):
    seed, n_cells, n_views, n_calls, adv = case
    progs = [Program.generate(seed, b, n_cells, n_views, n_calls, adv) for b in range(5)]
    out = elem_eval(ctx, progs, runs_cap=1 << 16)
    rt = Runtime(ctx)
    try:
        for b, p in enumerate(progs):
            buf = rt.buffer(p.n_cells, 4)
            for lo, hi in zip(p.view_lo, p.view_hi):
                buf.view(int(lo), int(hi))
            stuck_at = None
            for c in range(p.n_calls):
                try:
                    buf.call(p.calls[c])
                except CohError:
                    stuck_at = c
                    break
            r = out["results"][b]
            if r.status == 1:  # stuck
                assert stuck_at == r.stuck_call, (b, stuck_at, r.stuck_call)
            else:
                assert r.status == 0 and stuck_at is None, (b, r.status, stuck_at)
            log = rt.copy_log()
            mine = log[log["buffer"] == buf.id]
            runs = np.asarray(out["runs"][b][: r.n_runs])
            assert len(mine) == r.n_runs, (b, len(mine), r.n_runs)
            assert np.array_equal(mine["first"], runs[:, 0]) and np.array_equal(mine["last"], runs[:, 1]), b
            assert int((mine["last"] - mine["first"] + 1).sum()) == r.transfer_cells
            # a push (h2d) feeds a GPU component, a pull a CPU one: the copied cells were
            # invalid on the destination, so each direction matches its plane's runs
            planes = buf.planes()
            w = planes.shape[1]
            assert np.array_equal(planes, out["planes"][b][:, :w]), b
            nv = len(p.view_lo)
            assert [buf.view_state(v) for v in range(nv)] == list(out["view_abs"][b][:nv]), b
        if adv >= 1024:  # the all-adversarial case really exercises stuck calls
            assert any(out["results"][b].status == 1 for b in range(len(progs)))
        st = rt.stats()
        total = sum(int(r.transfer_cells) for r in out["results"][: len(progs)])
        assert st["h2d_bytes"] + st["d2h_bytes"] == 4 * total
        assert st["h2d_copies"] + st["d2h_copies"] == sum(int(r.n_runs) for r in out["results"][: len(progs)])
    finally:
        rt.close()


class _Dev:  # a device pointer as a torch tensor (CUDA array interface)
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def test_view_data_really_moves(ctx):
    """The bytes behind the copies, on two overlapping views a = [0, 2047], b = [1024, 4095]:
    a GPU read of b uploads b; a GPU write of b closes over a (shadow RW) and uploads the
    part of a the GPU lacked; the GPU's new data then comes back to the host when a CPU
    component reads b."""
    from paper_1910_11110_b200.elem import ElemCall

    def call(v, kind, site, eff, lo, hi):
        c = ElemCall()
        c.view, c.kind, c.site, c.n_body = v, kind, site, 1
        c.body[0].effect, c.body[0].site, c.body[0].lo, c.body[0].hi = eff, site, lo, hi
        return c

    rt = Runtime(ctx)
    try:
        buf = rt.buffer(4096, 4)
        a = buf.view(0, 2047)
        b = buf.view(1024, 4095)
        host = buf.host.view(np.float32)
        host[:] = np.arange(4096, dtype=np.float32)
        dev = torch.as_tensor(_Dev(buf.device_ptr, 4096), device="cuda")
        buf.call(call(b, 0, 1, 2, 0, 3071))  # GR(b), reads all of b
        rt.sync()
        assert torch.equal(dev[1024:].cpu(), torch.arange(1024, 4096, dtype=torch.float32))
        buf.call(call(b, 1, 1, 3, 0, 3071))  # GW(b), writes all of b: shadow GRW(a)
        rt.sync()
        assert torch.equal(dev.cpu(), torch.arange(4096, dtype=torch.float32))
        dev[1024:] = -1.0  # the GPU component's output
        torch.cuda.synchronize()
        buf.call(call(b, 0, 0, 2, 0, 3071))  # R(b) on the CPU
        rt.sync()
        assert (host[1024:] == -1.0).all() and np.array_equal(host[:1024], np.arange(1024, dtype=np.float32))
        log = [(int(x["first"]), int(x["last"]), int(x["h2d"])) for x in rt.copy_log()]
        assert log == [(1024, 4095, 1), (0, 1023, 1), (1024, 4095, 0)]
        assert buf.view_state(a) == 2 and buf.view_state(b) == 3  # a^ (I,V), b^ (V,V)
    finally:
        rt.close()


def test_view_argument_errors_and_stuck_text(ctx):
    """Construction errors (view outside its buffer, malformed call) and a stuck sync
    (data valid nowhere the view needs it) come back as the reference's error kinds."""
    from paper_1910_11110_b200.elem import ElemCall
    rt = Runtime(ctx)
    try:
        buf = rt.buffer(1000, 8)
        with pytest.raises(CohError):
            buf.view(10, 1000)  # hi past the buffer (program.hpp:65-68)
        v = buf.view(0, 99)
        w = buf.view(50, 149)
        bad = ElemCall()
        bad.view, bad.kind, bad.site, bad.n_body = 7, 0, 0, 0  # no such view
        with pytest.raises(CohError):
            buf.call(bad)
        # an adversarial body: R(v) on the CPU (v^ valid there: no sync) whose body reads
        # on the GPU, where nothing was ever copied -> stuck at v's first cell
        c = ElemCall()
        c.view, c.kind, c.site, c.n_body = v, 0, 0, 1
        c.body[0].effect, c.body[0].site, c.body[0].lo, c.body[0].hi = 2, 1, 0, 99
        with pytest.raises(CohError) as e:
            buf.call(c)
        assert "stuck" in str(e.value) and "cell 0" in str(e.value)
        assert rt.stats()["stuck_calls"] == 1 and len(rt.copy_log()) == 0
        # the same block with the read at the mode's site completes, and a GPU read of w
        # then uploads w's cells
        c.body[0].site = 0
        buf.call(c)
        g = ElemCall()
        g.view, g.kind, g.site, g.n_body = w, 0, 1, 1
        g.body[0].effect, g.body[0].site, g.body[0].lo, g.body[0].hi = 2, 1, 0, 99
        buf.call(g)
        assert [(int(x["first"]), int(x["last"]), int(x["h2d"])) for x in rt.copy_log()] == [(50, 149, 1)]
    finally:
        rt.close()
