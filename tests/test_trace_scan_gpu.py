"""The latency path (k_trace_scan: a block per single-array trace, calls spread over its
threads and combined by an associative scan of per-call state maps) against the C oracle
and the per-thread kernel, field for field: default and adversarial mixes, fuel cut-offs
anywhere in a pass, ragged lengths, traces longer than one pass, transfer bytes, defect
records (missing key, malformed kind), boundary words and the fused counters."""
import os

import numpy as np
import pytest

import oracle_ffi as o
import paper_1910_11110_b200 as coh
from test_trace_gpu import dev_eval, first_diff, same

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


class path:
    def __init__(self, which):
        self.which = which

    def __enter__(self):
        os.environ["COH_TE_PATH"] = self.which

    def __exit__(self, *a):
        os.environ.pop("COH_TE_PATH", None)


CASES = [
    # (seed, n_traces, n_calls, adv_per1024, fuel, array_bytes)
    (41, 1, 1000, 64, 10000, None),      # BASELINE C1 shape
    (42, 1, 1000, 1024, 10000, None),    # every call adversarial: early stuck
    (43, 7, 1000, 16, 300, None),        # fuel runs out mid-pass
    (44, 300, 100, 8, 10000, None),      # ragged length, many blocks
    (45, 5, 3000, 4, 10000, [4096]),     # several passes, transfer bytes
    (46, 3, 5000, 2, 20000, None),
    (47, 2, 1024, 0, 10000, None),       # exactly one pass
    (48, 2, 1025, 0, 3, None),           # fuel 3
    (49, 50, 64, 64, 0, None),           # fuel 0
    (50, 9, 2100, 1, 1500, [7]),         # fuel cut-off in the third pass
]


@pytest.mark.parametrize("cfg", CASES, ids=[f"s{c[0]}" for c in CASES])
def test_scan_vs_oracle_and_thread_kernel(ctx, cfg):
    seed, nt, nc, adv, fuel, ab = cfg
    recs = coh.gen_records_host(seed, 0, nt, nc, 1, adv)
    want, want_b = o.orc_eval(recs, nt, nc, 1, fuel, ab)
    with path("scan"):
        res, bnd = dev_eval(ctx, recs, nt, nc, 1, fuel, ab)
    assert same(res, want), first_diff(res, want)
    assert np.array_equal(bnd, want_b)
    with path("thread"):
        res_t, bnd_t = dev_eval(ctx, recs, nt, nc, 1, fuel, ab)
    assert same(res_t, res) and np.array_equal(bnd_t, bnd)


def test_scan_defect_records(ctx):
    rng = np.random.default_rng(5)
    nt, nc = 6, 700
    recs = coh.gen_records_host(7, 0, nt, nc, 1, 8).copy()
    for t in range(nt):  # one defect per trace at a random call: missing key or kind 3
        c = int(rng.integers(0, nc))
        idx = ((c // 8) * nt + t) * 8 + c % 8
        recs[idx] = coh.make_record(1, 0, 0, 0) if t % 2 else coh.make_record(0, 3, 1, 0)
    want, want_b = o.orc_eval(recs, nt, nc, 1, 10000)
    with path("scan"):
        res, bnd = dev_eval(ctx, recs, nt, nc, 1, 10000)
    assert same(res, want), first_diff(res, want)
    assert np.array_equal(bnd, want_b)
    assert (res["status"] != 0).all()


def test_scan_default_dispatch_and_counters(ctx):
    """C1's shape (one trace) takes the scan path by default; fused counters agree."""
    nt, nc = 4, 1000
    recs = coh.gen_records_host(3, 0, nt, nc, 1, 32)
    want, _ = o.orc_eval(recs, nt, nc, 1, 10000)
    d_rec = torch.from_numpy(recs.view(np.int16).copy()).cuda()
    d_res = torch.empty(nt * 64, dtype=torch.uint8, device="cuda")
    d_cnt = torch.full((16,), 7, dtype=torch.int64, device="cuda")
    ctx.eval_traces_counted(d_rec, nt, nc, 1, 10000, d_res, d_cnt, None,
                            stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    res = d_res.cpu().numpy().view(coh.RESULT_DTYPE)
    assert same(res, want)
    cnt = d_cnt.cpu().numpy().view(np.uint64)[:11]
    st = want["status"]
    exp = [(st == 1).sum(), (st == 2).sum(), (want["violations"] > 0).sum(), (st == 3).sum(),
           want["steps"].astype(np.uint64).sum(), want["transfers"].astype(np.uint64).sum(),
           want["transfer_bytes"].sum(), want["violations"].astype(np.uint64).sum(),
           want["calls_done"].astype(np.uint64).sum(), nt, ((want["stuck_flags"] & coh.FLAG_UNSAFE) != 0).sum()]
    assert [int(x) for x in cnt] == [int(x) for x in exp]
