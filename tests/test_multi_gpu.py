"""GPU tests of the multi-GPU trace path through the C ABI:
the NCCL communicator entry points on a one-rank communicator (the only shape a one-GPU
box admits), and the single-process multi-device step coh_eval_traces_multi."""
import numpy as np
import pytest

import oracle_ffi as o
import paper_1910_11110_b200 as coh

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NT, NC, NA, ADV, SEED = 20000, 128, 64, 64, 23


def _batch(ctx, s, first, n):
    d_rec = torch.empty(coh.records_elems(n, NC), dtype=torch.int16, device="cuda")
    ctx.gen_records(SEED, first, n, NC, NA, ADV, d_rec, s)
    return d_rec


def test_comm_init_rank_allreduce_one_rank(ctx):
    """ncclCommInitRank with world 1 (unique id from coh_comm_unique_id): the allreduce of
    the counters leaves them unchanged and equal to the oracle's."""
    s = torch.cuda.current_stream().cuda_stream
    d_rec = _batch(ctx, s, 0, NT)
    d_res = torch.empty(NT * 64, dtype=torch.uint8, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    comm = coh.Comm.init_rank(ctx, coh.comm_unique_id(), 1, 0)
    try:
        ctx.eval_traces_counted(d_rec, NT, NC, NA, 10000, d_res, d_cnt, None, stream=s)
        before = d_cnt.clone()
        comm.allreduce_counters(d_cnt, s)
        torch.cuda.synchronize()
    finally:
        comm.close()
    assert torch.equal(before, d_cnt)
    res, _ = o.orc_eval(o.orc_gen(SEED, 0, NT, NC, NA, ADV), NT, NC, NA)
    assert np.array_equal(d_cnt.cpu().numpy().view(np.uint64)[:11], coh.counters_host(res))


def test_eval_traces_multi_init_all(ctx):
    """ncclCommInitAll over the visible devices (one here): coh_eval_traces_multi over
    contiguous shards gives per-trace results equal to the oracle and whole-job counters."""
    n_dev = torch.cuda.device_count()
    ctxs = [ctx] + [coh.Context(d) for d in range(1, n_dev)]
    comms = coh.Comm.init_all(ctxs)
    try:
        shards, outs, cnts, streams = [], [], [], []
        for d in range(n_dev):
            with torch.cuda.device(d):
                first, n = coh.shard_split(d, n_dev, NT)
                s = torch.cuda.current_stream(d).cuda_stream
                shards.append((_batch(ctxs[d], s, first, n), n, NC, NA, 10000))
                outs.append(torch.empty(n * 64, dtype=torch.uint8, device=f"cuda:{d}"))
                cnts.append(torch.zeros(16, dtype=torch.int64, device=f"cuda:{d}"))
                streams.append(s)
        coh.eval_traces_multi(comms, shards, outs, cnts, streams)
        for d in range(n_dev):
            torch.cuda.synchronize(d)
    finally:
        for c in comms:
            c.close()
        for c in ctxs[1:]:
            c.close()
    res, _ = o.orc_eval(o.orc_gen(SEED, 0, NT, NC, NA, ADV), NT, NC, NA)
    got = np.concatenate([x.cpu().numpy() for x in outs])
    assert np.array_equal(got, res.view(np.uint8))
    for c in cnts:
        assert np.array_equal(c.cpu().numpy().view(np.uint64)[:11], coh.counters_host(res))


def test_comm_errors(ctx):
    with pytest.raises(coh.CohError) as e:
        coh.Comm.init_rank(ctx, coh.comm_unique_id(), 1, 3)  # rank out of range
    assert e.value.code == 6
