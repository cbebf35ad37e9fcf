"""GPU parity of multi-mode blocks (COH_BATCH_BLOCKS, k_trace_blocks): records with
COH_REC_CONT continue the previous record's DeclBlock.  Bit-exact against the C oracle
(itself pinned to the reference's own multi-mode DeclBlocks in test_oracle.py) and the
live reference; without CONT bits the blocks kernel equals the single-mode fast path."""
import numpy as np
import pytest

import oracle_ffi as o
import paper_1910_11110_b200 as coh

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev_eval(ctx, recs, nt, nc, na, fuel, flags, array_bytes=None, counted=False):
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.from_numpy(recs.view(np.int16).copy()).cuda()
    d_res = torch.empty(nt * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.empty(max(1, coh.boundary_words(nc) * nt), dtype=torch.int32, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    if counted:
        ctx.eval_traces_counted(d_rec, nt, nc, na, fuel, d_res, d_cnt, d_bnd, array_bytes=array_bytes, stream=s,
                                flags=flags)
    else:
        ctx.eval_traces(d_rec, nt, nc, na, fuel, d_res, d_bnd, array_bytes=array_bytes, stream=s, flags=flags)
    torch.cuda.synchronize()
    res = d_res.cpu().numpy().view(coh.RESULT_DTYPE)
    bnd = d_bnd.cpu().numpy().view(np.uint32)[: coh.boundary_words(nc) * nt]
    return res, bnd, d_cnt.cpu().numpy().view(np.uint64)[: len(coh.COUNTER_NAMES)]


@pytest.mark.parametrize("nt,nc,na,adv,fuel", [(5000, 256, 64, 16, 10000), (3000, 100, 7, 200, 10000),
                                               (4000, 64, 64, 64, 150), (2000, 37, 3, 900, 10000)])
def test_no_cont_equals_fast_path(ctx, nt, nc, na, adv, fuel):
    recs = o.orc_gen(3, 0, nt, nc, na, adv)
    a, ab, _ = dev_eval(ctx, recs, nt, nc, na, fuel, 0)
    b, bb, _ = dev_eval(ctx, recs, nt, nc, na, fuel, coh.BATCH_BLOCKS)
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    assert np.array_equal(ab, bb)


@pytest.mark.parametrize("nt,nc,na,adv,cont,dup,fuel,sizes", [
    (20000, 256, 64, 16, 300, 0, 10000, False), (8000, 96, 5, 200, 600, 40, 10000, True),
    (8000, 128, 64, 64, 450, 5, 300, False), (6000, 41, 12, 500, 800, 100, 10000, True)])
def test_blocks_vs_oracle(ctx, nt, nc, na, adv, cont, dup, fuel, sizes):
    recs = o.add_blocks(o.orc_gen(11, 0, nt, nc, na, adv), nt, nc, cont, 7, dup)
    ab = (np.arange(na, dtype=np.uint64) * 977 + 13) if sizes else None
    got, gb, cnt = dev_eval(ctx, recs, nt, nc, na, fuel, coh.BATCH_BLOCKS, array_bytes=ab, counted=True)
    want, wb = o.orc_eval(recs, nt, nc, na, fuel, array_bytes=ab, flags=coh.BATCH_BLOCKS)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    assert np.array_equal(gb, wb)
    assert np.array_equal(cnt, coh.counters_host(want))
    assert cnt[10] == 0  # is_unsafe never holds (Property 2)
    assert (recs & 1).sum() > nt  # multi-mode blocks were formed


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not built")
def test_blocks_vs_live_reference(ctx):
    nt, nc, na = 400, 64, 10
    recs = o.add_blocks(o.orc_gen(21, 0, nt, nc, na, 150), nt, nc, 500, 9, 30)
    got, gb, _ = dev_eval(ctx, recs, nt, nc, na, 10000, coh.BATCH_BLOCKS)
    want, wb = o.ref_eval(recs, nt, nc, na, 10000, mode=2)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    assert np.array_equal(gb, wb)


def test_unknown_flags_rejected(ctx):
    recs = o.orc_gen(1, 0, 4, 8, 2, 0)
    with pytest.raises(coh.CohError):
        dev_eval(ctx, recs, 4, 8, 2, 100, 6)


def test_generated_blocks_c2_scale_vs_oracle(ctx):
    """Device-generated multi-mode records (coh_gen_records_blocks == the host generator) at
    the C2 shape, 256K traces x 256 calls x 64 arrays: every trace equals the oracle."""
    nt, nc, na, adv, cont = 1 << 18, 256, 64, 1, 300
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.empty(coh.records_elems(nt, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records_blocks(1, 0, nt, nc, na, adv, cont, d_rec, s)
    d_res = torch.empty(nt * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.empty(coh.boundary_words(nc) * nt, dtype=torch.int32, device="cuda")
    ctx.eval_traces(d_rec, nt, nc, na, 10000, d_res, d_bnd, stream=s, flags=coh.BATCH_BLOCKS)
    torch.cuda.synchronize()
    recs = d_rec.cpu().numpy().view(np.uint16)
    assert np.array_equal(recs, coh.gen_records_blocks_host(1, 0, nt, nc, na, adv, cont))
    assert (recs & 1).mean() > 0.2
    want, wb = o.orc_eval(recs, nt, nc, na, 10000, flags=coh.BATCH_BLOCKS)
    assert np.array_equal(d_res.cpu().numpy(), want.view(np.uint8))
    assert np.array_equal(d_bnd.cpu().numpy().view(np.uint32), wb)
