"""GPU parity tests for the trace_eval kernel: bit-exact against the reference's golden
fixtures, the C oracle and (when oracle/_ref traveled) the live reference."""
import os

import numpy as np
import pytest

import oracle_ffi as o
import paper_1910_11110_b200 as coh

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def dev_eval(ctx, recs_np, nt, nc, na, fuel, array_bytes=None):
    d_rec = torch.from_numpy(recs_np.view(np.int16).copy()).cuda()
    d_res = torch.empty(max(nt, 1) * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.empty(max(coh.boundary_words(nc) * nt, 1), dtype=torch.int32, device="cuda")
    ctx.eval_traces(d_rec, nt, nc, na, fuel, d_res, d_bnd, array_bytes=array_bytes,
                    stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    res = d_res.cpu().numpy()[: nt * 64].view(coh.RESULT_DTYPE)
    bnd = d_bnd.cpu().numpy()[: coh.boundary_words(nc) * nt].view(np.uint32)
    return res, bnd


def same(a, b):
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def first_diff(a, b):
    idx = np.nonzero((a.view(np.uint8).reshape(-1, 64) != b.view(np.uint8).reshape(-1, 64)).any(1))[0]
    if not len(idx):
        return None
    i = idx[0]
    return i, a[i], b[i]


def golden():
    z = np.load(os.path.join(GOLDEN, "traces.npz"))
    for name in sorted({k.split(".")[0] for k in z.files}):
        seed, trace0, nt, nc, na, adv, fuel = (int(x) for x in z[f"{name}.params"])
        ab = z[f"{name}.array_bytes"]
        yield name, z[f"{name}.records"], nt, nc, na, fuel, (ab if ab.size else None), \
            z[f"{name}.results"].view(coh.RESULT_DTYPE), z[f"{name}.boundary"]


def test_golden_device_entry(ctx):
    for name, recs, nt, nc, na, fuel, ab, want, want_b in golden():
        res, bnd = dev_eval(ctx, recs, nt, nc, na, fuel, ab)
        assert same(res, want), (name, first_diff(res, want))
        assert np.array_equal(bnd, want_b), name


def test_golden_host_entry(ctx):
    for name, recs, nt, nc, na, fuel, ab, want, want_b in golden():
        res, bnd = ctx.eval_traces_host(recs, nt, nc, na, fuel, ab)
        assert same(res, want), (name, first_diff(res, want))
        assert np.array_equal(bnd, want_b), name


def test_golden_reads_like_reference(ctx):
    # c1_canonical: one array, 1000 canonical calls -> Done, every boundary OK
    # (Theorems 1-2); the stuck cases describe() like StuckInfo.
    for name, recs, nt, nc, na, fuel, ab, want, want_b in golden():
        res, bnd = dev_eval(ctx, recs, nt, nc, na, fuel, ab)
        if name == "c1_canonical":
            run = coh.annotated_run(res, bnd, 0, nt, na)
            assert run.status == "done" and len(run.boundary_ok) == 1000 and all(run.boundary_ok)
        if name == "c2_adversarial":
            stuck = [coh.annotated_run(res, bnd, t, nt, na) for t in range(nt)]
            texts = {r.stuck.describe() for r in stuck if r.stuck}
            assert any(t.startswith("gr ") and t.endswith("against the swapped pair") for t in texts)
            assert any(t.startswith("r ") and "need (V,*)" in t for t in texts)


def test_device_generator_matches_host(ctx):
    for seed, trace0, nt, nc, na, adv in [(1, 0, 3000, 256, 64, 1), (9, 77, 1001, 37, 5, 500), (3, 0, 17, 1, 1, 1024)]:
        d = torch.empty(coh.records_elems(nt, nc), dtype=torch.int16, device="cuda")
        ctx.gen_records(seed, trace0, nt, nc, na, adv, d, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy().view(np.uint16), coh.gen_records_host(seed, trace0, nt, nc, na, adv))


CONFIGS = [
    # (seed, n_traces, n_calls, n_arrays, adv_per1024, fuel, array_bytes)
    (21, 20000, 256, 64, 1, 10000, None),
    (22, 20000, 256, 64, 16, 10000, None),
    (23, 5000, 256, 64, 4, 700, None),          # fuel runs out mid-trace (check_fuel path)
    (24, 4000, 1000, 1, 8, 10000, None),
    (25, 6000, 33, 2, 60, 10000, None),
    (26, 6000, 31, 63, 30, 10000, None),
    (27, 3000, 7, 5, 300, 10000, None),
    (28, 3000, 1, 1, 1024, 10000, None),
    (29, 7000, 256, 64, 3, 10000, list(range(1, 65))),     # non-uniform bytes
    (30, 7000, 200, 33, 3, 500, [4096] * 33),              # uniform, scaled bytes, fuel
    (31, 1000, 64, 64, 1024, 10000, None),                 # all adversarial
    (32, 129, 2047, 3, 2, 20000, [8, 16, 24]),             # max length for non-uniform
    (33, 1000, 96, 64, 0, 1, None),                        # fuel 1
    (34, 1000, 96, 64, 0, 0, None),                        # fuel 0
]


@pytest.mark.parametrize("cfg", CONFIGS, ids=[f"s{c[0]}" for c in CONFIGS])
def test_kernel_vs_oracle(ctx, cfg):
    seed, nt, nc, na, adv, fuel, ab = cfg
    recs = coh.gen_records_host(seed, 0, nt, nc, na, adv)
    res, bnd = dev_eval(ctx, recs, nt, nc, na, fuel, ab)
    want, want_b = o.orc_eval(recs, nt, nc, na, fuel, ab)
    assert same(res, want), first_diff(res, want)
    assert np.array_equal(bnd, want_b)


@pytest.mark.parametrize("cfg", [CONFIGS[1], CONFIGS[2], CONFIGS[8], CONFIGS[3]], ids=["adv", "fuel", "bytes", "wide"])
def test_fused_counters_equal_sum_of_results(ctx, cfg):
    seed, nt, nc, na, adv, fuel, ab = cfg
    recs = coh.gen_records_host(seed, 0, nt, nc, na, adv)
    d_rec = torch.from_numpy(recs.view(np.int16).copy()).cuda()
    d_res = torch.empty(nt * 64, dtype=torch.uint8, device="cuda")
    d_cnt = torch.full((16,), 7, dtype=torch.int64, device="cuda")
    ctx.eval_traces_counted(d_rec, nt, nc, na, fuel, d_res, d_cnt, None, array_bytes=ab,
                            stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    res = d_res.cpu().numpy().view(coh.RESULT_DTYPE)
    cnt = d_cnt.cpu().numpy().view(np.uint64)[:11]
    want, _ = o.orc_eval(recs, nt, nc, na, fuel, ab)
    assert same(res, want)
    st = want["status"]
    exp = [(st == 1).sum(), (st == 2).sum(), (want["violations"] > 0).sum(), (st == 3).sum(),
           want["steps"].astype(np.uint64).sum(), want["transfers"].astype(np.uint64).sum(),
           want["transfer_bytes"].sum(), want["violations"].astype(np.uint64).sum(),
           want["calls_done"].astype(np.uint64).sum(), nt, ((want["stuck_flags"] & coh.FLAG_UNSAFE) != 0).sum()]
    assert [int(x) for x in cnt] == [int(x) for x in exp]


def test_defect_records(ctx):
    recs = np.zeros(coh.records_elems(2, 8), dtype=np.uint16)
    recs[0:8] = [0, 0, coh.make_record(0, 3, 0, 0), 0, 0, 0, 0, 0]
    recs[8:16] = [coh.make_record(a, 0, 0, 0) for a in (0, 1, 2, 5, 0, 0, 0, 0)]
    res, bnd = dev_eval(ctx, recs, 2, 8, 4, 10000)
    want, want_b = o.orc_eval(recs, 2, 8, 4)
    assert same(res, want) and np.array_equal(bnd, want_b)
    assert res["status"].tolist() == [3, 3]


def test_argument_errors(ctx):
    with pytest.raises(coh.CohError):
        ctx.eval_traces(0, 10, 8, 65, 100, 0)
    with pytest.raises(coh.CohError):
        ctx.eval_traces(0, 10, 4096, 3, 100, 0, array_bytes=[1, 2, 3])


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref not shipped")
def test_kernel_vs_live_reference_sample(ctx):
    nt, nc, na = 512, 256, 64
    recs = coh.gen_records_host(1, 0, nt, nc, na, 8)
    res, bnd = dev_eval(ctx, recs, nt, nc, na, 10000)
    want, want_b = o.ref_eval(recs, nt, nc, na, 10000)
    assert same(res, want), first_diff(res, want)
    assert np.array_equal(bnd, want_b)


def test_full_size_c2_properties(ctx):
    """BASELINE config 2 at full size (1M traces x 64 arrays x 256 calls): oracle on a
    sample of trace ids, counters == sum of per-trace fields, determinism, and shard
    invariance (the same ids evaluated as 4 contiguous shards give identical bytes)."""
    N, nc, na, adv, seed = 1 << 20, 256, 64, 1, 1
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.empty(coh.records_elems(N, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records(seed, 0, N, nc, na, adv, d_rec, s)
    d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.empty(coh.boundary_words(nc) * N, dtype=torch.int32, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    ctx.eval_traces_counted(d_rec, N, nc, na, 10000, d_res, d_cnt, d_bnd, stream=s)
    d_cnt2 = torch.zeros(16, dtype=torch.int64, device="cuda")
    ctx.reduce_counters(d_res, N, d_cnt2, s)
    torch.cuda.synchronize()
    assert torch.equal(d_cnt[:11], d_cnt2[:11])  # fused == separate reduction
    res = d_res.cpu().numpy().view(coh.RESULT_DTYPE)
    bnd = d_bnd.cpu().numpy().view(np.uint32)
    cnt = d_cnt.cpu().numpy().view(np.uint64)[:11]
    # counters
    st = res["status"]
    assert cnt[0] == (st == 1).sum() and cnt[1] == (st == 2).sum() and cnt[3] == (st == 3).sum()
    assert cnt[4] == res["steps"].astype(np.uint64).sum() and cnt[5] == res["transfers"].astype(np.uint64).sum()
    assert cnt[7] == res["violations"].astype(np.uint64).sum() and cnt[8] == res["calls_done"].astype(np.uint64).sum()
    assert cnt[9] == N
    # sample vs oracle (every 997th id, generated per id on the host)
    ids = np.arange(0, N, 997)
    for t in ids[:600]:
        r1 = coh.gen_records_host(seed, int(t), 1, nc, na, adv)
        w, wb = o.orc_eval(r1, 1, nc, na, 10000)
        assert same(res[t:t + 1], w), (t, first_diff(res[t:t + 1], w))
        assert np.array_equal(bnd[t::N], wb), t
    # determinism
    h1 = torch.sum(d_res.view(torch.int64)).item()
    ctx.eval_traces(d_rec, N, nc, na, 10000, d_res, d_bnd, stream=s)
    torch.cuda.synchronize()
    assert torch.sum(d_res.view(torch.int64)).item() == h1
    # shard invariance: 4 contiguous shards generated from (seed, trace0)
    shard = N // 4
    for k in range(4):
        r = torch.empty(coh.records_elems(shard, nc), dtype=torch.int16, device="cuda")
        ctx.gen_records(seed, k * shard, shard, nc, na, adv, r, s)
        o_res = torch.empty(shard * 64, dtype=torch.uint8, device="cuda")
        ctx.eval_traces(r, shard, nc, na, 10000, o_res, None, stream=s)
        torch.cuda.synchronize()
        assert torch.equal(o_res, d_res[k * shard * 64:(k + 1) * shard * 64]), k


def test_full_size_c2_every_trace_vs_oracle(ctx):
    """BASELINE config 2 at full size, every one of the 1M traces (256M calls) against the C
    oracle (run on all host cores in trace-id slices): results and boundary bits bit-exact."""
    import concurrent.futures as cf

    N, nc, na, adv, seed = 1 << 20, 256, 64, 1, 1
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.empty(coh.records_elems(N, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records(seed, 0, N, nc, na, adv, d_rec, s)
    d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
    d_bnd = torch.empty(coh.boundary_words(nc) * N, dtype=torch.int32, device="cuda")
    ctx.eval_traces(d_rec, N, nc, na, 10000, d_res, d_bnd, stream=s)
    torch.cuda.synchronize()
    recs = d_rec.cpu().numpy().view(np.uint16)
    res = d_res.cpu().numpy().view(coh.RESULT_DTYPE)
    bnd = d_bnd.cpu().numpy().view(np.uint32).reshape(coh.boundary_words(nc), N)
    k = max(1, min(32, os.cpu_count() or 1))
    cuts = [N * i // k for i in range(k + 1)]

    def check(i):
        a, b = cuts[i], cuts[i + 1]
        w, wb = o.orc_eval(recs, N, nc, na, 10000, t_begin=a, t_end=b)
        ok = np.array_equal(res[a:b].view(np.uint8), w.view(np.uint8))
        okb = np.array_equal(bnd[:, a:b], wb.reshape(coh.boundary_words(nc), b - a))
        return ok and okb

    with cf.ThreadPoolExecutor(k) as ex:
        assert all(ex.map(check, range(k)))


def test_c4_full_size_shards(ctx):
    """BASELINE config 4 at full size on one device: 64M traces evaluated as one batch and
    as 8 contiguous shards (each generated on the device from its id range) give the same
    per-trace results (order-free checksum of every record) and counters; a sample of the
    ids = 0 (mod 64) matches the oracle; fused counters equal the separate reduction."""
    from paper_1910_11110_b200 import shard
    N, nc, na, adv, seed, G = 1 << 26, 256, 64, 1, 1, 8
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.empty(coh.records_elems(N, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records(seed, 0, N, nc, na, adv, d_rec, s)
    d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
    d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    ctx.eval_traces_counted(d_rec, N, nc, na, 10000, d_res, d_cnt, None, stream=s)
    d_cnt2 = torch.zeros(16, dtype=torch.int64, device="cuda")
    ctx.reduce_counters(d_res, N, d_cnt2, s)
    torch.cuda.synchronize()
    assert torch.equal(d_cnt[:11], d_cnt2[:11])
    whole = shard.results_checksum(d_res)
    # SURVEY §8(d) C4 parity sample: every id = 0 (mod 64), 1M traces, against the C oracle
    # (all of them) and the reference itself (run_annotated over its std::map store, a
    # 32K-trace subset on the host threads); the records of the sample are cut out of the
    # device buffer (chunk-major layout: [chunk][trace][8])
    samp_rec = d_rec.view(-1, N, 8)[:, ::64, :].contiguous().cpu().numpy().view(np.uint16).reshape(-1)
    samp_res = d_res.view(N, 64)[::64].contiguous().cpu().numpy().reshape(-1).view(coh.RESULT_DTYPE)
    ns = N // 64
    w, _ = o.orc_eval(samp_rec, ns, nc, na, 10000)
    assert same(samp_res, w)
    if o.have_ref():
        m = 1 << 15
        wr, _ = o.ref_eval(samp_rec, ns, nc, na, 10000, t_begin=0, t_end=m)
        assert same(samp_res[:m], wr)
    del d_rec
    total, cnt_sum = 0, np.zeros(11, np.uint64)
    for g in range(G):
        first, cnt = shard.split_range(g, G, N)
        d_r = torch.empty(coh.records_elems(cnt, nc), dtype=torch.int16, device="cuda")
        ctx.gen_records(seed, first, cnt, nc, na, adv, d_r, s)
        d_o = torch.empty(cnt * 64, dtype=torch.uint8, device="cuda")
        d_c = torch.zeros(16, dtype=torch.int64, device="cuda")
        ctx.eval_traces_counted(d_r, cnt, nc, na, 10000, d_o, d_c, None, stream=s)
        torch.cuda.synchronize()
        assert torch.equal(d_o, d_res[first * 64:(first + cnt) * 64])
        total = (total + shard.results_checksum(d_o)) & ((1 << 64) - 1)
        cnt_sum += d_c.cpu().numpy().view(np.uint64)[:11]
        del d_r, d_o
    assert total == whole
    assert np.array_equal(cnt_sum, d_cnt.cpu().numpy().view(np.uint64)[:11])
    torch.cuda.empty_cache()


@pytest.mark.parametrize("nc", [100, 96, 64])  # ragged (no ring), single ring, double ring
def test_dynamic_batches_long_launch(ctx, nc):
    """Launches long enough for the dynamic warp batches (> 5 rounds per thread): every
    variant's results equal the same traces evaluated as small static launches (whose
    parity with the oracle the tests above establish), checked in full by checksum and on
    a sample against the oracle."""
    from paper_1910_11110_b200 import shard
    N, na, adv, seed = 1 << 20, 64, 8, 9
    s = torch.cuda.current_stream().cuda_stream
    d_rec = torch.empty(coh.records_elems(N, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records(seed, 0, N, nc, na, adv, d_rec, s)
    d_res = torch.empty(N * 64, dtype=torch.uint8, device="cuda")
    ctx.eval_traces(d_rec, N, nc, na, 10000, d_res, None, stream=s)
    torch.cuda.synchronize()
    whole = shard.results_checksum(d_res)
    parts = 0
    for g in range(16):  # 64K-trace launches: static striding
        first, cnt = shard.split_range(g, 16, N)
        d_r = torch.empty(coh.records_elems(cnt, nc), dtype=torch.int16, device="cuda")
        ctx.gen_records(seed, first, cnt, nc, na, adv, d_r, s)
        d_o = torch.empty(cnt * 64, dtype=torch.uint8, device="cuda")
        ctx.eval_traces(d_r, cnt, nc, na, 10000, d_o, None, stream=s)
        torch.cuda.synchronize()
        parts = (parts + shard.results_checksum(d_o)) & ((1 << 64) - 1)
    assert parts == whole
    res = d_res.cpu().numpy().view(coh.RESULT_DTYPE)
    for t in range(0, N, 4099)[:200]:
        w, _ = o.orc_eval(coh.gen_records_host(seed, t, 1, nc, na, adv), 1, nc, na, 10000)
        assert same(res[t:t + 1], w), t


def test_packed12_host_entry_equals_plain(ctx):
    """COH_BATCH_PACKED12: the host entry with 12-bit packed records (unpacked on the
    device per slice) returns exactly what the 16-bit records give, across slices."""
    nt, nc, na = (1 << 17) + 333, 96, 48
    recs = coh.gen_records_host(4, 0, nt, nc, na, 64)
    a, ab = ctx.eval_traces_host(recs, nt, nc, na)
    pk = coh.pack_records12(recs, nt, nc)
    assert pk.size == recs.size // 8 * 12
    b, bb = ctx.eval_traces_host(pk, nt, nc, na, flags=coh.BATCH_PACKED12)
    assert same(a, b) and np.array_equal(ab, bb)
    # COH_BATCH_OVERLAP is ignored by the host entry (its kernels read what its copies wrote)
    c, cb = ctx.eval_traces_host(pk, nt, nc, na, flags=coh.BATCH_PACKED12 | coh.BATCH_OVERLAP)
    assert same(a, c) and np.array_equal(ab, cb)
    with pytest.raises(coh.CohError):
        ctx.eval_traces_host(pk, nt, nc, na, flags=coh.BATCH_PACKED12 | coh.BATCH_BLOCKS)


@pytest.mark.parametrize("sizes,launches", [([20000, 1 << 20, 7000, 1 << 20], 300), ([20000, 7000], 260),
                                            ([1 << 20], 3)], ids=["mixed", "ring", "ticket"])
def test_overlapped_launch_stream(ctx, sizes, launches):
    """COH_BATCH_OVERLAP: a stream of back-to-back launches (each may start on the SMs its
    predecessor frees) with their own outputs gives every batch the results, boundary words
    and counters of a plain launch; more launches than the context's ring of launch slots,
    mixing batch sizes (short launches: static striding; long ones: the slot's ticket)."""
    s = torch.cuda.current_stream().cuda_stream
    nc, na = 256, 64
    recs = {}
    want = {}
    for n in set(sizes):
        d_rec = torch.empty(coh.records_elems(n, nc), dtype=torch.int16, device="cuda")
        ctx.gen_records(5, 0, n, nc, na, 8, d_rec, s)
        d_res = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
        d_bnd = torch.empty(coh.boundary_words(nc) * n, dtype=torch.int32, device="cuda")
        d_cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
        ctx.eval_traces_counted(d_rec, n, nc, na, 10000, d_res, d_cnt, d_bnd, stream=s)
        torch.cuda.synchronize()
        recs[n] = d_rec
        want[n] = (d_res.clone(), d_bnd.clone(), d_cnt.clone())
    outs = [(torch.empty(n * 64, dtype=torch.uint8, device="cuda"),
             torch.empty(coh.boundary_words(nc) * n, dtype=torch.int32, device="cuda"),
             torch.full((16,), 7, dtype=torch.int64, device="cuda")) for n in sizes]
    for k in range(launches):  # mixed / ring: > 256 launch slots
        i = k % len(sizes)
        n = sizes[i]
        ctx.eval_traces_counted(recs[n], n, nc, na, 10000, outs[i][0], outs[i][2], outs[i][1], stream=s,
                                flags=coh.BATCH_OVERLAP)
        if k % 37 == 36 or k == launches - 1:  # check the latest launch of every size
            torch.cuda.synchronize()
            for j, m in enumerate(sizes):
                assert torch.equal(outs[j][0], want[m][0]) and torch.equal(outs[j][1], want[m][1])
                assert torch.equal(outs[j][2][:11], want[m][2][:11])
    torch.cuda.synchronize()
    # the ring is clean: a plain launch after the stream counts from zero
    m = sizes[-1]
    d_cnt = torch.full((16,), 7, dtype=torch.int64, device="cuda")
    ctx.eval_traces_counted(recs[m], m, nc, na, 10000, outs[-1][0], d_cnt, outs[-1][1], stream=s)
    torch.cuda.synchronize()
    assert torch.equal(d_cnt[:11], want[m][2][:11])


@pytest.mark.parametrize("fuel,ab", [(700, None), (10000, list(range(1, 65))), (700, [4096] * 64)],
                         ids=["fuel", "bytes", "fuel_uniform_bytes"])
def test_overlap_flag_other_variants(ctx, fuel, ab):
    """COH_BATCH_OVERLAP on the kernel variants it does not change: fuel-limited batches
    (the slot store stays after the stop test) and non-uniform sizes (launched in order):
    back-to-back launches with their own outputs equal a plain launch."""
    s = torch.cuda.current_stream().cuda_stream
    n, nc, na = 30000, 256, 64
    d_rec = torch.empty(coh.records_elems(n, nc), dtype=torch.int16, device="cuda")
    ctx.gen_records(9, 0, n, nc, na, 16, d_rec, s)
    outs = [(torch.empty(n * 64, dtype=torch.uint8, device="cuda"),
             torch.empty(coh.boundary_words(nc) * n, dtype=torch.int32, device="cuda"),
             torch.zeros(16, dtype=torch.int64, device="cuda")) for _ in range(3)]
    ctx.eval_traces_counted(d_rec, n, nc, na, fuel, outs[0][0], outs[0][2], outs[0][1], array_bytes=ab, stream=s)
    for k in range(6):
        ob = outs[1 + (k & 1)]
        ctx.eval_traces_counted(d_rec, n, nc, na, fuel, ob[0], ob[2], ob[1], array_bytes=ab, stream=s,
                                flags=coh.BATCH_OVERLAP)
    torch.cuda.synchronize()
    recs = d_rec.cpu().numpy().view(np.uint16)
    want, want_b = o.orc_eval(recs, n, nc, na, fuel, ab)
    for res, bnd, cnt in outs:
        assert same(res.cpu().numpy().view(coh.RESULT_DTYPE), want)
        assert np.array_equal(bnd.cpu().numpy().view(np.uint32), want_b)
        assert torch.equal(cnt[:11], outs[0][2][:11])
