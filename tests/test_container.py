"""Container runtime (config C5): real cudaMemcpyAsync traffic equals the evaluator's
prediction (GPU kernel and CPU oracle) for random call chains; data really moves."""
import numpy as np
import pytest

import oracle_ffi as o

pytestmark = pytest.mark.gpu


def _rt(ctx):
    from paper_1910_11110_b200.container import Runtime

    return Runtime(ctx)


def test_paper_example_chain(ctx):
    # foo(R(vx), W(vy), RW(vz)) on the CPU after a GPU producer (PAPER.md:280-290 style)
    rt = _rt(ctx)
    x, y, z = (rt.vector(1 << 20) for _ in range(3))
    rt.call("gpu", [(x, "W"), (z, "RW")])   # GW(x), GRW(z): z uploaded first
    rt.call("cpu", [(x, "R"), (y, "W"), (z, "RW")])  # x, z downloaded
    rt.call("gpu", [(y, "R")])              # y uploaded
    rt.sync()
    st = rt.stats()
    assert st["h2d_copies"] == 2 and st["d2h_copies"] == 2
    assert np.all(x.host[:8] == 1.0)  # the GPU write of x came back to the host
    pred = rt.predicted()
    assert pred["transfer_bytes"] == st["h2d_bytes"] + st["d2h_bytes"]
    assert pred["status"] == 0 and pred["violations"] == 0


def test_random_chains_bytes_equal_prediction(ctx):
    rng = np.random.default_rng(7)
    for trial in range(6):
        rt = _rt(ctx)
        vecs = [rt.vector(int(rng.choice([1 << 12, 1 << 16, 1 << 18]))) for _ in range(4)]
        for _ in range(40):
            k = int(rng.integers(1, 4))
            idx = rng.choice(len(vecs), size=k, replace=False)
            site = "gpu" if rng.random() < 0.5 else "cpu"
            rt.call(site, [(vecs[i], ["R", "W", "RW"][int(rng.integers(0, 3))]) for i in idx])
        rt.sync()
        st = rt.stats()
        pred = rt.predicted()
        assert pred["transfer_bytes"] == st["h2d_bytes"] + st["d2h_bytes"], trial
        assert pred["transfers"] == st["h2d_copies"] + st["d2h_copies"], trial
        # the CPU oracle predicts the same
        recs, n = rt.records()
        want, _ = o.orc_eval(recs, 1, n, len(vecs), 1 << 30, [v.nbytes for v in vecs])
        assert want[0]["transfer_bytes"] == pred["transfer_bytes"]
        # runtime state == evaluator final store, per vector
        for v in vecs:
            nib = (int(pred["state"][v.id // 8]) >> (4 * (v.id % 8))) & 15
            assert v.state() == nib


def test_values_flow_between_sites(ctx):
    rt = _rt(ctx)
    x = rt.vector(1 << 16)
    rt.call("cpu", [(x, "W")])           # host: x = 1
    rt.call("gpu", [(x, "RW")])          # upload, device: x = 1.5
    rt.call("cpu", [(x, "RW")])          # download, host: x = 1.75
    rt.sync()
    assert np.allclose(x.host, 1.75)
    assert rt.stats()["h2d_copies"] == 1 and rt.stats()["d2h_copies"] == 1


def test_declared_twice_is_construction_error(ctx):
    import paper_1910_11110_b200 as coh

    rt = _rt(ctx)
    x = rt.vector(64)
    with pytest.raises(coh.CohError) as e:
        rt.call("cpu", [(x, "R"), (x, "W")])
    assert e.value.code == 1


@pytest.mark.parametrize("seed", [3, 11])
def test_async_host_components_same_data_and_bytes(ctx, seed):
    """Side streams + stream-ordered CPU components (coh_rt_set_async) reorder nothing the
    calculus orders: the same chain leaves byte-identical host and device data and moves
    exactly the same bytes as the synchronous runtime, equal to the evaluator's
    prediction."""
    import torch

    from paper_1910_11110_b200.container import Runtime

    outs = []
    for mode in (False, True):
        rng = np.random.default_rng(seed)
        rt = Runtime(ctx)
        if mode:
            rt.set_async(True)
        vecs = [rt.vector(1 << 22) for _ in range(4)]
        for _ in range(48):
            k = int(rng.integers(1, 4))
            idx = rng.choice(4, size=k, replace=False)
            site = "gpu" if rng.random() < 0.5 else "cpu"
            rt.call(site, [(vecs[i], ["R", "W", "RW"][int(rng.integers(0, 3))]) for i in idx])
        for v in vecs:  # bring every vector to the host (CPU reads)
            rt.call("cpu", [(v, "R")])
        rt.sync()
        st = rt.stats()
        pred = rt.predicted()
        assert pred["transfer_bytes"] == st["h2d_bytes"] + st["d2h_bytes"]
        outs.append(([v.host.copy() for v in vecs], st["h2d_bytes"], st["d2h_bytes"]))
        rt.close()
    (h0, u0, d0), (h1, u1, d1) = outs
    assert (u0, d0) == (u1, d1)
    for a, b in zip(h0, h1):
        assert np.array_equal(a, b)
    del torch
