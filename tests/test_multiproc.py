"""World-size-2 gloo tests of the multi-GPU host logic (config C4): trace-id sharding,
per-rank evaluation, and the counter allreduce.  The per-rank evaluator here is the CPU
oracle (no GPU in this container); on the GPU box the same host code drives trace_eval."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ffi as o
import paper_1910_11110_b200 as coh
from paper_1910_11110_b200 import shard

N_PER, NC, NA, ADV, SEED = 300, 96, 16, 40, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t0, n = shard.shard_range(rank, world, N_PER)
    recs = coh.gen_records_host(SEED, t0, n, NC, NA, ADV)
    res, bnd = o.orc_eval(recs, n, NC, NA)
    cnt = torch.from_numpy(shard.counters_from_results(res).view(np.int64).copy())
    shard.allreduce_counters(cnt)
    # strong-scaling split of the same job also sums to the same counters
    f0, fn = shard.split_range(rank, world, world * N_PER)
    recs2 = coh.gen_records_host(SEED, f0, fn, NC, NA, ADV)
    res2, _ = o.orc_eval(recs2, fn, NC, NA)
    cnt2 = torch.from_numpy(shard.counters_from_results(res2).view(np.int64).copy())
    shard.allreduce_counters(cnt2)
    np.save(os.path.join(outdir, f"res{rank}.npy"), res.view(np.uint8))
    if rank == 0:
        np.save(os.path.join(outdir, "cnt.npy"), cnt.numpy())
        np.save(os.path.join(outdir, "cnt2.npy"), cnt2.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_counters_equal_single_process(world):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        total = world * N_PER
        recs = coh.gen_records_host(SEED, 0, total, NC, NA, ADV)
        res, _ = o.orc_eval(recs, total, NC, NA)
        want = shard.counters_from_results(res).view(np.int64)
        assert np.array_equal(np.load(os.path.join(d, "cnt.npy")), want)
        assert np.array_equal(np.load(os.path.join(d, "cnt2.npy")), want)
        # per-trace results of the shards are the same bytes as the unsharded run
        got = np.concatenate([np.load(os.path.join(d, f"res{r}.npy")) for r in range(world)])
        assert np.array_equal(got, res.view(np.uint8))


def test_split_range_partitions():
    for world in (1, 2, 3, 8):
        for total in (0, 1, 7, 1000, 1 << 20):
            spans = [shard.split_range(r, world, total) for r in range(world)]
            assert sum(n for _, n in spans) == total
            pos = 0
            for first, n in spans:
                assert first == pos
                pos += n


def test_results_checksum_adds_over_shards():
    """The C4 cross-G check: the checksum of a batch equals the (mod 2^64) sum of the
    checksums of any contiguous split of it, and changes when one record does."""
    import torch

    from paper_1910_11110_b200 import shard
    rng = np.random.default_rng(4)
    res = torch.from_numpy(rng.integers(0, 256, 64 * 1000, dtype=np.uint8))
    whole = shard.results_checksum(res)
    for world in (1, 2, 3, 8):
        parts = [shard.split_range(r, world, 1000) for r in range(world)]
        total = sum(shard.results_checksum(res[64 * f:64 * (f + c)]) for f, c in parts) & ((1 << 64) - 1)
        assert total == whole
    res[64 * 517 + 9] ^= 1
    assert shard.results_checksum(res) != whole


def _worker_cabi(rank, world, port, outdir):
    """The same step through the product's C ABI host entry points: coh_shard_split for
    the rank's contiguous trace ids and coh_counters_host for its counter vector (the
    vector the device kernel computes), summed over the ranks with gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = world * N_PER + 3  # ragged: the shards differ by one trace
    t0, n = coh.shard_split(rank, world, total)
    assert (t0, n) == shard.split_range(rank, world, total)
    recs = o.orc_gen(SEED, t0, n, NC, NA, ADV)
    res, _ = o.orc_eval(recs, n, NC, NA)
    mine = coh.counters_host(res)
    assert np.array_equal(mine, shard.counters_from_results(res))
    cnt = torch.from_numpy(mine.view(np.int64).copy())
    shard.allreduce_counters(cnt)
    if rank == 0:
        np.save(os.path.join(outdir, "cnt.npy"), cnt.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_cabi_sharded_counters_world2():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_cabi, args=(world, _free_port(), d), nprocs=world, join=True)
        total = world * N_PER + 3
        res, _ = o.orc_eval(o.orc_gen(SEED, 0, total, NC, NA, ADV), total, NC, NA)
        assert np.array_equal(np.load(os.path.join(d, "cnt.npy")).view(np.uint64), coh.counters_host(res))


def test_cabi_shard_split_and_errors():
    for world in (1, 2, 3, 8):
        for total in (0, 1, 7, 1000, 1 << 26):
            assert [coh.shard_split(r, world, total) for r in range(world)] == \
                [shard.split_range(r, world, total) for r in range(world)]
    with pytest.raises(coh.CohError):
        coh.shard_split(2, 2, 10)
    with pytest.raises(coh.CohError):
        coh.shard_split(0, 0, 10)
    assert np.array_equal(coh.counters_host(np.zeros(0, coh.RESULT_DTYPE)), np.zeros(len(coh.COUNTER_NAMES), np.uint64))


def test_nccl_binds_at_run_time():
    """The library loads without linking NCCL; the communicator entry points bind
    libnccl.so.2 at run time (a unique id needs no GPU)."""
    v = coh.nccl_version()
    assert v is not None and v >= 22000
    assert len(coh.comm_unique_id()) == 128
