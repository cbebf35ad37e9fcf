"""Multi-GPU sharding for config C4: traces are independent, so rank r owns
the contiguous trace-id range [r*N, (r+1)*N) and generates its records on its own device
(no scatter).  The only exchange is one allreduce (sum) of the COH_N_COUNTERS vector —
integer sums, so the result is exact and independent of rank count and order.  Element
buffers (C3) shard by buffer id the same way, with no exchange at all."""
from __future__ import annotations

import numpy as np

from ._ffi import COUNTER_NAMES

N_COUNTERS = len(COUNTER_NAMES)


def shard_range(rank: int, world: int, per_rank: int) -> tuple[int, int]:
    """(first trace id, count) of a rank's weak-scaling shard."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * per_rank, per_rank


def split_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """(first trace id, count) of a rank's strong-scaling shard of `total` traces
    (contiguous, sizes differ by at most one)."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def counters_from_results(results: np.ndarray) -> np.ndarray:
    """The COH_N_COUNTERS vector of a batch of coh_trace_result records (host side; the
    device computes the same vector inside trace_eval)."""
    st = results["status"]
    out = np.zeros(N_COUNTERS, np.uint64)
    out[0] = (st == 1).sum()
    out[1] = (st == 2).sum()
    out[2] = (results["violations"] > 0).sum()
    out[3] = (st == 3).sum()
    out[4] = results["steps"].astype(np.uint64).sum()
    out[5] = results["transfers"].astype(np.uint64).sum()
    out[6] = results["transfer_bytes"].astype(np.uint64).sum()
    out[7] = results["violations"].astype(np.uint64).sum()
    out[8] = results["calls_done"].astype(np.uint64).sum()
    out[9] = len(results)
    out[10] = ((results["stuck_flags"] & 0x10) != 0).sum()
    return out


def allreduce_counters(counters, group=None):
    """Sum the counter vector over all ranks (NCCL on GPU tensors, gloo on CPU tensors).
    `counters` is an int64 torch tensor holding the uint64 counters bit-for-bit."""
    import torch.distributed as dist

    dist.all_reduce(counters[:N_COUNTERS], op=dist.ReduceOp.SUM, group=group)
    return counters


_MIX = (0x9E3779B97F4A7C15, 0xC2B2AE3D27D4EB4F, 0x165667B19E3779F9, 0x27D4EB2F165667C5,
        0x94D049BB133111EB, 0xBF58476D1CE4E5B9, 0x2545F4914F6CDD1D, 0x5851F42D4C957F2D)


def results_checksum(d_results) -> int:
    """Order-free 64-bit checksum of a batch of coh_trace_result records on the device
    (a torch uint8 tensor): a 64-bit mix of each 64-byte record, summed with wraparound
    over the records.  Shards of any size and count add up (mod 2^64) to the value of
    the whole batch, so per-trace equality between G = 1 and G = 8 is
    one integer compare."""
    import torch

    x = d_results.view(torch.int64).view(-1, 8)
    h = torch.zeros(x.shape[0], dtype=torch.int64, device=x.device)
    for k, mul in enumerate(_MIX):
        h ^= x[:, k] * (mul - (1 << 64) if mul >= 1 << 63 else mul)
        h = h * 0x5851F42D4C957F2D + k
    return int(h.sum().item()) & ((1 << 64) - 1)
