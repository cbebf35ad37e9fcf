"""General block programs and schedule sweeps: the acceptance corpus
(gen_well_declared programs, every schedule of <= max_decisions opaque answers) evaluated
with one GPU thread per run."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._ffi import CohError, lib

LEAF_DTYPE = np.dtype([("seed", "<u8"), ("schedule", "<u4"), ("sched_len", "u1"), ("status", "u1"),
                       ("blocks_done", "u1"), ("boundary_ok", "u1"), ("steps", "<u4"), ("consumed", "u1"),
                       ("overflowed", "u1"), ("stuck_key", "u1"), ("stuck_info", "u1"), ("store", "<u8")])
assert LEAF_DTYPE.itemsize == 32


class GenLimits(C.Structure):
    """GenLimits (testkit.hpp:279-287), same field order and defaults."""
    _fields_ = [("max_blocks", C.c_uint32), ("max_body_depth", C.c_uint32), ("max_vars", C.c_uint32),
                ("max_buffer_len", C.c_uint32), ("max_loop_unroll", C.c_uint32), ("allow_arrays", C.c_uint32),
                ("allow_overlaps", C.c_uint32), ("pad", C.c_uint32)]

    def __init__(self, **kw):
        d = dict(max_blocks=3, max_body_depth=2, max_vars=3, max_buffer_len=6, max_loop_unroll=2, allow_arrays=1,
                 allow_overlaps=1, pad=0)
        d.update(kw)
        super().__init__(**d)


class _Stats(C.Structure):
    _fields_ = [("programs", C.c_uint64), ("runs", C.c_uint64), ("done", C.c_uint64), ("stuck", C.c_uint64),
                ("fuel_exhausted", C.c_uint64), ("runs_with_violation", C.c_uint64), ("nodes", C.c_uint64),
                ("conflicts", C.c_uint64), ("device_ms", C.c_double), ("launches", C.c_uint64)]


class EnumStats(C.Structure):
    _fields_ = [("programs", C.c_uint64), ("done", C.c_uint64), ("stuck", C.c_uint64), ("fuel_exhausted", C.c_uint64),
                ("unsafe", C.c_uint64), ("steps", C.c_uint64)]


def _register(L):
    vp = C.c_void_p
    L.coh_enum_straight_line.restype = C.c_int
    L.coh_enum_straight_line.argtypes = [vp, C.c_uint32, C.c_int32, vp, vp, C.c_uint64]
    L.coh_gen_program_text.restype = C.c_int
    L.coh_gen_program_text.argtypes = [C.c_uint64, vp, C.c_char_p, C.c_size_t]
    L.coh_sweep.restype = C.c_int
    L.coh_sweep.argtypes = [vp, C.c_uint64, C.c_uint32, vp, C.c_uint32, C.c_int32, vp, C.c_uint64, vp]


_register(lib())


def gen_program_text(seed: int, limits: GenLimits | None = None) -> str:
    lim = limits or GenLimits()
    buf = C.create_string_buffer(1 << 16)
    rc = lib().coh_gen_program_text(seed, C.addressof(lim), buf, len(buf))
    if rc < 0:
        raise CohError(6, "program text buffer too small")
    return buf.value.decode()


def sweep(ctx, seed0: int, n_seeds: int, max_decisions: int = 6, fuel: int = 10000, leaves_cap: int = 0,
          limits: GenLimits | None = None):
    lim = limits or GenLimits()
    leaves = np.zeros(max(1, leaves_cap), LEAF_DTYPE)
    st = _Stats()
    rc = lib().coh_sweep(ctx._h, seed0, n_seeds, C.addressof(lim), max_decisions, fuel,
                         leaves.ctypes.data if leaves_cap else None, leaves_cap, C.addressof(st))
    ctx._check(rc, "coh_sweep")
    stats = {k: getattr(st, k) for k, _ in st._fields_}
    return leaves[: min(leaves_cap, stats["runs"])], stats


def enum_straight_line(ctx, max_len: int = 4, fuel: int = 16):
    """Acceptance criterion 1 on the GPU: (stats dict, per-program RunStatus array) for every
    straight-line program of length <= max_len over the ten effect forms on one scalar."""
    st = EnumStats()
    n = sum(10 ** k for k in range(max_len + 1))
    statuses = np.zeros(n, np.uint8)
    rc = lib().coh_enum_straight_line(ctx._h, max_len, fuel, C.addressof(st), statuses.ctypes.data, n)
    ctx._check(rc, "coh_enum_straight_line")
    return {k: int(getattr(st, k)) for k, _ in st._fields_}, statuses
