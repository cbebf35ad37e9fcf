"""Element-granular programs (overlapping views over bit planes): ctypes structures and a
Python mirror of the reference's declaration vocabulary (buffer, views, DeclBlock with one
mode and element bodies).  Evaluation goes through coh_elem_eval (CUDA)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._ffi import CohError, lib

MAX_VIEWS = 16
READ, WRITE = 2, 3


class ElemOp(C.Structure):
    _fields_ = [("effect", C.c_uint8), ("site", C.c_uint8), ("pad", C.c_uint16), ("lo", C.c_uint32), ("hi", C.c_uint32)]


class ElemCall(C.Structure):
    _fields_ = [("view", C.c_uint32), ("kind", C.c_uint8), ("site", C.c_uint8), ("n_body", C.c_uint8),
                ("pad", C.c_uint8), ("body", ElemOp * 2)]


class ElemProgram(C.Structure):
    _fields_ = [("n_cells", C.c_uint32), ("n_views", C.c_uint32), ("view_lo", C.c_void_p), ("view_hi", C.c_void_p),
                ("n_calls", C.c_uint32), ("fuel", C.c_int32), ("calls", C.c_void_p), ("frag_seed", C.c_uint64),
                ("frag_log2", C.c_uint32), ("pad", C.c_uint32)]


class ElemResult(C.Structure):
    _fields_ = [("status", C.c_uint8), ("stuck_effect", C.c_uint8), ("stuck_flags", C.c_uint8), ("pad", C.c_uint8),
                ("stuck_call", C.c_uint32), ("stuck_index", C.c_uint32), ("calls_done", C.c_uint32),
                ("violations", C.c_uint32), ("transfers", C.c_uint32), ("steps", C.c_uint64),
                ("transfer_cells", C.c_uint64), ("n_runs", C.c_uint64), ("vpu_cells", C.c_uint64)]

    def as_tuple(self):
        return tuple(getattr(self, k) for k, _ in self._fields_ if k != "pad")


class ElemStats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("alg_bytes", C.c_uint64), ("launches", C.c_uint64), ("tiles", C.c_uint64),
                ("stages", C.c_uint32), ("pad", C.c_uint32)]


assert C.sizeof(ElemCall) == 32 and C.sizeof(ElemResult) == 56 and C.sizeof(ElemProgram) == 56


class Program:
    """One buffer `b` of n_cells, views v0..v{k-1} (absolute inclusive ranges) and calls."""

    def __init__(self, n_cells: int, view_lo, view_hi, calls, fuel: int = 10000, frag_log2: int = 0,
                 frag_seed: int = 0):
        """frag_log2 > 0: a pre-fragmented start, 2^-frag_log2 of the cells already
        coherent at (V,V) (coh_elem_program.frag_*; SURVEY §8(d) C3's rho)."""
        self.n_cells = int(n_cells)
        self.frag_log2, self.frag_seed = int(frag_log2), int(frag_seed)
        self.view_lo = np.ascontiguousarray(view_lo, dtype=np.uint32)
        self.view_hi = np.ascontiguousarray(view_hi, dtype=np.uint32)
        if isinstance(calls, C.Array):
            self.calls = calls
        else:
            self.calls = (ElemCall * max(1, len(calls)))()
            for i, c in enumerate(calls):
                view, kind, site, body = c
                x = self.calls[i]
                x.view, x.kind, x.site, x.n_body = view, kind, site, len(body)
                for k, (eff, s, lo, hi) in enumerate(body):
                    x.body[k].effect, x.body[k].site, x.body[k].lo, x.body[k].hi = eff, s, lo, hi
            self._n_calls = len(calls)
        self.n_calls = getattr(self, "_n_calls", len(self.calls))
        self.fuel = int(fuel)

    @classmethod
    def generate(cls, seed: int, prog_id: int, n_cells: int, n_views: int, n_calls: int, adv_per1024: int,
                 fuel: int = 1 << 30, frag_log2: int = 0):
        lo = np.zeros(n_views, np.uint32)
        hi = np.zeros(n_views, np.uint32)
        calls = (ElemCall * max(1, n_calls))()
        rc = lib().coh_elem_gen(seed, prog_id, n_cells, n_views, n_calls, adv_per1024, lo.ctypes.data, hi.ctypes.data,
                                C.addressof(calls))
        if rc:
            raise CohError(rc, "coh_elem_gen")
        p = cls(n_cells, lo, hi, calls, fuel, frag_log2, (seed * 0x9E3779B97F4A7C15 + prog_id) & ((1 << 64) - 1))
        p.n_calls = n_calls
        return p

    @classmethod
    def from_bytes(cls, n_cells, view_lo, view_hi, calls_bytes, n_calls, fuel):
        calls = (ElemCall * max(1, n_calls))()
        C.memmove(C.addressof(calls), bytes(calls_bytes), 32 * n_calls)
        p = cls(n_cells, view_lo, view_hi, calls, fuel)
        p.n_calls = n_calls
        return p

    def struct(self) -> ElemProgram:
        return ElemProgram(self.n_cells, len(self.view_lo), self.view_lo.ctypes.data, self.view_hi.ctypes.data,
                           self.n_calls, self.fuel, C.addressof(self.calls), self.frag_seed, self.frag_log2, 0)


def program_array(programs):
    arr = (ElemProgram * len(programs))()
    for i, p in enumerate(programs):
        arr[i] = p.struct()
    return arr


def _register(L):
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    L.coh_elem_eval.restype = C.c_int
    L.coh_elem_eval.argtypes = [vp, vp, u32, vp, vp, u32, vp, vp, u32, vp, u64, vp]
    L.coh_elem_gen.restype = C.c_int
    L.coh_elem_gen.argtypes = [u64, u64, u32, u32, u32, u32, vp, vp, vp]


_register(lib())


def elem_eval(ctx, programs, want_planes=True, runs_cap=4096, download_runs=True):
    """Evaluate element programs on the device.  Returns dict of numpy outputs.  runs_cap
    transfer ranges per program are written on the device; download_runs=False leaves
    them there (the C3 measurement: every range written, none copied to the host)."""
    n = len(programs)
    arr = program_array(programs)
    res = (ElemResult * n)()
    pw = max((p.n_cells + 31) // 32 for p in programs)
    bw = max(1, max((p.n_calls + 31) // 32 for p in programs))
    planes = np.zeros((n, 2, pw), np.uint32) if want_planes else None
    vabs = np.zeros((n, MAX_VIEWS), np.uint8)
    bnd = np.zeros((n, bw), np.uint32)
    runs = np.zeros((n, max(1, runs_cap), 2), np.uint32) if download_runs else None
    stats = ElemStats()
    rc = lib().coh_elem_eval(ctx._h, C.addressof(arr), n, C.addressof(res),
                             planes.ctypes.data if want_planes else None, pw, vabs.ctypes.data, bnd.ctypes.data, bw,
                             runs.ctypes.data if (runs_cap and download_runs) else None, runs_cap,
                             C.addressof(stats))
    ctx._check(rc, "coh_elem_eval")
    return {"results": res, "planes": planes, "view_abs": vabs, "boundary": bnd, "runs": runs, "stats": stats}
