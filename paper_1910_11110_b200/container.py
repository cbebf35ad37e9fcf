"""Coherent containers (VectorPU-style API on the calculus, config C5).

    rt = Runtime(ctx)
    x = rt.vector(1 << 28)                 # float32, pinned host + device copies
    rt.call("gpu", [(x, "W")])             # GW(x): built-in GPU component
    rt.call("cpu", [(x, "R"), (y, "RW")])  # R(x), RW(y) on the CPU: downloads x first
    rt.stats()                             # bytes really moved by cudaMemcpyAsync
    rt.predicted_bytes()                   # the evaluator's prediction for the same calls

Modes follow PAPER.md Table 1: R/W/RW on the host, GR/GW/GRW on the device."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _ffi
from ._ffi import CohError, lib

KIND = {"R": 0, "W": 1, "RW": 2}
SITE = {"cpu": 0, "local": 0, "gpu": 1, "remote": 1}


class _Arg(C.Structure):
    _fields_ = [("vec", C.c_uint32), ("kind", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("h2d_copies", C.c_uint64),
                ("d2h_copies", C.c_uint64), ("calls", C.c_uint64), ("syncs_elided", C.c_uint64),
                ("stuck_calls", C.c_uint64), ("copy_ms", C.c_double)]


class _Touch(C.Structure):
    _fields_ = [("rt", C.c_void_p), ("n", C.c_uint32), ("vec", C.c_uint32 * 8), ("kind", C.c_uint32 * 8),
                ("bytes", C.c_uint64 * 8), ("checksum", C.c_double)]


def _register(L):
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    L.coh_rt_create.restype = C.c_int
    L.coh_rt_create.argtypes = [vp, C.POINTER(vp)]
    L.coh_rt_destroy.restype = None
    L.coh_rt_destroy.argtypes = [vp]
    L.coh_rt_vector.restype = C.c_int
    L.coh_rt_vector.argtypes = [vp, C.c_size_t, C.POINTER(u32)]
    L.coh_rt_host_ptr.restype = vp
    L.coh_rt_host_ptr.argtypes = [vp, u32]
    L.coh_rt_device_ptr.restype = vp
    L.coh_rt_device_ptr.argtypes = [vp, u32]
    L.coh_rt_state.restype = C.c_int
    L.coh_rt_state.argtypes = [vp, u32, C.POINTER(C.c_uint8)]
    L.coh_rt_call.restype = C.c_int
    L.coh_rt_call.argtypes = [vp, u32, vp, u32, vp, vp]
    L.coh_rt_sync.restype = C.c_int
    L.coh_rt_sync.argtypes = [vp]
    L.coh_rt_get_stats.restype = C.c_int
    L.coh_rt_get_stats.argtypes = [vp, vp]
    L.coh_rt_set_async.restype = C.c_int
    L.coh_rt_set_async.argtypes = [vp, C.c_int]


def _register_views(L):
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    L.coh_rt_buffer.restype = C.c_int
    L.coh_rt_buffer.argtypes = [vp, u32, u32, C.POINTER(u32)]
    L.coh_rt_view.restype = C.c_int
    L.coh_rt_view.argtypes = [vp, u32, u32, u32, C.POINTER(u32)]
    L.coh_rt_call_view.restype = C.c_int
    L.coh_rt_call_view.argtypes = [vp, u32, vp, vp, vp]
    L.coh_rt_view_state.restype = C.c_int
    L.coh_rt_view_state.argtypes = [vp, u32, u32, C.POINTER(C.c_uint8)]
    L.coh_rt_buffer_planes.restype = C.c_int
    L.coh_rt_buffer_planes.argtypes = [vp, u32, vp]
    L.coh_rt_buffer_host_ptr.restype = vp
    L.coh_rt_buffer_host_ptr.argtypes = [vp, u32]
    L.coh_rt_buffer_device_ptr.restype = vp
    L.coh_rt_buffer_device_ptr.argtypes = [vp, u32]
    L.coh_rt_copy_log.restype = C.c_int
    L.coh_rt_copy_log.argtypes = [vp, vp, u64, C.POINTER(u64)]


_register(lib())
_register_views(lib())
COPY_DTYPE = np.dtype([("buffer", "<u4"), ("first", "<u4"), ("last", "<u4"), ("h2d", "<u4")])
_TOUCH = {0: C.cast(lib().coh_rt_touch_cpu, C.c_void_p).value, 1: C.cast(lib().coh_rt_touch_gpu, C.c_void_p).value}


class Vector:
    def __init__(self, rt, vid, nbytes):
        self.rt, self.id, self.nbytes = rt, vid, nbytes

    @property
    def host(self) -> np.ndarray:
        """float32 view of the pinned host copy (valid only where the runtime says so)."""
        p = lib().coh_rt_host_ptr(self.rt._h, self.id)
        return np.ctypeslib.as_array((C.c_float * (self.nbytes // 4)).from_address(p))

    @property
    def device_ptr(self) -> int:
        return lib().coh_rt_device_ptr(self.rt._h, self.id)

    def state(self) -> int:
        s = C.c_uint8()
        lib().coh_rt_state(self.rt._h, self.id, C.byref(s))
        return s.value


class Buffer:
    """A mother vector with element-granular validity and views (pvector<T>(mother, lo,
    hi)): calls are coh_elem_call records on its views, executed with
    the copies of exactly the cells the element evaluator predicts."""

    def __init__(self, rt, bid, n_cells, elem_bytes):
        self.rt, self.id, self.n_cells, self.elem_bytes = rt, bid, n_cells, elem_bytes
        self.views: list[tuple[int, int]] = []

    def view(self, lo: int, hi: int) -> int:
        vi = C.c_uint32()
        self.rt.ctx._check(lib().coh_rt_view(self.rt._h, self.id, lo, hi, C.byref(vi)), "coh_rt_view")
        self.views.append((lo, hi))
        return vi.value

    def call(self, call, component=None):
        """One component call (an elem.ElemCall on this buffer's views); component: None
        (coherence only) or (fn pointer, user pointer).  Raises CohError when stuck."""
        fn, user = component if component is not None else (None, None)
        self.rt.ctx._check(lib().coh_rt_call_view(self.rt._h, self.id, C.addressof(call), fn, user), "coh_rt_call_view")

    def view_state(self, v: int) -> int:
        s = C.c_uint8()
        lib().coh_rt_view_state(self.rt._h, self.id, v, C.byref(s))
        return s.value

    def planes(self) -> np.ndarray:
        w = (self.n_cells + 31) // 32
        out = np.zeros((2, w), np.uint32)
        self.rt.ctx._check(lib().coh_rt_buffer_planes(self.rt._h, self.id, out.ctypes.data), "coh_rt_buffer_planes")
        return out

    @property
    def host(self) -> np.ndarray:
        p = lib().coh_rt_buffer_host_ptr(self.rt._h, self.id)
        return np.ctypeslib.as_array((C.c_uint8 * (self.n_cells * self.elem_bytes)).from_address(p))

    @property
    def device_ptr(self) -> int:
        return lib().coh_rt_buffer_device_ptr(self.rt._h, self.id)


class Runtime:
    def __init__(self, ctx: "_ffi.Context"):
        self.ctx = ctx
        h = C.c_void_p()
        rc = lib().coh_rt_create(ctx._h, C.byref(h))
        if rc:
            raise CohError(rc, "coh_rt_create")
        self._h = h
        self._keep: list = []  # component user data, kept until sync
        self.vectors: list[Vector] = []
        self.log: list[tuple[int, list[tuple[int, int]]]] = []   # (site, [(vec, kind)]) per call

    def close(self):
        if getattr(self, "_h", None):
            lib().coh_rt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def vector(self, n_floats: int) -> Vector:
        nbytes = 4 * int(n_floats)
        if nbytes % 16:
            raise ValueError("vectors are multiples of 4 floats")
        vid = C.c_uint32()
        self.ctx._check(lib().coh_rt_vector(self._h, nbytes, C.byref(vid)), "coh_rt_vector")
        v = Vector(self, vid.value, nbytes)
        self.vectors.append(v)
        return v

    def call(self, site: str, args, component="builtin"):
        """One component call: args = [(Vector, "R"|"W"|"RW"), ...]; component "builtin"
        (trivial CPU loop / GPU kernel), None (coherence only) or a ctypes-compatible
        function pointer taking (void* user, void* stream)."""
        s = SITE[site]
        arr = (_Arg * max(1, len(args)))()
        for i, (v, k) in enumerate(args):
            arr[i].vec, arr[i].kind = v.id, KIND[k]
        fn, user = None, None
        if component == "builtin":
            t = _Touch()
            t.rt, t.n = self._h, len(args)
            for i, (v, k) in enumerate(args):
                t.vec[i], t.kind[i], t.bytes[i] = v.id, KIND[k], v.nbytes
            fn, user = _TOUCH[s], C.addressof(t)
            self._keep.append(t)  # stays valid until sync (asynchronous CPU components)
        elif component is not None:
            fn, user = component
        rc = lib().coh_rt_call(self._h, s, C.addressof(arr), len(args), fn, user)
        self.ctx._check(rc, "coh_rt_call")
        self.log.append((s, [(v.id, KIND[k]) for v, k in args]))

    def buffer(self, n_cells: int, elem_bytes: int = 4) -> Buffer:
        bid = C.c_uint32()
        self.ctx._check(lib().coh_rt_buffer(self._h, n_cells, elem_bytes, C.byref(bid)), "coh_rt_buffer")
        return Buffer(self, bid.value, n_cells, elem_bytes)

    def copy_log(self) -> np.ndarray:
        """Every copy issued so far (COPY_DTYPE: buffer, first / last cell, h2d)."""
        n = C.c_uint64()
        lib().coh_rt_copy_log(self._h, None, 0, C.byref(n))
        out = np.zeros(n.value, COPY_DTYPE)
        if n.value:
            lib().coh_rt_copy_log(self._h, out.ctypes.data, n.value, C.byref(n))
        return out

    def sync(self):
        self.ctx._check(lib().coh_rt_sync(self._h), "coh_rt_sync")
        self._keep = []

    def set_async(self, on: bool = True):
        """CPU components as stream-ordered host functions (coh_rt_set_async): calls return
        at once; host data is final after sync()."""
        self.ctx._check(lib().coh_rt_set_async(self._h, int(on)), "coh_rt_set_async")

    def stats(self) -> dict:
        st = _Stats()
        lib().coh_rt_get_stats(self._h, C.addressof(st))
        return {k: (float if k == "copy_ms" else int)(getattr(st, k)) for k, _ in st._fields_}

    def records(self) -> np.ndarray:
        """The executed calls as one whole-array trace (include/cohere_b200.h records):
        each (vector, mode) argument becomes one canonical-body call record (a
        multi-argument block is split into single-mode blocks; for canonical bodies the
        copies are identical)."""
        recs = [_ffi.make_record(a, k, s, 0) for s, args in self.log for a, k in args]
        n = len(recs)
        out = np.zeros(_ffi.records_elems(1, n), np.uint16)
        out[:n] = recs  # one trace: record i at [(i/8)*1 + 0]*8 + i%8 == i
        return out, n

    def predicted(self):
        """Evaluator prediction (coh_eval_traces_host on the GPU) for the executed calls."""
        recs, n = self.records()
        nv = len(self.vectors)
        res, _ = self.ctx.eval_traces_host(recs, 1, n, max(1, nv), fuel=1 << 30,
                                           array_bytes=[v.nbytes for v in self.vectors] or None,
                                           want_boundary=False)
        return res[0]
