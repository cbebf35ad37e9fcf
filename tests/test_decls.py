"""Declarations (program.hpp:141-226) through the C ABI: arrays with byte sizes and
buffers with views, numbered in declaration order, filling a trace batch and an element
program; construction defects are ConstructionError (COH_E_CONSTRUCTION).  Host only."""
import ctypes as C

import numpy as np

from paper_1910_11110_b200._ffi import COH_E_CONSTRUCTION, lib


class Batch(C.Structure):  # coh_trace_batch
    _fields_ = [("records", C.c_void_p), ("n_traces", C.c_uint64), ("n_calls", C.c_uint32),
                ("n_arrays", C.c_uint32), ("fuel", C.c_int32), ("flags", C.c_uint32),
                ("array_bytes", C.c_void_p)]


class Prog(C.Structure):  # coh_elem_program
    _fields_ = [("n_cells", C.c_uint32), ("n_views", C.c_uint32), ("view_lo", C.c_void_p), ("view_hi", C.c_void_p),
                ("n_calls", C.c_uint32), ("fuel", C.c_int32), ("calls", C.c_void_p), ("frag_seed", C.c_uint64),
                ("frag_log2", C.c_uint32), ("pad", C.c_uint32)]


def _lib():
    L = lib()
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    L.coh_decls_create.argtypes = [C.POINTER(vp)]
    L.coh_decls_destroy.argtypes = [vp]
    L.coh_decls_destroy.restype = None
    L.coh_decls_error.argtypes = [vp]
    L.coh_decls_error.restype = C.c_char_p
    L.coh_decls_array.argtypes = [vp, u64, C.POINTER(u32)]
    L.coh_decls_buffer.argtypes = [vp, u32, C.POINTER(u32)]
    L.coh_decls_view.argtypes = [vp, u32, u32, u32, C.POINTER(u32)]
    L.coh_decls_trace_batch.argtypes = [vp, vp]
    L.coh_decls_elem_program.argtypes = [vp, u32, vp]
    return L


def test_decls_fill_batch_and_program():
    L = _lib()
    d = C.c_void_p()
    assert L.coh_decls_create(C.byref(d)) == 0
    try:
        i = C.c_uint32()
        for k, nb in enumerate((4, 8, 4096)):
            assert L.coh_decls_array(d, nb, C.byref(i)) == 0 and i.value == k
        b = Batch()
        assert L.coh_decls_trace_batch(d, C.byref(b)) == 0
        assert b.n_arrays == 3
        assert list(np.ctypeslib.as_array((C.c_uint64 * 3).from_address(b.array_bytes))) == [4, 8, 4096]
        buf = C.c_uint32()
        assert L.coh_decls_buffer(d, 100, C.byref(buf)) == 0
        for lo, hi, want in ((0, 49, 0), (40, 99, 1)):
            assert L.coh_decls_view(d, buf, lo, hi, C.byref(i)) == 0 and i.value == want
        p = Prog()
        assert L.coh_decls_elem_program(d, buf, C.byref(p)) == 0
        assert (p.n_cells, p.n_views) == (100, 2)
        assert list(np.ctypeslib.as_array((C.c_uint32 * 2).from_address(p.view_hi))) == [49, 99]
        # construction defects (program.hpp:57-68)
        assert L.coh_decls_view(d, buf, 60, 100, C.byref(i)) == COH_E_CONSTRUCTION
        assert b"fit" in L.coh_decls_error(d)
        assert L.coh_decls_view(d, buf, 9, 3, C.byref(i)) == COH_E_CONSTRUCTION
        assert L.coh_decls_buffer(d, 0, C.byref(i)) == COH_E_CONSTRUCTION
        for _ in range(61):
            assert L.coh_decls_array(d, 1, C.byref(i)) == 0
        assert L.coh_decls_array(d, 1, C.byref(i)) == COH_E_CONSTRUCTION  # the 65th
    finally:
        L.coh_decls_destroy(d)
