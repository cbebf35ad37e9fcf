"""Test-side loader for the CPU oracles (oracle/).  Never imported by the product.

  oracle/_build/libcohere_oracle.so  plain-C restatement (cohere_oracle.c)
  oracle/_ref/libcohere_ref.so       the unmodified reference headers compiled in place
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# The ABI record layouts of include/cohere_b200.h, restated here so that the checker side
# (tests, the bench's reference arm) never imports or loads the product package.
RESULT_DTYPE = np.dtype(
    [("state", "<u4", (8,)), ("transfer_bytes", "<u8"), ("steps", "<u4"), ("transfers", "<u4"),
     ("calls_done", "<u4"), ("violations", "<u4"), ("stuck_call", "<u4"), ("status", "u1"),
     ("stuck_array", "u1"), ("stuck_effect", "u1"), ("stuck_flags", "u1")])
assert RESULT_DTYPE.itemsize == 64


class _Outcome(C.Structure):  # coh_call_outcome
    _fields_ = [(n, C.c_uint8) for n in ("status", "state_after", "steps", "transfers", "viol_before",
                                          "viol_after", "stuck_effect", "stuck_flags")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def records_elems(n_traces: int, n_calls: int) -> int:
    return ((n_calls + 7) // 8) * n_traces * 8


def boundary_words(n_calls: int) -> int:
    return (n_calls + 31) // 32

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libcohere_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcohere_ref.so")

_orc = None
_ref = None


def oracle():
    global _orc
    if _orc is None:
        L = C.CDLL(ORACLE_SO)
        u64, u32, i32, vp = C.c_uint64, C.c_uint32, C.c_int32, C.c_void_p
        L.orc_apply_cell.restype = C.c_int
        L.orc_apply_cell.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_leq.restype = C.c_int
        L.orc_leq.argtypes = [C.c_int, C.c_int]
        L.orc_call_outcome.restype = C.c_int
        L.orc_call_outcome.argtypes = [u32, u32, C.POINTER(_Outcome)]
        L.orc_eval_traces.restype = C.c_int
        L.orc_eval_traces.argtypes = [vp, u64, u64, u64, u32, u32, i32, vp, vp, vp]
        L.orc_eval_traces_ex.restype = C.c_int
        L.orc_eval_traces_ex.argtypes = [vp, u64, u64, u64, u32, u32, i32, vp, u32, vp, vp]
        L.orc_gen_records.restype = C.c_int
        L.orc_gen_records.argtypes = [u64, u64, u64, u32, u32, u32, vp]
        _orc = L
    return _orc


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def reference():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        u64, u32, i32, vp = C.c_uint64, C.c_uint32, C.c_int32, C.c_void_p
        L.ref_eval_traces.restype = C.c_int
        L.ref_eval_traces.argtypes = [vp, u64, u64, u64, u32, u32, i32, vp, vp, vp, C.c_int, C.c_int]
        L.ref_call_outcome.restype = C.c_int
        L.ref_call_outcome.argtypes = [u32, u32, C.POINTER(_Outcome)]
        L.ref_selfcheck.restype = C.c_int
        L.ref_selfcheck.argtypes = [vp, u64, u32, u32, i32]
        L.ref_overlap_closure.restype = C.c_int
        L.ref_overlap_closure.argtypes = [vp, u32, u32, vp, vp, u32, vp, u32, vp, vp]
        L.ref_registry_query.restype = C.c_int
        L.ref_registry_query.argtypes = [vp, u32, vp, u32, vp, u32, vp, C.c_int]
        _ref = L
    return _ref


def _ab(array_bytes):
    if array_bytes is None:
        return None, None
    a = np.ascontiguousarray(np.asarray(array_bytes, dtype=np.uint64))
    return a, a.ctypes.data


def orc_eval(records, n_total, n_calls, n_arrays, fuel=10000, array_bytes=None, t_begin=0, t_end=None, flags=0):
    t_end = n_total if t_end is None else t_end
    m = t_end - t_begin
    out = np.zeros(m, dtype=RESULT_DTYPE)
    bnd = np.zeros(boundary_words(n_calls) * m, dtype=np.uint32)
    keep, abp = _ab(array_bytes)
    rc = oracle().orc_eval_traces_ex(records.ctypes.data, n_total, t_begin, t_end, n_calls, n_arrays, fuel, abp, flags,
                                     out.ctypes.data, bnd.ctypes.data)
    assert rc == 0
    return out, bnd


def ref_eval(records, n_total, n_calls, n_arrays, fuel=10000, array_bytes=None, t_begin=0, t_end=None,
             threads=None, mode=0):
    t_end = n_total if t_end is None else t_end
    m = t_end - t_begin
    out = np.zeros(m, dtype=RESULT_DTYPE)
    bnd = np.zeros(boundary_words(n_calls) * m, dtype=np.uint32)
    keep, abp = _ab(array_bytes)
    rc = reference().ref_eval_traces(records.ctypes.data, n_total, t_begin, t_end, n_calls, n_arrays, fuel, abp,
                                     out.ctypes.data, bnd.ctypes.data, threads or os.cpu_count(), mode)
    assert rc == 0
    return out, bnd


def orc_outcome(call_type, state):
    o = _Outcome()
    oracle().orc_call_outcome(call_type, state, C.byref(o))
    return o.as_dict()


def ref_outcome(call_type, state):
    o = _Outcome()
    reference().ref_call_outcome(call_type, state, C.byref(o))
    return o.as_dict()


def orc_gen(seed, trace0, n_traces, n_calls, n_arrays, adv):
    out = np.zeros(records_elems(n_traces, n_calls), dtype=np.uint16)
    oracle().orc_gen_records(seed, trace0, n_traces, n_calls, n_arrays, adv, out.ctypes.data)
    return out


# ---- element programs -------------------------------------------------------------------
def _elem_fn(lib, name):
    f = getattr(lib, name)
    f.restype = C.c_int
    f.argtypes = [C.c_void_p] * 7 + [C.c_uint64]
    return f


def elem_run(which, program, runs_cap=4096):
    """Run one element program on the C oracle ('orc') or the reference ('ref')."""
    from paper_1910_11110_b200.elem import ElemResult

    lib_, name = (oracle(), "orc_elem_run") if which == "orc" else (reference(), "ref_elem_run")
    f = _elem_fn(lib_, name)
    st = program.struct()
    r = ElemResult()
    pw = (program.n_cells + 31) // 32
    L = np.zeros(pw, np.uint32)
    R = np.zeros(pw, np.uint32)
    va = np.zeros(16, np.uint8)
    b = np.zeros(max(1, (program.n_calls + 31) // 32), np.uint32)
    runs = np.zeros((max(1, runs_cap), 2), np.uint32)
    rc = f(C.addressof(st), C.addressof(r), L.ctypes.data, R.ctypes.data, va.ctypes.data, b.ctypes.data,
           runs.ctypes.data, runs_cap)
    return rc, r, L, R, va, b, runs[: min(r.n_runs, runs_cap)]


# ---- general programs / sweeps ----------------------------------------------------------
def ref_program_text(seed):
    L = reference()
    L.ref_gen_program_text.restype = C.c_int
    L.ref_gen_program_text.argtypes = [C.c_uint64, C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(1 << 16)
    assert L.ref_gen_program_text(seed, buf, len(buf)) == 0
    return buf.value.decode()


def ref_sweep_leaves(seed0, n, max_dec=6, fuel=10000, cap=1 << 20):
    from paper_1910_11110_b200.sweep import LEAF_DTYPE

    L = reference()
    L.ref_sweep_leaves.restype = C.c_int64
    L.ref_sweep_leaves.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32, C.c_void_p, C.c_uint64]
    out = np.zeros(cap, LEAF_DTYPE)
    got = L.ref_sweep_leaves(seed0, n, max_dec, fuel, out.ctypes.data, cap)
    assert 0 <= got <= cap
    return out[:got]


def ref_sweep_stats(seed0, n, max_dec=6, fuel=10000):
    L = reference()
    L.ref_sweep_stats.restype = C.c_int
    L.ref_sweep_stats.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32, C.c_void_p]
    out = np.zeros(6, np.uint64)
    L.ref_sweep_stats(seed0, n, max_dec, fuel, out.ctypes.data)
    return dict(zip(["runs", "done", "stuck", "fuel_exhausted", "bad_boundary_programs", "oracle_disagreements"],
                    (int(x) for x in out)))


def add_blocks(records, n_traces, n_calls, cont_per1024, seed, dup_per1024=0):
    """Multi-mode blocks for tests: set COH_REC_CONT (bit 0) on call i > 0 of each trace with
    probability cont_per1024/1024 when its array is not yet in the current block (and, with
    probability dup_per1024/1024, even when it is: a construction defect)."""
    rng = np.random.default_rng(seed)
    r = records.copy().reshape(-1, n_traces, 8)
    for t in range(n_traces):
        cur = set()
        for i in range(n_calls):
            c, k = divmod(i, 8)
            a = (int(r[c, t, k]) >> 8) & 63
            if i > 0 and rng.integers(0, 1024) < cont_per1024 and (a not in cur or rng.integers(0, 1024) < dup_per1024):
                r[c, t, k] |= 1
                cur.add(a)
            else:
                cur = {a}
    return r.reshape(-1)


STEP_DTYPE = np.dtype([("call", "<u4"), ("rule", "u1"), ("array", "u1"), ("head", "u1"), ("delta", "u1")])


def ref_trace_steps(records, n_calls, n_arrays, fuel=10000, flags=0, cap=1 << 16):
    """The reference's TraceMode::Full step list of one trace (records in call order)."""
    L = reference()
    L.ref_trace_steps.restype = C.c_int
    L.ref_trace_steps.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_int32, C.c_uint32, C.c_void_p, C.c_uint32,
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    out = np.zeros(cap, STEP_DTYPE)
    n, st = C.c_uint32(), C.c_uint32()
    r = np.ascontiguousarray(records, dtype=np.uint16)
    assert L.ref_trace_steps(r.ctypes.data, n_calls, n_arrays, fuel, flags, out.ctypes.data, cap, C.byref(n), C.byref(st)) == 0
    return out[: min(n.value, cap)], st.value
