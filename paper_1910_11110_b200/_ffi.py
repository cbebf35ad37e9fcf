"""ctypes binding of include/cohere_b200.h (the product C ABI)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("COH_B200_LIB") or os.path.join(_HERE, "lib", "libcohere_b200.so")

COH_OK, COH_E_CONSTRUCTION, COH_E_DEFECT, COH_E_OVERLAP_CONFLICT, COH_E_CUDA, COH_E_NCCL, COH_E_ARG = range(7)
_ERR_NAMES = {
    1: "ConstructionError",
    2: "DefectError",
    3: "OverlapInferenceError",
    4: "CudaError",
    5: "NcclError",
    6: "ArgumentError",
}

# struct coh_trace_result (64 bytes)
RESULT_DTYPE = np.dtype(
    [
        ("state", "<u4", (8,)),
        ("transfer_bytes", "<u8"),
        ("steps", "<u4"),
        ("transfers", "<u4"),
        ("calls_done", "<u4"),
        ("violations", "<u4"),
        ("stuck_call", "<u4"),
        ("status", "u1"),
        ("stuck_array", "u1"),
        ("stuck_effect", "u1"),
        ("stuck_flags", "u1"),
    ]
)
assert RESULT_DTYPE.itemsize == 64

STEP_DTYPE = np.dtype([("call", "<u4"), ("rule", "u1"), ("array", "u1"), ("head", "u1"), ("delta", "u1")])
assert STEP_DTYPE.itemsize == 8

COUNTER_NAMES = (
    "stuck_traces",
    "fuel_exhausted_traces",
    "violating_traces",
    "defect_traces",
    "steps",
    "transfers",
    "transfer_bytes",
    "violating_blocks",
    "completed_blocks",
    "traces",
    "unsafe_traces",
)
BATCH_BLOCKS = 1  # COH_BATCH_BLOCKS: records carry COH_REC_CONT (multi-mode blocks)
BATCH_PACKED12 = 2  # COH_BATCH_PACKED12: host records packed 12 bits per call (coh_eval_traces_host)
BATCH_OVERLAP = 4  # COH_BATCH_OVERLAP: may start before the previous kernel on the stream ends (own outputs)
REC_CONT = 1      # COH_REC_CONT
FLAG_UNSAFE = 0x10
N_COUNTERS = len(COUNTER_NAMES)


class CohError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERR_NAMES.get(code, 'Error')} ({code}): {msg}")
        self.code = code


class _Batch(C.Structure):
    _fields_ = [
        ("records", C.c_void_p),
        ("n_traces", C.c_uint64),
        ("n_calls", C.c_uint32),
        ("n_arrays", C.c_uint32),
        ("fuel", C.c_int32),
        ("flags", C.c_uint32),
        ("array_bytes", C.c_void_p),
    ]


class _Outcome(C.Structure):
    _fields_ = [
        ("status", C.c_uint8),
        ("state_after", C.c_uint8),
        ("steps", C.c_uint8),
        ("transfers", C.c_uint8),
        ("viol_before", C.c_uint8),
        ("viol_after", C.c_uint8),
        ("stuck_effect", C.c_uint8),
        ("stuck_flags", C.c_uint8),
    ]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None


def lib():
    """Load the CUDA library; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise RuntimeError(
                f"cohere-b200 CUDA library missing at {lib_path}; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(lib_path)
        vp, u64, u32, i32, i = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_int
        sig = {
            "coh_ctx_create": (i, [i, C.POINTER(vp)]),
            "coh_ctx_destroy": (None, [vp]),
            "coh_last_error": (C.c_char_p, [vp]),
            "coh_version": (C.c_char_p, []),
            "coh_calltable_describe": (i, [u32, u32, C.POINTER(_Outcome)]),
            "coh_calltable_program": (i, [u32, C.POINTER(C.c_uint8)]),
            "coh_gen_records": (i, [vp, u64, u64, u64, u32, u32, u32, vp, vp]),
            "coh_gen_records_host": (i, [u64, u64, u64, u32, u32, u32, vp]),
            "coh_gen_records_blocks": (i, [vp, u64, u64, u64, u32, u32, u32, u32, vp, vp]),
            "coh_gen_records_blocks_host": (i, [u64, u64, u64, u32, u32, u32, u32, vp]),
            "coh_eval_traces": (i, [vp, C.POINTER(_Batch), vp, vp, vp]),
            "coh_eval_traces_host": (i, [vp, C.POINTER(_Batch), vp, vp]),
            "coh_eval_traces_counted": (i, [vp, C.POINTER(_Batch), vp, vp, vp, vp]),
            "coh_reduce_counters": (i, [vp, vp, u64, vp, vp]),
            "coh_launch_count": (u64, [vp]),
            "coh_host_alloc": (vp, [C.c_size_t]),
            "coh_host_free": (None, [vp]),
            "coh_measure_link": (i, [vp, C.c_size_t, i, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
            "coh_nccl_version": (i, [C.POINTER(i)]),
            "coh_comm_unique_id": (i, [vp]),
            "coh_comm_init_rank": (i, [vp, vp, i, i, C.POINTER(vp)]),
            "coh_comm_init_all": (i, [C.POINTER(vp), i, C.POINTER(vp)]),
            "coh_comm_destroy": (None, [vp]),
            "coh_comm_allreduce_counters": (i, [vp, vp, vp]),
            "coh_eval_traces_multi": (i, [C.POINTER(vp), i, vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                          C.POINTER(vp)]),
            "coh_shard_split": (i, [u32, u32, u64, C.POINTER(u64), C.POINTER(u64)]),
            "coh_counters_host": (i, [vp, u64, vp]),
            "coh_pack_records12": (i, [vp, u64, u32, vp]),
            "coh_trace_steps": (i, [vp, vp, u32, u32, i32, u32, vp, u32, C.POINTER(u32), C.POINTER(u32)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def make_record(array: int, kind: int, site: int, variant: int) -> int:
    """One whole-array call record (include/cohere_b200.h COH_MAKE_REC): call type in
    bits 2-7 (kind | site << 2 | variant << 3), array id in bits 8-13."""
    return ((array & 63) << 8) | ((kind & 3) << 2) | ((site & 1) << 4) | ((variant & 7) << 5)


def record_fields(recs: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """(array, kind, site, variant) of packed records."""
    r = recs.astype(np.uint32)
    return (r >> 8) & 63, (r >> 2) & 3, (r >> 4) & 1, (r >> 5) & 7


def records_elems(n_traces: int, n_calls: int) -> int:
    return ((n_calls + 7) // 8) * n_traces * 8


def boundary_words(n_calls: int) -> int:
    return (n_calls + 31) // 32


def calltable_describe(call_type: int, state: int) -> dict:
    o = _Outcome()
    rc = lib().coh_calltable_describe(call_type, state, C.byref(o))
    if rc:
        raise CohError(rc, "coh_calltable_describe")
    return o.as_dict()


def calltable_program(call_type: int) -> list[int]:
    ops = (C.c_uint8 * 8)()
    n = lib().coh_calltable_program(call_type, ops)
    if n < 0:
        raise CohError(-n, "coh_calltable_program")
    return list(ops[:n])


def gen_records_host(seed: int, trace0: int, n_traces: int, n_calls: int, n_arrays: int, adv_per1024: int) -> np.ndarray:
    out = np.zeros(records_elems(n_traces, n_calls), dtype=np.uint16)
    rc = lib().coh_gen_records_host(seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, out.ctypes.data)
    if rc:
        raise CohError(rc, "coh_gen_records_host")
    return out


def gen_records_blocks_host(seed: int, trace0: int, n_traces: int, n_calls: int, n_arrays: int, adv_per1024: int,
                            cont_per1024: int) -> np.ndarray:
    """coh_gen_records_blocks_host: the synthetic records with COH_REC_CONT block marks."""
    out = np.zeros(records_elems(n_traces, n_calls), dtype=np.uint16)
    rc = lib().coh_gen_records_blocks_host(seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, cont_per1024,
                                           out.ctypes.data)
    if rc:
        raise CohError(rc, "coh_gen_records_blocks_host")
    return out


def pack_records12(records: np.ndarray, n_traces: int, n_calls: int, out: np.ndarray | None = None) -> np.ndarray:
    """coh_pack_records12: call-major 16-bit records -> the COH_BATCH_PACKED12 host form."""
    n = ((n_calls + 7) // 8) * n_traces * 12
    if out is None:
        out = np.zeros(n, np.uint8)
    r = np.ascontiguousarray(records, dtype=np.uint16)
    rc = lib().coh_pack_records12(r.ctypes.data, n_traces, n_calls, out.ctypes.data)
    if rc:
        raise CohError(rc, "coh_pack_records12")
    return out


def _ptr(x) -> int:
    """Raw address of a torch tensor / numpy array / int."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


class Context:
    """One device context (coh_ctx): compiled call table on the device, launch geometry."""

    def __init__(self, device: int = 0):
        self._L = lib()
        h = C.c_void_p()
        rc = self._L.coh_ctx_create(device, C.byref(h))
        if rc:
            raise CohError(rc, f"coh_ctx_create(device={device}) failed (no CUDA device?)")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._L.coh_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str):
        if rc:
            msg = self._L.coh_last_error(self._h)
            raise CohError(rc, f"{what}: {msg.decode() if msg else ''}")

    @property
    def launch_count(self) -> int:
        return int(self._L.coh_launch_count(self._h))

    @staticmethod
    def _batch(records, n_traces, n_calls, n_arrays, fuel, array_bytes, flags=0):
        b = _Batch()
        b.records = _ptr(records)
        b.n_traces = n_traces
        b.n_calls = n_calls
        b.n_arrays = n_arrays
        b.fuel = fuel
        b.flags = flags
        if array_bytes is not None:
            ab = np.ascontiguousarray(np.asarray(array_bytes, dtype=np.uint64))
            b.array_bytes = ab.ctypes.data
            b._keep = ab
        else:
            b.array_bytes = None
        return b

    def gen_records(self, seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, d_records, stream=0):
        self._check(
            self._L.coh_gen_records(self._h, seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, _ptr(d_records), _ptr(stream)),
            "coh_gen_records",
        )

    def gen_records_blocks(self, seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, cont_per1024, d_records,
                           stream=0):
        self._check(self._L.coh_gen_records_blocks(self._h, seed, trace0, n_traces, n_calls, n_arrays, adv_per1024,
                                                   cont_per1024, _ptr(d_records), _ptr(stream)),
                    "coh_gen_records_blocks")

    def eval_traces(self, d_records, n_traces, n_calls, n_arrays, fuel, d_results, d_boundary=None, array_bytes=None, stream=0,
                    flags=0):
        """Device-buffer entry point (coh_eval_traces); all pointers are device addresses."""
        b = self._batch(d_records, n_traces, n_calls, n_arrays, fuel, array_bytes, flags)
        self._check(
            self._L.coh_eval_traces(self._h, C.byref(b), _ptr(d_results), _ptr(d_boundary), _ptr(stream)),
            "coh_eval_traces",
        )

    def eval_traces_counted(self, d_records, n_traces, n_calls, n_arrays, fuel, d_results, d_counters, d_boundary=None,
                            array_bytes=None, stream=0, flags=0):
        """coh_eval_traces with the COH_N_COUNTERS reduction fused into the kernel."""
        b = self._batch(d_records, n_traces, n_calls, n_arrays, fuel, array_bytes, flags)
        self._check(
            self._L.coh_eval_traces_counted(self._h, C.byref(b), _ptr(d_results), _ptr(d_boundary), _ptr(d_counters),
                                            _ptr(stream)),
            "coh_eval_traces_counted",
        )

    def eval_traces_host(self, records: np.ndarray, n_traces, n_calls, n_arrays, fuel=10000, array_bytes=None,
                         results: np.ndarray | None = None, boundary: np.ndarray | None = None, want_boundary=True,
                         flags=0):
        """Host-buffer entry point (coh_eval_traces_host): H2D, kernel and D2H inside the call."""
        if flags & BATCH_PACKED12:
            if records.dtype != np.uint8 or records.size < records_elems(n_traces, n_calls) // 8 * 12:
                raise ValueError("packed records must be uint8, 12 bytes per 8-call chunk")
        elif records.dtype != np.uint16 or records.size < records_elems(n_traces, n_calls):
            raise ValueError("records must be uint16 in the call-major interleaved layout")
        if results is None:
            results = np.zeros(n_traces, dtype=RESULT_DTYPE)
        if boundary is None and want_boundary:
            boundary = np.zeros(boundary_words(n_calls) * n_traces, dtype=np.uint32)
        b = self._batch(records, n_traces, n_calls, n_arrays, fuel, array_bytes, flags)
        self._check(
            self._L.coh_eval_traces_host(self._h, C.byref(b), _ptr(results), _ptr(boundary) if want_boundary else None),
            "coh_eval_traces_host",
        )
        return results, boundary

    def trace_steps(self, records: np.ndarray, n_calls: int, n_arrays: int, fuel: int = 10000, flags: int = 0,
                    cap: int = 1 << 16):
        """TraceMode::Full for one trace (coh_trace_steps): (steps, status); records in call
        order.  steps is a STEP_DTYPE array (call, rule, array, head, delta)."""
        r = np.ascontiguousarray(records, dtype=np.uint16)
        out = np.zeros(cap, STEP_DTYPE)
        n, st = C.c_uint32(), C.c_uint32()
        rc = self._L.coh_trace_steps(self._h, r.ctypes.data, n_calls, n_arrays, fuel, flags, out.ctypes.data, cap,
                                     C.byref(n), C.byref(st))
        if rc > 0:
            self._check(rc, "coh_trace_steps")
        return out[: min(n.value, cap)], st.value

    def measure_link(self, nbytes: int, reps: int = 3) -> tuple[float, float]:
        h2d, d2h = C.c_double(), C.c_double()
        self._check(self._L.coh_measure_link(self._h, nbytes, reps, C.byref(h2d), C.byref(d2h)), "coh_measure_link")
        return h2d.value, d2h.value

    def reduce_counters(self, d_results, n_traces, d_counters, stream=0):
        self._check(self._L.coh_reduce_counters(self._h, _ptr(d_results), n_traces, _ptr(d_counters), _ptr(stream)),
                    "coh_reduce_counters")


# ---- multi-GPU (include/cohere_b200.h "multi-GPU") --------------------------------------
COMM_ID_BYTES = 128


def shard_split(rank: int, world: int, total: int) -> tuple[int, int]:
    """(first trace id, count) of a rank's contiguous share of `total` traces (C ABI)."""
    f, n = C.c_uint64(), C.c_uint64()
    rc = lib().coh_shard_split(rank, world, total, C.byref(f), C.byref(n))
    if rc:
        raise CohError(rc, "coh_shard_split")
    return f.value, n.value


def counters_host(results: np.ndarray) -> np.ndarray:
    """The COH_N_COUNTERS vector of a host batch of coh_trace_result records (C ABI)."""
    r = np.ascontiguousarray(results)
    out = np.zeros(N_COUNTERS, np.uint64)
    rc = lib().coh_counters_host(r.ctypes.data if len(r) else None, len(r), out.ctypes.data)
    if rc:
        raise CohError(rc, "coh_counters_host")
    return out


def nccl_version() -> int | None:
    v = C.c_int()
    return v.value if lib().coh_nccl_version(C.byref(v)) == 0 else None


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * COMM_ID_BYTES)()
    rc = lib().coh_comm_unique_id(buf)
    if rc:
        raise CohError(rc, "coh_comm_unique_id (NCCL unavailable?)")
    return bytes(buf)


class Comm:
    """An NCCL communicator bound to one Context (coh_comm): the counter allreduce of the
    multi-GPU trace path."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self._h, self._L = ctx, handle, lib()

    @classmethod
    def init_rank(cls, ctx: Context, unique_id: bytes, world: int, rank: int) -> "Comm":
        h = C.c_void_p()
        idb = (C.c_uint8 * COMM_ID_BYTES).from_buffer_copy(unique_id)
        ctx._check(lib().coh_comm_init_rank(ctx._h, idb, world, rank, C.byref(h)), "coh_comm_init_rank")
        return cls(ctx, h)

    @classmethod
    def init_all(cls, ctxs: list) -> list:
        n = len(ctxs)
        hs = (C.c_void_p * n)(*[c._h.value for c in ctxs])
        out = (C.c_void_p * n)()
        ctxs[0]._check(lib().coh_comm_init_all(hs, n, out), "coh_comm_init_all")
        return [cls(c, C.c_void_p(out[d])) for d, c in enumerate(ctxs)]

    def allreduce_counters(self, d_counters, stream=0):
        self.ctx._check(self._L.coh_comm_allreduce_counters(self._h, _ptr(d_counters), _ptr(stream)),
                        "coh_comm_allreduce_counters")

    def close(self):
        if getattr(self, "_h", None):
            self._L.coh_comm_destroy(self._h)
            self._h = None


def eval_traces_multi(comms: list, shards: list, d_results: list, d_counters: list, streams: list,
                      d_boundary: list | None = None):
    """coh_eval_traces_multi: shards[d] = (d_records, n_traces, n_calls, n_arrays, fuel)."""
    n = len(comms)
    batches = (_Batch * n)()
    for d, (rec, nt, nc, na, fuel) in enumerate(shards):
        batches[d] = Context._batch(rec, nt, nc, na, fuel, None)
    arr = lambda xs: (C.c_void_p * n)(*[_ptr(x) for x in xs])  # noqa: E731
    rc = lib().coh_eval_traces_multi((C.c_void_p * n)(*[c._h.value for c in comms]), n, batches, arr(d_results),
                                     arr(d_boundary) if d_boundary is not None else None, arr(d_counters),
                                     arr(streams))
    comms[0].ctx._check(rc, "coh_eval_traces_multi")
