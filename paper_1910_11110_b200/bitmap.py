"""Bit-plane primitives over device planes: range set / clear, first
zero, zero-run extraction and the per-view abstraction check (include/cohere_b200.h
coh_bitmap_*).  Planes are int32 torch tensors on the device (torch is the allocator);
ranges are RANGE_DTYPE records."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._ffi import lib

RANGE_DTYPE = np.dtype([("word_off", "<u8"), ("lo", "<u4"), ("hi", "<u4")])


def _register(L):
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    for name in ("coh_bitmap_range_set", "coh_bitmap_range_clear"):
        getattr(L, name).restype = C.c_int
        getattr(L, name).argtypes = [vp, vp, vp, u32, vp]
    L.coh_bitmap_first_zero.restype = C.c_int
    L.coh_bitmap_first_zero.argtypes = [vp, vp, vp, u32, vp, vp]
    L.coh_bitmap_extract_zero_runs.restype = C.c_int
    L.coh_bitmap_extract_zero_runs.argtypes = [vp, vp, vp, u32, vp, vp, u64, vp, vp]
    L.coh_bitmap_view_check.restype = C.c_int
    L.coh_bitmap_view_check.argtypes = [vp, vp, vp, vp, vp, u32, vp, vp]


_register(lib())


def _ranges(ranges: np.ndarray):
    import torch
    assert ranges.dtype == RANGE_DTYPE
    return torch.from_numpy(np.ascontiguousarray(ranges).view(np.uint8).copy()).cuda()


def range_set(ctx, words, ranges: np.ndarray, value: bool = True, stream: int = 0):
    fn = lib().coh_bitmap_range_set if value else lib().coh_bitmap_range_clear
    d = _ranges(ranges)
    ctx._check(fn(ctx._h, words.data_ptr(), d.data_ptr(), len(ranges), stream), "coh_bitmap_range_set/clear")


def first_zero(ctx, words, ranges: np.ndarray, stream: int = 0) -> np.ndarray:
    import torch
    d = _ranges(ranges)
    out = torch.empty(max(1, len(ranges)), dtype=torch.int32, device="cuda")
    ctx._check(lib().coh_bitmap_first_zero(ctx._h, words.data_ptr(), d.data_ptr(), len(ranges), out.data_ptr(), stream),
               "coh_bitmap_first_zero")
    torch.cuda.synchronize()
    return out.cpu().numpy()[: len(ranges)].view(np.uint32)


def zero_runs(ctx, words, ranges: np.ndarray, cap: int = 1 << 20, stream: int = 0):
    """(run_off [n+1], starts, ends): runs of range k are starts/ends[run_off[k]:run_off[k+1]]."""
    import torch
    d = _ranges(ranges)
    st = torch.empty(max(1, cap), dtype=torch.int32, device="cuda")
    en = torch.empty(max(1, cap), dtype=torch.int32, device="cuda")
    off = torch.empty(len(ranges) + 1, dtype=torch.int64, device="cuda")
    ctx._check(lib().coh_bitmap_extract_zero_runs(ctx._h, words.data_ptr(), d.data_ptr(), len(ranges), st.data_ptr(),
                                                  en.data_ptr(), cap, off.data_ptr(), stream),
               "coh_bitmap_extract_zero_runs")
    torch.cuda.synchronize()
    o = off.cpu().numpy().view(np.uint64)
    m = int(min(o[-1], cap))
    return o, st.cpu().numpy()[:m].view(np.uint32), en.cpu().numpy()[:m].view(np.uint32)


def view_check(ctx, L, R, ranges: np.ndarray, abs_pair: np.ndarray, stream: int = 0) -> np.ndarray:
    import torch
    d = _ranges(ranges)
    a = torch.from_numpy(np.ascontiguousarray(abs_pair, np.uint8)).cuda()
    ok = torch.empty(max(1, len(ranges)), dtype=torch.uint8, device="cuda")
    ctx._check(lib().coh_bitmap_view_check(ctx._h, L.data_ptr(), R.data_ptr(), d.data_ptr(), a.data_ptr(), len(ranges),
                                           ok.data_ptr(), stream), "coh_bitmap_view_check")
    torch.cuda.synchronize()
    return ok.cpu().numpy()[: len(ranges)].astype(bool)
