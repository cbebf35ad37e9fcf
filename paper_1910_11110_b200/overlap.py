"""Batched overlap registry and mode closure on the GPU: the
reference's OverlapRegistry::query and infer_overlap_closure (overlap.hpp:33-244) over
many views and many blocks at once.  Views and modes are numpy records (VIEW_DTYPE,
MODE_DTYPE = coh_view / coh_mode of include/cohere_b200.h); torch is only the device
allocator."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._ffi import CohError, lib

VIEW_DTYPE = np.dtype([("buffer", "<u4"), ("lo", "<i4"), ("hi", "<i4"), ("name_rank", "<u4")])
MODE_DTYPE = np.dtype([("var", "<u4"), ("kind", "u1"), ("site", "u1"), ("flags", "u1"), ("pad", "u1")])
FLAG_VIEW, FLAG_SHADOW = 1, 2
STATUS_OK, STATUS_LIMIT = -1, -2


def _register(L):
    vp, u32 = C.c_void_p, C.c_uint32
    L.coh_registry_build.restype = C.c_int
    L.coh_registry_build.argtypes = [vp, vp, u32, C.POINTER(vp), vp]
    L.coh_registry_destroy.restype = None
    L.coh_registry_destroy.argtypes = [vp]
    L.coh_registry_query.restype = C.c_int
    L.coh_registry_query.argtypes = [vp, vp, vp, u32, vp, u32, vp, vp]
    L.coh_overlap_closure.restype = C.c_int
    L.coh_overlap_closure.argtypes = [vp, vp, vp, vp, u32, vp, u32, vp, vp, vp]


_register(lib())


def _dev(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).cuda()


class Registry:
    """build_registry over `views` (VIEW_DTYPE, declaration order = index) on ctx's device."""

    def __init__(self, ctx, views: np.ndarray, stream: int = 0):
        assert views.dtype == VIEW_DTYPE
        self.ctx, self.n = ctx, len(views)
        self._views = _dev(views)
        h = C.c_void_p()
        rc = lib().coh_registry_build(ctx._h, self._views.data_ptr() if self.n else None, self.n, C.byref(h), stream)
        ctx._check(rc, "coh_registry_build")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().coh_registry_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, probes: np.ndarray, stride: int = 64, stream: int = 0):
        """(hits [n, stride] name-sorted, counts [n]) of OverlapRegistry::query(view)."""
        import torch
        n = len(probes)
        d_p = torch.from_numpy(np.ascontiguousarray(probes, np.uint32).view(np.int32)).cuda()
        d_h = torch.zeros(max(1, n * stride), dtype=torch.int32, device="cuda")
        d_c = torch.zeros(max(1, n), dtype=torch.int32, device="cuda")
        rc = lib().coh_registry_query(self.ctx._h, self._h, d_p.data_ptr(), n, d_h.data_ptr(), stride, d_c.data_ptr(),
                                      stream)
        self.ctx._check(rc, "coh_registry_query")
        torch.cuda.synchronize()
        return d_h.cpu().numpy()[: n * stride].view(np.uint32).reshape(n, stride), d_c.cpu().numpy()[:n].view(np.uint32)

    def closure(self, modes: np.ndarray, block_off: np.ndarray, stride: int = 32, stream: int = 0):
        """(out [n_blocks, stride] MODE_DTYPE, counts, status) of infer_overlap_closure per block."""
        import torch
        assert modes.dtype == MODE_DTYPE
        nb = len(block_off) - 1
        d_m = _dev(modes) if len(modes) else torch.zeros(8, dtype=torch.uint8, device="cuda")
        d_o = torch.from_numpy(np.ascontiguousarray(block_off, np.uint32).view(np.int32)).cuda()
        d_out = torch.zeros(max(1, nb * stride) * 8, dtype=torch.uint8, device="cuda")
        d_cnt = torch.zeros(max(1, nb), dtype=torch.int32, device="cuda")
        d_st = torch.zeros(max(1, nb), dtype=torch.int32, device="cuda")
        rc = lib().coh_overlap_closure(self.ctx._h, self._h, d_m.data_ptr(), d_o.data_ptr(), nb, d_out.data_ptr(), stride,
                                       d_cnt.data_ptr(), d_st.data_ptr(), stream)
        self.ctx._check(rc, "coh_overlap_closure")
        torch.cuda.synchronize()
        out = d_out.cpu().numpy()[: nb * stride * 8].view(MODE_DTYPE).reshape(nb, stride)
        return out, d_cnt.cpu().numpy()[:nb].view(np.uint32), d_st.cpu().numpy()[:nb]


def gen_workload(seed: int, n_buffers: int, buf_len: int, n_views: int, n_blocks: int, modes_per_block: int,
                 n_scalars: int = 4, max_view_len: int | None = None, p_same_site: float = 0.85):
    """Synthetic registry + blocks: views with random names (name order != declaration
    order), intervals of length 1..max_view_len, blocks whose modes pick views of one
    buffer (so they overlap), kinds R/W/RW, mostly one site per block (some conflicts)."""
    rng = np.random.default_rng(seed)
    mvl = max_view_len or buf_len
    views = np.zeros(n_views, VIEW_DTYPE)
    views["buffer"] = rng.integers(0, n_buffers, n_views)
    ln = rng.integers(1, mvl + 1, n_views)
    views["lo"] = rng.integers(0, buf_len, n_views)
    views["hi"] = np.minimum(views["lo"] + ln - 1, buf_len - 1)
    views["name_rank"] = rng.permutation(n_views)
    by_buf = [np.nonzero(views["buffer"] == b)[0] for b in range(n_buffers)]
    modes, off = [], [0]
    for _ in range(n_blocks):
        b = int(rng.integers(0, n_buffers))
        pool = by_buf[b] if len(by_buf[b]) else np.arange(n_views)
        k = int(rng.integers(1, modes_per_block + 1))
        chosen = rng.choice(pool, size=min(k, len(pool)), replace=False)
        site0 = int(rng.integers(0, 2))
        for v in chosen:
            site = site0 if rng.random() < p_same_site else 1 - site0
            modes.append((int(v), int(rng.integers(0, 3)), site, FLAG_VIEW, 0))
        if n_scalars and rng.random() < 0.3:
            modes.append((int(rng.integers(0, n_scalars)), int(rng.integers(0, 3)), int(rng.integers(0, 2)), 0, 0))
        off.append(len(modes))
    return views, np.array(modes, MODE_DTYPE), np.array(off, np.uint32)


def gen_workload_fast(seed: int, n_buffers: int, buf_len: int, n_views: int, n_blocks: int, modes_per_block: int,
                      max_view_len: int, p_same_site: float = 0.9):
    """Vectorised generator for large batches (the bench): each block declares k in
    [1, modes_per_block] distinct views of one buffer (consecutive in that buffer's view
    list from a random start), random kinds, mostly one site."""
    rng = np.random.default_rng(seed)
    views = np.zeros(n_views, VIEW_DTYPE)
    buf = np.sort(rng.integers(0, n_buffers, n_views)).astype(np.uint32)
    views["buffer"] = buf
    views["lo"] = rng.integers(0, buf_len, n_views)
    views["hi"] = np.minimum(views["lo"] + rng.integers(0, max_view_len, n_views), buf_len - 1)
    views["name_rank"] = rng.permutation(n_views)
    start = np.searchsorted(buf, np.arange(n_buffers)).astype(np.int64)
    count = np.bincount(buf, minlength=n_buffers).astype(np.int64)
    nonempty = np.nonzero(count)[0]
    b = nonempty[rng.integers(0, len(nonempty), n_blocks)]
    k = np.minimum(rng.integers(1, modes_per_block + 1, n_blocks), count[b])
    off = np.zeros(n_blocks + 1, np.uint32)
    off[1:] = np.cumsum(k)
    blk = np.repeat(np.arange(n_blocks), k)
    j = np.arange(off[-1]) - np.repeat(off[:-1].astype(np.int64), k)
    r0 = rng.integers(0, 1 << 30, n_blocks)
    cb = count[b][blk]
    modes = np.zeros(int(off[-1]), MODE_DTYPE)
    modes["var"] = start[b][blk] + (r0[blk] + j) % cb
    modes["kind"] = rng.integers(0, 3, len(modes))
    site0 = rng.integers(0, 2, n_blocks)[blk]
    flip = rng.random(len(modes)) >= p_same_site
    modes["site"] = np.where(flip, 1 - site0, site0)
    modes["flags"] = FLAG_VIEW
    return views, modes, off
