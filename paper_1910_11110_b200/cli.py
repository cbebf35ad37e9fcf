"""Command-line front end mirroring the reference tool (tools/cohere_main.cpp): subcommands
check / run / infer / translate over a program file, flags --raw --json --no-overlap
--fuel --schedule, the same stdout / stderr text and exit codes.  Everything goes through
coh_cli (include/cohere_b200.h); `run` executes on the GPU.

    python -m paper_1910_11110_b200.cli run samples/write_read.coh
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys

from ._ffi import CohError, lib


class _Opts(C.Structure):
    _fields_ = [("raw", C.c_int), ("json", C.c_int), ("no_overlap", C.c_int), ("fuel", C.c_int32),
                ("schedule", C.c_char_p), ("trace", C.c_int)]


def _register(L):
    vp = C.c_void_p
    L.coh_cli.restype = C.c_int
    L.coh_cli.argtypes = [vp, C.c_char_p, C.c_char_p, C.POINTER(_Opts), C.c_char_p, C.c_size_t, C.c_char_p,
                          C.c_size_t, C.POINTER(C.c_int)]


_register(lib())
lib().coh_cli_batch.restype = C.c_int
lib().coh_cli_batch.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_uint32, C.POINTER(_Opts), C.c_int, C.c_char_p,
                                C.c_size_t, C.c_void_p, C.c_char_p, C.c_size_t, C.c_void_p, C.c_void_p]


def run_cli_batch(command: str, srcs, raw: bool = False, json: bool = False, no_overlap: bool = False,
                  threads: int = 0) -> list[tuple[str, str, int]]:
    """(stdout, stderr, exit code) of `command` (check / infer / translate) for every program
    text, evaluated on the host threads (coh_cli_batch)."""
    import numpy as np

    n = len(srcs)
    o = _Opts(int(raw), int(json), int(no_overlap), 10000, None, 0)
    arr = (C.c_char_p * max(1, n))(*[s.encode() for s in srcs])
    cap = max(1 << 16, 256 * n)
    while True:
        out, err = C.create_string_buffer(cap), C.create_string_buffer(cap)
        oo, eo = np.zeros(n + 1, np.uint64), np.zeros(n + 1, np.uint64)
        codes = np.zeros(max(1, n), np.int32)
        rc = lib().coh_cli_batch(command.encode(), arr, n, C.byref(o), threads, out, cap, oo.ctypes.data, err, cap,
                                 eo.ctypes.data, codes.ctypes.data)
        if rc < 0:
            cap = -rc + 16
            continue
        if rc:
            raise CohError(rc, f"coh_cli_batch({command})")
        ob, eb = out.raw, err.raw
        return [(ob[oo[i]:oo[i + 1]].decode(), eb[eo[i]:eo[i + 1]].decode(), int(codes[i])) for i in range(n)]


def run_cli(command: str, src: str, ctx=None, raw: bool = False, json: bool = False, no_overlap: bool = False,
            fuel: int = 10000, schedule: str | None = None, trace: bool = False) -> tuple[str, str, int]:
    """(stdout, stderr, exit code) of the reference CLI's `command` on program text `src`."""
    o = _Opts(int(raw), int(json), int(no_overlap), fuel, schedule.encode() if schedule else None, int(trace))
    cap = 1 << 16
    while True:
        out, err, code = C.create_string_buffer(cap), C.create_string_buffer(cap), C.c_int(0)
        rc = lib().coh_cli(ctx._h if ctx is not None else None, command.encode(), src.encode(), C.byref(o), out, cap,
                           err, cap, C.byref(code))
        if rc < 0:
            cap = -rc + 1
            continue
        if rc:
            raise CohError(rc, f"coh_cli({command}): {err.value.decode()}")
        return out.value.decode(), err.value.decode(), code.value


def main(argv: list[str] | None = None) -> int:
    p = argparse.ArgumentParser(prog="cohere", description="valid-invalid coherence calculus tool")
    sub = p.add_subparsers(dest="cmd", required=True)
    for name, run_flags in (("check", False), ("run", True), ("trace", True), ("infer", False), ("translate", False)):
        s = sub.add_parser(name)
        s.add_argument("file")
        s.add_argument("--raw", action="store_true")
        s.add_argument("--json", action="store_true")
        s.add_argument("--no-overlap", action="store_true")
        if run_flags:
            s.add_argument("--fuel", type=int, default=10000)
            s.add_argument("--schedule", default="")
        if name == "run":
            s.add_argument("--trace", action="store_true")
    a = p.parse_args(argv)
    try:
        src = open(a.file, encoding="utf-8").read()
    except OSError:
        sys.stderr.write(f"error: cannot read '{a.file}'\n")
        return 2
    ctx = None
    if a.cmd in ("run", "trace"):
        from ._ffi import Context
        ctx = Context(0)
    out, err, code = run_cli(a.cmd, src, ctx, a.raw, a.json, a.no_overlap, getattr(a, "fuel", 10000),
                             getattr(a, "schedule", "") or None, getattr(a, "trace", False))
    sys.stdout.write(out)
    sys.stderr.write(err)
    return code


if __name__ == "__main__":
    sys.exit(main())
