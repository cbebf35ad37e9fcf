"""Acceptance criterion 1 statuses from the REFERENCE itself (oracle/_ref ref_enum_straight_line:
enumerate_raw_programs + run, testkit.hpp:241-268).  Run where /root/reference exists:

    make -C oracle && python tests/golden/make_golden_enum.py

Output (committed): enum4.npy, the RunStatus of each of the 11111 programs, in the
reference's enumeration order."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]
import oracle_ffi as o  # noqa: E402


def ref_enum(max_len=4, fuel=16):
    R = o.reference()
    R.ref_enum_straight_line.restype = C.c_int
    R.ref_enum_straight_line.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_long, C.POINTER(C.c_long)]
    st = np.zeros(200000, np.uint8)
    unsafe = C.c_long()
    n = R.ref_enum_straight_line(max_len, fuel, st.ctypes.data, len(st), C.byref(unsafe))
    return st[:n], unsafe.value


if __name__ == "__main__":
    st, unsafe = ref_enum()
    print(len(st), "programs", int((st == 0).sum()), "done", int((st == 1).sum()), "stuck", unsafe, "unsafe")
    np.save(os.path.join(HERE, "enum4.npy"), st)
