"""Regenerate the golden fixtures from the REFERENCE itself (oracle/_ref/libcohere_ref.so =
/root/reference/proj/include compiled in place by oracle/Makefile).  Run in the build
container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Outputs (committed):
  calltable.json  every (call type, start state) block outcome, via ref_call_outcome
                  (translate_block + run(Full) from that store, SURVEY Appendix A probe)
  traces.npz      named trace batches: records, per-trace results, boundary bitmaps,
                  produced by the reference's run_annotated loop (ref_eval_traces mode 0)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_ffi as o  # noqa: E402
import paper_1910_11110_b200 as coh  # noqa: E402

# name: (seed, trace0, n_traces, n_calls, n_arrays, adv_per1024, fuel, array_bytes)
CASES = {
    "c1_canonical": (0, 0, 1, 1000, 1, 0, 10000, None),
    "c1_adversarial": (0, 0, 64, 1000, 1, 16, 10000, None),
    "c2_default_mix": (1, 0, 256, 256, 64, 1, 10000, None),
    "c2_adversarial": (1, 1000, 256, 256, 64, 64, 10000, None),
    "fuel_limited_bytes": (7, 0, 256, 256, 64, 2, 300, [64 * (a + 1) for a in range(64)]),
    "ragged_small": (9, 3, 300, 37, 5, 200, 50, None),
    "all_adversarial": (13, 0, 128, 64, 7, 1024, 10000, None),
    "no_calls": (5, 0, 16, 0, 3, 0, 10, None),
    "zero_fuel": (5, 0, 16, 9, 3, 0, 0, None),
}


def main():
    assert o.have_ref(), "build oracle/_ref first (make -C oracle)"
    table = {}
    for t in range(64):
        if (t & 3) == 3:
            continue  # mode kind 3 is not a reference AccessMode::Kind
        for s in range(16):
            table[f"{t}:{s}"] = o.ref_outcome(t, s)
    with open(os.path.join(HERE, "calltable.json"), "w") as f:
        json.dump(table, f, indent=0, sort_keys=True)

    arrays = {}
    for name, (seed, trace0, nt, nc, na, adv, fuel, ab) in CASES.items():
        recs = coh.gen_records_host(seed, trace0, nt, nc, na, adv)
        res, bnd = o.ref_eval(recs, nt, nc, na, fuel, ab)
        arrays[f"{name}.params"] = np.array([seed, trace0, nt, nc, na, adv, fuel], dtype=np.int64)
        arrays[f"{name}.array_bytes"] = np.array(ab if ab else [], dtype=np.uint64)
        arrays[f"{name}.records"] = recs
        arrays[f"{name}.results"] = res.view(np.uint8)
        arrays[f"{name}.boundary"] = bnd
        st = np.bincount(res["status"], minlength=4)
        print(f"{name}: traces={nt} calls={nc} arrays={na} status(done,stuck,fuel,defect)={st.tolist()}")
    np.savez_compressed(os.path.join(HERE, "traces.npz"), **arrays)


if __name__ == "__main__":
    main()
