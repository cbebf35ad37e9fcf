"""Acceptance-sweep fixtures from the REFERENCE (oracle/_ref): the program text of every
acceptance seed (as a digest), the leaves of all_schedules_run for seeds 0..999 at fuel
10000 and 0..299 at fuel 25, and the acceptance aggregate for seeds 0..9999 (criterion 4:
85335 schedule-distinct runs).  Run in the build container:
    make -C oracle && python tests/golden/make_golden_sweep.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_ffi as o  # noqa: E402


def main():
    h = hashlib.sha256()
    for seed in range(10000):
        h.update(o.ref_program_text(seed).encode())
    stats = o.ref_sweep_stats(0, 10000)
    with open(os.path.join(HERE, "sweep.json"), "w") as f:
        json.dump({"program_text_sha256_0_9999": h.hexdigest(), "acceptance_0_9999": stats}, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "sweep_leaves.npz"),
                        fuel10000=o.ref_sweep_leaves(0, 1000), fuel25=o.ref_sweep_leaves(0, 300, fuel=25))
    print(stats)


if __name__ == "__main__":
    main()
