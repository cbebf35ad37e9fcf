"""Host mirror of the reference vocabulary for reading batched results.

Names and text follow namespace cohere so parity tests read like the reference's tests:
  RunStatus names        semantics.hpp:222-230 ("done", "stuck", "fuel-exhausted")
  EffectKind names       validity.hpp:37-46 ("push", "pull", "r", "w", "noop")
  ValidityPair text      validity.hpp:30-32 ("(V,I)")
  StuckInfo::describe    semantics.hpp:68-75
  AnnotatedRun fields    modes.hpp:95-103
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

RUN_STATUS_NAMES = {0: "done", 1: "stuck", 2: "fuel-exhausted", 3: "defect"}
EFFECT_NAMES = {0: "push", 1: "pull", 2: "r", 3: "w", 4: "noop"}
# effect_signature pre-patterns (validity.hpp:79-99) rendered by pre_to_string
_PRE = {0: "(V,*)", 1: "(*,V)", 2: "(V,*)", 3: "(*,*)", 4: "(*,*)"}


def pair_str(bits: int) -> str:
    """to_string(ValidityPair): bit0 = local Valid, bit1 = remote Valid."""
    return "(" + ("V" if bits & 1 else "I") + "," + ("V" if bits & 2 else "I") + ")"


@dataclass
class StuckInfo:
    key: str          # "a3" (concrete) or "a3^" (abstract), to_string(VarKey)
    effect: int
    site: int         # 0 local, 1 remote
    actual: int       # stored pair bits, unswapped

    def describe(self) -> str:
        out = ("g" if self.site else "") + EFFECT_NAMES[self.effect] + " " + self.key + ": have " + \
            pair_str(self.actual) + ", need " + _PRE[self.effect]
        if self.site:
            out += " against the swapped pair"
        return out


def describe_stuck(r) -> str:
    flags = int(r["stuck_flags"])
    key = f"a{int(r['stuck_array'])}" + ("^" if flags & 2 else "")
    return StuckInfo(key, int(r["stuck_effect"]), flags & 1, (flags >> 2) & 3).describe()


@dataclass
class AnnotatedRun:
    status: str
    store: dict = field(default_factory=dict)   # "a0" -> "(V,I)", "a0^" -> "(V,V)"
    stuck: StuckInfo | None = None
    boundary_ok: list = field(default_factory=list)
    steps: int = 0
    transfers: int = 0
    transfer_bytes: int = 0


def annotated_run(results: np.ndarray, boundary: np.ndarray | None, t: int, n_traces: int, n_arrays: int) -> AnnotatedRun:
    """Unpack trace t of a batch into the reference's AnnotatedRun shape."""
    r = results[t]
    store = {}
    for a in range(n_arrays):
        nib = (int(r["state"][a // 8]) >> (4 * (a % 8))) & 15
        store[f"a{a}"] = pair_str(nib & 3)
        store[f"a{a}^"] = pair_str(nib >> 2)
    status = RUN_STATUS_NAMES[int(r["status"])]
    stuck = None
    if status == "stuck":
        flags = int(r["stuck_flags"])
        stuck = StuckInfo(f"a{int(r['stuck_array'])}" + ("^" if flags & 2 else ""), int(r["stuck_effect"]),
                          flags & 1, (flags >> 2) & 3)
    bok = []
    if boundary is not None:
        for i in range(int(r["calls_done"])):
            w = int(boundary[(i // 32) * n_traces + t])
            bok.append(bool((w >> (i % 32)) & 1))
    return AnnotatedRun(status, store, stuck, bok, int(r["steps"]), int(r["transfers"]), int(r["transfer_bytes"]))
