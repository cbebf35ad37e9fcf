"""cohere-b200: B200-native batched evaluator of the access-mode calculus of arXiv 1910.11110.

The compute path is the in-tree CUDA library ``lib/libcohere_b200.so`` (sm_100a) behind the
C ABI in ``include/cohere_b200.h``; this module is a thin ctypes binding over it plus a
host-side mirror of the reference vocabulary (``cohere::RunStatus``, ``EffectKind``, ``Site``,
``StuckInfo::describe``, ``AnnotatedRun``) so tests read like the reference's own tests.

There is no CPU fallback: importing works without a GPU (the call-table compiler and host
generator are host code), but every evaluation goes through the CUDA library and raises if it
is missing or fails.
"""
from ._ffi import (  # noqa: F401
    BATCH_BLOCKS,
    BATCH_OVERLAP,
    BATCH_PACKED12,
    pack_records12,
    COUNTER_NAMES,
    FLAG_UNSAFE,
    REC_CONT,
    RESULT_DTYPE,
    CohError,
    Comm,
    Context,
    comm_unique_id,
    counters_host,
    eval_traces_multi,
    nccl_version,
    shard_split,
    calltable_describe,
    calltable_program,
    gen_records_blocks_host,
    gen_records_host,
    lib,
    lib_path,
    make_record,
    record_fields,
    records_elems,
    boundary_words,
)
from .reference_api import (  # noqa: F401
    EFFECT_NAMES,
    RUN_STATUS_NAMES,
    AnnotatedRun,
    StuckInfo,
    annotated_run,
    describe_stuck,
    pair_str,
)

__all__ = [
    "BATCH_BLOCKS",
    "FLAG_UNSAFE",
    "REC_CONT",
    "Context",
    "CohError",
    "Comm",
    "comm_unique_id",
    "counters_host",
    "eval_traces_multi",
    "nccl_version",
    "shard_split",
    "RESULT_DTYPE",
    "COUNTER_NAMES",
    "calltable_describe",
    "calltable_program",
    "gen_records_host",
    "make_record",
    "record_fields",
    "records_elems",
    "boundary_words",
    "annotated_run",
    "AnnotatedRun",
    "StuckInfo",
    "describe_stuck",
    "lib",
    "lib_path",
]
