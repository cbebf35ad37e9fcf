"""The INTEGRATION.md shim (include/cohere_b200_shim.hpp), compiled against the reference's
own headers (oracle/Makefile -> oracle/_ref/shim_test, built where /root/reference exists
and shipped with the snapshot): AnnotatedProgram -> records -> AnnotatedProgram round
trip on the CPU, and run_annotated_batch on the GPU equal to cohere::run_annotated."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_test")

needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/shim_test not built (no reference here)")


@needs_bin
def test_shim_encode_round_trip():
    r = subprocess.run([BIN, "encode"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout


@needs_bin
@pytest.mark.gpu
def test_shim_run_annotated_batch_equals_reference():
    r = subprocess.run([BIN, "run"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
