"""The header-only VectorPU facade (include/cohere_b200_vectorpu.hpp): vector<T>,
pvector<T>(mother, lo, hi) and the R/W/RW/GR/GW/GRW accessors over the C ABI.  CPU: the
header compiles on its own (g++, no CUDA headers).  GPU: a VectorPU-style program (CPU
write, GPU read, GPU update of a view, CPU read) built with nvcc against the in-tree
library moves exactly one upload of the vector and one download of the view."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")
LIB = os.path.join(ROOT, "paper_1910_11110_b200", "lib")


def test_facade_header_compiles():
    src = '#include "cohere_b200_vectorpu.hpp"\nint main() { return 0; }\n'
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.cpp")
        open(p, "w").write(src)
        r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra", "-I", INC, p],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_facade_program_moves_exactly_the_predicted_cells():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "vpu_demo")
        r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17",
                            "-I", INC, os.path.join(ROOT, "tests", "cpp", "vpu_demo.cu"), "-o", exe, "-L", LIB,
                            "-lcohere_b200", f"-Xlinker=-rpath={LIB}"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
