#!/bin/bash
# compute-sanitizer over the kernels changed in round 2's second session, plus the host
# sanitizer build on the GPU tests' host side.  usage: bash scripts/sanitize_gpu.sh OUT
OUT=${1:-gpurun_out/sanitizer.txt}
CS="compute-sanitizer --target-processes all --error-exitcode 9"
{
echo "# compute-sanitizer runs on one B200 (round 2, second session)"
echo; echo "## memcheck: smoke()"
timeout 600 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo; echo "## memcheck: overlapped launch streams (launch-slot ring wrap, ticket path), fused counters"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_trace_gpu.py -q -p no:cacheprovider -k "overlapped and (ring or ticket) or fused_counters" 2>&1 | tail -2
echo; echo "## memcheck: zero-run primitives (collect / place with programmatic dependent launch), element path"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_bitmap.py tests/test_elem_gpu.py -q -p no:cacheprovider -k "not 16777216 and not 2p24 and not large" 2>&1 | tail -2
echo; echo "## racecheck: zero-run primitives (dense u16 staging) and the element apply"
timeout 1500 $CS --tool racecheck python -m pytest tests/test_bitmap.py -q -p no:cacheprovider -k "not 16777216" 2>&1 | tail -2
echo; echo "## host ASan + UBSan (lib/variants/asan.so): GPU tests' host side"
SAN_LOG=none timeout 1500 bash scripts/host_sanitize.sh -m gpu -k "not 1048576 and not c4 and not full and not 67108864 and not 2p24 and not large and not 16777216 and not shim and not facade" 2>&1 | tail -2
echo "(tests that run a separately built binary in a subprocess -- the shim test, the C++ facade build -- are left out: the preloaded ASan runtime is inherited by nvcc and by binaries that are not instrumented)"
} > "$OUT" 2>&1
