#!/bin/bash
# Host code under AddressSanitizer + UndefinedBehaviorSanitizer: builds
# lib/variants/asan.so (make asan) and runs the CPU test suite against it with the ASan
# runtime preloaded into Python.  On a GPU box, pass extra pytest args (e.g. -m gpu -k ...)
# to cover the host side of GPU entry points too.
# usage: bash scripts/host_sanitize.sh [pytest args...]  (default: -m "not gpu")
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -C "$ROOT/paper_1910_11110_b200/csrc" asan -j8 > /tmp/host_sanitize_make.log 2>&1 || { tail -20 /tmp/host_sanitize_make.log; exit 1; }
ASAN_RT=$(/usr/bin/g++ -print-file-name=libasan.so)
UBSAN_RT=$(/usr/bin/g++ -print-file-name=libubsan.so)
export COH_B200_LIB="$ROOT/paper_1910_11110_b200/lib/variants/asan.so"
# protect_shadow_gap=0: the CUDA driver maps memory in the shadow gap; Python's own
# allocations are not leak-checked (detect_leaks=0); any UB report aborts the test run
# reports also go to files (pytest captures the test's stderr and a halting report exits
# before pytest could print it): ${SAN_LOG:-/tmp/host_sanitize}.asan.PID / .ubsan.PID
LOG=${SAN_LOG:-/tmp/host_sanitize}
export ASAN_OPTIONS="protect_shadow_gap=0:detect_leaks=0:halt_on_error=1"
export UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1"
if [ "$LOG" != "none" ]; then
  ASAN_OPTIONS="$ASAN_OPTIONS:log_path=$LOG.asan"
  UBSAN_OPTIONS="$UBSAN_OPTIONS:log_path=$LOG.ubsan"
fi
args=("$@")
[ ${#args[@]} -eq 0 ] && args=(-m "not gpu")
cd "$ROOT" && LD_PRELOAD="$ASAN_RT $UBSAN_RT" python -m pytest tests/ -x -q -p no:cacheprovider "${args[@]}"
