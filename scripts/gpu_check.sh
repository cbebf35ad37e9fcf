#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of trace_eval.
# usage (from repo root, under gpurun): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.txt
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/ncu_launch_bench_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_eval -s 2 -c 1 \
  -o $OUT/prof_trace_eval_$TAG -f python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_full_$TAG.txt 2>&1
echo done
