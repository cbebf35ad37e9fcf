#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full captures of the top kernels,
# whole-run element-path DRAM sums.
# usage (from repo root, under gpurun): bash scripts/gpu_check.sh TAG [quick]
set -u
TAG=${1:-r01}
MODE=${2:-full}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
[ "$MODE" = "quick" ] && { echo done; exit 0; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --bitmap-buffers 32 --container-log2-floats 24 \
  --c4-traces 0 --sweep-seeds 1000 --overlap-views 65536 --overlap-blocks 65536 --checker-programs 0 > $OUT/ncu_launch_bench_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_eval -s 2 -c 1 \
  -o $OUT/prof_trace_eval_$TAG -f python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --bitmap-buffers 0 \
  --container-log2-floats 0 --c4-traces 0 --sweep-seeds 0 --overlap-views 0 --checker-programs 0 > $OUT/ncu_full_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elem_pass1 -s 40 -c 1 \
  -o $OUT/prof_elem_pass1_$TAG -f python scripts/bench_elem.py --reps 1 --buffers 256 --frag-log2 16 > $OUT/ncu_elem_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elem_apply -s 20 -c 1 \
  -o $OUT/prof_elem_apply_$TAG -f python scripts/bench_elem.py --reps 1 --buffers 256 --frag-log2 16 >> $OUT/ncu_elem_$TAG.txt 2>&1
for k in 0 16 8 1; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --cache-control none --csv --log-file $OUT/ncu_elem_whole_k${k}_$TAG.csv python scripts/bench_elem.py --reps 1 --frag-log2 $k \
    > $OUT/ncu_elem_whole_k${k}_$TAG.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_runs_collect -s 1 -c 1 \
  -o $OUT/prof_runs_collect_$TAG -f python scripts/runs_rho.py 16 > $OUT/ncu_prims_$TAG.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_runs_place -s 1 -c 1 \
  -o $OUT/prof_runs_place_$TAG -f python scripts/runs_rho.py 1 full >> $OUT/ncu_prims_$TAG.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace_blocks -c 1 \
  -o $OUT/prof_trace_blocks_$TAG -f python -m pytest tests/test_trace_blocks_gpu.py -q -m gpu -k "vs_oracle and 20000" >> $OUT/ncu_prims_$TAG.txt 2>&1
echo done
