python scripts/te_debug.py > gpurun_out/te_debug.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_dbl.txt 2>&1
COH_TE_SINGLE=1 timeout 600 python -m pytest tests/test_trace_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu_single.txt 2>&1
for v in 0 1; do COH_TE_SINGLE=$v timeout 300 python bench.py --no-cpu-baseline --bitmap-buffers 0 --e2e-steps 0 > gpurun_out/bench_te_single$v.json 2> gpurun_out/bench_te_single$v.err; done
