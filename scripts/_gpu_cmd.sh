python scripts/te_debug.py > gpurun_out/te_debug.txt 2>&1
timeout 600 python -m pytest tests/test_trace_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu_te.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --bitmap-buffers 0 --sweep-seeds 0 --overlap-views 0 --container-log2-floats 0 --e2e-steps 0 > gpurun_out/bench_te.json 2> gpurun_out/bench_te.err
