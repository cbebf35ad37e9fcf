timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r02c.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --container-log2-floats 0 --sweep-seeds 0 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
