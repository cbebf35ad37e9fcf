timeout 600 python -m pytest tests/test_sweep.py -x -q -m gpu > gpurun_out/pytest_gpu_sw.txt 2>&1
timeout 600 python bench.py --steps 10 --no-cpu-baseline --bitmap-buffers 0 --overlap-views 0 --container-log2-floats 0 --e2e-steps 0 > gpurun_out/bench_sw.json 2> gpurun_out/bench_sw.err
