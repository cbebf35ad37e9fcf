timeout 600 python -m pytest tests/test_container.py -x -q -m gpu > gpurun_out/pytest_gpu_ct.txt 2>&1
timeout 600 python bench.py --steps 20 --no-cpu-baseline --bitmap-buffers 0 --sweep-seeds 0 --overlap-views 0 --e2e-steps 0 > gpurun_out/bench_ct.json 2> gpurun_out/bench_ct.err
