timeout 600 python -m pytest tests/test_bitmap.py tests/test_elem_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu_bm.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --container-log2-floats 0 --sweep-seeds 0 --overlap-views 0 --e2e-steps 0 --steps 20 > gpurun_out/bench_bm.json 2> gpurun_out/bench_bm.err
