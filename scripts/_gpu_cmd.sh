timeout 600 python -m pytest tests/test_elem_gpu.py tests/test_container.py -x -q -m gpu > gpurun_out/pytest_gpu_elem.txt 2>&1
timeout 300 python scripts/bench_elem.py --reps 5 > gpurun_out/bench_elem_pdl.json 2>&1
