python scripts/te_debug.py > gpurun_out/te_debug.txt 2>&1
bash scripts/gpu_check.sh r01z quick
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace_eval -s 2 -c 1 -o gpurun_out/prof_trace_eval_r01z -f python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --bitmap-buffers 0 > gpurun_out/ncu_full_r01z.txt 2>&1
