make -s >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_multirank.py -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -10
