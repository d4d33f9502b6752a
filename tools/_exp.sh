make -s >/dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
