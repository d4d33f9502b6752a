make -s >/dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
timeout 2000 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_fuzz.py -q -k "G" > gpurun_out/mc.log 2>&1; tail -2 gpurun_out/mc.log
