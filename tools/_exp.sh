make -s >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
