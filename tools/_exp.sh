make -s >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
