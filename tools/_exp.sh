make -s >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_robust.py -q -m gpu > gpurun_out/t_edge.log 2>&1; tail -3 gpurun_out/t_edge.log
