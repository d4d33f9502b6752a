make -s >/dev/null 2>&1
timeout 3000 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frontend.py -q -x > gpurun_out/memcheck_par.log 2>&1; echo rc=$?; tail -4 gpurun_out/memcheck_par.log
