make -s >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "pdl_dependent or concurrent" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -8
