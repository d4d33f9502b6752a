make -s >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -k "group_size or fuzz" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
timeout 900 python tools/sweep.py --sections H --out gpurun_out/sweepH > /dev/null 2>&1; grep "^| [0-9]" gpurun_out/sweepH.md
