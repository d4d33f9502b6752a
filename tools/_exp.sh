make -s >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_frontend.py -q -x 2>&1 | tail -3
timeout 900 python tools/sweep.py --sections D --out gpurun_out/sweepD 2>&1 | tail -8
