#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
timeout 600 python tools/sweep.py --sections T --out gpurun_out/sweepT > gpurun_out/sweepT.log 2>&1; cat gpurun_out/sweepT.md
