#!/bin/bash
# scratch: LAYOUT-TC with the CTA-level fix-up: tests + sweep T (vs GQSA_CTA_FIX=0)
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_robust.py tests/test_gpu_fixup_modes.py -m gpu -q -x > gpurun_out/pytest_tc.log 2>&1; tail -2 gpurun_out/pytest_tc.log
timeout 900 python tools/sweep.py --out gpurun_out/sweepT1 --sections T > gpurun_out/sweepT1.log 2>&1; grep "| tc" gpurun_out/sweepT1.md
GQSA_CTA_FIX=0 timeout 900 python tools/sweep.py --out gpurun_out/sweepT0 --sections T > gpurun_out/sweepT0.log 2>&1; grep "| tc" gpurun_out/sweepT0.md
