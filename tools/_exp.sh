#!/bin/bash
# scratch: TC kernel with the look-back fix-up: tests + sweep T
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --out gpurun_out/sweepT --sections T > gpurun_out/sweepT.log 2>&1; sed -n '/^## T/,$p' gpurun_out/sweepT.md | head -14
