#!/bin/bash
# scratch: CTA-level fix-up with the look-back collector (c1 collects): tests + timing
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python tools/ab.py --rounds 2 "base||--x-ready 0" 2>&1 | tee gpurun_out/ab_lb.log
timeout 300 python tools/trace_layer.py --rows 4096 --cols 4096 --launches 6 > gpurun_out/trace_4096_lb.log 2>&1; tail -7 gpurun_out/trace_4096_lb.log
timeout 600 python tools/stack_bench.py --sections E --settings W4S50 --forms merged,grouped --batches 1,2 > gpurun_out/stack_lb.log 2>&1; grep '"section"' gpurun_out/stack_lb.log
