#!/bin/bash
# scratch: slice-aligned CTA ranges (GQSA_CTA_SLICEK=1) for dependent launches: parity + timing
cd /root/repo
mkdir -p gpurun_out
GQSA_CTA_SLICEK=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_slicek.log 2>&1; tail -3 gpurun_out/pytest_slicek.log
timeout 1200 python tools/ab.py --rounds 1 "base||--x-ready 0" "slicek|GQSA_CTA_SLICEK=1|--x-ready 0" "slicek_ts32|GQSA_CTA_SLICEK=1 GQSA_TARGET_SLOTS=32|--x-ready 0" "slicek_ts64|GQSA_CTA_SLICEK=1 GQSA_TARGET_SLOTS=64|--x-ready 0" "base_b8||--x-ready 0 --batch 8" "slicek_b8|GQSA_CTA_SLICEK=1|--x-ready 0 --batch 8" 2>&1 | tee gpurun_out/ab_slicek.log
GQSA_CTA_SLICEK=1 timeout 300 python tools/trace_layer.py --rows 4096 --cols 4096 --launches 6 > gpurun_out/trace_4096_slicek.log 2>&1; tail -7 gpurun_out/trace_4096_slicek.log
for cfg in "base|" "slicek|GQSA_CTA_SLICEK=1" "slicek_ts64|GQSA_CTA_SLICEK=1 GQSA_TARGET_SLOTS=64"; do
  name=${cfg%%|*}; envs=${cfg#*|}
  env $envs timeout 600 python tools/stack_bench.py --sections E --settings W4S50 --forms merged --batches 1,8 > gpurun_out/stack_$name.log 2>&1; echo "$name"; grep '"section"' gpurun_out/stack_$name.log
done
