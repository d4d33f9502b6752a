#!/bin/bash
# scratch: CTA-level fix-up A/B (GQSA_CTA_FIX=1 default vs 0)
cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_cfix.log 2>&1; tail -3 gpurun_out/pytest_gpu_cfix.log
for r in 1 2; do
for v in 1 0; do
  GQSA_CTA_FIX=$v timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 10 --x-ready 0 > gpurun_out/ab_cfix$v.json 2>gpurun_out/ab_cfix$v.err
  python -c "
import json;d=json.load(open('gpurun_out/ab_cfix$v.json'));print('cfix=$v xr0', d['us_per_step'], [ (l['shape'], l['us']) for l in d['layers']])" || tail -3 gpurun_out/ab_cfix$v.err
done
done
for v in 1 0; do
  GQSA_CTA_FIX=$v timeout 600 python tools/stack_bench.py --sections E --settings W4S50 --forms merged,grouped --batches 1,8 > gpurun_out/stack_cfix$v.log 2>&1; echo cfix=$v; tail -12 gpurun_out/stack_cfix$v.log
done
