#!/bin/bash
# scratch: CTA fix-up: publish before collect (no cross-CTA wait chains): tests + timing
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 10 > gpurun_out/bench_ro.json 2> gpurun_out/bench_ro.err; python -c "
import json;d=json.load(open('gpurun_out/bench_ro.json'));print('2000', d['us_per_step'], d['value']);[print(l['shape'], l['us'], l['us_x_ready']) for l in d['layers']]" || tail -5 gpurun_out/bench_ro.err
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 10 --x-ready 0 --no-layers > gpurun_out/bench_ro0.json 2> gpurun_out/bench_ro0.err; python -c "
import json;d=json.load(open('gpurun_out/bench_ro0.json'));print('xr0', d['us_per_step'], d['value'])" || tail -5 gpurun_out/bench_ro0.err
timeout 300 python tools/trace_layer.py --rows 4096 --cols 4096 --launches 6 > gpurun_out/trace_4096_ro.log 2>&1; tail -7 gpurun_out/trace_4096_ro.log
timeout 600 python tools/stack_bench.py --sections E --settings W4S50 --forms merged --batches 1,8 > gpurun_out/stack_ro.log 2>&1; grep '"section"' gpurun_out/stack_ro.log
