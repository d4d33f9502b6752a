#!/bin/bash
# scratch: warp-level look-back (pipelined launches): tests + timing
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 10 > gpurun_out/bench_lb2.json 2> gpurun_out/bench_lb2.err; python -c "
import json;d=json.load(open('gpurun_out/bench_lb2.json'));print('2000', d['us_per_step'], d['value']);[print(l['shape'], l['us'], l['us_x_ready']) for l in d['layers']]" || tail -5 gpurun_out/bench_lb2.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 --no-layers > gpurun_out/bench_lb20.json 2> gpurun_out/bench_lb20.err; python -c "
import json;d=json.load(open('gpurun_out/bench_lb20.json'));print('20', d['us_per_step'], d['value'])" || tail -5 gpurun_out/bench_lb20.err
done
timeout 600 python tools/stack_bench.py --sections E --settings W4S50 --forms merged --batches 1 > gpurun_out/stack_lb2.log 2>&1; grep '"section"' gpurun_out/stack_lb2.log
