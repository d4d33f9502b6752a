#!/bin/bash
cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log | head
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 10 --batch 8 --x-ready 0 > gpurun_out/bench_tpw8.json 2> gpurun_out/bench_tpw8.err; python -c "
import json;d=json.load(open('gpurun_out/bench_tpw8.json'));print('B8', d['us_per_step']);[print(l['shape'], l['us'], l['us_x_ready']) for l in d['layers']]" || tail -5 gpurun_out/bench_tpw8.err
