#!/bin/bash
# round evidence: tests, smoke, bench lines (driver command, 2000 steps, default), e2e breakdown,
# ncu launch list of the driver command + one full capture of the dominant kernel
cd /root/repo
mkdir -p gpurun_out
make -s >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; cat gpurun_out/bench_driver.json; tail -3 gpurun_out/bench_driver.err
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_2000.json 2> gpurun_out/bench_2000.err; cat gpurun_out/bench_2000.json
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_long.json 2> gpurun_out/bench_long.err; cat gpurun_out/bench_long.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; cat gpurun_out/e2e_probe.log
# (compute-sanitizer is closed on the GPU pool since this round; profiles/r02_*check.log are the
#  last runs, over tests/sanitize_small.py on the pre-CTA-fix-up build)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gqsa --csv --log-file gpurun_out/launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-layers --e2e-steps 2 > gpurun_out/bench_ncu.log 2>&1; tail -2 gpurun_out/bench_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gqsa_stream -s 40 -c 1 -o gpurun_out/bench_full -f python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-layers --e2e-steps 2 > gpurun_out/bench_full.log 2>&1; tail -2 gpurun_out/bench_full.log
