#!/bin/bash
# round evidence: tests, smoke, bench lines (driver command and a long run),
# ncu launch list of the driver command + one full capture of the dominant kernel
cd /root/repo
R=${R:-r02}
mkdir -p gpurun_out
make -s >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; cat gpurun_out/bench_driver.json; tail -3 gpurun_out/bench_driver.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_long.json 2> gpurun_out/bench_long.err; cat gpurun_out/bench_long.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gqsa --csv --log-file gpurun_out/launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-layers --e2e-steps 2 > gpurun_out/bench_ncu.log 2>&1; tail -2 gpurun_out/bench_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gqsa_stream -s 40 -c 1 -o gpurun_out/bench_full -f python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-layers --e2e-steps 2 > gpurun_out/bench_full.log 2>&1; tail -2 gpurun_out/bench_full.log
