# round-end evidence: tests, smoke, bench line, ncu launch list + full capture, sweeps
make -s >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gqsa -s 27 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_ncu.log 2>&1; tail -2 gpurun_out/bench_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gqsa_streamk -s 60 -c 3 -o gpurun_out/bench_full python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_full.log 2>&1; tail -2 gpurun_out/bench_full.log
timeout 1200 python tools/sweep.py --out gpurun_out/r01_sweep > gpurun_out/sweep.log 2>&1; tail -3 gpurun_out/sweep.log
timeout 1500 python tools/stack_bench.py --out gpurun_out/r01_stack > gpurun_out/stack.log 2>&1; tail -3 gpurun_out/stack.log
