# ad-hoc GPU experiment driver (edited per session)
make -s >/dev/null 2>&1
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gqsa -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gqsa --launch-skip 40 --launch-count 3 -o gpurun_out/bench_full -f python bench.py --steps 10 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out
