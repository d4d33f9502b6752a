# scratch: first run of the LAYOUT v3 register-streaming kernel
make -s >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py -x -q -m gpu > gpurun_out/t1.log 2>&1; tail -15 gpurun_out/t1.log
timeout 300 python bench.py --steps 2000 --warmup 20 --cpu-budget 2 > gpurun_out/b_grouped.json 2> gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b_grouped.json'));print('grouped', d['us_per_step'], d['value'], d['roofline']['frac'], [ (l['shape'], l['us']) for l in d['layers']], d['e2e']['value'], d['cpu_baseline']['gpu_parity'])"; tail -3 gpurun_out/b.err
timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --path launches > gpurun_out/b_launch.json 2>> gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b_launch.json'));print('launches', d['us_per_step'], d['value'])"
timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --x-ready 1 > gpurun_out/b_xr.json 2>> gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b_xr.json'));print('grouped x_ready', d['us_per_step'], d['value'])"
