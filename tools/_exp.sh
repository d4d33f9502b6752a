make -s >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-budget 3 > gpurun_out/b20.json 2> gpurun_out/b20.err; python -c "
import json;d=json.load(open('gpurun_out/b20.json'));print('steps20', d['us_per_step'], d['value'], d['roofline']['frac'], d['cpu_baseline']['gpu_parity'], d['clocks'])"; tail -3 gpurun_out/b20.err
timeout 300 python bench.py --steps 20000 --warmup 200 --no-cpu-baseline > gpurun_out/b20k.json 2>> gpurun_out/b20.err; python -c "
import json;d=json.load(open('gpurun_out/b20k.json'));print('steps20000', d['us_per_step'], d['value'], d['roofline']['frac'], [ (l['shape'], l['us']) for l in d['layers']], d['e2e']['value'])"
