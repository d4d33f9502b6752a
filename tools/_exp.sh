make -s >/dev/null 2>&1
timeout 600 python bench.py --allgather fused --steps 2000 --warmup 50 --no-cpu-baseline --e2e-steps 10 > gpurun_out/f.json 2> gpurun_out/f.err; python -c "
import json; d=json.loads(open('gpurun_out/f.json').readline()); print(d['value'], d['us_per_step'], d['config'])" ; tail -5 gpurun_out/f.err
