make -s >/dev/null 2>&1
for b in 2 8; do timeout 600 python bench.py --batch $b --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 50 2>gpurun_out/err.txt | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('B=$b', d['value'], d['us_per_step'], [l['us'] for l in d['layers']], d['e2e']['value'])" || tail -3 gpurun_out/err.txt; done
for p in chain; do timeout 600 python bench.py --path chain --batch 2 --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 50 2>gpurun_out/err.txt | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('chain B=2', d['value'], d['us_per_step'])" || tail -3 gpurun_out/err.txt; done
