make -s >/dev/null 2>&1
for cfg in "GQSA_CTAS_PER_SM=1" "GQSA_CTAS_PER_SM=2 GQSA_WARPS=8 GQSA_FEW=0"; do
  env $cfg timeout 300 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 10 2>gpurun_out/err.txt | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$cfg', d['value'], d['us_per_step'], [l['us'] for l in d['layers']])" || tail -3 gpurun_out/err.txt
done
