make -s >/dev/null 2>&1
for cfg in "GQSA_TARGET_SLOTS=64" "GQSA_TARGET_SLOTS=128" "GQSA_TARGET_SLOTS=256" "GQSA_TARGET_SLOTS=32"; do
  env $cfg timeout 300 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 10 2>gpurun_out/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$cfg', d['value'], d['us_per_step'], [l['us'] for l in d['layers']])" || tail -5 gpurun_out/err.txt
done
