#!/bin/bash
# A/B timing of experimental library builds (paper_2412_17560_b200/lib/var/<name>.so):
#   tools/ab.sh "A B" [rounds] [bench args...]   -- alternates the builds, prints us/step per run
names=$1; rounds=${2:-3}; shift 2
for r in $(seq 1 $rounds); do
  for v in $names; do
    GQSA_LIB_PATH=paper_2412_17560_b200/lib/var/$v.so timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 10 "$@" > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
    python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', d['us_per_step'], [ (l['shape'], l['us']) for l in d['layers']])" || tail -2 gpurun_out/ab_$v.err
  done
done
