#!/bin/bash
# scratch: dependent launches -- is the cross-CTA fix-up tail slowed by the next launch's prologue loads?
cd /root/repo
mkdir -p gpurun_out
for cfg in "base|" "nopdl|GQSA_DEP_PDL=0" "waitfirst|GQSA_DEP_WAIT_FIRST=1"; do
  name=${cfg%%|*}; envs=${cfg#*|}
  echo "== $name"
  env $envs timeout 300 python tools/trace_layer.py --rows 4096 --cols 4096 --launches 6 > gpurun_out/trace_4096_$name.log 2>&1; tail -7 gpurun_out/trace_4096_$name.log
done
timeout 1200 python tools/ab.py --rounds 1 "base||--x-ready 0" "nopdl|GQSA_DEP_PDL=0|--x-ready 0" "waitfirst|GQSA_DEP_WAIT_FIRST=1|--x-ready 0" 2>&1 | tee gpurun_out/ab_dep.log
for cfg in "base|" "nopdl|GQSA_DEP_PDL=0" "waitfirst|GQSA_DEP_WAIT_FIRST=1"; do
  name=${cfg%%|*}; envs=${cfg#*|}
  env $envs timeout 600 python tools/stack_bench.py --sections E --settings W4S50 --forms merged --batches 1 > gpurun_out/stack_$name.log 2>&1; echo "$name $(grep '"B": 1' gpurun_out/stack_$name.log)"
done
