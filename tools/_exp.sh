make -s >/dev/null 2>&1
timeout 600 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 2000 2>gpurun_out/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print(d['value'], d['us_per_step'], d['e2e'])" || tail -5 gpurun_out/err.txt
timeout 1500 python tools/stack_bench.py --out gpurun_out/r01_stack > gpurun_out/stack.log 2>&1; tail -60 gpurun_out/stack.log | grep "^|"
