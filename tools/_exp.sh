make -s >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hostio" 2>&1 | tail -2
timeout 600 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 2000 2>gpurun_out/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print(d['value'], d['us_per_step'], d['e2e'])" || tail -5 gpurun_out/err.txt
