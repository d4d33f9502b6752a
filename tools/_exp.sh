make -s >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "hostio" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -5
timeout 600 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 2000 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['e2e'])"
