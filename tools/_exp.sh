make -s >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head
timeout 600 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 200 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], [(l['us'], l['us_p10_p50_p90']) for l in d['layers']])"
