make -s >/dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
timeout 900 python tools/sweep.py --sections H --out gpurun_out/sweepH > /dev/null 2>&1; grep "^|" gpurun_out/sweepH.md
timeout 600 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 200 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], [l['us'] for l in d['layers']])"
