make -s >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_chain.py -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
timeout 300 python tools/trace_chain.py 2>&1 | tail -4
for P in chain launches; do timeout 300 python bench.py --path $P --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$P', d['value'], d['us_per_step'])"; done
timeout 1500 python tools/stack_bench.py --batches 1 --out gpurun_out/stk > gpurun_out/stack.log 2>&1; grep "^| W4S50" gpurun_out/stack.log
