make -s >/dev/null 2>&1
GQSA_XCLUSTER=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "exact_integer or realistic" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E |FAILED|Error" gpurun_out/t.log | head -5
for xc in 0 2 4; do GQSA_XCLUSTER=$xc timeout 300 python bench.py --steps 5000 --warmup 100 --no-cpu-baseline --e2e-steps 10 2>gpurun_out/err.txt | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('XC=$xc', d['value'], d['us_per_step'], [l['us'] for l in d['layers']])" || tail -3 gpurun_out/err.txt; done
