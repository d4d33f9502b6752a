make -s >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_chain.py -q 2>&1 | tail -2
timeout 1500 python tools/stack_bench.py --batches 1 --out gpurun_out/r01_stack_b1 > gpurun_out/stack.log 2>&1; grep "^| W" gpurun_out/stack.log | head -14
