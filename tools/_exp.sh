make -s >/dev/null 2>&1
timeout 1800 python tools/stack_bench.py --out gpurun_out/r01_stack > gpurun_out/stack.log 2>&1; grep -A20 "## G" gpurun_out/r01_stack.md
