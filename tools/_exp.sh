make -s >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 900 python tools/sweep.py --sections A --quick --out gpurun_out/sweepA > /dev/null 2>&1; grep "^| W" gpurun_out/sweepA.md
