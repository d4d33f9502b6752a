# ad-hoc GPU experiment driver (edited per session)
make -s >/dev/null 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
python tools/sweep.py --out gpurun_out/r01_sweep > gpurun_out/sweep.log 2>&1; grep "^|" gpurun_out/sweep.log | head -20
