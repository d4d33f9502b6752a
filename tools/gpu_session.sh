# ad-hoc GPU experiment driver (edited per session)
make -s >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for s in "4096 4096" "14336 4096" "4096 14336"; do set -- $s; for b in 3 4 8; do python tools/prof_layer.py --rows $1 --cols $2 --batch $b --launches 50 --time | grep -v plan; done; for w in 8 12; do GQSA_WARPS=$w python tools/prof_layer.py --rows $1 --cols $2 --batch 2 --launches 50 --time | grep -v plan | sed "s/^/w=$w /"; done; done
