# ad-hoc GPU experiment driver (edited per session)
make -s >/dev/null 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for st in 2 4; do for s in "4096 4096" "14336 4096" "4096 14336"; do set -- $s; GQSA_STAGES=$st python tools/prof_layer.py --rows $1 --cols $2 --launches 50 --time | grep -v plan | sed "s/^/st=$st /"; done; done > gpurun_out/pair.log 2>&1
python tools/trace_layer.py --rows 14336 --cols 4096 > gpurun_out/trace_pair.log 2>&1
cat gpurun_out/pair.log
