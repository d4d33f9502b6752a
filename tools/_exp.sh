run() { for sh in "4096 4096" "14336 4096" "4096 14336"; do set -- $sh; python tools/prof_layer.py --rows $1 --cols $2 --launches 1 --time 2>&1 | tail -1 | sed "s/^/$TAG /"; done; }
TAG=np1 run
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
ncu --set full --import-source on --clock-control none -k regex:gqsa_streamk -s 6 -c 1 -o gpurun_out/l14336b python tools/prof_layer.py --rows 14336 --cols 4096 --launches 8 > /dev/null 2>&1
