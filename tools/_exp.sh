make -s >/dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gqsa_streamk -s 6 -c 1 -o gpurun_out/l14336 python tools/prof_layer.py --rows 14336 --cols 4096 --launches 8 > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
