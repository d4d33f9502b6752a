make -s >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py tests/test_gpu_frontend.py tests/test_gpu_fuzz.py -x -q -m gpu > gpurun_out/t1.log 2>&1; tail -2 gpurun_out/t1.log
tools/ab.sh "A D" 2
for v in D; do echo $v; GQSA_LIB_PATH=paper_2412_17560_b200/lib/var/$v.so timeout 300 python tools/trace_step.py 2>&1 | grep -E "exit-to-exit|phase|per tile|fixup|last exit|warps="; done
