mkdir -p gpurun_out
SVB_LIB=build/alt/libsvb.so timeout 600 python tools/syc_passes.py 32 > gpurun_out/g24_syc_rb5.txt 2>&1; tail -2 gpurun_out/g24_syc_rb5.txt
SVB_LIB=build/alt/libsvb.so SVB_JIT_STRICT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c64" > gpurun_out/g24_tests.log 2>&1; tail -3 gpurun_out/g24_tests.log
SVB_LIB=build/alt/libsvb.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "syc" > gpurun_out/g24_full.log 2>&1; tail -3 gpurun_out/g24_full.log
