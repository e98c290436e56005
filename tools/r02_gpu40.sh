mkdir -p gpurun_out
timeout 600 python tools/syc_passes.py 32 2>&1 | tail -1
SVB_LIB=build/alt/libsvb.so SVB_TRACE=1 timeout 600 python tools/syc_passes.py 32 > gpurun_out/g40_m14.txt 2>&1; tail -1 gpurun_out/g40_m14.txt; grep "jit pass" gpurun_out/g40_m14.txt | tail -3
