mkdir -p gpurun_out
timeout 600 python tools/c64_probe.py > gpurun_out/g25_main.txt 2>&1; tail -1 gpurun_out/g25_main.txt
SVB_LIB=build/alt/libsvb.so timeout 600 python tools/c64_probe.py > gpurun_out/g25_alt.txt 2>&1; tail -1 gpurun_out/g25_alt.txt
SVB_LIB=build/alt/libsvb.so SVB_JIT_OPTS=-DSVB_NO_FFMA2 timeout 600 python tools/syc_passes.py 32 > gpurun_out/g25_syc_rb5_noffma2.txt 2>&1; tail -1 gpurun_out/g25_syc_rb5_noffma2.txt
SVB_JIT_OPTS=-DSVB_NO_FFMA2 timeout 600 python tools/syc_passes.py 32 > gpurun_out/g25_syc_rb4_noffma2.txt 2>&1; tail -1 gpurun_out/g25_syc_rb4_noffma2.txt
