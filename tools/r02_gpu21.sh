mkdir -p gpurun_out
./tools/mb/fmabench > gpurun_out/g21_fma.txt 2>&1; cat gpurun_out/g21_fma.txt
timeout 600 python tools/syc_passes.py 32 > gpurun_out/g21_syc_main.txt 2>&1; tail -2 gpurun_out/g21_syc_main.txt
SVB_LIB=build/alt/libsvb.so timeout 600 python tools/syc_passes.py 32 > gpurun_out/g21_syc_alt.txt 2>&1; tail -2 gpurun_out/g21_syc_alt.txt
