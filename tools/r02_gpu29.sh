mkdir -p gpurun_out
timeout 900 python tools/batch_pass_probe.py > gpurun_out/g29_passes_main.txt 2>&1; grep "_24x" gpurun_out/g29_passes_main.txt | cut -c1-300
SVB_LIB=build/alt/libsvb.so timeout 900 python tools/batch_pass_probe.py > gpurun_out/g29_passes_alt.txt 2>&1; grep "_24x" gpurun_out/g29_passes_alt.txt | cut -c1-300
timeout 900 python tools/batch_time.py 3 > gpurun_out/g29_bt_main.txt 2>&1; tail -1 gpurun_out/g29_bt_main.txt
SVB_LIB=build/alt/libsvb.so timeout 900 python tools/batch_time.py 3 > gpurun_out/g29_bt_alt.txt 2>&1; tail -1 gpurun_out/g29_bt_alt.txt
