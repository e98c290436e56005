# round-2 GPU call 1: full-size parity, GPU suite, Sycamore c64 pass baseline + ncu
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/g1_fullsize.log 2>&1; echo rc=$? >> gpurun_out/g1_fullsize.log
tail -3 gpurun_out/g1_fullsize.log
timeout 300 python tools/syc_passes.py > gpurun_out/g1_syc.log 2>&1; tail -3 gpurun_out/g1_syc.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 6 --launch-count 1 -o gpurun_out/g1_syc32_c64_pass -f python tools/one_syc.py > gpurun_out/g1_ncu_syc.log 2>&1; echo ncu_rc=$?
timeout 1200 python -m pytest tests -q -x -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/g1_gpu.log 2>&1; echo rc=$? >> gpurun_out/g1_gpu.log
tail -3 gpurun_out/g1_gpu.log
