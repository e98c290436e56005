mkdir -p gpurun_out
timeout 600 python tools/syc_passes.py 32 > gpurun_out/g26_syc.txt 2>&1; tail -1 gpurun_out/g26_syc.txt
timeout 600 python tools/c64_probe.py > gpurun_out/g26_c64.txt 2>&1; tail -1 gpurun_out/g26_c64.txt
SVB_JIT_STRICT=1 timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/g26_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/g26_gpu_tests.log; tail -4 gpurun_out/g26_gpu_tests.log
