mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_advice.py tests/test_gpu_reference_suite.py -q > gpurun_out/g2_tests.log 2>&1; echo rc=$? >> gpurun_out/g2_tests.log
tail -30 gpurun_out/g2_tests.log
tail -40 gpurun_out/reference_suite.log
