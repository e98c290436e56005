mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/g20_tests.log 2>&1; echo rc=$? >> gpurun_out/g20_tests.log; tail -3 gpurun_out/g20_tests.log
SVB_BATCH_PROFILE=1 timeout 1500 python tools/batch_ab.py > gpurun_out/g20_ab.txt 2>&1; cat gpurun_out/g20_ab.txt
SVB_BATCH_PROFILE=1 timeout 900 python tools/batch_probe.py > gpurun_out/g20_probe.json 2> gpurun_out/g20_probe.err; cat gpurun_out/g20_probe.json; grep "batch_run" gpurun_out/g20_probe.err | tail -12
