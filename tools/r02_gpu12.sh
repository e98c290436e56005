mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_batch.py tests/test_gpu_sampling_large.py tests/test_gpu_pblock.py -q > gpurun_out/g12_tests.log 2>&1; echo rc=$? >> gpurun_out/g12_tests.log; tail -4 gpurun_out/g12_tests.log
rm -rf /root/.cache/svb_jit
timeout 1200 python tools/batch_probe.py > gpurun_out/g12_batch.json 2> gpurun_out/g12_batch.err; cat gpurun_out/g12_batch.json; tail -3 gpurun_out/g12_batch.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense_tc6 --launch-count 1 -o gpurun_out/g12_tc6 -f python tools/one_dense.py 6 > gpurun_out/g12_ncu6.log 2>&1; echo ncu6=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense_tcp --launch-count 1 -o gpurun_out/g12_tcp5 -f python tools/one_dense.py 5 > gpurun_out/g12_ncu5.log 2>&1; echo ncu5=$?
