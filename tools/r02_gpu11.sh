mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_batch.py -q -x > gpurun_out/g11_tests.log 2>&1; echo rc=$? >> gpurun_out/g11_tests.log; tail -3 gpurun_out/g11_tests.log
timeout 600 python tools/dense_bench.py 30 5 2>&1 | grep '"c64"' | grep tensor > gpurun_out/g11_dense.jsonl; cat gpurun_out/g11_dense.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense_tcp --launch-count 1 -o gpurun_out/g11_tcp5 -f python tools/one_dense.py 5 > gpurun_out/g11_ncu5.log 2>&1; echo ncu5=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense_tc6 --launch-count 1 -o gpurun_out/g11_tc6 -f python tools/one_dense.py 6 > gpurun_out/g11_ncu6.log 2>&1; echo ncu6=$?
timeout 900 python tools/batch_bench.py > gpurun_out/g11_batch.json 2> gpurun_out/g11_batch.err; cat gpurun_out/g11_batch.json; tail -3 gpurun_out/g11_batch.err
