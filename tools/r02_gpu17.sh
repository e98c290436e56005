mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dense.py -q -x > gpurun_out/g17_tests.log 2>&1; echo rc=$? >> gpurun_out/g17_tests.log; tail -5 gpurun_out/g17_tests.log
timeout 600 python tools/dense_bench.py 30 5 2>&1 | grep '"c64"' | grep tensor > gpurun_out/g17_dense_tma.jsonl; cat gpurun_out/g17_dense_tma.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense_tma --launch-count 1 -o gpurun_out/g17_tma5 -f python tools/one_dense.py 5 > gpurun_out/g17_ncu.log 2>&1; echo ncu=$?
