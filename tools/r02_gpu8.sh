mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x > gpurun_out/g8_tests.log 2>&1; echo rc=$? >> gpurun_out/g8_tests.log; tail -5 gpurun_out/g8_tests.log
timeout 600 python tools/dense_bench.py 30 5 2>&1 | grep '"c64"' | grep tensor > gpurun_out/g8_dense_pipe.jsonl; cat gpurun_out/g8_dense_pipe.jsonl
SVB_TC_NOPIPE=1 timeout 600 python tools/dense_bench.py 30 5 2>&1 | grep '"c64"' | grep tensor > gpurun_out/g8_dense_nopipe.jsonl; cat gpurun_out/g8_dense_nopipe.jsonl
