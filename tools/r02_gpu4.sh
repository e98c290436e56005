mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_batch.py -q -x > gpurun_out/g4_tests.log 2>&1; echo rc=$? >> gpurun_out/g4_tests.log
tail -15 gpurun_out/g4_tests.log
timeout 600 python tools/dense_bench.py 30 5 > gpurun_out/g4_dense_bench.jsonl 2> gpurun_out/g4_dense_bench.err; cat gpurun_out/g4_dense_bench.jsonl; tail -3 gpurun_out/g4_dense_bench.err
timeout 900 python tools/batch_bench.py > gpurun_out/g4_batch.json 2> gpurun_out/g4_batch.err; cat gpurun_out/g4_batch.json; tail -5 gpurun_out/g4_batch.err
