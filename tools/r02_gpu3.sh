mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x > gpurun_out/g3_dense.log 2>&1; echo rc=$? >> gpurun_out/g3_dense.log
tail -30 gpurun_out/g3_dense.log
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -q > gpurun_out/g3_ref.log 2>&1; echo rc=$? >> gpurun_out/g3_ref.log
tail -3 gpurun_out/g3_ref.log; grep -E "passed|failed" gpurun_out/reference_suite.log | tail -12
timeout 600 python tools/dense_bench.py 30 5 > gpurun_out/g3_dense_bench.jsonl 2> gpurun_out/g3_dense_bench.err; cat gpurun_out/g3_dense_bench.jsonl; tail -5 gpurun_out/g3_dense_bench.err
